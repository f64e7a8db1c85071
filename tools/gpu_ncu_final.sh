#!/bin/bash
# GPU call: ncu launch list of the default bench command and one --set full capture of each psi pass
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
CMD2="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 300 $CMD2 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^psi_kernel -s 0 -c 2 -o gpurun_out/prof $CMD2 > gpurun_out/ncu_full.log 2>&1
echo done
