#!/bin/bash
# GPU call: the new tests, then the ncu evidence of the final state (launch list of the headline
# bench; one full capture of the KDE kernel)
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -k "tile_shape or sort_is_exact" > gpurun_out/pytest_new.log 2>&1; echo "exit $?" >> gpurun_out/pytest_new.log
C="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 300 $C > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $C > gpurun_out/ncu_launch.log 2>&1
C1="python bench.py --workload kde --steps 1 --warmup 0"
timeout 300 $C1 > gpurun_out/plain_kde.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kde_kernel -c 1 -o gpurun_out/prof_kde $C1 > gpurun_out/ncu_kde.log 2>&1
echo done
