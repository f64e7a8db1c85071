#!/bin/bash
# One GPU call: tests, smoke, bench, then ncu launch list + full capture of the psi pass.
set -u
mkdir -p gpurun_out
nvidia-smi -q -d CLOCK > gpurun_out/clock_q.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1; nproc > gpurun_out/nproc.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
if [ "${NCU:-1}" = "1" ]; then
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
CMD2="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 300 $CMD2 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:psi_kernel -s 0 -c 2 -o gpurun_out/prof $CMD2 > gpurun_out/ncu_full.log 2>&1
fi
echo done
