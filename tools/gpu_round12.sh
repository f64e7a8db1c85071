#!/bin/bash
# GPU call: ncu captures of the block sort kernels and of the centred psi kernel (traffic, pipes)
set -u
mkdir -p gpurun_out
C1="python tools/run_sort.py 16384"
timeout 120 $C1 > gpurun_out/plain_sort.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sort_ -s 2 -c 2 -o gpurun_out/prof_sort $C1 > gpurun_out/ncu_sort.log 2>&1
C2="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 300 $C2 > gpurun_out/plain_psi.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:psi_kernel -s 0 -c 2 -o gpurun_out/prof_psi $C2 > gpurun_out/ncu_psi.log 2>&1
echo done
