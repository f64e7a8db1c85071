#!/bin/bash
# Last GPU call: the GPU suite, smoke and the headline bench on the final build; a separate ncu
# capture of the psi4 pass (the second psi_kernel launch of a step: captured alone, its metrics are valid)
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python tools/psi_graph_time.py 16384 32768 49152 65536 100000 131072 > gpurun_out/psi_graph.jsonl 2> gpurun_out/psi_graph.err
CMD2="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^psi_kernel -s 1 -c 1 -o gpurun_out/prof_psi4 $CMD2 > gpurun_out/ncu_psi4.log 2>&1
echo done
