#!/bin/bash
# GPU call after the scheduler change: the full GPU suite, smoke, the headline bench, graph-timed
# passes (default scheduler against PLUGIN_PSI_TAIL=0, two alternating runs), then the launch list
# and the ncu captures of both passes (tools/gpu_ncu_final.sh)
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python tools/parity_report.py > gpurun_out/parity_report.jsonl 2> gpurun_out/parity_report.err
NS="16384 32768 49152 65536 100000 131072 262144 1048576"
: > gpurun_out/psi_graph_ab.jsonl
for rep in 1 2; do
  timeout 600 python tools/psi_graph_time.py $NS | sed 's/"lib": "libplugin.so"/"sched": "default"/' >> gpurun_out/psi_graph_ab.jsonl
  PLUGIN_PSI_TAIL=0 timeout 600 python tools/psi_graph_time.py $NS | sed 's/"lib": "libplugin.so"/"sched": "whole"/' >> gpurun_out/psi_graph_ab.jsonl
done
timeout 600 python tools/latency.py > gpurun_out/latency.jsonl 2> gpurun_out/latency.err
bash tools/gpu_ncu_final.sh
echo done
