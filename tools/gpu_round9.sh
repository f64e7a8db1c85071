#!/bin/bash
# GPU call: full tests (centred form fix + block sort), parity report, A/B, latency, phases, breakdown
set -u
mkdir -p gpurun_out
timeout 120 python tools/sanitize_smoke.py > gpurun_out/entry_smoke.log 2>&1; echo "exit $?" >> gpurun_out/entry_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
bash tools/ab_center.sh > gpurun_out/ab.log 2>&1
PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/libplugin_ftime.so timeout 300 python tools/fused_phases.py 128 512 1024 2048 > gpurun_out/fused_phases.jsonl 2> gpurun_out/fused_phases.err
timeout 300 python tools/breakdown.py > gpurun_out/breakdown.jsonl 2> gpurun_out/breakdown.err
timeout 600 python tools/latency.py > gpurun_out/latency.jsonl 2> gpurun_out/latency.err
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo done
