#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf --timeout 600 -k "batch or fused or sort or toy or two_point or small" > gpurun_out/pytest_batch.log 2>&1; echo "exit $?" >> gpurun_out/pytest_batch.log
timeout 300 python bench.py --workload batch > gpurun_out/bench_batch.json 2> gpurun_out/bench_batch.err
PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/libplugin_ftime.so timeout 300 python tools/fused_phases.py 128 1024 > gpurun_out/fused_phases.jsonl 2> gpurun_out/fused_phases.err
echo done
