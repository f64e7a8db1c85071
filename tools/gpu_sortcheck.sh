#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -rf --timeout 600 -k "sort or fused or small or toy or two_point or kde_sweep" > gpurun_out/pytest_sort.log 2>&1; echo "exit $?" >> gpurun_out/pytest_sort.log
PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/libplugin_ftime.so timeout 300 python tools/fused_phases.py 128 512 1024 2048 > gpurun_out/fused_phases.jsonl 2> gpurun_out/fused_phases.err
timeout 600 python tools/latency.py > gpurun_out/latency.jsonl 2> gpurun_out/latency.err
echo done
