#!/bin/bash
set -u
mkdir -p gpurun_out
PLUGIN_BATCH_R_REPORT=4 timeout 300 python bench.py --workload batch > gpurun_out/ab_batch_r4.json 2>&1
PLUGIN_BATCH_R_REPORT=2 PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/libplugin_batch2.so timeout 300 python bench.py --workload batch > gpurun_out/ab_batch_r2.json 2>&1
PLUGIN_BATCH_R_REPORT=1 PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/libplugin_batch1.so timeout 300 python bench.py --workload batch > gpurun_out/ab_batch_r1.json 2>&1
echo done
