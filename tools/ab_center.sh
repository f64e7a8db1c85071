#!/bin/bash
# A/B of the centred-FMA pair formulation (default build) against difference-first (PSI_CENTER=0)
set -u
mkdir -p gpurun_out
for lib in libplugin.so libplugin_nocenter.so; do
  PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_center_$lib.json 2>&1
  PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/$lib timeout 300 python tools/parity_report.py > gpurun_out/parity_$lib.jsonl 2>&1
done
echo done
