#!/bin/bash
# A/B of the r=4 hybrid exp (PSI_HYB4=1 build, centred form) against the default library
set -u
mkdir -p gpurun_out
for lib in libplugin.so libplugin_hyb4.so; do
  PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$lib.json 2>&1
  PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/$lib timeout 300 python tools/parity_report.py > gpurun_out/parity_$lib.jsonl 2>&1
done
echo done
