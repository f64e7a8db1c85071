#!/bin/bash
# A/B of the fp32 chunk length of the psi pass (PSI_CH) with parity reports
set -u
mkdir -p gpurun_out
for lib in libplugin.so libplugin_ch128.so libplugin_ch128u16.so libplugin_ch32.so; do
  PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_ch_$lib.json 2>&1
  PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/$lib timeout 300 python tools/parity_report.py > gpurun_out/parity_ch_$lib.jsonl 2>&1
done
echo done
