#!/bin/bash
# A/B of the r=4 FMA-pipe-exp variant (PSI_HYB4=1 build) against the default library
set -u
mkdir -p gpurun_out
for lib in libplugin.so libplugin_hyb4.so; do
  PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$lib.json 2>&1
done
PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/libplugin_hyb4.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "baseline_configs or small_sweep or adversarial" > gpurun_out/ab_hyb4_parity.log 2>&1
echo done
