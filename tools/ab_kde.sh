#!/bin/bash
# A/B of the KDE kernel occupancy (KDE_OCC=3 build) against the default library
set -u
mkdir -p gpurun_out
for lib in libplugin.so libplugin_kde3.so; do
  PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/$lib timeout 300 python bench.py --workload kde --steps 10 --warmup 3 > gpurun_out/ab_kde_$lib.json 2>&1
done
PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/libplugin_kde3.so timeout 900 python -m pytest tests/test_gpu_kde.py -m gpu -q > gpurun_out/ab_kde3_parity.log 2>&1
echo done
