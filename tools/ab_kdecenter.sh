#!/bin/bash
# A/B of the centred KDE terms (default) against difference-first (KDE_CENTER=0)
set -u
mkdir -p gpurun_out
for lib in libplugin.so libplugin_kdenocenter.so; do
  PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/$lib timeout 300 python bench.py --workload kde --steps 10 --warmup 3 > gpurun_out/ab_kde_$lib.json 2>&1
done
timeout 900 python -m pytest tests/test_gpu_kde.py -m gpu -q -rf > gpurun_out/kde_tests.log 2>&1
echo done
