#!/bin/bash
# A/B of the KDE hybrid fraction (KDE_POLY16 = 3, 4, 5 default, 6)
set -u
mkdir -p gpurun_out
for lib in libplugin.so libplugin_kdep3.so libplugin_kdep4.so libplugin_kdep6.so; do
  PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/$lib timeout 300 python bench.py --workload kde --steps 10 --warmup 3 > gpurun_out/ab_kde_$lib.json 2>&1
done
PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/libplugin_kdep4.so timeout 900 python -m pytest tests/test_gpu_kde.py -m gpu -q -rf > gpurun_out/kde_tests_p4.log 2>&1
echo done
