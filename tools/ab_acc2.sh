#!/bin/bash
# A/B: one vs two accumulators per row for R = 1 tiles (cfg2 passes, the batch kernel)
set -u
mkdir -p gpurun_out
for lib in libplugin.so libplugin_acc1.so; do
  for rep in 1 2; do
    PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/$lib timeout 300 python bench.py --config 2 --steps 50 --no-cpu-baseline > gpurun_out/ab_acc2_cfg2_${lib}_$rep.json 2>&1
    PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/$lib timeout 300 python bench.py --workload batch > gpurun_out/ab_acc2_batch_${lib}_$rep.json 2>&1
  done
done
echo done
