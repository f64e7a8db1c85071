#!/bin/bash
# tile-shape sweep at mid-size n: CTA tiles R = 1, 2, 4 (T = 256 R), pass time alone
set -u
mkdir -p gpurun_out
NS="3000 5000 8192 12000 16384 24000 40000 65000 100000 130000"
for r in 1 2 4; do
  PLUGIN_PSI_R=$r timeout 300 python tools/psi_time.py $NS > gpurun_out/ab_tiles_r$r.jsonl 2>&1
done
timeout 300 python tools/psi_time.py $NS > gpurun_out/ab_tiles_default.jsonl 2>&1
echo done
