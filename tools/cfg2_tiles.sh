#!/bin/bash
# tile-size experiment at cfg2 (n = 16384): per-step breakdown for R = 1, 2, 4 (PLUGIN_PSI_R)
for r in 1 2 4; do
  echo "R=$r"; PLUGIN_PSI_R=$r timeout 300 python tools/breakdown.py 2>&1 | head -1
done
