#!/bin/bash
# A/B at mid n: R = 1, 2 tiles at 3 CTAs/SM (default build) vs 4 CTAs/SM (<= 64 registers,
# tools/ab/libplugin_occ4.so), rows per thread forced by PLUGIN_PSI_R; CUDA-graph replays
out=gpurun_out/${1:-ab}_occ.jsonl
: > $out
NS="${NS:-8192 12000 16384 24576 32768 49152 65536}"
for R in 1 2; do
  PLUGIN_PSI_R=$R python tools/psi_graph_time.py $NS >> $out
  PLUGIN_PSI_R=$R PLUGIN_LIB_PATH=tools/ab/libplugin_occ4.so python tools/psi_graph_time.py $NS >> $out
done
PLUGIN_PSI_R=4 python tools/psi_graph_time.py 32768 49152 65536 >> $out
