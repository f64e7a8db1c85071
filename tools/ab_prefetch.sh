#!/bin/bash
# A/B: psi tiles with the next tile index fetched one tile ahead and all of a tile's loads issued
# together (current build) vs the previous build (tools/ab/libplugin_head.so); CUDA graphs
out=gpurun_out/${1:-ab}_prefetch.jsonl
: > $out
NS="${NS:-4096 8192 16384 32768 65536 131072 1048576}"
for rep in 1 2; do
  python tools/psi_graph_time.py $NS >> $out
  PLUGIN_LIB_PATH=tools/ab/libplugin_head.so python tools/psi_graph_time.py $NS >> $out
done
