#!/bin/bash
# A/B at the headline size: current build (tile centre without role swap, grouped-pass launches)
# vs tools/ab/libplugin_tiles.so (61b2655: centre with role swap); CUDA-graph replays
out=gpurun_out/${1:-ab}_swap.jsonl
: > $out
for rep in 1 2; do
  python tools/psi_graph_time.py 1048576 131072 16384 >> $out
  PLUGIN_LIB_PATH=tools/ab/libplugin_tiles.so python tools/psi_graph_time.py 1048576 131072 16384 >> $out
done
