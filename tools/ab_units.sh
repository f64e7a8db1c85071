#!/bin/bash
# A/B: work-unit psi kernel (libplugin.so) vs the round-1 tile scheduler (tools/ab/libplugin_tiles.so,
# built from 61b2655), device times from CUDA-graph replays (tools/psi_graph_time.py)
out=gpurun_out/${1:-ab}_units.jsonl
: > $out
NS="${NS:-4096 8192 12000 16384 24576 32768 65536 131072 262144 1048576}"
python tools/psi_graph_time.py $NS >> $out
PLUGIN_LIB_PATH=tools/ab/libplugin_tiles.so python tools/psi_graph_time.py $NS >> $out
