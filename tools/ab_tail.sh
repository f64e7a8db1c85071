#!/bin/bash
# A/B: whole tiles (default) vs the tail split of the last S + tiles mod S tiles into column quarters
# (PLUGIN_PSI_TAIL=1); CUDA-graph replays
out=gpurun_out/${1:-ab}_tail.jsonl
: > $out
NS="${NS:-8192 16384 24576 32768 65536 131072 262144 1048576}"
for rep in 1 2; do
  python tools/psi_graph_time.py $NS >> $out
  PLUGIN_PSI_TAIL=1 python tools/psi_graph_time.py $NS | sed "s/\"lib\": \"libplugin.so\"/\"lib\": \"tail_split\"/" >> $out
done
