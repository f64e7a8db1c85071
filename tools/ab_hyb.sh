#!/bin/bash
# A/B at cfg4: FMA-pipe exps for 1/8 of the psi4 pairs (PSI_HYB4) and 1/16 of the psi6 pairs
# (PSI_HYB6), with the chunk loop unrolled 16x (default) or 8x; CUDA-graph replays of each pass
out=gpurun_out/${1:-ab}_hyb.jsonl
: > $out
for rep in 1 2; do
  for v in "" base_u8 hyb4_u16 hyb4_u8 hyb46_u8 hyb46_u16; do
    if [ -z "$v" ]; then python tools/psi_graph_time.py 1048576 >> $out;
    else PLUGIN_LIB_PATH=tools/ab/libplugin_$v.so python tools/psi_graph_time.py 1048576 >> $out; fi
  done
done
