# A/B (variant not kept; profiles/r04h_ab_units_fx_drow.jsonl): equal-work chunk units for R = 1, 2
# (592 CTAs, each a contiguous run of 64-column chunks through one or two tiles) with per-(row,
# chunk) fixed point (libplugin.so then) or fp64 row sums and one block reduction per run
# (libplugin_drow.so, -DPSI_UNITS_DROW=1) against the whole-tile scheduler (libplugin_tiles.so);
# CUDA-graph times of the passes and of plugin_h
set -u
mkdir -p gpurun_out
NS="${NS:-4096 8192 12288 16384 24576 32768 49152 65536}"
for rep in 1 2; do
  for lib in libplugin.so libplugin_drow.so libplugin_tiles.so; do
    PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/$lib python tools/psi_graph_time.py $NS >> gpurun_out/ab_units2.jsonl
  done
done
