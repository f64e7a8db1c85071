# A/B: psi pass j-loop unroll at the cfg4 size (R = 4 psi6, R = 8 psi4): 16 (kept) vs 8 (1.2% / 1.8% slower)
set -u
for rep in 1 2; do
  for lib in libplugin.so libplugin_u8.so; do  # libplugin_u8.so: -DPSI_UNROLL=8
    PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/$lib python tools/psi_graph_time.py 1048576 | sed "s/^{/{\"variant\": \"$lib\", /" >> gpurun_out/ab_unroll.jsonl
  done
done
