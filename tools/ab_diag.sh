# A/B: banded diagonal tiles (psi_tile_sum<..., DIAG>, default) against full-square diagonal tiles
# (-DPSI_DIAG_BAND=0): the batch workload; and, when the pass kernel used it too (not kept: psi6 at
# n = 12288 went 25.8 -> 28.6 us), the R = 1 passes (n = 4096 ... 12288)
set -u
mkdir -p gpurun_out
for rep in 1 2; do
  for lib in libplugin.so libplugin_nodiag.so; do
    PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/$lib timeout 300 python bench.py --workload batch --steps 5 | sed "s/^{/{\"lib\": \"$lib\", /" >> gpurun_out/ab_diag_batch.jsonl
    PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/$lib python tools/psi_graph_time.py 4096 8192 12288 >> gpurun_out/ab_diag_graph.jsonl
  done
done
