# A/B: programmatic dependent launch of the multi-kernel sequence (default) against plain launches
# (PLUGIN_NO_PDL=1): CUDA-graph times of the passes and of plugin_h, n = 4096 ... 2^20
set -u
mkdir -p gpurun_out
for rep in 1 2; do
  for v in 0 1; do
    PLUGIN_NO_PDL=$v python tools/psi_graph_time.py 4096 16384 32768 131072 1048576 | sed "s/^{/{\"no_pdl\": $v, /" >> gpurun_out/ab_pdl.jsonl
  done
done
