#!/bin/bash
# A/B of the pass scheduler (PLUGIN_PSI_TAIL): 0 whole tiles from one counter (default), 1 remainder
# tiles (tiles mod 148) as 64-column slices, 2 slices + per-SM quota of the whole tiles.  The GPU
# suite under mode 2 and under the default, then CUDA-graph pass times per n, two alternating runs.
set -u
mkdir -p gpurun_out
tag=${1:-ab}
PLUGIN_PSI_TAIL=2 timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/${tag}_pytest_mode2.log 2>&1; echo "pytest exit $?" >> gpurun_out/${tag}_pytest_mode2.log
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/${tag}_pytest_default.log 2>&1; echo "pytest exit $?" >> gpurun_out/${tag}_pytest_default.log
out=gpurun_out/${tag}_smq.jsonl
: > $out
NS="${NS:-4096 8192 12000 16384 24576 32768 49152 65536 100000 131072 262144}"
for rep in 1 2; do
  for m in 0 1 2; do
    PLUGIN_PSI_TAIL=$m timeout 600 python tools/psi_graph_time.py $NS | sed "s/\"lib\": \"libplugin.so\"/\"mode\": $m/" >> $out
  done
done
for m in 0 2; do
  PLUGIN_PSI_TAIL=$m timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_mode$m.json 2> gpurun_out/${tag}_bench_mode$m.err
done
echo done
