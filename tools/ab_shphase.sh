#!/bin/bash
# A/B: the quota scheduler's phase in a register (default build) vs in shared memory
# (-DPSI_SMQ_SHARED_PHASE, tools/ab/libplugin_shphase.so); graph-timed passes, two alternating runs;
# the scheduler-mode GPU test on the variant
set -u
mkdir -p gpurun_out
V=$PWD/tools/ab/libplugin_shphase.so
PLUGIN_LIB_PATH=$V timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "scheduler_modes or shards_sum or full_size_sampled" > gpurun_out/shphase_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/shphase_pytest.log
out=gpurun_out/shphase_ab.jsonl
: > $out
for rep in 1 2; do
  timeout 300 python tools/psi_graph_time.py 32768 49152 65536 100000 >> $out
  PLUGIN_LIB_PATH=$V timeout 300 python tools/psi_graph_time.py 32768 49152 65536 100000 >> $out
  PLUGIN_PSI_TAIL=2 timeout 300 python tools/psi_graph_time.py 131072 262144 | sed 's/"lib": "libplugin.so"/"lib": "libplugin.so forced mode 2"/' >> $out
  PLUGIN_PSI_TAIL=2 PLUGIN_LIB_PATH=$V timeout 300 python tools/psi_graph_time.py 131072 262144 | sed 's/"lib": "libplugin_shphase.so"/"lib": "libplugin_shphase.so forced mode 2"/' >> $out
  PLUGIN_PSI_TAIL=0 timeout 300 python tools/psi_graph_time.py 131072 262144 | sed 's/"lib": "libplugin.so"/"lib": "libplugin.so whole"/' >> $out
done
echo done
