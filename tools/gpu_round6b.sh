#!/bin/bash
# GPU round 6 work with the cfg5 oracle resuming in the background for the rest of the call.
set -u
mkdir -p gpurun_out/ckpt/cfg5 gpurun_out/golden
cp tests/golden/checkpoints/cfg5/*.json gpurun_out/ckpt/cfg5/ 2>/dev/null
python -c "import oracle; oracle.build(force=True)"
timeout ${ORACLE_SECONDS:-3400} nice -n 10 python -m oracle.make_golden 5 --ckpt-root gpurun_out/ckpt --out-dir gpurun_out/golden > gpurun_out/oracle_cfg5.log 2>&1 &
ORA=$!
bash tools/gpu_round6.sh
wait $ORA
echo "oracle exit $?" >> gpurun_out/oracle_cfg5.log
