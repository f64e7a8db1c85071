#!/bin/bash
# The cfg5 oracle on the host cores (resumed from the committed checkpoints) while one
# compute-sanitizer tool runs over every entry point on the GPU.
set -u
mkdir -p gpurun_out/ckpt/cfg5 gpurun_out/golden
cp tests/golden/checkpoints/cfg5/*.json gpurun_out/ckpt/cfg5/ 2>/dev/null
python -c "import oracle; oracle.build(force=True)"
timeout ${ORACLE_SECONDS:-3200} python -m oracle.make_golden 5 --ckpt-root gpurun_out/ckpt --out-dir gpurun_out/golden > gpurun_out/oracle_cfg5.log 2>&1 &
ORA=$!
TOOL=${TOOL:-memcheck} bash tools/gpu_sanitize.sh
wait $ORA
echo "oracle exit $?" >> gpurun_out/oracle_cfg5.log
echo done
