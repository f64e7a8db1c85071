#!/bin/bash
# The cfg5 oracle on the host cores (resumed), with short GPU work: the changed tests, the
# latency table (oracle paused), one compute-sanitizer tool.
set -u
mkdir -p gpurun_out/ckpt/cfg5 gpurun_out/golden
cp tests/golden/checkpoints/cfg5/*.json gpurun_out/ckpt/cfg5/ 2>/dev/null
python -c "import oracle; oracle.build(force=True)"
timeout ${ORACLE_SECONDS:-3150} python -m oracle.make_golden 5 --ckpt-root gpurun_out/ckpt --out-dir gpurun_out/golden > gpurun_out/oracle_cfg5.log 2>&1 &
ORA=$!
kill -STOP $ORA
timeout 600 python -m pytest tests/test_gpu_kde.py tests/test_gpu_parity.py -m gpu -q -rf --timeout 600 -k "prepare or fused or small or two_point or toy" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/latency.py > gpurun_out/latency.jsonl 2> gpurun_out/latency.err
kill -CONT $ORA
TOOL=${TOOL:-memcheck} bash tools/gpu_sanitize.sh
wait $ORA
echo "oracle exit $?" >> gpurun_out/oracle_cfg5.log
echo done
