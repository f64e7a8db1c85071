#!/bin/bash
# Long fp64 oracle run of BASELINE config 5 on the GPU box's host cores (checkpointed).
mkdir -p gpurun_out/ckpt gpurun_out/golden
if [ -d tests/golden/checkpoints/cfg5 ]; then mkdir -p gpurun_out/ckpt/cfg5 && cp tests/golden/checkpoints/cfg5/*.json gpurun_out/ckpt/cfg5/ ; fi
nproc > gpurun_out/oracle_nproc.txt
python -c "import oracle; oracle.build(force=True)"
timeout ${ORACLE_SECONDS:-9000} python -m oracle.make_golden 5 --ckpt-root gpurun_out/ckpt --out-dir gpurun_out/golden > gpurun_out/oracle_cfg5.log 2>&1
echo "exit $?" >> gpurun_out/oracle_cfg5.log
