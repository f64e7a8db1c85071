#!/bin/bash
# GPU call: fused-path phase times, per-step breakdown, latency table (graphs incl. the fused
# launch), the headline bench; the cfg5 oracle (if unfinished) resumes in the background.
set -u
mkdir -p gpurun_out/ckpt/cfg5 gpurun_out/golden
if [ ! -f tests/golden/cfg5.json ]; then
  cp tests/golden/checkpoints/cfg5/*.json gpurun_out/ckpt/cfg5/ 2>/dev/null
  python -c "import oracle; oracle.build(force=True)"
  timeout ${ORACLE_SECONDS:-3300} nice -n 10 python -m oracle.make_golden 5 --ckpt-root gpurun_out/ckpt --out-dir gpurun_out/golden > gpurun_out/oracle_cfg5.log 2>&1 &
  ORA=$!
fi
PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/libplugin_ftime.so timeout 300 python tools/fused_phases.py 128 512 1024 2048 > gpurun_out/fused_phases.jsonl 2> gpurun_out/fused_phases.err
timeout 300 python tools/breakdown.py > gpurun_out/breakdown.jsonl 2> gpurun_out/breakdown.err
timeout 600 python tools/latency.py > gpurun_out/latency.jsonl 2> gpurun_out/latency.err
if [ -n "${ORA:-}" ]; then kill -STOP $ORA; fi
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ -n "${ORA:-}" ]; then kill -CONT $ORA; wait $ORA; echo "oracle exit $?" >> gpurun_out/oracle_cfg5.log; fi
echo done
