#!/bin/bash
# GPU call: full GPU tests, parity report, benches, latency table, ncu of the small-n path;
# the cfg5 oracle resumes in the background (nice 19) while the GPU parts run.
set -u
mkdir -p gpurun_out/ckpt/cfg5 gpurun_out/golden
cp tests/golden/checkpoints/cfg5/*.json gpurun_out/ckpt/cfg5/ 2>/dev/null
python -c "import oracle; oracle.build(force=True)"
if [ "${ORACLE:-1}" = "1" ]; then
  nice -n 19 python -m oracle.make_golden 5 --ckpt-root gpurun_out/ckpt --out-dir gpurun_out/golden > gpurun_out/oracle_cfg5.log 2>&1 &
  ORA=$!
fi
timeout 120 python tools/sanitize_smoke.py > gpurun_out/entry_smoke.log 2>&1; echo "exit $?" >> gpurun_out/entry_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/parity_report.py > gpurun_out/parity_report.jsonl 2> gpurun_out/parity_report.err
timeout 600 python tools/latency.py > gpurun_out/latency.jsonl 2> gpurun_out/latency.err
if [ "${ORACLE:-1}" = "1" ]; then kill -STOP $ORA 2>/dev/null; fi   # quiet host for the timed benches
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --workload kde > gpurun_out/bench_kde.json 2> gpurun_out/bench_kde.err
if [ "${ORACLE:-1}" = "1" ]; then kill -CONT $ORA 2>/dev/null; fi
C2="python tools/run_small.py 1024"
timeout 120 $C2 > gpurun_out/plain_small.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:plugin_fused -s 2 -c 1 -o gpurun_out/prof_fused $C2 > gpurun_out/ncu_fused.log 2>&1
C3="python tools/latency.py --reps 20"
timeout 300 $C3 > gpurun_out/plain_lat.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_latency.csv $C3 > gpurun_out/ncu_lat.log 2>&1
sleep ${ORACLE_EXTRA:-0}
if [ "${ORACLE:-1}" = "1" ]; then kill $ORA 2>/dev/null; sleep 2; kill -9 $ORA 2>/dev/null; tail -2 gpurun_out/oracle_cfg5.log; fi
echo done
