#!/bin/bash
# GPU call: tests, smoke, benches (plugin, kde, skip), latency table, ncu captures.
set -u
mkdir -p gpurun_out
timeout 120 python tools/sanitize_smoke.py > gpurun_out/entry_smoke.log 2>&1; rc=$?; echo "entry smoke exit $rc" >> gpurun_out/entry_smoke.log
if [ $rc -ne 0 ]; then echo "entry smoke failed: stopping"; exit 1; fi
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
timeout 300 python bench.py --workload kde > gpurun_out/bench_kde.json 2> gpurun_out/bench_kde.err
timeout 300 python bench.py --skip-underflow --config 4 > gpurun_out/bench_skip4.json 2> gpurun_out/bench_skip4.err
timeout 600 python bench.py --skip-underflow --config 5 --steps 3 > gpurun_out/bench_skip5.json 2> gpurun_out/bench_skip5.err
timeout 600 python tools/latency.py > gpurun_out/latency.jsonl 2> gpurun_out/latency.err
timeout 300 python bench.py --workload q32 --config 3 --steps 3 > gpurun_out/bench_q32.json 2> gpurun_out/bench_q32.err
timeout 300 python bench.py --workload dpi --stages 3 --config 4 --steps 3 > gpurun_out/bench_dpi.json 2> gpurun_out/bench_dpi.err
PLUGIN_KDE_MUFU_ONLY=1 timeout 300 python bench.py --workload kde > gpurun_out/bench_kde_mufu.json 2> gpurun_out/bench_kde_mufu.err
if [ "${NCU:-1}" = "1" ]; then
C1="python bench.py --workload kde --steps 1 --warmup 0"
timeout 300 $C1 > gpurun_out/plain_kde.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kde_kernel -c 1 -o gpurun_out/prof_kde $C1 > gpurun_out/ncu_kde.log 2>&1
C2="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 300 $C2 > gpurun_out/plain_psi4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:psi_kernel -s 1 -c 1 -o gpurun_out/prof_psi4 $C2 > gpurun_out/ncu_psi4.log 2>&1
C3="python tools/latency.py --reps 20"
timeout 300 $C3 > gpurun_out/plain_lat.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_latency.csv $C3 > gpurun_out/ncu_lat.log 2>&1
fi
echo done
