#!/bin/bash
# GPU call: full GPU tests, KDE occupancy A/B, ncu of the q32 pass (one tool per call: no sanitizer here).
set -u
mkdir -p gpurun_out
timeout 120 python tools/sanitize_smoke.py > gpurun_out/entry_smoke.log 2>&1; echo "exit $?" >> gpurun_out/entry_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/parity_report.py > gpurun_out/parity_report.jsonl 2> gpurun_out/parity_report.err
bash tools/ab_kde.sh > gpurun_out/ab.log 2>&1
C1="python bench.py --workload q32 --config 2 --steps 1 --warmup 0"
timeout 300 $C1 > gpurun_out/plain_q32.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:psi_q32 -c 1 -o gpurun_out/prof_q32 $C1 > gpurun_out/ncu_q32.log 2>&1

echo done
