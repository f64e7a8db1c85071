#!/bin/bash
# compute-sanitizer over one small call of every entry point; TOOL = memcheck | racecheck | synccheck
set -u
mkdir -p gpurun_out
TOOL=${TOOL:-memcheck}
timeout 120 python tools/sanitize_smoke.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $TOOL --error-exitcode 9 python tools/sanitize_smoke.py > gpurun_out/sanitize_$TOOL.log 2>&1
echo "exit $?" >> gpurun_out/sanitize_$TOOL.log
