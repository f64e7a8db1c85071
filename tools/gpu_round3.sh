#!/bin/bash
# GPU call: KDE bench + ncu, r=4 hybrid-exp A/B, fused-kernel ncu; the cfg5 oracle resumes in
# the background on the host cores (nice 19) and is stopped before the call ends.
set -u
mkdir -p gpurun_out/ckpt/cfg5 gpurun_out/golden
cp tests/golden/checkpoints/cfg5/*.json gpurun_out/ckpt/cfg5/ 2>/dev/null
python -c "import oracle; oracle.build(force=True)"
nice -n 19 python -m oracle.make_golden 5 --ckpt-root gpurun_out/ckpt --out-dir gpurun_out/golden > gpurun_out/oracle_cfg5.log 2>&1 &
ORA=$!
timeout 300 python bench.py --workload kde > gpurun_out/bench_kde.json 2> gpurun_out/bench_kde.err
PLUGIN_KDE_MUFU_ONLY=1 timeout 300 python bench.py --workload kde > gpurun_out/bench_kde_mufu.json 2> gpurun_out/bench_kde_mufu.err
bash tools/ab_hyb4.sh > gpurun_out/ab.log 2>&1
C1="python bench.py --workload kde --steps 1 --warmup 0"
timeout 300 $C1 > gpurun_out/plain_kde.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kde_kernel -c 1 -o gpurun_out/prof_kde $C1 > gpurun_out/ncu_kde.log 2>&1
C2="python tools/run_small.py 1024"
timeout 120 $C2 > gpurun_out/plain_small.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:plugin_fused -s 2 -c 1 -o gpurun_out/prof_fused $C2 > gpurun_out/ncu_fused.log 2>&1
# give the oracle the rest of the call, then stop it (it checkpoints per row chunk)
sleep ${ORACLE_EXTRA:-1500}
kill $ORA 2>/dev/null; sleep 2; kill -9 $ORA 2>/dev/null
tail -2 gpurun_out/oracle_cfg5.log
echo done
