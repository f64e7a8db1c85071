#!/bin/bash
# GPU call: validate the centred pair formulation (full GPU tests incl. cfg5, parity report, A/B)
set -u
mkdir -p gpurun_out
timeout 120 python tools/sanitize_smoke.py > gpurun_out/entry_smoke.log 2>&1; echo "exit $?" >> gpurun_out/entry_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
bash tools/ab_center.sh > gpurun_out/ab.log 2>&1
PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/libplugin_nocenter.so timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -k "baseline or adversarial or sweep" > gpurun_out/pytest_nocenter.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo done
