# small-n evidence: the single-launch tests, latency per call, in-kernel phases
# (needs paper_1505_02100_b200/libplugin_ftime.so built with -DPLUGIN_FUSED_TIMING)
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or small or graph or sweep or toy or discretised or data_errors or second_device or concurrent" 2>&1 | tail -3
python tools/fused_grid.py > gpurun_out/small_fused_pipelined.jsonl 2>&1
PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/libplugin_ftime.so python tools/fused_phases.py 128 256 512 1024 2048 > gpurun_out/small_fused_phases.jsonl 2>&1
python tools/latency.py --reps 100 > gpurun_out/small_latency.jsonl 2>&1
