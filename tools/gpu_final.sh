#!/bin/bash
# Final GPU call of the round: every GPU test, smoke, parity report, every bench workload, latency.
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 300 python tools/parity_report.py > gpurun_out/parity_report.jsonl 2> gpurun_out/parity_report.err
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err
timeout 300 python bench.py --workload kde > gpurun_out/bench_kde.json 2> gpurun_out/bench_kde.err
timeout 300 python bench.py --skip-underflow --config 4 > gpurun_out/bench_skip4.json 2> gpurun_out/bench_skip4.err
timeout 600 python bench.py --skip-underflow --config 5 --steps 3 > gpurun_out/bench_skip5.json 2> gpurun_out/bench_skip5.err
timeout 300 python bench.py --workload q32 --config 3 --steps 3 > gpurun_out/bench_q32.json 2> gpurun_out/bench_q32.err
timeout 300 python bench.py --workload dpi --stages 3 --config 4 --steps 3 > gpurun_out/bench_dpi.json 2> gpurun_out/bench_dpi.err
timeout 300 python bench.py --workload batch > gpurun_out/bench_batch.json 2> gpurun_out/bench_batch.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 600 python tools/latency.py > gpurun_out/latency.jsonl 2> gpurun_out/latency.err
timeout 300 python tools/breakdown.py > gpurun_out/breakdown.jsonl 2> gpurun_out/breakdown.err
timeout 600 python tools/discrete_report.py > gpurun_out/discrete.jsonl 2> gpurun_out/discrete.err
timeout 300 python tools/rounded_report.py > gpurun_out/rounded.jsonl 2> gpurun_out/rounded.err
timeout 300 python tools/fused_grid.py > gpurun_out/fused_pipelined.jsonl 2> gpurun_out/fused_pipelined.err
timeout 900 python tools/psi_graph_time.py 2048 4096 8192 16384 32768 65536 131072 262144 1048576 > gpurun_out/psi_graph.jsonl 2> gpurun_out/psi_graph.err
bash tools/gpu_ncu_final.sh
echo done
