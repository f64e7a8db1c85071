#!/usr/bin/env python
"""Benchmark of the PLUGIN hot path (arXiv 1505.02100, Alg. 1) on B200.

`python bench.py --gpus N --steps K --warmup W [--impl ours|reference] [--config C]`

One step = one whole PLUGIN run (Step I, sort, the Step IV pass psi6, g2, the Step VI
pass psi4, h) on BASELINE config C (default 4: n = 1,048,576 i.i.d. N(3, 2^2), seed 3),
the configuration BASELINE.json quotes at 1/2/4/8 GPUs.  Metric: pairwise K4/K6
evaluations per second, 2 * n(n-1)/2 per step (unique pairs of both passes, Eq. 6/7),
over the whole job (all ranks).  N > 1: launched by torchrun, one rank per GPU, tile
shards + one 32-byte NCCL allreduce per pass (strong scaling: n is fixed).

Timing: per step CUDA events on the launching stream, L2 flushed (256 MiB write)
between steps outside the events, barrier + synchronize around the timed region,
max over ranks.  Clocks sampled with nvidia-smi during the timed region.
`--impl reference` times the fp64 CPU oracle (oracle/) on a bounded row sample of the
same workload on the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "pairwise K4/K6 evaluations/sec (GPairs/s) and end-to-end h time vs FMA/SFU roofline, 1-8 GPUs"
UNIT = "GPairs/s"
MUFU_EX2_PER_CLK_PER_SM = 16      # measured: tools/probe/mufu_probe.cu (profiles/r01_mufu_probe.jsonl)
FMA_LANE_OPS_PER_CLK_PER_SM = 128  # FP32 lane-ops (packed FFMA2 = 2), measured 124-128 (r01_mufu_probe.jsonl)
EX2_FMA_LANE_OPS = 8               # simd.cuh ex2_fma2: an FMA-pipe 2^x costs 8 FP32 lane-ops per lane


def dual_pipe_bound(fp32_ops: float) -> float:
    """Pairs (terms) per clock per SM when a fraction phi of the exps runs on the FMA pipe
    (ex2_fma2) and the rest on MUFU.EX2, at the best phi: min(16 / (1 - phi), 128 / (k + 8 phi)) is
    largest where both pipes saturate, phi = (128 - 16 k) / (128 + 16 * 8).  k = FP32 lane-ops per
    pair besides the exp: 7 (psi6), 6 (psi4), 3 (KDE, centred)."""
    phi = (FMA_LANE_OPS_PER_CLK_PER_SM - MUFU_EX2_PER_CLK_PER_SM * fp32_ops) / (
        FMA_LANE_OPS_PER_CLK_PER_SM + MUFU_EX2_PER_CLK_PER_SM * EX2_FMA_LANE_OPS)
    phi = max(0.0, phi)
    return min(MUFU_EX2_PER_CLK_PER_SM / (1.0 - phi), FMA_LANE_OPS_PER_CLK_PER_SM / (fp32_ops + EX2_FMA_LANE_OPS * phi))


# Q32.32 pass (q32.cu): the ALU pipe binds (ncu on an all-in-range pass, profiles/r02_prof_q32_summary.txt:
# ALU 64% of peak, FMA/IMAD 26%, XU 0%); 169 ALU-pipe thread-instructions per in-range pair
# (sm__inst_executed_pipe_alu x 32 / pairs) at 64 ALU lanes/clk/SM (16 per SMSP, rt 2)
Q32_ALU_INST_PER_PAIR = 169.0
ALU_LANES_PER_CLK_PER_SM = 64
# kernels of one step, n > 32768 (group.cu: from kGroupMinN = 32768 the distinct-value count and
# compaction run after Step I, and each pass launches the fp32 tile pass and the grouped exact
# pass, one of which returns at once)
KERNELS_PER_STEP = 23             # distributed API: 12 radix sort, step1, 2 group, 2 x (psi, group psi, export, finalize)
KERNELS_PER_PLUGIN_H = 19         # plugin_h: 12 radix sort, step1, 2 group, 2 x (psi, group psi) (finalize in the last CTA)


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--workload", default="plugin", choices=["plugin", "kde", "q32", "dpi", "batch"],
                    help="plugin: Alg. 1 (the headline); kde: Eq. 1-2 on a 65536-point curve (NEXT 1); "
                         "q32: Alg. 1 with the Q32.32 pair passes (NEXT 2); dpi: the l-stage plug-in (NEXT 3)")
    ap.add_argument("--stages", type=int, default=3, help="dpi workload: l")
    ap.add_argument("--batch", type=int, default=4096, help="batch workload: samples of n = 1024")
    ap.add_argument("--kde-points", type=int, default=65536)
    ap.add_argument("--skip-underflow", action="store_true",
                    help="plugin workload, 1 GPU: PLUGIN_SKIP_UNDERFLOW (bit-identical result; reports the "
                         "effective rate, the roofline over the pairs actually evaluated)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU time of the oracle sample")
    return ap.parse_args()


def _workload(k, n):
    from paper_1505_02100_b200 import inputs
    c = inputs.CONFIGS[k]
    return (f"cfg{k}: n={n} float32 {c['dist']} seed {c['seed']}; full PLUGIN per step "
            f"(Step I, sort, psi6 pass, g2, psi4 pass, h)")


class ClockSampler:
    """nvidia-smi sampling of SM clock and throttle reasons during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            p = [s.strip() for s in line.split(",")]
            if len(p) >= 7:
                self.rows.append(p)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "power_w_max": max((float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()), default=None)}


def _traffic(n, name="psi_traffic.json", m=None):
    """DRAM bytes per launch of a kernel from its committed ncu --set full capture (same sizes only)."""
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            t = json.load(f)
    except OSError:
        return None
    if t.get("n") != n or (m is not None and t.get("m") != m):
        return None
    return t["dram_bytes_read_per_launch"] + t["dram_bytes_write_per_launch"]


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_oracle_sample(k: int, seconds: float, threads: int = 0):
    """Time the oracle (as it stands) on rows [0, m) of both passes of config k."""
    import numpy as np

    import oracle
    from paper_1505_02100_b200 import inputs
    x = inputs.config_data(k)
    n = x.size
    s1 = oracle.step1(x)
    z = oracle.zscore(x, s1["mean"], s1["sigma"])
    g1 = oracle.g1_bandwidth(oracle.psi8_ns(1.0), n)
    gold = os.path.join(ROOT, "tests", "golden", f"cfg{k}.json")
    g2 = json.load(open(gold))["g2_z"] if os.path.exists(gold) else g1
    # calibrate on a small sample, then size the timed sample to ~`seconds`
    m0 = max(1, min(n, 64))
    t0 = time.perf_counter()
    oracle.psi_sum_rows(z, g1, 6, 0, m0, threads)
    rate = oracle.pair_count_rows(n, 0, m0) / max(time.perf_counter() - t0, 1e-6)
    target_pairs = rate * seconds / 2
    m = m0
    while m < n and oracle.pair_count_rows(n, 0, m) < target_pairs:
        m = min(n, m * 2)
    pairs = 0
    t0 = time.perf_counter()
    for r, g in ((6, g1), (4, g2)):
        oracle.psi_sum_rows(z, g, r, 0, m, threads)
        pairs += oracle.pair_count_rows(n, 0, m)
    dt = time.perf_counter() - t0
    cores = threads if threads > 0 else oracle.lib().oracle_max_threads()
    return {"value": pairs / dt / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"cfg{k} rows [0,{m}) of both passes ({pairs} pairs, {dt:.1f} s, fp64, OpenMP)",
            "seconds": dt, "pairs": pairs}


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    vals = []
    info = None
    secs = max(1.0, min(a.cpu_seconds, 120.0 / max(1, a.steps + a.warmup)))
    for i in range(a.warmup + a.steps):
        info = cpu_oracle_sample(a.config, secs)
        if i >= a.warmup:
            vals.append(info["value"])
    v = statistics.median(vals)
    from paper_1505_02100_b200 import inputs
    n = inputs.CONFIGS[a.config]["n"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": info["seconds"] * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": _workload(a.config, n), "sample": info["sample"]},
            "cpu_baseline": {k: info[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)
    return 0


def psi_pairs_evaluated(xh, g, tile=2048):
    """Pairs the psi pass evaluates with PLUGIN_SKIP_UNDERFLOW (the rule of psi.cu): every
    diagonal tile, and off-diagonal tiles unless (xs[j0] - xs[i0+T-1]) s (1 - 1e-5) > 13.25."""
    import numpy as np
    xs = np.sort(xh.astype(np.float32)).astype(np.float64)
    n = xs.size
    nb = -(-n // tile)
    s = float(np.float32(1.0 / g))
    first = xs[np.arange(nb) * tile]
    last = xs[np.minimum(np.arange(nb) * tile + tile - 1, n - 1)]
    rows = np.minimum(tile, n - np.arange(nb) * tile).astype(np.float64)
    tot = 0.0
    for bi in range(nb):
        gap = first[bi + 1:] - last[bi]
        keep = ~(gap * s * (1 - 1e-5) > 13.25)
        tot += 2.0 * rows[bi] * float(np.sum(rows[bi + 1:][keep])) / 2.0  # unique pairs (i<j) of kept tiles
        tot += rows[bi] * (rows[bi] - 1) / 2.0
    return tot


def run_skip(a):
    """1 GPU, plugin_h_ex(PLUGIN_SKIP_UNDERFLOW): effective pair rate, bit-identical result."""
    import torch

    from paper_1505_02100_b200 import inputs
    from paper_1505_02100_b200 import plugin as P
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    xh = inputs.config_data(a.config)
    n = xh.size
    x = torch.from_numpy(xh).to(dev)
    ws = P.workspace(n, dev)
    out = P.new_result(dev)
    ref = P.read_result(P.plugin_h(x, out=out, ws=ws))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(a.warmup):
        P.plugin_h(x, out=out, ws=ws, flags=P.PLUGIN_SKIP_UNDERFLOW)
    torch.cuda.synchronize(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    clk = ClockSampler(0)
    clk.start()
    time.sleep(0.3)
    for s in range(a.steps):
        flush.fill_(s & 0xff)
        ev[s][0].record(stream)
        P.plugin_h(x, out=out, ws=ws, flags=P.PLUGIN_SKIP_UNDERFLOW)
        ev[s][1].record(stream)
    torch.cuda.synchronize(dev)
    clocks = clk.stop()
    res = P.read_result(out)
    same = all(res[k] == ref[k] for k in ref if ref[k] == ref[k])
    ms = sum(e0.elapsed_time(e1) for e0, e1 in ev) / a.steps
    pairs = n * (n - 1) // 2
    ev6 = psi_pairs_evaluated(xh, res["g1"], P.plugin_tile_edge(n, 6))
    ev4 = psi_pairs_evaluated(xh, res["g2"], P.plugin_tile_edge(n, 4))
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    f_meas = clocks.get("sm_mhz") or 1965.0
    peak = MUFU_EX2_PER_CLK_PER_SM * sms * f_meas * 1e6 / 1e9
    line = {"metric": METRIC + " [effective, PLUGIN_SKIP_UNDERFLOW]", "value": 2 * pairs / (ms / 1e3) / 1e9,
            "unit": UNIT, "n_gpus": 1, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": _workload(a.config, n) + " with PLUGIN_SKIP_UNDERFLOW", "n": n,
                       "pairs_per_step_effective": 2 * pairs, "pairs_evaluated": {"psi6": ev6, "psi4": ev4},
                       "bit_identical_to_full": same},
            "roofline": {"bound": "alu", "achieved": (ev6 + ev4) / (ms / 1e3) / 1e9, "peak": peak, "unit": UNIT,
                         "frac": (ev6 + ev4) / (ms / 1e3) / 1e9 / peak, "traffic": None,
                         "kernel": "whole step over evaluated pairs (includes sort/Step I)"},
            "h": res["h"], "status": res["status"], "clocks": clocks, "gpu_launches": KERNELS_PER_PLUGIN_H * a.steps}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(a):
    import torch
    import torch.distributed as dist

    from paper_1505_02100_b200 import distributed as D
    from paper_1505_02100_b200 import inputs
    from paper_1505_02100_b200 import plugin as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    xh = inputs.config_data(a.config)
    n = xh.size
    x = torch.from_numpy(xh).to(dev)
    ws = P.workspace(n, dev)
    out = P.new_result(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    pairs_pass = n * (n - 1) // 2

    def step(events=None):
        return D.plugin_h_distributed(x, out=out, ws=ws, events=events)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    kev = [{f"psi{r}": (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for r in (6, 4)}
           for _ in range(a.steps)]
    clk = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clk.start()
    time.sleep(0.3)
    wall0 = time.perf_counter()
    for s in range(a.steps):
        flush.fill_(s & 0xff)                      # L2 flush, outside the events
        ev[s][0].record(stream)
        step(kev[s])
        ev[s][1].record(stream)
    torch.cuda.synchronize(dev)
    wall = time.perf_counter() - wall0
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    k6 = [k["psi6"][0].elapsed_time(k["psi6"][1]) for k in kev]
    k4 = [k["psi4"][0].elapsed_time(k["psi4"][1]) for k in kev]
    t = torch.tensor([sum(step_ms), sum(k6), sum(k4)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tot_ms, k6_ms, k4_ms = t.tolist()
    res = P.read_result(out)

    # end to end through the public API with host buffers (H2D of X and D2H of the result inside)
    e2e = None
    if world > 1:
        # every rank: pinned X -> device, the distributed step, result -> host; max over ranks
        xpin = torch.from_numpy(xh).pin_memory()
        ts = []
        for _ in range(max(3, min(a.steps, 10))):
            flush.fill_(1)
            torch.cuda.synchronize(dev)
            dist.barrier()
            t0 = time.perf_counter()
            x.copy_(xpin, non_blocking=True)
            P.read_result(D.plugin_h_distributed(x, out=out, ws=ws))
            ts.append(time.perf_counter() - t0)
        tm = torch.tensor([statistics.median(ts)], dtype=torch.float64, device=dev)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        e2e = {"value": 2 * pairs_pass / tm.item() / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": 4 * n * world, "d2h_bytes_per_step": P.RESULT_BYTES * world,
               "seconds_per_step": tm.item(), "api": "distributed.plugin_h_distributed (per rank: H2D of X, "
                                                     "D2H of the result; max over ranks)"}
    if world == 1:
        xpin = torch.from_numpy(xh).pin_memory()
        wsh = P.workspace(n, dev, host=True)
        P.plugin_h_host(xpin, wsh)
        torch.cuda.synchronize(dev)
        ts = []
        for _ in range(max(3, min(a.steps, 10))):
            flush.fill_(1)
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            P.plugin_h_host(xpin, wsh)
            ts.append(time.perf_counter() - t0)
        e2e = {"value": 2 * pairs_pass / statistics.median(ts) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": P.RESULT_BYTES,
               "seconds_per_step": statistics.median(ts), "api": "plugin_h_host (C ABI)"}

    if rank == 0:
        ms = tot_ms / a.steps
        value = 2 * pairs_pass / (ms / 1e3) / 1e9
        # roofline of the dominant kernel: the psi pass (MUFU.EX2-bound, 1 ex2 per pair)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        f_meas = clocks.get("sm_mhz") or 1965.0
        peak = MUFU_EX2_PER_CLK_PER_SM * sms * f_meas * 1e6 / 1e9          # GPairs/s per GPU
        per_launch_pairs = pairs_pass / world
        k_ms = (k6_ms + k4_ms) / (2 * a.steps)
        achieved = per_launch_pairs / (k_ms / 1e3) / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": _workload(a.config, n), "n": n, "pairs_per_step": 2 * pairs_pass,
                       "l2": "flushed between steps (256 MiB write, outside the events); X (4n bytes) is L2/smem-"
                             "resident within a step by design",
                       "parallelism": f"tile-triangle shards x{world}, 1 NCCL allreduce (32 B) per pass"
                       if world > 1 else "single GPU"},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": UNIT, "frac": achieved / peak,
                         "traffic": _traffic(n), "kernel": "psi_kernel (r=6 and r=4 pass average)",
                         "peak_basis": f"{MUFU_EX2_PER_CLK_PER_SM} MUFU.EX2/clk/SM x {sms} SMs x measured median "
                                       f"SM clock {f_meas:.0f} MHz (1 ex2 per pair)",
                         "frac_at_1965MHz": achieved / (MUFU_EX2_PER_CLK_PER_SM * sms * 1.965),
                         # the same against the dual-pipe bound (some exps on the FMA pipe, both pipes
                         # saturated): 17.07 (psi6) / 18.29 (psi4) pairs/clk/SM; the passes evaluate all
                         # exps on MUFU, so this is the headroom a hybrid exp could take
                         "frac_dual_pipe": achieved / (2.0 / (1.0 / dual_pipe_bound(7) + 1.0 / dual_pipe_bound(6))
                                                       * sms * f_meas * 1e6 / 1e9),
                         "dual_pipe_pairs_per_clk_per_sm": {"psi6": dual_pipe_bound(7), "psi4": dual_pipe_bound(6)}},
            "passes": {"psi6_gpairs_s": per_launch_pairs * world / (k6_ms / a.steps / 1e3) / 1e9,
                       "psi4_gpairs_s": per_launch_pairs * world / (k4_ms / a.steps / 1e3) / 1e9,
                       "psi6_ms": k6_ms / a.steps, "psi4_ms": k4_ms / a.steps},
            "h_ms_device": ms, "h": res["h"], "status": res["status"],
            "clocks": clocks, "gpu_launches": KERNELS_PER_STEP * a.steps, "wall_s": wall,
        }
        if e2e:
            line["e2e"] = e2e
        if not a.no_cpu_baseline and world == 1:
            cb = cpu_oracle_sample(a.config, a.cpu_seconds)
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            # also one thread, and the CPU model
            cb1 = cpu_oracle_sample(a.config, min(3.0, a.cpu_seconds / 4), threads=1)
            cpu_oracle_sample(a.config, 0.05, threads=cb["cores"])  # restore the OpenMP team size
            line["cpu_baseline"]["single_thread_value"] = cb1["value"]
            line["cpu_baseline"]["cpu_model"] = cpu_model()
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


KDE_H = {4: 0.1326215, 5: 0.05}   # fixed bandwidths (cfg4: its PLUGIN h rounded), as tests/test_gpu_kde.py


def _kde_setup(k, m):
    import numpy as np

    from paper_1505_02100_b200 import inputs
    xh = inputs.config_data(k)
    h = KDE_H.get(k, 0.1)
    pts = np.linspace(float(xh.min()) - 4 * h, float(xh.max()) + 4 * h, m).astype(np.float32)
    return xh, h, pts


def kde_terms_visited(xh, h, pts, block=1024):
    """Terms kde_eval evaluates: per block of 1024 points, the sorted samples within the
    fp32 underflow cutoff of the block's [min, max] (the same rule as kde.cu)."""
    import numpy as np
    xs = np.sort(xh.astype(np.float64))
    kf = float(np.float32(-1.4426950408889634 / (2 * h * h)))
    cut = (126.5 / abs(kf)) ** 0.5 * (1 + 1e-6)
    tot = 0
    for b in range(0, pts.size, block):
        p = pts[b:b + block].astype(np.float64)
        lo = np.searchsorted(xs, p.min() - cut, "left")
        hi = np.searchsorted(xs, p.max() + cut, "right")
        tot += int(p.size) * max(0, int(hi - lo))
    return int(tot)


def run_kde(a):
    """Eq. 1-2 (NEXT 1): f(x_k, h) at a sorted 65536-point curve over BASELINE config k."""
    import torch

    from paper_1505_02100_b200 import plugin as P
    xh, h, pts = _kde_setup(a.config, a.kde_points)
    n, m = xh.size, pts.size
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    x = torch.from_numpy(xh).to(dev)
    p = torch.from_numpy(pts).to(dev)
    ws = P.kde_workspace(n, m, dev)
    f = torch.empty(m, dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(a.warmup):
        P.kde_eval(x, h, p, out=f, ws=ws)
    torch.cuda.synchronize(dev)
    def evs():
        return [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev = [evs() for _ in range(a.steps)]
    clk = ClockSampler(0)
    clk.start()
    time.sleep(0.3)
    for s in range(a.steps):
        flush.fill_(s & 0xff)
        ev[s][0].record(stream)
        P.kde_prepare(x, ws)                                   # = kde_eval, split so the
        ev[s][1].record(stream)                                #   kernel can be timed alone
        P.kde_eval_prepared(n, h, p, ws, out=f)
        ev[s][2].record(stream)
    torch.cuda.synchronize(dev)
    clocks = clk.stop()
    ms = statistics.median([e[0].elapsed_time(e[2]) for e in ev])
    k_ms = statistics.median([e[1].elapsed_time(e[2]) for e in ev])
    visited = kde_terms_visited(xh, h, pts)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    f_meas = clocks.get("sm_mhz") or 1965.0
    mufu_only = os.environ.get("PLUGIN_KDE_MUFU_ONLY") == "1"
    # MUFU-only: 16 ex2/clk/SM.  Hybrid (default, centred terms of 3 FP32 lane-ops):
    # 12 of 16 terms on MUFU, 4 of 16 with an 8-lane-op FMA-pipe exp2:
    # min(16 / (12/16), 128 / (3 + 8 * 4/16)) = 21.33 terms/clk/SM (MUFU-bound)
    per_clk = MUFU_EX2_PER_CLK_PER_SM if mufu_only else 16.0 / (12.0 / 16.0)
    peak = per_clk * sms * f_meas * 1e6 / 1e9
    achieved = visited / (k_ms / 1e3) / 1e9
    # end to end from host memory: H2D of X and the points, D2H of the curve
    xpin, ppin = torch.from_numpy(xh).pin_memory(), torch.from_numpy(pts).pin_memory()
    fh = torch.empty(m, dtype=torch.float64).pin_memory()
    ts = []
    for _ in range(max(3, min(a.steps, 10))):
        flush.fill_(1)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        x.copy_(xpin, non_blocking=True)
        p.copy_(ppin, non_blocking=True)
        P.kde_eval(x, h, p, out=f, ws=ws)
        fh.copy_(f, non_blocking=True)
        torch.cuda.synchronize(dev)
        ts.append(time.perf_counter() - t0)
    line = {"metric": "KDE terms/sec (Eq. 1-2, effective n*m)", "value": n * m / (ms / 1e3) / 1e9,
            "unit": "GTerms/s", "n_gpus": 1, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"kde: cfg{a.config} n={n}, h={h}, {m} sorted points over [min-4h, max+4h]",
                       "terms_visited": visited, "terms_effective": n * m,
                       "l2": "flushed between steps (256 MiB write, outside the events)"},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "GTerms/s",
                         "frac": achieved / peak,
                         "traffic": None if mufu_only else _traffic(n, "kde_traffic.json", m),
                         "kernel": "kde_kernel",
                         "kernel_ms": k_ms, "prepare_ms": ms - k_ms,
                         "peak_basis": (f"{per_clk:.2f} terms/clk/SM x {sms} SMs x {f_meas:.0f} MHz ("
                                        + ("MUFU.EX2-bound, 1 ex2 per visited term" if mufu_only else
                                           "12/16 of the exps on MUFU.EX2 (the binding pipe), 4/16 on the FMA "
                                           "pipe, centred terms") + ")"),
                         "variant": "mufu_only" if mufu_only else "hybrid",
                         # the LP optimum of the centred 3-op term (5/16 FMA-pipe exps, both pipes saturated)
                         "frac_dual_pipe": achieved / (dual_pipe_bound(3) * sms * f_meas * 1e6 / 1e9),
                         "dual_pipe_terms_per_clk_per_sm": dual_pipe_bound(3)},
            "e2e": {"value": n * m / statistics.median(ts) / 1e9, "unit": "GTerms/s",
                    "h2d_bytes_per_step": 4 * (n + m), "d2h_bytes_per_step": 8 * m,
                    "seconds_per_step": statistics.median(ts)},
            "clocks": clocks, "gpu_launches": 14 * a.steps}
    print(json.dumps(line), flush=True)
    return 0


def run_variant(a):
    """1 GPU, one step = plugin_h_q32 (q32) or plugin_dpi(l) (dpi) on config k; pair rate over the
    unique pairs of all passes of the step."""
    import torch

    from paper_1505_02100_b200 import inputs
    from paper_1505_02100_b200 import plugin as P
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    xh = inputs.config_data(a.config)
    n = xh.size
    x = torch.from_numpy(xh).to(dev)
    if a.workload == "q32":
        out = P.new_result(dev)
        ws = torch.empty(P.lib().plugin_q32_workspace_bytes(n) + 256, dtype=torch.uint8, device=dev)
        ws = ws[(-ws.data_ptr()) % 256:][:P.lib().plugin_q32_workspace_bytes(n)]
        step = lambda: P.plugin_h_q32(x, out=out, ws=ws)  # noqa: E731
        passes, launches = 2, 21    # 12 radix sort, Step I, 2 group, encode, rg1, 2 x (pass, finalize)
    else:
        out = torch.empty(P.DPI_RESULT_BYTES, dtype=torch.uint8, device=dev)
        ws = P.workspace(n, dev)
        step = lambda: P.plugin_dpi(x, a.stages, out=out, ws=ws)  # noqa: E731
        passes, launches = a.stages, 16 + 3 * a.stages  # 12 radix sort, Step I, 2 group, init, l x (pass, group pass, finalize)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    clk = ClockSampler(0)
    clk.start()
    time.sleep(0.3)
    for s in range(a.steps):
        flush.fill_(s & 0xff)
        ev[s][0].record(stream)
        step()
        ev[s][1].record(stream)
    torch.cuda.synchronize(dev)
    clocks = clk.stop()
    ms = statistics.median([e0.elapsed_time(e1) for e0, e1 in ev])
    pairs = passes * n * (n - 1) // 2
    res = P.read_result(out) if a.workload == "q32" else P.read_dpi_result(out)
    what = ("Alg. 1 with both pair passes in Q32.32 fixed point (plugin_h_q32)" if a.workload == "q32"
            else f"{a.stages}-stage direct plug-in (plugin_dpi), passes r = {2 * a.stages + 2}..4")
    line = {"metric": f"pair evaluations/sec, {a.workload} variant", "value": pairs / (ms / 1e3) / 1e9,
            "unit": UNIT, "n_gpus": 1, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "q32.32 (int64)" if a.workload == "q32" else "f32", "data": "synthetic",
            "config": {"workload": f"cfg{a.config} n={n}: {what}", "pairs_per_step": pairs},
            "h": res["h"], "status": res["status"], "clocks": clocks, "gpu_launches": launches * a.steps}
    if a.workload == "dpi":
        # per pass r: min(16 MUFU.EX2, 128 / (4 + r/2) FP32 lane-ops) pairs/clk/SM (centred form:
        # u, t, a, r/2 Horner steps in t, the accumulate); the step's bound is their harmonic mix
        rs = [2 * j + 2 for j in range(a.stages, 0, -1)]
        per_clk = len(rs) / sum(1.0 / min(16.0, 128.0 / (4 + r // 2)) for r in rs)
        mhz = clocks.get("sm_mhz") or 1965.0
        peak = per_clk * 148 * mhz * 1e6 / 1e9
        line["roofline"] = {"bound": "alu", "achieved": line["value"], "peak": peak, "unit": UNIT,
                            "frac": line["value"] / peak, "traffic": None,
                            "kernel": "whole step (sort, Step I, the l pair passes)",
                            "peak_basis": f"{per_clk:.2f} pairs/clk/SM (passes r = {rs}: min(16 MUFU, 128/(4 + r/2) FMA))"
                                          f" x 148 SMs x {mhz:.0f} MHz"}
    if a.workload == "q32":
        # in-range pairs (|u| <= 7: the long path of q32_term; the others leave after two multiplies)
        # counted on the host from the z-scores, at the ALU-pipe bound of an in-range pair
        import numpy as np
        z = np.sort((xh.astype(np.float64) - res["mean"]) / res["sigma"])
        inrange = 0
        for gz in (res["g1_z"], res["g2_z"]):
            inrange += int((np.searchsorted(z, z + 7.0 * gz, side="right") - np.arange(z.size) - 1).sum())
        mhz = clocks.get("sm_mhz") or 1965.0
        per_clk = ALU_LANES_PER_CLK_PER_SM / Q32_ALU_INST_PER_PAIR
        peak = per_clk * 148 * mhz * 1e6 / 1e9
        achieved = inrange / (ms / 1e3) / 1e9
        line["roofline"] = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "GPairs/s (in-range)",
                            "frac": achieved / peak, "traffic": None,
                            "kernel": "whole step (sort, Step I, encode, the two Q32.32 passes)",
                            "in_range_pairs": inrange, "pairs": pairs,
                            "peak_basis": f"{per_clk:.3f} in-range pairs/clk/SM = {ALU_LANES_PER_CLK_PER_SM} ALU "
                                          f"lanes/clk/SM / {Q32_ALU_INST_PER_PAIR:.0f} ALU-pipe instructions per "
                                          f"in-range pair (ncu) x 148 SMs x {mhz:.0f} MHz"}
    print(json.dumps(line), flush=True)
    return 0


def run_batch(a):
    """plugin_h_batch over a.batch independent N(0,1) samples of n = 1024 (the paper's largest
    size, Table 2): whole-algorithm throughput for many small problems, one CTA per sample."""
    import numpy as np
    import torch

    from paper_1505_02100_b200 import plugin as P
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    n, count = 1024, a.batch
    xh = np.random.default_rng(123).standard_normal(n * count).astype(np.float32)
    x = torch.from_numpy(xh).to(dev)
    offs = torch.arange(0, n * (count + 1), n, dtype=torch.int64, device=dev)
    out = torch.empty(count * P.RESULT_BYTES, dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(a.warmup):
        P.plugin_h_batch(x, offs, out=out)
    torch.cuda.synchronize(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    clk = ClockSampler(0)
    clk.start()
    time.sleep(0.3)
    for s in range(a.steps):
        flush.fill_(s & 0xff)
        ev[s][0].record(stream)
        P.plugin_h_batch(x, offs, out=out)
        ev[s][1].record(stream)
    torch.cuda.synchronize(dev)
    clocks = clk.stop()
    ms = statistics.median([e0.elapsed_time(e1) for e0, e1 in ev])
    pairs = count * n * (n - 1)  # both passes, unique pairs
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    f_meas = clocks.get("sm_mhz") or 1965.0
    peak = MUFU_EX2_PER_CLK_PER_SM * sms * f_meas * 1e6 / 1e9
    # the batch kernel's tiles (T = 256, n a multiple of T here): nb (nb - 1) / 2 off-diagonal tiles
    # of T^2 pairs; each diagonal tile evaluates its 64-wide diagonal squares in both orders and the
    # 64-column chunks right of them once (psi_tile_sum<..., DIAG>): 64^2 B (B + 1) / 2, B = T / 64
    T = 256
    nbt = -(-n // T)
    B = T // 64
    evaluated = count * 2 * (nbt * (nbt - 1) // 2 * T * T + nbt * 64 * 64 * B * (B + 1) // 2)
    res = P.read_results(out, 2)
    line = {"metric": "pairwise K4/K6 evaluations/sec, batches of independent samples", "value": pairs / (ms / 1e3) / 1e9,
            "unit": UNIT, "n_gpus": 1, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"plugin_h_batch: {count} samples of n = {n} N(0,1), full PLUGIN each",
                       "us_per_sample": ms * 1e3 / count, "pairs_per_step": pairs},
            "roofline": {"bound": "alu", "achieved": evaluated / (ms / 1e3) / 1e9, "peak": peak, "unit": UNIT,
                         "frac": evaluated / (ms / 1e3) / 1e9 / peak, "traffic": None,
                         "kernel": "plugin_batch_kernel (whole step)",
                         "peak_basis": f"{MUFU_EX2_PER_CLK_PER_SM} MUFU.EX2/clk/SM x {sms} SMs x {f_meas:.0f} MHz"},
            "h_first": res[0]["h"], "status_first": res[0]["status"], "clocks": clocks, "gpu_launches": a.steps}
    print(json.dumps(line), flush=True)
    return 0


def launch_plan(gpus: int, env: dict, device_count: int) -> tuple[str, str]:
    """How the repo arm runs N GPUs: ("run", "") when the process is already one of N ranks
    (or N = 1 without a launcher), ("reexec", "") when N > 1 was asked without torchrun (re-run
    under torch.distributed.run, one rank per GPU), ("error", why) when the request cannot be
    honoured -- never one rank labelled N."""
    ws = env.get("WORLD_SIZE")
    if ws is not None:
        if int(ws) != gpus:
            return "error", f"--gpus {gpus} but WORLD_SIZE={ws}"
        return "run", ""
    if gpus <= 1:
        return "run", ""
    if device_count < gpus:
        return "error", f"--gpus {gpus} needs {gpus} visible CUDA devices, found {device_count}"
    return "reexec", ""


def _reexec_under_torchrun(gpus: int) -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    a = _args()
    if a.impl == "reference":
        return run_reference(a)
    if a.workload != "plugin" or a.skip_underflow:
        if a.gpus != 1 or int(os.environ.get("WORLD_SIZE", "1")) != 1:
            print(f"bench.py: the {a.workload}{' --skip-underflow' if a.skip_underflow else ''} workload runs on "
                  "one GPU only (--gpus 1)", file=sys.stderr)
            return 2
    else:
        import torch
        plan, why = launch_plan(a.gpus, dict(os.environ), torch.cuda.device_count())
        if plan == "error":
            print(f"bench.py: {why}", file=sys.stderr)
            return 2
        if plan == "reexec":
            return _reexec_under_torchrun(a.gpus)
    if a.workload == "kde":
        return run_kde(a)
    if a.workload in ("q32", "dpi"):
        return run_variant(a)
    if a.workload == "batch":
        return run_batch(a)
    if a.skip_underflow:
        return run_skip(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
