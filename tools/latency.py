"""End-to-end latency of one PLUGIN run (Alg. 1, X resident -> h) at the paper's sizes.

Table 2 of the paper times the full algorithm for n = 128..1024 on unpublished
data; SURVEY §8(d) proposes N(0,1) samples with seeds 100..107 as the stand-in.  Also BASELINE
configs 1-3.  For each n: device time per call (CUDA events around back-to-back calls on one
stream, median), for the default path (one cluster launch when n <= 2048) and the forced
multi-kernel path, the multi-kernel path replayed from a CUDA graph, and the host-visible time
of plugin_h_host (H2D of X, the run, D2H of the result, synchronise).
usage: python tools/latency.py [--reps 200] > gpurun_out/latency.json
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1505_02100_b200 import inputs  # noqa: E402
from paper_1505_02100_b200 import plugin as P  # noqa: E402


def dev_time(fn, reps):
    st = torch.cuda.current_stream()
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts), min(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=200)
    a = ap.parse_args()
    cases = [(f"paper n={n} N(0,1) seed {100 + k}", inputs.normal(n, 100 + k)) for k, n in
             enumerate(range(128, 1025, 128))]
    cases += [(f"n={n} N(0,1) seed 7", inputs.normal(n, 7)) for n in (2048, 4096, 8192)]
    cases += [(f"cfg{k}", inputs.config_data(k)) for k in (1, 2, 3)]
    rows = []
    for name, xh in cases:
        n = xh.size
        x = torch.from_numpy(xh).cuda()
        ws = P.workspace(n, x.device)
        out = P.new_result(x.device)
        row = {"case": name, "n": n, "pairs_per_run": n * (n - 1)}
        med, mn = dev_time(lambda: P.plugin_h(x, out=out, ws=ws), a.reps)
        row["default_us"], row["default_min_us"] = med, mn
        h_default = P.read_result(out)["h"]
        med, mn = dev_time(lambda: P.plugin_h(x, out=out, ws=ws, flags=P.PLUGIN_MULTI_KERNEL), a.reps)
        row["multi_kernel_us"], row["multi_kernel_min_us"] = med, mn
        # CUDA graph of the multi-kernel sequence (capturable: no allocation, no sync inside)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            P.plugin_h(x, out=out, ws=ws, flags=P.PLUGIN_MULTI_KERNEL)
        torch.cuda.current_stream().wait_stream(s)
        with torch.cuda.graph(g):
            P.plugin_h(x, out=out, ws=ws, flags=P.PLUGIN_MULTI_KERNEL)
        med, mn = dev_time(g.replay, a.reps)
        row["graph_multi_kernel_us"], row["graph_multi_kernel_min_us"] = med, mn
        # the default path (one cluster launch for n <= 2048) captured in a graph too
        try:
            g2 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g2):
                P.plugin_h(x, out=out, ws=ws)
            med, mn = dev_time(g2.replay, a.reps)
            row["graph_default_us"], row["graph_default_min_us"] = med, mn
        except Exception as e:  # report, do not hide: the header claims capturability
            row["graph_default_error"] = repr(e)
        # the library's own graph API (plugin_graph_create / _launch)
        pg = P.PluginGraph(x, out=out, ws=ws)
        med, mn = dev_time(lambda: pg.launch(), a.reps)
        row["plugin_graph_us"], row["plugin_graph_min_us"] = med, mn
        # device time per call with the queue kept full: 50 back-to-back plugin_graph_launch
        # between two events (the host-side call overhead overlaps the previous run)
        med, mn = dev_time(lambda: [pg.launch() for _ in range(50)], max(10, a.reps // 10))
        row["plugin_graph_pipelined_us"], row["plugin_graph_pipelined_min_us"] = med / 50, mn / 50
        med, mn = dev_time(lambda: [P.plugin_h(x, out=out, ws=ws) for _ in range(50)], max(10, a.reps // 10))
        row["default_pipelined_us"], row["default_pipelined_min_us"] = med / 50, mn / 50
        pg.close()
        row["h"] = h_default
        row["same_h_all_paths"] = P.read_result(out)["h"] == h_default
        xpin = torch.from_numpy(xh).pin_memory()
        wsh = P.workspace(n, x.device, host=True)
        for _ in range(10):
            P.plugin_h_host(xpin, wsh)
        ts = []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            P.plugin_h_host(xpin, wsh)
            ts.append((time.perf_counter() - t0) * 1e6)
        row["host_e2e_us"], row["host_e2e_min_us"] = statistics.median(ts), min(ts)
        rows.append(row)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
