"""Device time of one psi pass (Steps IV/VI) per n, free of host overhead: 20 psi_r_shard
calls (the pass kernel + its 1-thread export kernel) captured in a CUDA graph and replayed
between two events; the export-only time (an empty shard) is measured the same way and
subtracted.  Also plugin_h (Alg. 1 end to end, X resident) as a graph.  N(0,1) samples,
g of Algorithm 1.  usage: python tools/psi_graph_time.py 4096 16384 ... > out.jsonl
(PLUGIN_PSI_R / PLUGIN_LIB_PATH select A/B variants)"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1505_02100_b200 import inputs  # noqa: E402
from paper_1505_02100_b200 import plugin as P  # noqa: E402

REPS = 20


def graph_us(fn, reps=REPS, trials=15):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    ts = []
    for it in range(trials + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        if it >= 2:
            ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    return statistics.median(ts)


def main():
    for n in map(int, sys.argv[1:]):
        x = torch.from_numpy(inputs.normal(n, 7)).cuda()
        ws = P.workspace(n, x.device)
        out = P.new_result(x.device)
        P.plugin_step1(x, out, ws)
        part = P.new_partial(x.device)
        P.psi_r_shard(n, 6, 0, 1, out, part, ws)
        P.plugin_after_psi6(part, out)
        torch.cuda.synchronize()
        row = {"n": n, "units": P.plugin_num_tiles(n, 6), "R_env": os.environ.get("PLUGIN_PSI_R", ""),
               "lib": os.path.basename(P.LIB_PATH)}
        row["T6"], row["T4"] = P.plugin_tile_edge(n, 6), P.plugin_tile_edge(n, 4)
        # an empty shard (rank 0 of units + 1 ranks owns [0, 0)) runs only the export kernel
        world = P.plugin_num_tiles(n, 6) + 1
        assert P.plugin_shard_tiles(n, 6, 0, world) == (0, 0)
        export = graph_us(lambda: P.psi_r_shard(n, 6, 0, world, out, part, ws))
        row["export_us"] = round(export, 2)
        pairs = n * (n - 1) / 2
        for r in (6, 4):
            t = graph_us(lambda: P.psi_r_shard(n, r, 0, 1, out, part, ws)) - export
            row[f"psi{r}_us"] = round(t, 2)
            row[f"psi{r}_frac"] = round(pairs / (t * 1e-6) / 4.65312e12, 4)  # 16 ex2/clk/SM x 148 x 1965 MHz
        xo = P.new_result(x.device)
        row["plugin_h_us"] = round(graph_us(lambda: P.plugin_h(x, out=xo, ws=ws), reps=5), 2)
        # the preparation alone: sort + Step I (+ the distinct count from n = 32768)
        row["step1_sort_us"] = round(graph_us(lambda: P.plugin_step1(x, xo, ws), reps=10), 2)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
