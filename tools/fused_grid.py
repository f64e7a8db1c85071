"""Device time per plugin_h call at small n (the fused single launch), queue kept full: 50
back-to-back plugin_graph_launch between two events, median of 15 (A/B helper for the grid size,
PLUGIN_FUSED_CLUSTER).  usage: python tools/fused_grid.py > out.jsonl"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1505_02100_b200 import inputs  # noqa: E402
from paper_1505_02100_b200 import plugin as P  # noqa: E402

for n in (128, 256, 512, 1024, 2048):
    x = torch.from_numpy(inputs.normal(n, 100 + n)).cuda()
    pg = P.PluginGraph(x)
    for _ in range(20):
        pg.launch()
    torch.cuda.synchronize()
    ts = []
    for _ in range(15):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            pg.launch()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / 50)
    print(json.dumps({"n": n, "cluster_env": os.environ.get("PLUGIN_FUSED_CLUSTER", ""), "us_per_call": statistics.median(ts),
                      "h": P.read_result(pg.out)["h"]}), flush=True)
    pg.close()
