"""Device time of the preparation kernels from CUDA-graph replays (no host overhead): plugin_sort
alone and plugin_step1 (memset + sort + Step I-III, + the distinct count from n = 32768), and the
sort's exactness.  usage: python tools/prep_time.py 2048 4096 16384 ... > out.jsonl
(PLUGIN_LIB_PATH selects an A/B variant)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1505_02100_b200 import inputs  # noqa: E402
from paper_1505_02100_b200 import plugin as P  # noqa: E402
from psi_graph_time import graph_us  # noqa: E402

for n in map(int, sys.argv[1:]):
    xh = inputs.normal(n, 3)
    x = torch.from_numpy(xh).cuda()
    ws = P.workspace(n, x.device)
    out = P.new_result(x.device)
    y = P.plugin_sort(x, ws)
    torch.cuda.synchronize()
    ok = bool(np.array_equal(y.cpu().numpy(), np.sort(xh)))
    row = {"n": n, "lib": os.path.basename(P.LIB_PATH), "exact": ok,
           "sort_us": round(graph_us(lambda: P.plugin_sort(x, ws), reps=10), 2),
           "step1_sort_us": round(graph_us(lambda: P.plugin_step1(x, out, ws), reps=10), 2)}
    print(json.dumps(row), flush=True)
