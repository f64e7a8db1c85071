"""Device time of plugin_sort (CUDA events, median of 20) at sizes n:
python tools/sort_time.py 40000 131072 1048576 4194304"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1505_02100_b200 import inputs  # noqa: E402
from paper_1505_02100_b200 import plugin as P  # noqa: E402

for n in map(int, sys.argv[1:]):
    xh = inputs.normal(n, 3)
    x = torch.from_numpy(xh).cuda()
    ws = P.workspace(n, x.device)
    ts = []
    for it in range(23):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        y = P.plugin_sort(x, ws)
        e1.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    ok = bool(np.array_equal(y.cpu().numpy(), np.sort(xh)))
    print(json.dumps({"n": n, "sort_us": round(statistics.median(ts), 2), "exact": ok}), flush=True)
