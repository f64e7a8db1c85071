"""Run plugin_h on one BASELINE config a few times (for ncu launch lists).
usage: python tools/run_cfg.py K [REPS]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1505_02100_b200 import inputs  # noqa: E402
from paper_1505_02100_b200 import plugin as P  # noqa: E402

k = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
x = torch.from_numpy(inputs.config_data(k)).cuda()
ws = P.workspace(x.numel(), x.device)
out = P.new_result(x.device)
for _ in range(reps):
    P.plugin_h(x, out=out, ws=ws)
torch.cuda.synchronize()
print(P.read_result(out)["h"])
