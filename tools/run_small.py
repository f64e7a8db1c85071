"""A few plugin_h calls at a small n (default cfg1, n = 1024), for ncu captures of the fused path."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1505_02100_b200 import inputs  # noqa: E402
from paper_1505_02100_b200 import plugin as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
x = torch.from_numpy(inputs.config_data(1) if n == 1024 else inputs.normal(n, 7)).cuda()
ws = P.workspace(n, x.device)
out = P.new_result(x.device)
for _ in range(5):
    P.plugin_h(x, out=out, ws=ws)
print(P.read_result(out)["h"])
