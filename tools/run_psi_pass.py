"""One psi_r pass (host bandwidth) at a BASELINE config, for ncu captures of a single pass kernel:
python tools/run_psi_pass.py CONFIG R [G_SCALE]   (g = G_SCALE * the Alg. 1 bandwidth of that pass)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1505_02100_b200 import inputs  # noqa: E402
from paper_1505_02100_b200 import plugin as P  # noqa: E402

k, r = int(sys.argv[1]), int(sys.argv[2])
x = torch.from_numpy(inputs.config_data(k)).cuda()
res = P.plugin_h_sync(x)
g = res["g1"] if r == 6 else res["g2"]
print(P.psi_r(x, g, r).item(), P.read_result(P.plugin_h(x))["h"])
