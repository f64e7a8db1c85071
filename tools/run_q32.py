"""psi_r_q32 on a sample whose pairs are all in range of the Q32.32 exp (|u| <= 7: the long path
of q32_term), for ncu: the instruction mix per in-range pair behind bench.py's q32 roofline.
usage: python tools/run_q32.py [n] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1505_02100_b200 import inputs  # noqa: E402
from paper_1505_02100_b200 import plugin as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
z = np.clip(inputs.normal(n, 9).astype(np.float64), -3.4, 3.4)  # |z_i - z_j| <= 6.8: u = |d| / 1 <= 7
zq = np.round(z * 2.0 ** 32).astype(np.int64)
zt = torch.from_numpy(zq).cuda()
for _ in range(reps):
    tot = P.psi_r_q32(zt, 1 << 32, 6)   # rg = 1: g_z = 1
print(n, tot)
