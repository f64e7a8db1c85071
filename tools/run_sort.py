"""plugin_sort a few times at n (default 16384): the target of ncu captures of the sort kernels."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1505_02100_b200 import inputs  # noqa: E402
from paper_1505_02100_b200 import plugin as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
x = torch.from_numpy(inputs.normal(n, 3)).cuda()
ws = P.workspace(n, x.device)
for _ in range(3):
    y = P.plugin_sort(x, ws)
torch.cuda.synchronize()
print(float(y[0]), float(y[-1]))
