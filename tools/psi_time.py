"""Device time of the psi passes alone (psi_r_shard over all work items + its export kernel;
CUDA events around 10 back-to-back calls, so the host-side call overhead overlaps; median of 20)
at sizes n, N(0,1) samples, the bandwidths of Algorithm 1:
python tools/psi_time.py 4096 16384 50000 ...   (PLUGIN_PSI_R / PLUGIN_PSI_WARP select tiles)"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1505_02100_b200 import inputs  # noqa: E402
from paper_1505_02100_b200 import plugin as P  # noqa: E402


def main():
    for n in map(int, sys.argv[1:]):
        x = torch.from_numpy(inputs.normal(n, 7)).cuda()
        ws = P.workspace(n, x.device)
        out = P.new_result(x.device)
        P.plugin_step1(x, out, ws)
        row = {"n": n, "units6": P.plugin_num_tiles(n, 6), "T6": P.plugin_tile_edge(n, 6), "T4": P.plugin_tile_edge(n, 4),
               "R_env": os.environ.get("PLUGIN_PSI_R", "")}
        for r in (6, 4):
            ts = []
            part = P.new_partial(x.device)
            reps = 10 if n < 200000 else 1
            for it in range(23):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    P.psi_r_shard(n, r, 0, 1, out, part, ws)
                e1.record()
                torch.cuda.synchronize()
                if it >= 3:
                    ts.append(e0.elapsed_time(e1) * 1e3 / reps)
            (P.plugin_after_psi6 if r == 6 else P.plugin_after_psi4)(part, out)
            med = statistics.median(ts)
            row[f"psi{r}_us"] = round(med, 2)
            row[f"psi{r}_gpairs_s"] = round(n * (n - 1) / 2 / med / 1e3, 1)
        row["h"] = P.read_result(out)["h"]
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
