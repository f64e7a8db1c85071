"""Where the time of one PLUGIN run goes, per step, for BASELINE configs 2-4 (CUDA events around
the multi-GPU building blocks on one GPU: Step I + sort, each pass, each finalize).
usage: python tools/breakdown.py > gpurun_out/breakdown.jsonl"""
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
    for k in (2, 3, 4):
        xh = inputs.config_data(k)
        n = xh.size
        x = torch.from_numpy(xh).cuda()
        ws = P.workspace(n, x.device)
        out = P.new_result(x.device)
        part = P.new_partial(x.device)
        names = ["step1_sort", "psi6", "after6", "psi4", "after4"]
        reps = 20 if k < 4 else 3
        rows = {m: [] for m in names}
        for it in range(reps + 2):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
            ev[0].record()
            P.plugin_step1(x, out, ws)
            ev[1].record()
            P.psi_r_shard(n, 6, 0, 1, out, part, ws)
            ev[2].record()
            P.plugin_after_psi6(part, out)
            ev[3].record()
            P.psi_r_shard(n, 4, 0, 1, out, part, ws)
            ev[4].record()
            P.plugin_after_psi4(part, out)
            ev[5].record()
            torch.cuda.synchronize()
            if it >= 2:
                for i, m in enumerate(names):
                    rows[m].append(ev[i].elapsed_time(ev[i + 1]) * 1e3)
        med = {m: statistics.median(v) for m, v in rows.items()}
        print(json.dumps({"config": k, "n": n, "us": med, "total_us": sum(med.values()),
                          "h": P.read_result(out)["h"]}), flush=True)


if __name__ == "__main__":
    main()
