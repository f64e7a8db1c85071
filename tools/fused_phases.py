"""Phase times of the fused single-launch path (a -DPLUGIN_FUSED_TIMING build, loaded through
PLUGIN_LIB_PATH): sort (ranks + cluster barrier), Step I-III, each pass, each partial exchange (DSMEM + cluster barrier), each finalize, for CTA 0.
usage: PLUGIN_LIB_PATH=.../libplugin_ftime.so python tools/fused_phases.py [n ...]"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1505_02100_b200 import inputs  # noqa: E402
from paper_1505_02100_b200 import plugin as P  # noqa: E402

NAMES = ["load_tables", "slice_keys", "rank_sync_reload", "step1_red", "step1_fin", "pass6", "bsum6", "sync6", "final6", "pass4", "bsum4", "sync4", "final4"]


def main():
    for n in [int(a) for a in sys.argv[1:]] or [128, 512, 1024, 2048]:
        x = torch.from_numpy(inputs.normal(n, 7)).cuda()
        ws = P.workspace(n, x.device)
        # the timing slots follow the 2 * 1024 Fx128 partials of the fused region (abi.cu layout:
        # ctrl | step1 partials | xs | tmp | radix histograms | result | fused | group arrays)
        def up(v):
            return (v + 255) // 256 * 256
        off = up(512) + up(16 * 592) + 2 * up(4 * max(n, 1)) + up(4 * 256 * max(1, -(-n // 2048))) + up(P.RESULT_BYTES)
        acc = {k: [] for k in NAMES}
        for it in range(30):
            P.plugin_h(x, ws=ws)
            torch.cuda.synchronize()
            t = ws[off + 2 * 1024 * 16: off + 2 * 1024 * 16 + 8 * (len(NAMES) + 1)].clone().view(torch.int64).cpu().tolist()
            if it >= 5:
                for i, k in enumerate(NAMES):
                    acc[k].append((t[i + 1] - t[i]) / 1e3)
        print(json.dumps({"n": n, "us": {k: statistics.median(v) for k, v in acc.items()},
                          "total_us": sum(statistics.median(v) for v in acc.values())}), flush=True)


if __name__ == "__main__":
    main()
