"""One small call of every compute entry point of libplugin.so, for compute-sanitizer
(memcheck / racecheck / synccheck).  usage: compute-sanitizer --tool memcheck python tools/sanitize_smoke.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1505_02100_b200 import inputs  # noqa: E402
from paper_1505_02100_b200 import plugin as P  # noqa: E402


def main():
    small = torch.from_numpy(inputs.mixture(1000, 1)).cuda()      # fused single-launch path
    mid = torch.from_numpy(inputs.mixture(9000, 2)).cuda()        # multi-kernel path, ragged tiles
    r1 = P.read_result(P.plugin_h(small))
    r2 = P.read_result(P.plugin_h(small, flags=P.PLUGIN_MULTI_KERNEL | P.PLUGIN_SKIP_UNDERFLOW))
    r3 = P.read_result(P.plugin_h(mid, flags=P.PLUGIN_SKIP_UNDERFLOW))
    r4 = P.plugin_h_sync(mid)
    psi = [P.psi_r(mid, 0.3, r).item() for r in (4, 6, 8)]
    d = P.read_dpi_result(P.plugin_dpi(mid, 3))
    f = P.kde_eval(mid, 0.2, torch.linspace(-8, 8, 3000, device="cuda")).cpu()
    ws = P.workspace(mid.numel())
    out = P.new_result()
    P.plugin_step1(mid, out, ws)
    part = P.new_partial()
    P.psi_r_shard(mid.numel(), 6, 1, 3, out, part, ws)
    P.plugin_after_psi6(part, out)
    torch.cuda.synchronize()
    print("ok", r1["h"], r2["h"], r3["h"], r4["h"], psi, d["h"], float(f.sum()))


if __name__ == "__main__":
    main()
