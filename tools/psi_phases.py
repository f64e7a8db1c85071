"""Phase times of the psi pass kernel per CTA, from a -DPSI_TIMING build (PLUGIN_LIB_PATH):
%globaltimer at kernel entry, after the first tile-index atomic, after the first tile's staging,
after its sum, at loop exit and at the end; the CTA's SM and tile count.  Prints one JSON line per
n with percentiles (us, relative to the earliest CTA entry) and per-SM tile counts.
usage: PLUGIN_LIB_PATH=.../libplugin_ptime.so python tools/psi_phases.py 4096 16384 ..."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1505_02100_b200 import inputs  # noqa: E402
from paper_1505_02100_b200 import plugin as P  # noqa: E402


def pct(a):
    a = np.asarray(a, dtype=np.float64)
    return {"min": round(float(a.min()), 3), "p50": round(float(np.median(a)), 3), "max": round(float(a.max()), 3)}


def main():
    L = P.lib()
    f = L.plugin_debug_psi_timing
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_void_p, ctypes.c_int]
    for n in map(int, sys.argv[1:]):
        x = torch.from_numpy(inputs.normal(n, 7)).cuda()
        ws = P.workspace(n, x.device)
        out = P.new_result(x.device)
        P.plugin_step1(x, out, ws)
        part = P.new_partial(x.device)
        for r in (6, 4):
            for _ in range(5):
                P.psi_r_shard(n, r, 0, 1, out, part, ws)
            torch.cuda.synchronize()
            buf = np.zeros(4096 * 8, dtype=np.uint64)
            assert f(buf.ctypes.data, 4096) == 0
            # the CTAs of this launch: entry time set and within 1 ms of the latest entry
            t = buf.reshape(-1, 8).astype(np.int64)
            live = t[t[:, 0] > 0]
            live = live[live[:, 0] > live[:, 0].max() - 1_000_000]
            t0 = live[:, 0].min()
            us = (live[:, :6] - t0) / 1e3
            work = live[live[:, 7] > 0]
            wus = (work[:, :6] - t0) / 1e3
            per_sm = np.bincount(live[:, 6].astype(np.int64), weights=live[:, 7], minlength=148)
            ctas_sm = np.bincount(live[:, 6].astype(np.int64), minlength=148)
            row = {
                "n": n, "r": r, "ctas": int(len(live)), "tiles": int(live[:, 7].sum()),
                "entry": pct(us[:, 0]),
                "atomic": pct(wus[:, 1] - wus[:, 0]),
                "setup": pct(wus[:, 2] - wus[:, 1]),
                "tile": pct(wus[:, 3] - wus[:, 2]),
                "exit": pct(us[:, 4]),
                "end": pct(us[:, 5]),
                "tiles_per_sm": {str(k): int(v) for k, v in zip(*np.unique(per_sm[:148], return_counts=True))},
                "ctas_per_sm": {str(k): int(v) for k, v in zip(*np.unique(ctas_sm[:148], return_counts=True))},
            }
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
