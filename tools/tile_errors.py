"""Per-tile errors of the psi pass on a sample (dev probe): the GPU's exact fixed-point sum of a
tile alone (psi_r_shard with one tile per rank) against the oracle's block sum of the same
pairs, for the diagonal tiles, the first off-diagonals and a random set; one JSON line per tile.
usage: python tools/tile_errors.py CONFIG(4r|1..5) [r] [extra_random]"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_1505_02100_b200 import inputs  # noqa: E402
from paper_1505_02100_b200 import plugin as P  # noqa: E402
from paper_1505_02100_b200.distributed import from_limbs  # noqa: E402


def tile_coords(t, nb):
    lo, hi = 0, nb - 1
    while lo < hi:
        mid = (lo + hi + 1) // 2
        if mid * nb - mid * (mid - 1) // 2 <= t:
            lo = mid
        else:
            hi = mid - 1
    return lo, lo + (t - (lo * nb - lo * (lo - 1) // 2))


def main():
    name = sys.argv[1]
    r = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    extra = int(sys.argv[3]) if len(sys.argv) > 3 else 200
    g_all = json.load(open(os.path.join(ROOT, "tests", "golden", f"cfg{name}.json")))
    x = inputs.rounded_data(name) if name in inputs.ROUNDED else inputs.config_data(int(name))
    n = x.size
    g = g_all["g1"] if r == 6 else g_all["g2"]
    xd = torch.from_numpy(x).cuda()
    ws = P.workspace(n)
    P.plugin_step1(xd, P.new_result(), ws)
    res = P.plugin_result()
    res.status, res.n, res.g1, res.g2 = 0, n, g, g
    dres = torch.frombuffer(bytearray(bytes(res)), dtype=torch.uint8).cuda()
    zs = np.sort(oracle.widen(x))
    ntiles, T = P.plugin_num_tiles(n, r), P.plugin_tile_edge(n, r)
    nb = -(-n // T)
    off = lambda b: b * nb - b * (b - 1) // 2  # noqa: E731
    picks = set(off(b) for b in range(nb)) | set(off(b) + 1 for b in range(nb - 1))
    picks |= set(np.random.default_rng(0).integers(0, ntiles, extra).tolist())
    phi0 = 1 / math.sqrt(2 * math.pi)
    for t in sorted(picks):
        part = P.new_partial()
        P.psi_r_shard(n, r, t, ntiles, dres, part, ws)
        got = from_limbs(part.cpu().tolist()) / 2.0 ** 64 * phi0
        bi, bj = tile_coords(t, nb)
        rows, cols = (bi * T, min(n, bi * T + T)), (bj * T, min(n, bj * T + T))
        w = 1.0 if bi == bj else 2.0
        ref = w * oracle.psi_block_sum(zs, g, r, *rows, *cols)
        print(json.dumps({"t": t, "bi": bi, "bj": bj, "x_rows": [float(zs[rows[0]]), float(zs[rows[1] - 1])],
                          "x_cols": [float(zs[cols[0]]), float(zs[cols[1] - 1])], "got": got, "ref": ref,
                          "err": got - ref}), flush=True)


if __name__ == "__main__":
    main()
