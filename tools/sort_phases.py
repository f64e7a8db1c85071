"""Phase times of the preparation kernels (sort_block_kernel, sort_merge_kernel, step1_kernel) from
a -DSORT_TIMING build (PLUGIN_LIB_PATH): %globaltimer marks per CTA, in us relative to the first
block-sort CTA's entry, max over CTAs.  usage: PLUGIN_LIB_PATH=... python tools/sort_phases.py 2048 16384"""
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

NAMES = {0: "blk_entry", 1: "blk_loaded", 2: "blk_warpsort", 3: "blk_runs_stored", 4: "blk_merge256",
         5: "blk_merge512", 6: "blk_merge1024", 7: "blk_end", 8: "mrg_entry", 9: "mrg_filled", 10: "mrg_end",
         11: "last_cta_filled", 12: "last_cta_step1_end"}


def main():
    L = P.lib()
    for f in (L.plugin_debug_sort_timing, L.plugin_debug_step1_timing):
        f.restype = ctypes.c_int
        f.argtypes = [ctypes.c_void_p]
    for n in map(int, sys.argv[1:]):
        x = torch.from_numpy(inputs.normal(n, 3)).cuda()
        ws = P.workspace(n, x.device)
        out = P.new_result(x.device)
        for _ in range(5):
            P.plugin_step1(x, out, ws)
        torch.cuda.synchronize()
        sb = np.zeros(64 * 16, dtype=np.uint64)
        s1 = np.zeros(64 * 4, dtype=np.uint64)
        assert L.plugin_debug_sort_timing(sb.ctypes.data) == 0
        assert L.plugin_debug_step1_timing(s1.ctypes.data) == 0
        sb = sb.reshape(64, 16).astype(np.int64)
        s1 = s1.reshape(64, 4).astype(np.int64)
        nblk = (n + 2047) // 2048
        t0 = sb[:nblk, 0].min()
        row = {"n": n}
        for k, name in NAMES.items():
            rows = sb[:nblk, k] if k < 8 else sb[:, k]
            rows = rows[rows > t0 - 1]
            if len(rows):
                row[name] = round(float((rows.max() - t0) / 1e3), 3)
        s = s1[s1[:, 0] > t0 - 1]
        for k, name in enumerate(("s1_entry", "s1_blocksum", "s1_counter", "s1_end")):
            v = s[:, k]
            v = v[v > 0]
            if len(v):
                row[name] = round(float((v.max() - t0) / 1e3), 3)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
