"""Relative errors of the GPU path against the oracle's golden values for the BASELINE configs
(tests/golden/cfg*.json, written by oracle.make_golden), one JSON line per config; the
evidence behind BASELINE.md §4's error column.  usage: python tools/parity_report.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1505_02100_b200 import inputs  # noqa: E402
from paper_1505_02100_b200 import plugin as P  # noqa: E402

KEYS = ("sigma", "g1", "psi6", "g2", "psi4", "h", "psi6_z", "psi4_z", "h_z")


def main():
    for k in (1, 2, 3, 4, 5):
        path = os.path.join(ROOT, "tests", "golden", f"cfg{k}.json")
        if not os.path.exists(path):
            print(json.dumps({"config": k, "golden": "missing"}), flush=True)
            continue
        g = json.load(open(path))
        x = inputs.config_data(k)
        assert inputs.sha256_f32(x) == g["sha256"]
        r = P.plugin_h_sync(torch.from_numpy(x).cuda())
        row = {"config": k, "n": int(x.size), "status": r["status"],
               "rel_err": {key: (r[key] - g[key]) / abs(g[key]) for key in KEYS},
               "gpu": {key: r[key] for key in KEYS}, "oracle": {key: g[key] for key in KEYS}}
        row["max_abs_rel_err_psi6_psi4_h"] = max(abs(row["rel_err"][q]) for q in ("psi6", "psi4", "h"))
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
