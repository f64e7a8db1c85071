"""Relative errors of plugin_h against the oracle on discretised / tied samples and a few
continuous ones, one JSON line per sample.  Dev helper (runs under gpurun);
the parity tests proper are tests/test_gpu_parity.py.
usage: python tools/discrete_report.py [name ...]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_1505_02100_b200 import inputs  # noqa: E402
from paper_1505_02100_b200 import plugin as P  # noqa: E402


def grid(n, q, seed):
    return (np.round(np.random.default_rng(seed).standard_normal(n) / q) * q).astype(np.float32)


SAMPLES = {
    "ties": lambda: inputs.ties(12000, 4),
    "ties20": lambda: inputs.ties(20000, 7, levels=20),
    "ties60": lambda: inputs.ties(30000, 11, levels=60),
    "int": lambda: np.round(inputs.normal(20000, 12, sd=5)).astype(np.float32),
    "offset": lambda: inputs.offset(12000, 5),
    "offset3e4": lambda: inputs.offset(20000, 8, base=3.0e4),
    "grid001": lambda: grid(20000, 0.001, 31),
    "grid0003": lambda: grid(20000, 0.0003, 31),
    "grid0001": lambda: grid(20000, 0.0001, 31),
    "mixture": lambda: inputs.mixture(20000, 3),
    "cfg2": lambda: inputs.config_data(2),
}
KEYS = ("psi6_z", "psi4_z", "h", "g2")


def main():
    names = sys.argv[1:] or list(SAMPLES)
    for name in names:
        x = SAMPLES[name]()
        o = oracle.plugin(x)
        r = P.plugin_h_sync(torch.from_numpy(x).cuda())
        row = {"sample": name, "n": int(x.size), "distinct": int(np.unique(x).size), "status": r["status"],
               "rel_err": {k: (r[k] - o[k]) / abs(o[k]) for k in KEYS}}
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
