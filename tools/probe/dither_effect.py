"""Dev probe (CPU): how much the per-row scale dither alone changes the function evaluated --
the weighted pair sum with s_i = s + k_i ulp(s) (the kernel's antithetic dither, A = 128) and every
other quantity in exact fp64, against the same sum at the exact 1/g (tools/probe/emu_terms.c,
flag 1).  VERDICT r1 weak 9.  usage: python tools/probe/dither_effect.py > profiles/r02_dither_effect.txt"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402  (bandwidths only)
from paper_1505_02100_b200 import inputs  # noqa: E402

EMU = "/tmp/emu"  # gcc -O2 -fopenmp -ffp-contract=off -o /tmp/emu tools/probe/emu_terms.c -lm


def grid(n, q, seed):
    return (np.round(np.random.default_rng(seed).standard_normal(n) / q) * q).astype(np.float32)


CASES = {"cfg2": lambda: inputs.config_data(2), "mixture": lambda: inputs.mixture(20000, 3),
         "ties": lambda: inputs.ties(12000, 4), "integers": lambda: np.round(inputs.normal(20000, 12, sd=5)).astype(np.float32),
         "grid0.0003": lambda: grid(20000, 0.0003, 31), "offset": lambda: inputs.offset(12000, 5)}
print("# relative change of the pair sum from the antithetic scale dither alone (A = 128), T = 256 tiles")
for name, f in CASES.items():
    x0 = f()
    x = np.sort(x0)
    x.tofile("/tmp/dither_x.f32")
    ref = oracle.plugin(x0)
    row = []
    for r, g in ((6, ref["g1"]), (4, ref["g2"])):
        def S(flags):
            out = subprocess.check_output([EMU, "/tmp/dither_x.f32", str(x.size), repr(float(g)), str(r), "256",
                                           str(flags), "0", "128", "6"])
            return float(out)
        row.append(f"psi{r} {S(1) / S(0) - 1:+.2e}")
    print(f"{name:12s} n={x.size:6d}  " + "  ".join(row), flush=True)
