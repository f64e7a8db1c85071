"""Command line front end of libplugin.so (the verbs SURVEY §5 keeps from SPEC S:458-462).

  python -m paper_1505_02100_b200 bandwidth FILE [--stages L] [--q32] [--skip-underflow]
  python -m paper_1505_02100_b200 compare FILE --h-ref H [--stages L] [--q32]
  python -m paper_1505_02100_b200 kde FILE --h H --grid LO HI M [--out CURVE.npy]

FILE: a sample as .npy (any real dtype), or raw little-endian float32 (.f32 / .bin), or text
(one number per line).  The sample is converted to float32 and run on cuda:0; the result is
one JSON object on stdout.  `compare` reports |h - h_ref| / |h_ref| against a
reference bandwidth the user supplies.  Everything runs in the CUDA library; there is no CPU path.
"""
from __future__ import annotations

import argparse
import json
import math
import sys

import numpy as np


def _load(path: str) -> np.ndarray:
    if path.endswith(".npy"):
        x = np.load(path)
    elif path.endswith((".f32", ".bin")):
        x = np.fromfile(path, dtype="<f4")
    else:
        x = np.loadtxt(path, ndmin=1)
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64).ravel().astype(np.float32))


def _bandwidth(P, torch, x, stages: int, q32: bool, skip: bool) -> dict:
    xt = torch.from_numpy(x).cuda()
    if q32:
        if stages != 2:
            raise SystemExit("--q32 implements Algorithm 1 (stages = 2) only")
        r = P.read_result(P.plugin_h_q32(xt))
        r["datapath"] = "q32.32"
    elif stages != 2:
        r = P.read_dpi_result(P.plugin_dpi(xt, stages))
        r["datapath"] = "f32 pairs, fp64 sums"
    else:
        r = P.read_result(P.plugin_h(xt, flags=P.PLUGIN_SKIP_UNDERFLOW if skip else 0))
        r["datapath"] = "f32 pairs, fp64 sums"
    r["status_name"] = P.STATUS_NAMES.get(r["status"], str(r["status"]))
    r["stages"] = stages
    return r


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1505_02100_b200")
    sub = ap.add_subparsers(dest="verb", required=True)
    for verb in ("bandwidth", "compare"):
        p = sub.add_parser(verb)
        p.add_argument("file")
        p.add_argument("--stages", type=int, default=2, help="direct plug-in stages (Alg. 1 = 2)")
        p.add_argument("--q32", action="store_true", help="the paper's Q32.32 datapath for the pair sums")
        p.add_argument("--skip-underflow", action="store_true")
        if verb == "compare":
            p.add_argument("--h-ref", type=float, required=True)
    p = sub.add_parser("kde")
    p.add_argument("file")
    p.add_argument("--h", type=float, required=True)
    p.add_argument("--grid", type=float, nargs=3, metavar=("LO", "HI", "M"), required=True)
    p.add_argument("--out", default=None, help="write the curve (float64) as .npy")
    a = ap.parse_args(argv)

    import torch

    from . import plugin as P
    if not torch.cuda.is_available():
        raise SystemExit("no CUDA device: libplugin.so has no CPU path")
    x = _load(a.file)
    if a.verb in ("bandwidth", "compare"):
        r = _bandwidth(P, torch, x, a.stages, a.q32, a.skip_underflow)
        if a.verb == "compare":
            r["h_ref"] = a.h_ref
            r["rel_diff"] = abs(r["h"] - a.h_ref) / abs(a.h_ref) if a.h_ref else math.inf
        print(json.dumps(r, default=float))
        return 0 if r["status"] == P.PLUGIN_OK else 1
    lo, hi, m = a.grid
    pts = torch.linspace(lo, hi, int(m), device="cuda", dtype=torch.float32)
    f = P.kde_eval(torch.from_numpy(x).cuda(), a.h, pts).cpu().numpy()
    if a.out:
        np.save(a.out, f)
    g = pts.cpu().numpy().astype(np.float64)
    mass = float(np.sum((f[1:] + f[:-1]) * np.diff(g)) / 2) if f.size > 1 else float("nan")
    print(json.dumps({"n": int(x.size), "h": a.h, "points": int(m), "trapezoid_mass": mass,
                      "max_density": float(f.max()) if f.size else None, "out": a.out}))
    return 0


if __name__ == "__main__":
    sys.exit(main())
