"""Write tests/golden/cfg{k}.json: the oracle's Alg. 1 values on BASELINE config k.

Calls only oracle/ (and the seeded input generators).  Long configs checkpoint per
row chunk under tests/golden/checkpoints/ so a run can resume.
usage: python -m oracle.make_golden 1 2 3 [--threads T] [--ckpt-root DIR] [--out-dir DIR]
"""
import argparse
import hashlib
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402
from paper_1505_02100_b200 import inputs  # noqa: E402


def _src_hash():
    h = hashlib.sha256()
    for f in ("plugin_oracle.c", "oracle.py"):
        with open(os.path.join(ROOT, "oracle", f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+", help="BASELINE config numbers 1..5, or a rounded variant of inputs.ROUNDED (e.g. 4r)")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--ckpt-root", default=os.path.join(ROOT, "tests", "golden", "checkpoints"))
    ap.add_argument("--out-dir", default=os.path.join(ROOT, "tests", "golden"))
    a = ap.parse_args()
    for k in a.configs:
        if k in inputs.ROUNDED:
            x = inputs.rounded_data(k)
            sha = inputs.sha256_f32(x)
        else:
            k = int(k)
            x = inputs.config_data(k)
            sha = inputs.sha256_f32(x)
            assert sha == inputs.SHA256[k], f"cfg{k} input hash mismatch"
        ck = os.path.join(a.ckpt_root, f"cfg{k}")
        os.makedirs(ck, exist_ok=True)
        t0 = time.time()
        res = oracle.plugin(x, threads=a.threads, checkpoint_dir=ck, log=lambda m: print(m, flush=True))
        res = {k2: (float(v) if not isinstance(v, (dict, str)) else v) for k2, v in res.items()}
        res.update({"config": k, "sha256": sha, "oracle_src": _src_hash(), "cpu": cpu_model(),
                    "wall_seconds": time.time() - t0,
                    "written_by": "python -m oracle.make_golden (oracle/ only)"})
        os.makedirs(a.out_dir, exist_ok=True)
        out = os.path.join(a.out_dir, f"cfg{k}.json")
        with open(out, "w") as f:
            json.dump(res, f, indent=1, sort_keys=True)
        print(f"cfg{k}: h={res['h']!r} psi6_z={res['psi6_z']!r} psi4_z={res['psi4_z']!r} ({res['wall_seconds']:.1f}s)", flush=True)


if __name__ == "__main__":
    main()
