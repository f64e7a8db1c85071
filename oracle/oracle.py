"""fp64 CPU oracle for the two-stage Gaussian PLUGIN selector (arXiv 1505.02100, Alg. 1).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product package ``paper_1505_02100_b200`` never imports it and
shares no code with it.

Layout: the O(n) / O(n^2) loops are plain C in ``plugin_oracle.c`` (built to
``liboracle.so`` with gcc, ``-fno-fast-math -ffp-contract=off``); every O(1)
scalar step is written below in plain Python floats (IEEE binary64), one
function per step of Algorithm 1, in the paper's notation.

Readings of the paper taken here (listed in DESIGN.md §3):
  R1  K^6, K^4 in Steps III/V are the 6th/4th derivatives of phi (P:93 vs P:101).
  R2  Step V keeps the printed minus sign: g2 = (-2K4(0)/(mu2 psi6 n))^(1/7), psi6 < 0.
  R3  Step I's V is the sample variance; it is evaluated by its definition
      sum (X-mean)^2/(n-1) (two-pass, Neumaier); the printed one-pass form is
      also returned and agrees to rounding on benign data.
  R4  The z-score of Eq. 3 uses Step I's sigma (n-1 denominator), so sigma_z = 1.
  R5  The main path is the paper's z-score path (Fig. 2, Eq. 3-4); a raw-unit
      path (no z-score) is available as a cross-check (Eq. 4 "easily proofed").
"""
from __future__ import annotations

import ctypes
import hashlib
import json
import math
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "plugin_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

# ---- constants of Algorithm 1, as printed --------------------------------------------
PI = math.pi
K6_0 = -15.0 / math.sqrt(2.0 * PI)        # Step III:  K^6(0) = -15/sqrt(2 pi)
K4_0 = 3.0 / math.sqrt(2.0 * PI)          # Step V,  P:113: K^4(0) = 3/sqrt(2 pi)
MU2 = 1.0                                  # mu_2(K) = 1
R_K = 1.0 / (2.0 * math.sqrt(PI))         # Step VII: R(K) = 1/(2 sqrt(pi))


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (OpenMP, strict IEEE fp64)."""
    if not force and os.path.exists(_LIB) and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC):
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    cmd = ["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-shared", "-fPIC",
           "-std=c11", "-o", tmp, _SRC, "-lm"]
    subprocess.check_call(cmd)
    os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        d, i64, i32 = ctypes.c_double, ctypes.c_int64, ctypes.c_int
        P = ctypes.c_void_p
        for name in ("oracle_phi", "oracle_K6", "oracle_K4"):
            getattr(L, name).restype = d
            getattr(L, name).argtypes = [d]
        L.oracle_K.restype = d
        L.oracle_K.argtypes = [i32, d]
        L.oracle_K_hermite.restype = d
        L.oracle_K_hermite.argtypes = [i32, d]
        L.oracle_step1.restype = i32
        L.oracle_step1.argtypes = [P, i64, P]
        L.oracle_zscore.restype = None
        L.oracle_zscore.argtypes = [P, i64, d, d, P]
        L.oracle_widen.restype = None
        L.oracle_widen.argtypes = [P, i64, P]
        L.oracle_psi_rows.restype = None
        L.oracle_psi_rows.argtypes = [P, i64, d, i32, i64, i64, i32, P]
        L.oracle_psi_block.restype = None
        L.oracle_psi_block.argtypes = [P, i64, d, i32, i64, i64, i64, i64, i32, P]
        L.oracle_psi_literal_sum.restype = d
        L.oracle_psi_literal_sum.argtypes = [P, i64, d, i32]
        L.oracle_kde.restype = None
        L.oracle_kde.argtypes = [P, i64, d, P, i64, i32, P]
        L.oracle_q32_mul.restype = i64
        L.oracle_q32_mul.argtypes = [i64, i64]
        L.oracle_q32_exp.restype = i64
        L.oracle_q32_exp.argtypes = [i64]
        L.oracle_q32_term.restype = i64
        L.oracle_q32_term.argtypes = [i64, i64, i32]
        L.oracle_q32_psi_sum.restype = None
        L.oracle_q32_psi_sum.argtypes = [P, i64, i64, i32, i32, P]
        L.oracle_max_threads.restype = i32
        L.oracle_max_threads.argtypes = []
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _f32(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float32))


def K(r: int, u: float) -> float:
    """K^(r)(u): r in {4, 6} as printed in Alg. 1 Steps IV/VI; other even r by Hermite recurrence."""
    return lib().oracle_K(int(r), float(u))


def K_hermite(r: int, u: float) -> float:
    """K^(r)(u) = He_r(u) phi(u) by the Hermite recurrence, any even r >= 0."""
    return lib().oracle_K_hermite(int(r), float(u))


def phi(u: float) -> float:
    """Eq. 2."""
    return lib().oracle_phi(float(u))


# ---- Step I --------------------------------------------------------------------------
class OracleError(ValueError):
    def __init__(self, code: str, msg: str):
        super().__init__(f"{code}: {msg}")
        self.code = code


def step1(x) -> dict:
    """Alg. 1 Step I: V and sigma of the float32 sample (fp64)."""
    x = _f32(x)
    out = np.empty(6, dtype=np.float64)
    rc = lib().oracle_step1(_ptr(x), x.size, _ptr(out))
    if rc == 1:
        raise OracleError("E_INVALID", "n < 2")
    if rc == 2:
        raise OracleError("E_NONFINITE", "non-finite sample value")
    if rc == 3:
        raise OracleError("E_DEGENERATE", "V <= 0")
    return {"sum": out[0], "sum_sq": out[1], "mean": out[2], "var_onepass": out[3],
            "var": out[4], "sigma": out[5]}


def zscore(x, mean: float, sigma: float) -> np.ndarray:
    """Eq. 3: Z_i = (X_i - mu)/sigma in fp64."""
    x = _f32(x)
    z = np.empty(x.size, dtype=np.float64)
    lib().oracle_zscore(_ptr(x), x.size, float(mean), float(sigma), _ptr(z))
    return z


def widen(x) -> np.ndarray:
    x = _f32(x)
    z = np.empty(x.size, dtype=np.float64)
    lib().oracle_widen(_ptr(x), x.size, _ptr(z))
    return z


# ---- Steps II, III, V, VII, Eq. 4 (scalar) -------------------------------------------
def psi8_ns(sigma: float) -> float:
    """Step II: Psi8^NS = 105 / (32 sqrt(pi) sigma^9)."""
    return 105.0 / (32.0 * math.sqrt(PI) * sigma ** 9)


def g1_bandwidth(psi8: float, n: int) -> float:
    """Step III: g1 = (-2 K^6(0) / (mu2 Psi8 n))^(1/9)."""
    return (-2.0 * K6_0 / (MU2 * psi8 * n)) ** (1.0 / 9.0)


def g2_bandwidth(psi6: float, n: int) -> float:
    """Step V: g2 = (-2 K^4(0) / (mu2 Psi6 n))^(1/7); needs Psi6 < 0 (R2)."""
    if not psi6 < 0.0:
        raise OracleError("E_DOMAIN", f"psi6 = {psi6!r} is not < 0")
    return (-2.0 * K4_0 / (MU2 * psi6 * n)) ** (1.0 / 7.0)


def h_bandwidth(psi4: float, n: int) -> float:
    """Step VII: h = (R(K) / (mu2^2 Psi4 n))^(1/5); needs Psi4 > 0."""
    if not psi4 > 0.0:
        raise OracleError("E_DOMAIN", f"psi4 = {psi4!r} is not > 0")
    return (R_K / (MU2 ** 2 * psi4 * n)) ** (1.0 / 5.0)


# ---- Steps IV and VI (the O(n^2) sums) -------------------------------------------------
def _neumaier(values):
    s = 0.0
    c = 0.0
    for v in values:
        t = s + v
        if abs(s) >= abs(v):
            c += (s - t) + v
        else:
            c += (v - t) + s
        s = t
    return s + c


def row_chunks(n: int, nchunks: int = 64):
    """Fixed row-chunk boundaries (a function of n only) so results never depend
    on checkpointing or thread count."""
    step = max(1, -(-n // nchunks))
    return [(i, min(n, i + step)) for i in range(0, n, step)]


def pair_count_rows(n: int, i0: int, i1: int) -> int:
    """Number of (i, j>i) pairs with i in [i0, i1)."""
    i1 = min(i1, n)
    if i1 <= i0:
        return 0
    m = i1 - i0
    return m * (n - 1) - (i0 + i1 - 1) * m // 2


def psi_sum_rows(z: np.ndarray, g: float, r: int, i0: int, i1: int, threads: int = 0):
    """sum_{i0<=i<i1} sum_{j>i} K^(r)((z_i - z_j)/g) as a Neumaier (sum, comp) pair."""
    z = np.ascontiguousarray(z, dtype=np.float64)
    out = np.zeros(2, dtype=np.float64)
    lib().oracle_psi_rows(_ptr(z), z.size, float(g), int(r), int(i0), int(i1), int(threads), _ptr(out))
    return float(out[0]), float(out[1])


def psi_halved_sum(z: np.ndarray, g: float, r: int, threads: int = 0, checkpoint: str | None = None,
                   log=None) -> float:
    """T_r = sum_{i<j} K^(r)((z_i - z_j)/g), the bracketed sum of Eq. 6/7.

    Rows are processed in fixed chunks; with ``checkpoint`` each finished chunk is
    recorded in a JSON file so a long run can resume."""
    z = np.ascontiguousarray(z, dtype=np.float64)
    n = z.size
    chunks = row_chunks(n)
    key = {"sha256_z": hashlib.sha256(z.tobytes()).hexdigest(), "g": g.hex() if isinstance(g, float) else float(g).hex(),
           "r": int(r), "n": int(n)}
    parts = []
    if checkpoint and os.path.exists(checkpoint):
        with open(checkpoint) as f:
            st = json.load(f)
        if st.get("key") == key:
            parts = [float.fromhex(p) for p in st["parts"]]
    for k in range(len(parts), len(chunks)):
        i0, i1 = chunks[k]
        t0 = time.time()
        s, c = psi_sum_rows(z, g, r, i0, i1, threads)
        parts.append(s + c)
        if log:
            log(f"[oracle] r={r} chunk {k + 1}/{len(chunks)} rows [{i0},{i1}) {time.time() - t0:.1f}s")
        if checkpoint:
            tmp = checkpoint + ".tmp"
            with open(tmp, "w") as f:
                json.dump({"key": key, "parts": [p.hex() for p in parts]}, f)
            os.replace(tmp, checkpoint)
    return _neumaier(parts)


def K_at_zero(r: int) -> float:
    """K^(r)(0): the printed constants for r = 6, 4, else (-1)^(r/2) (r-1)!! phi(0)."""
    if r == 6:
        return K6_0
    if r == 4:
        return K4_0
    dfact = 1.0
    for k in range(r - 1, 0, -2):
        dfact *= k
    return (-1.0) ** (r // 2) * dfact / math.sqrt(2.0 * PI)


def psi_from_halved_sum(T: float, n: int, g: float, r: int) -> float:
    """Eq. 6/7: Psi_r(g) = (2 T + n K^(r)(0)) / (n^2 g^(r+1))."""
    return (2.0 * T + n * K_at_zero(r)) / (n * n * g ** (r + 1))


def psi(z, g: float, r: int, threads: int = 0, checkpoint: str | None = None, log=None) -> float:
    """Psi_r(g) over data z via the halved sums (Eq. 6 for r=6, Eq. 7 for r=4)."""
    z = np.ascontiguousarray(z, dtype=np.float64)
    T = psi_halved_sum(z, g, r, threads, checkpoint, log)
    return psi_from_halved_sum(T, z.size, g, r)


def psi_block_sum(z, g: float, r: int, i0: int, i1: int, j0: int, j1: int, threads: int = 0) -> float:
    """sum_{i0<=i<i1} sum_{j0<=j<j1} K^(r)((z_i - z_j)/g): a block of the double sum of Steps IV/VI."""
    z = np.ascontiguousarray(z, dtype=np.float64)
    out = np.zeros(2, dtype=np.float64)
    lib().oracle_psi_block(_ptr(z), z.size, float(g), int(r), int(i0), int(i1), int(j0), int(j1), int(threads),
                           _ptr(out))
    return float(out[0]) + float(out[1])


def psi_literal(z, g: float, r: int) -> float:
    """Alg. 1 Step IV/VI as printed: (n^2 g^(r+1))^-1 sum_i sum_j K^(r)((z_i-z_j)/g)."""
    z = np.ascontiguousarray(z, dtype=np.float64)
    n = z.size
    return lib().oracle_psi_literal_sum(_ptr(z), n, float(g), int(r)) / (n * n * g ** (r + 1))


# ---- the l-stage direct plug-in family of Alg. 1 ----------------
def psi_ns(r: int, sigma: float) -> float:
    """Normal-scale functional Psi_r^NS = (-1)^(r/2) r! / ((2 sigma)^(r+1) (r/2)! sqrt(pi))
    (Wand & Jones; Step II, is r = 8)."""
    return (-1.0) ** (r // 2) * math.factorial(r) / ((2.0 * sigma) ** (r + 1) * math.factorial(r // 2)
                                                     * math.sqrt(PI))


def dpi(x, stages: int, threads: int = 0) -> dict:
    """l-stage direct plug-in (Alg. 1 is l = 2), z-score path (Eq. 3-4):
    Psi_{2l+4} <- Psi^NS;  for j = l..1:  g_j = (-2 K^(2j+2)(0) / (mu2 Psi_{2j+4} n))^(1/(2j+5)),
    Psi_{2j+2} <- Psi_hat_{2j+2}(g_j);  h = (R(K) / (mu2^2 Psi_4 n))^(1/5) sigma."""
    x = _f32(x)
    n = int(x.size)
    s1 = step1(x)
    sigma = s1["sigma"]
    z = zscore(x, s1["mean"], sigma)
    psi_next = psi_ns(2 * stages + 4, 1.0)
    res = {"n": n, "stages": stages, "sigma": sigma, "psi_ns_z": psi_next, "g_z": {}, "psi_z": {}}
    for j in range(stages, 0, -1):
        r = 2 * j + 2
        num = -2.0 * K_at_zero(r)
        if not num / psi_next > 0.0:
            raise OracleError("E_DOMAIN", f"stage {j}: Psi_{r + 2} = {psi_next!r} has the wrong sign")
        g = (num / (MU2 * psi_next * n)) ** (1.0 / (r + 3))
        psi_next = psi(z, g, r, threads)
        res["g_z"][j] = g
        res["psi_z"][j] = psi_next
    h_z = h_bandwidth(psi_next, n)
    res["h_z"] = h_z
    res["h"] = h_z * sigma
    return res


# ---- the paper's Q32.32 fixed-point datapath ---------
Q32_ONE = 1 << 32


def q32_encode(v) -> np.ndarray:
    """Q2: real -> Q32.32 raw int64, round to nearest, ties away from zero."""
    v = np.asarray(v, dtype=np.float64)
    s = v * float(Q32_ONE)                       # exact (power-of-two scaling)
    return (np.sign(s) * np.floor(np.abs(s) + 0.5)).astype(np.int64)


def q32_mul(a: int, b: int) -> int:
    return lib().oracle_q32_mul(int(a), int(b))


def q32_exp(x: int) -> int:
    return lib().oracle_q32_exp(int(x))


def q32_term(d: int, rg: int, r: int) -> int:
    return lib().oracle_q32_term(int(d), int(rg), int(r))


def q32_psi_sum(zq, rg: int, r: int, threads: int = 0) -> int:
    """sum_{i<j} term(z_i - z_j) in Q32.32 raw units, as an exact Python int (int128)."""
    zq = np.ascontiguousarray(zq, dtype=np.int64)
    out = np.zeros(2, dtype=np.int64)
    lib().oracle_q32_psi_sum(_ptr(zq), zq.size, int(rg), int(r), int(threads), _ptr(out))
    return int(out[1]) * (1 << 64) + (int(out[0]) & ((1 << 64) - 1))


def q32_psi(zq, g: float, r: int, threads: int = 0) -> dict:
    """Psi_r(g) of Steps IV/VI with the pair sum in Q32.32 (z units): rg = encode(1/g) (the
    hoisted reciprocal of Fig. 5), S = 2 sum_{i<j} term + n term(0), then
    Psi = phi(0) (S / 2^32) / (n^2 g^(r+1)) in fp64."""
    zq = np.ascontiguousarray(zq, dtype=np.int64)
    n = zq.size
    rg = int(q32_encode(1.0 / g))
    half = q32_psi_sum(zq, rg, r, threads)
    total = 2 * half + n * q32_term(0, rg, r)
    return {"rg": rg, "half_sum": half, "total": total,
            "psi": (total / float(Q32_ONE)) / math.sqrt(2.0 * PI) / (n * n * g ** (r + 1))}


def q32_plugin(x, threads: int = 0) -> dict:
    """Alg. 1 with the Steps IV/VI pair sums in Q32.32 (the paper's datapath, "fast" loop of
    Fig. 5) on the z-scored sample (Eq. 3, encoded to Q32.32); the O(1) steps in fp64."""
    x = _f32(x)
    n = int(x.size)
    s1 = step1(x)
    sigma = s1["sigma"]
    zq = q32_encode(zscore(x, s1["mean"], sigma))
    g1_z = g1_bandwidth(psi8_ns(1.0), n)
    p6 = q32_psi(zq, g1_z, 6, threads)
    g2_z = g2_bandwidth(p6["psi"], n)
    p4 = q32_psi(zq, g2_z, 4, threads)
    h_z = h_bandwidth(p4["psi"], n)
    return {"n": n, "sigma": sigma, "g1_z": g1_z, "psi6_z": p6["psi"], "g2_z": g2_z, "psi4_z": p4["psi"],
            "h_z": h_z, "h": h_z * sigma, "S6_q32": p6["total"], "S4_q32": p4["total"],
            "rg1": p6["rg"], "rg2": p4["rg"]}


# ---- Eq. 1-2: the kernel density estimate that h is for ----------
def kde(x, h: float, points, threads: int = 0) -> np.ndarray:
    """Eq. 1 with Eq. 2: f(x_k, h) = (1/(n h)) sum_i K((x_k - X_i)/h), fp64.

    ``x`` is the float32 sample, ``points`` the evaluation points (float32 values
    are widened exactly, as the GPU reads them)."""
    x = _f32(x)
    if not (h > 0.0 and math.isfinite(h)):
        raise OracleError("E_INVALID", f"h = {h!r} must be finite and > 0")
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64))
    f = np.empty(pts.size, dtype=np.float64)
    lib().oracle_kde(_ptr(x), x.size, float(h), _ptr(pts), pts.size, int(threads), _ptr(f))
    return f


# ---- the whole Algorithm 1 -------------------------------------------------------------
def _pow_int(b: float, k: int) -> float:
    """b^k by repeated multiplication (keeps exact 2^k scaling)."""
    out = 1.0
    for _ in range(k):
        out *= b
    return out


def plugin(x, threads: int = 0, literal: bool = False, raw_path: bool = False,
           checkpoint_dir: str | None = None, log=None) -> dict:
    """Algorithm 1 on the z-scored sample (Eq. 3-4), fp64.

    Returns every intermediate in z units (``*_z``) and raw data units.
    ``literal`` also evaluates the unhalved double sums;
    ``raw_path`` also runs Alg. 1 on the raw data without the z-score.
    """
    x = _f32(x)
    n = int(x.size)
    t0 = time.time()
    s1 = step1(x)                                  # Step I
    sigma = s1["sigma"]
    z = zscore(x, s1["mean"], sigma)               # Eq. 3
    psi8_z = psi8_ns(1.0)                          # Step II with sigma_z = 1
    g1_z = g1_bandwidth(psi8_z, n)                 # Step III
    ck6 = os.path.join(checkpoint_dir, "psi6.json") if checkpoint_dir else None
    ck4 = os.path.join(checkpoint_dir, "psi4.json") if checkpoint_dir else None
    psi6_z = psi(z, g1_z, 6, threads, ck6, log)    # Step IV via Eq. 6
    g2_z = g2_bandwidth(psi6_z, n)                 # Step V
    psi4_z = psi(z, g2_z, 4, threads, ck4, log)    # Step VI via Eq. 7
    h_z = h_bandwidth(psi4_z, n)                   # Step VII
    h = h_z * sigma                                # Eq. 4
    res = {
        "n": n, "mean": s1["mean"], "var": s1["var"], "var_onepass": s1["var_onepass"], "sigma": sigma,
        "psi8_z": psi8_z, "g1_z": g1_z, "psi6_z": psi6_z, "g2_z": g2_z, "psi4_z": psi4_z, "h_z": h_z,
        # raw data units: g scale like sigma, Psi_r like sigma^-(r+1)
        "psi8_ns": psi8_z / _pow_int(sigma, 9), "g1": g1_z * sigma, "psi6": psi6_z / _pow_int(sigma, 7),
        "g2": g2_z * sigma, "psi4": psi4_z / _pow_int(sigma, 5), "h": h,
    }
    if literal:
        res["psi6_z_literal"] = psi_literal(z, g1_z, 6)
        res["psi4_z_literal"] = psi_literal(z, g2_z, 4)
    if raw_path:
        w = widen(x)
        p8 = psi8_ns(sigma)
        g1r = g1_bandwidth(p8, n)
        p6r = psi(w, g1r, 6, threads)
        g2r = g2_bandwidth(p6r, n)
        p4r = psi(w, g2r, 4, threads)
        res["raw_path"] = {"psi8_ns": p8, "g1": g1r, "psi6": p6r, "g2": g2r, "psi4": p4r,
                           "h": h_bandwidth(p4r, n)}
    res["seconds"] = time.time() - t0
    res["threads"] = threads if threads > 0 else lib().oracle_max_threads()
    return res
