"""Pins for the fp64 oracle (oracle/), each against something other than the oracle itself:
closed forms, the definition of K as a derivative of phi (mpmath), textbook identities,
moment identities, the quadrature identity, exact rational arithmetic and a 50-digit
brute force.  CPU only (-m "not gpu")."""
import json
import math
import os
from fractions import Fraction

import mpmath as mp
import numpy as np
import pytest
from scipy import integrate, special

from paper_1505_02100_b200 import inputs

HERE = os.path.dirname(os.path.abspath(__file__))
SQ2PI = math.sqrt(2 * math.pi)


# ---------------------------------------------------------------- K^(4), K^(6)
def test_K_at_zero_matches_printed_constants(oracle_mod):
    # Alg. 1 Step III and Step V
    assert oracle_mod.K(6, 0.0) == pytest.approx(-15 / SQ2PI, rel=1e-15)
    assert oracle_mod.K(4, 0.0) == pytest.approx(3 / SQ2PI, rel=1e-15)
    assert oracle_mod.K6_0 == pytest.approx(-5.984134206021490, rel=1e-15)
    assert oracle_mod.K4_0 == pytest.approx(1.196826841204298, rel=1e-15)


def test_K_at_one_closed_form(oracle_mod):
    # He6(1) = 1-15+45-15 = 16, He4(1) = 1-6+3 = -2
    assert oracle_mod.K(6, 1.0) == pytest.approx(16 * math.exp(-0.5) / SQ2PI, rel=1e-14)
    assert oracle_mod.K(4, 1.0) == pytest.approx(-2 * math.exp(-0.5) / SQ2PI, rel=1e-14)


@pytest.mark.parametrize("r", [4, 6])
@pytest.mark.parametrize("u", [0.0, 0.3, -0.7, 1.3, 2.2, -3.1, 4.5, 7.0])
def test_K_is_rth_derivative_of_phi(oracle_mod, r, u):
    # Reading R1 (P:93 'K^6(0)' vs P:101 'K^(6)'): K^(r) = d^r/du^r phi(u), phi of Eq. 2.
    mp.mp.dps = 40
    phi = lambda v: mp.exp(-v * v / 2) / mp.sqrt(2 * mp.pi)
    ref = float(mp.diff(phi, mp.mpf(u), r))
    assert oracle_mod.K(r, u) == pytest.approx(ref, rel=1e-12, abs=1e-14)


@pytest.mark.parametrize("u", [0.0, 0.5, 1.1, 2.0, 3.7])
def test_K6_is_second_finite_difference_of_K4(oracle_mod, u):
    h = 1e-3
    fd = (oracle_mod.K(4, u + h) - 2 * oracle_mod.K(4, u) + oracle_mod.K(4, u - h)) / (h * h)
    assert fd == pytest.approx(oracle_mod.K(6, u), abs=2e-5)


@pytest.mark.parametrize("u", [0.0, 0.4, 1.2, 2.5])
def test_K4_is_fourth_finite_difference_of_phi(oracle_mod, u):
    h = 1e-2
    p = [oracle_mod.phi(u + k * h) for k in (-2, -1, 0, 1, 2)]
    fd = (p[0] - 4 * p[1] + 6 * p[2] - 4 * p[3] + p[4]) / h ** 4
    assert fd == pytest.approx(oracle_mod.K(4, u), abs=2e-4)


@pytest.mark.parametrize("r", [4, 6])
def test_K_matches_scipy_hermite(oracle_mod, r):
    for u in np.linspace(-6, 6, 41):
        ref = special.eval_hermitenorm(r, u) * math.exp(-u * u / 2) / SQ2PI
        assert oracle_mod.K(r, float(u)) == pytest.approx(ref, rel=1e-12, abs=1e-15)


def test_K_zeros(oracle_mod):
    # He4 roots: u^2 = 3 -+ sqrt(6);  He6 roots (Abramowitz & Stegun Table 25.10 scaled): 0.61670659, 1.88917588, 3.32425743
    for u in (math.sqrt(3 - math.sqrt(6)), math.sqrt(3 + math.sqrt(6))):
        assert abs(oracle_mod.K(4, u)) < 1e-14
    for u in (0.6167065901925941, 1.889175877753711, 3.324257433552119):
        assert abs(oracle_mod.K(6, u)) < 1e-12


@pytest.mark.parametrize("r,k,val", [(4, 0, 0), (4, 2, 0), (4, 4, 24), (6, 0, 0), (6, 2, 0), (6, 4, 0), (6, 6, 720)])
def test_K_moments(oracle_mod, r, k, val):
    # int u^k phi^(r)(u) du = 0 for k < r (even), = r! for k = r  (integration by parts)
    v, _ = integrate.quad(lambda u: u ** k * oracle_mod.K(r, u), -40, 40, limit=400, epsabs=1e-13)
    assert v == pytest.approx(val, abs=1e-9)


def test_K_even(oracle_mod):
    for u in (0.1, 0.77, 2.5, 9.0):
        assert oracle_mod.K(6, u) == oracle_mod.K(6, -u)
        assert oracle_mod.K(4, u) == oracle_mod.K(4, -u)


# ---------------------------------------------------------------- Step I
def _exact_var(x32):
    fr = [Fraction(float(v)) for v in x32]
    n = len(fr)
    s1, s2 = sum(fr), sum(v * v for v in fr)
    return s1, s2, s2 / (n - 1) - s1 * s1 / (n * (n - 1))


def test_step1_toy_exact_rational(oracle_mod):
    x = inputs.TOY.astype(np.float32)
    s1, s2, v = _exact_var(x)
    r = oracle_mod.step1(x)
    assert r["sum"] == float(s1) and r["sum_sq"] == float(s2)
    assert r["var"] == pytest.approx(float(v), rel=2e-16)
    assert r["var_onepass"] == pytest.approx(float(v), rel=1e-15)
    # the paper's decimal values: sum 14.7, sum of squares 36.57, V = 9.55875/7
    assert float(Fraction("36.57") / 7 - Fraction("14.7") ** 2 / 56) == pytest.approx(1.3655357142857143, rel=1e-16)
    assert r["var"] == pytest.approx(1.3655357142857143, rel=1e-7)   # float32 cast of 1.1, 1.9, 2.8, 2.9


@pytest.mark.parametrize("a,b", [(0.0, 1.0), (-3.5, 2.25), (1e3, 1e3 + 0.5)])
def test_step1_two_points(oracle_mod, a, b):
    r = oracle_mod.step1(np.array([a, b], np.float32))
    assert r["var"] == pytest.approx((a - b) ** 2 / 2, rel=1e-15)


def test_step1_random_exact(oracle_mod):
    x = inputs.normal(1000, 7, mean=5.0, sd=3.0)
    s1, s2, v = _exact_var(x)
    assert oracle_mod.step1(x)["var"] == pytest.approx(float(v), rel=1e-14)


def test_step1_errors(oracle_mod):
    with pytest.raises(oracle_mod.OracleError, match="E_INVALID"):
        oracle_mod.step1(np.array([1.0], np.float32))
    with pytest.raises(oracle_mod.OracleError, match="E_NONFINITE"):
        oracle_mod.step1(np.array([1.0, np.nan, 2.0], np.float32))
    with pytest.raises(oracle_mod.OracleError, match="E_NONFINITE"):
        oracle_mod.step1(np.array([1.0, np.inf], np.float32))
    with pytest.raises(oracle_mod.OracleError, match="E_DEGENERATE"):
        oracle_mod.step1(np.full(10, 2.5, np.float32))


# ---------------------------------------------------------------- Steps II, III, V, VII
def test_step2_is_textbook_normal_scale_psi8(oracle_mod):
    # Wand & Jones normal-scale functional: psi_r^NS = (-1)^(r/2) r! / ((2 sigma)^(r+1) (r/2)! sqrt(pi))
    for sigma in (1.0, 0.37, 2.5):
        ref = math.factorial(8) / ((2 * sigma) ** 9 * math.factorial(4) * math.sqrt(math.pi))
        assert oracle_mod.psi8_ns(sigma) == pytest.approx(ref, rel=1e-14)
    assert oracle_mod.psi8_ns(1.0) == pytest.approx(1.851247071016075, rel=1e-15)


@pytest.mark.parametrize("n,expect", [(2, 1.1392399750248389), (100, 0.7376337352101906), (1024, 0.5696199875124194),
                                      (1048576, 0.2636983710255757)])
def test_step3_g1_closed_form(oracle_mod, n, expect):
    # z units: g1 = (-2 K6(0)/(Psi8 n))^(1/9) = (32 sqrt(2) / (7 n))^(1/9)
    g1 = oracle_mod.g1_bandwidth(oracle_mod.psi8_ns(1.0), n)
    assert g1 == pytest.approx((32 * math.sqrt(2) / (7 * n)) ** (1 / 9), rel=1e-14)
    assert g1 == pytest.approx(expect, rel=1e-14)


def test_step5_step7_closed_forms(oracle_mod):
    n = 1000
    psi6 = -0.55
    assert oracle_mod.g2_bandwidth(psi6, n) == pytest.approx((6 / SQ2PI / (0.55 * n)) ** (1 / 7), rel=1e-14)
    assert oracle_mod.h_bandwidth(0.21, n) == pytest.approx((1 / (2 * math.sqrt(math.pi)) / (0.21 * n)) ** 0.2, rel=1e-14)
    with pytest.raises(oracle_mod.OracleError, match="E_DOMAIN"):
        oracle_mod.g2_bandwidth(0.1, n)
    with pytest.raises(oracle_mod.OracleError, match="E_DOMAIN"):
        oracle_mod.h_bandwidth(-0.1, n)


# ---------------------------------------------------------------- Steps IV / VI
@pytest.mark.parametrize("r", [4, 6])
@pytest.mark.parametrize("g", [0.3, 1.0, 2.7])
def test_psi_single_point(oracle_mod, r, g):
    # n = 1: only the diagonal term: Psi = K(0) / g^(r+1)
    k0 = -15 / SQ2PI if r == 6 else 3 / SQ2PI
    assert oracle_mod.psi(np.array([0.42]), g, r) == pytest.approx(k0 / g ** (r + 1), rel=1e-14)


@pytest.mark.parametrize("r", [4, 6])
def test_psi_two_points(oracle_mod, r):
    # n = 2: Psi = (2 K(0) + 2 K(d/g)) / (4 g^(r+1))   (Step IV/VI written out)
    z = np.array([-1.0, 1.0])
    g = 2.0
    k0 = -15 / SQ2PI if r == 6 else 3 / SQ2PI
    kd = (16 if r == 6 else -2) * math.exp(-0.5) / SQ2PI   # K(1)
    assert oracle_mod.psi(z, g, r) == pytest.approx((2 * k0 + 2 * kd) / (4 * g ** (r + 1)), rel=1e-14)


@pytest.mark.parametrize("r", [4, 6])
def test_psi_all_equal_differences(oracle_mod, r):
    # all points equal: every u = 0 -> Psi = K(0)/g^(r+1)
    k0 = -15 / SQ2PI if r == 6 else 3 / SQ2PI
    assert oracle_mod.psi(np.full(33, 1.25), 0.8, r) == pytest.approx(k0 / 0.8 ** (r + 1), rel=1e-13)


@pytest.mark.parametrize("r", [4, 6])
def test_halved_equals_literal(oracle_mod, r):
    # Eq. 5-7 vs the double sum of Steps IV/VI
    z = np.random.default_rng(3).standard_normal(300)
    for g in (0.2, 0.6, 1.5):
        assert oracle_mod.psi(z, g, r) == pytest.approx(oracle_mod.psi_literal(z, g, r), rel=1e-13)


def _quadrature_psi(X, g, s):
    """(-1)^s int (fhat^(s)_h(x))^2 dx with h = g/sqrt(2); fhat^(s) from scipy Hermite."""
    h = g / math.sqrt(2)
    n = len(X)

    def fs(x):
        u = (x - X) / h
        # d^s/dx^s phi((x - Xi)/h) = h^-s phi^(s)(u), phi^(s) = (-1)^s He_s phi
        return np.sum((-1) ** s * special.eval_hermitenorm(s, u) * np.exp(-u * u / 2) / SQ2PI) / (n * h ** (s + 1))

    lo, hi = X.min() - 14 * h, X.max() + 14 * h
    xs = np.linspace(lo, hi, 200001)
    vals = np.array([fs(x) for x in xs]) if n < 3 else None
    if vals is None:
        u = (xs[:, None] - X[None, :]) / h
        vals = np.sum((-1) ** s * special.eval_hermitenorm(s, u) * np.exp(-u * u / 2) / SQ2PI, axis=1) / (n * h ** (s + 1))
    return (-1) ** s * integrate.simpson(vals * vals, x=xs)


@pytest.mark.parametrize("n,seed", [(7, 1), (50, 2), (120, 3)])
@pytest.mark.parametrize("g", [0.15, 0.6])
def test_quadrature_identity(oracle_mod, n, seed, g):
    # phi_a * phi_b = phi_sqrt(a^2+b^2)  =>  Psi_2s(g) = (-1)^s int (fhat^(s)_{g/sqrt2})^2 dx
    X = np.random.default_rng(seed).standard_normal(n)
    for r, s in ((4, 2), (6, 3)):
        q = _quadrature_psi(X, g, s)
        assert oracle_mod.psi(X, g, r) == pytest.approx(q, rel=1e-9)


# ---------------------------------------------------------------- whole Algorithm 1
def _mp_plugin(x32):
    """Alg. 1 at 50 digits on the raw data (no z-score), K^(r) as mpmath derivatives of phi."""
    mp.mp.dps = 50
    X = [mp.mpf(float(v)) for v in x32]
    n = len(X)
    S1 = mp.fsum(X)
    S2 = mp.fsum(v * v for v in X)
    V = S2 / (n - 1) - S1 ** 2 / (n * (n - 1))
    sig = mp.sqrt(V)
    phi = lambda v: mp.exp(-v * v / 2) / mp.sqrt(2 * mp.pi)
    cache = {}

    def K(r, u):
        key = (r, mp.nstr(u, 45))
        if key not in cache:
            cache[key] = mp.diff(phi, u, r)
        return cache[key]

    def psi(r, g):
        return mp.fsum(K(r, abs(a - b) / g) for a in X for b in X) / (n * n * g ** (r + 1))

    psi8 = 105 / (32 * mp.sqrt(mp.pi) * sig ** 9)
    g1 = (-2 * K(6, mp.mpf(0)) / (psi8 * n)) ** (mp.mpf(1) / 9)
    p6 = psi(6, g1)
    g2 = (-2 * K(4, mp.mpf(0)) / (p6 * n)) ** (mp.mpf(1) / 7)
    p4 = psi(4, g2)
    h = (1 / (2 * mp.sqrt(mp.pi)) / (p4 * n)) ** (mp.mpf(1) / 5)
    return {"sigma": sig, "g1": g1, "psi6": p6, "g2": g2, "psi4": p4, "h": h}


@pytest.mark.parametrize("case", ["toy", "n3", "n5", "n16", "mixture12"])
def test_plugin_vs_50_digit_bruteforce(oracle_mod, case):
    if case == "toy":
        x = inputs.TOY.astype(np.float32)
    elif case == "mixture12":
        x = inputs.mixture(12, 5)
    else:
        x = inputs.normal(int(case[1:]), 11, mean=-1.0, sd=0.7)
    ref = _mp_plugin(x)
    o = oracle_mod.plugin(x)
    for k in ("sigma", "g1", "psi6", "g2", "psi4", "h"):
        assert o[k] == pytest.approx(float(ref[k]), rel=1e-12), k


def test_plugin_toy_matches_survey_50_digit_values(oracle_mod):
    with open(os.path.join(HERE, "golden", "toy.json")) as f:
        gold = json.load(f)["decimal_input_values_50_digits"]
    o = oracle_mod.plugin(inputs.TOY.astype(np.float32))
    # the survey evaluated exact decimals; float32 input moves values by ~1e-8
    for k in ("var", "sigma", "g1_z", "psi6_z", "g2_z", "psi4_z", "h_z", "h"):
        assert o[k] == pytest.approx(gold[k], rel=5e-7), k


@pytest.mark.parametrize("a,b", [(0.0, 1.0), (-2.0, 5.5), (100.0, 100.25)])
def test_plugin_two_points_universal(oracle_mod, a, b):
    # n = 2: z = +-1/sqrt(2) for any a != b, so the z-intermediates are universal and h = c |a - b|
    o = oracle_mod.plugin(np.array([a, b], np.float32))
    assert o["h"] == pytest.approx(0.74338814253112600 * abs(b - a), rel=1e-13)
    assert o["g1_z"] == pytest.approx(1.1392399750248389, rel=1e-14)
    assert o["psi6_z"] == pytest.approx(-0.37169296176652702, rel=1e-13)
    assert o["g2_z"] == pytest.approx(1.1818151934988414, rel=1e-13)
    assert o["psi4_z"] == pytest.approx(0.109827711778942, rel=1e-12)
    assert o["h_z"] == pytest.approx(1.0513095932748618, rel=1e-13)


def test_plugin_two_points_mp(oracle_mod):
    ref = _mp_plugin(np.array([0.0, 1.0], np.float32))
    assert float(ref["h"]) == pytest.approx(0.74338814253112600, rel=1e-15)


def test_raw_path_equals_z_path(oracle_mod):
    for x in (inputs.normal(500, 1, 3.0, 2.0), inputs.mixture(400, 2), inputs.TOY.astype(np.float32)):
        o = oracle_mod.plugin(x, raw_path=True, literal=True)
        raw = o["raw_path"]
        for k in ("g1", "psi6", "g2", "psi4", "h"):
            assert o[k] == pytest.approx(raw[k], rel=1e-12), k
        assert o["psi6_z"] == pytest.approx(o["psi6_z_literal"], rel=1e-13)
        assert o["psi4_z"] == pytest.approx(o["psi4_z_literal"], rel=1e-13)


@pytest.mark.parametrize("k", [3, -5, 10])
def test_pow2_scale_equivariance_bit_exact(oracle_mod, k):
    x = inputs.normal(700, 4, 1.0, 3.0)
    o = oracle_mod.plugin(x)
    o2 = oracle_mod.plugin((x * np.float32(2.0 ** k)).astype(np.float32))
    assert o2["h"] == o["h"] * 2.0 ** k
    assert o2["psi6_z"] == o["psi6_z"] and o2["psi4_z"] == o["psi4_z"]
    assert o2["g1"] == o["g1"] * 2.0 ** k and o2["g2"] == o["g2"] * 2.0 ** k


def test_scale_equivariance_general(oracle_mod):
    # dyadic data times 3 stays exact in float32, so h(3X) = 3 h(X) to rounding
    x = (np.round(inputs.normal(600, 5) * 64) / 64).astype(np.float32)
    o, o3 = oracle_mod.plugin(x), oracle_mod.plugin((x * 3).astype(np.float32))
    assert o3["h"] == pytest.approx(3 * o["h"], rel=1e-12)


def test_shift_invariance(oracle_mod):
    x = (np.round(inputs.normal(600, 6) * 256) / 256).astype(np.float32)
    o, o2 = oracle_mod.plugin(x), oracle_mod.plugin((x + 37.0).astype(np.float32))
    assert o2["h"] == pytest.approx(o["h"], rel=1e-12)


def test_permutation_invariance(oracle_mod):
    x = inputs.mixture(800, 8)
    p = np.random.default_rng(0).permutation(x.size)
    assert oracle_mod.plugin(x[p])["h"] == pytest.approx(oracle_mod.plugin(x)["h"], rel=1e-13)


def test_sign_invariants(oracle_mod):
    # Psi4 > 0 and Psi6 < 0 for every sample (quadrature identity)
    for seed in range(6):
        for x in (inputs.normal(300, seed), inputs.mixture(300, seed), inputs.ties(300, seed)):
            o = oracle_mod.plugin(x)
            assert o["psi6_z"] < 0 < o["psi4_z"]
            assert o["g1"] > 0 and o["g2"] > 0 and o["h"] > 0


def test_thread_count_determinism(oracle_mod):
    x = inputs.config_data(1)
    assert oracle_mod.plugin(x, threads=1)["h"] == oracle_mod.plugin(x, threads=8)["h"]


@pytest.mark.parametrize("r,g", [(4, 0.5), (6, 0.8), (4, 0.9)])
def test_normal_sample_expectation(oracle_mod, r, g):
    # E[Psi_r(g)] for N(0, s^2) data (fixed g): phi^(r)(0)[g^-(r+1)/n + (1-1/n)(g^2+2s^2)^-(r+1)/2]
    n, s = 4096, 1.0
    vals = []
    for seed in range(4):
        x = inputs.normal(n, 100 + seed)
        vals.append(oracle_mod.psi(oracle_mod.widen(x), g, r))
    k0 = -15 / SQ2PI if r == 6 else 3 / SQ2PI
    expect = k0 * (g ** -(r + 1) / n + (1 - 1 / n) * (g * g + 2 * s * s) ** (-(r + 1) / 2))
    assert np.mean(vals) == pytest.approx(expect, rel=0.1 if r == 4 else 0.3)


def test_config_inputs_sha256():
    for k in (1, 2, 3):
        assert inputs.sha256_f32(inputs.config_data(k)) == inputs.SHA256[k]


def test_block_sums_partition_the_double_sum(oracle_mod):
    # the rectangular blocks used for sampled full-size parity add up to the literal double sum,
    # and full = 2 * (upper blocks) + (diagonal blocks)  (Eq. 5-7)
    z = np.random.default_rng(12).standard_normal(301)
    n, g = z.size, 0.45
    cuts = [0, 77, 150, 301]
    for r in (4, 6):
        lit = oracle_mod.lib().oracle_psi_literal_sum(z.ctypes.data, n, g, r)
        blocks = {(a, b): oracle_mod.psi_block_sum(z, g, r, cuts[a], cuts[a + 1], cuts[b], cuts[b + 1])
                  for a in range(3) for b in range(3)}
        assert sum(blocks.values()) == pytest.approx(lit, rel=1e-13)
        sym = sum(2 * v if a < b else v for (a, b), v in blocks.items() if a <= b)
        assert sym == pytest.approx(lit, rel=1e-13)
