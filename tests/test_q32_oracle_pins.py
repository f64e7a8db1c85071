"""Pins for the oracle's Q32.32 fixed-point datapath (Fig. 5 "fast" loop;
SURVEY §8(f) NEXT 2; definitions Q1-Q7 in DESIGN.md §14), each against something other than
the oracle's C code: Python's exact integers and fractions, mpmath exp, the fp64 oracle's
K^(r), a literal all-ordered-pairs double sum, and the paper's own accuracy bound on h
(Table 4, max relative error 4.2e-6).  CPU only (-m "not gpu")."""
import math
import random
from fractions import Fraction

import mpmath as mp
import numpy as np
import pytest

from paper_1505_02100_b200 import inputs

ONE = 1 << 32


def test_mul_is_floor_of_exact_product(oracle_mod):
    rng = random.Random(0)
    for _ in range(20000):
        a = rng.randrange(-(1 << 50), 1 << 50)
        b = rng.randrange(-(1 << 45), 1 << 45)
        got = oracle_mod.q32_mul(a, b)
        exact = Fraction(a * b, ONE)
        assert got == math.floor(exact)
        assert Fraction(got) <= exact < Fraction(got) + 1
    assert oracle_mod.q32_mul(2 * ONE, ONE // 2) == ONE
    assert oracle_mod.q32_mul(3 * ONE, ONE // 4) == 3 * ONE // 4


def test_encode_rounds_half_away(oracle_mod):
    assert oracle_mod.q32_encode([1.5])[0] == 0x0000_0001_8000_0000
    assert oracle_mod.q32_encode([-0.5])[0] == -(1 << 31)
    half_ulp = 2.0 ** -33
    assert oracle_mod.q32_encode([half_ulp])[0] == 1 and oracle_mod.q32_encode([-half_ulp])[0] == -1
    rng = np.random.default_rng(1)
    v = rng.normal(0, 3, 5000)
    q = oracle_mod.q32_encode(v)
    assert np.all(np.abs(q / ONE - v) <= 2.0 ** -33)


def test_exp_against_mpmath(oracle_mod):
    mp.mp.dps = 40
    rng = random.Random(2)
    xs = [0, -1, -ONE // 2, -21 * ONE] + [rng.randrange(-21 * ONE, 1) for _ in range(4000)]
    for x in xs:
        ref = mp.exp(mp.mpf(x) / ONE)
        got = oracle_mod.q32_exp(x)
        # truncated Q2.62 Taylor (|w| <= ln2/2, remainder 2^-37) + the final right shift (floor)
        assert abs(mp.mpf(got) / ONE - ref) <= mp.mpf(2) ** -31, (x, got, ref)
    assert oracle_mod.q32_exp(0) == ONE                                   # e^0 = 1 exactly
    assert oracle_mod.q32_exp(-21 * ONE - 1) == 0                          # underflow clamp (ledger)


def test_exp_monotone(oracle_mod):
    grid = np.linspace(-21, 0, 20001)
    vals = [oracle_mod.q32_exp(int(v * ONE)) for v in grid]
    assert all(b >= a for a, b in zip(vals, vals[1:]))


@pytest.mark.parametrize("r", [4, 6])
def test_term_against_fp64_kernel(oracle_mod, r):
    rg = int(oracle_mod.q32_encode([1 / 0.37])[0])
    phi0 = 1 / math.sqrt(2 * math.pi)
    for d in np.linspace(-5, 5, 801):
        dq = int(oracle_mod.q32_encode([d])[0])
        u = abs(dq) * rg / ONE / ONE
        t = u * u
        got = oracle_mod.q32_term(dq, rg, r) / ONE
        ref = oracle_mod.K(r, u) / phi0
        if t > 42.0 + 1e-6:
            assert got == 0.0          # e^{-t/2} below the clamp e^-21 (Q3)
            continue
        # e^{-t/2} carries <= 2^-31 absolute (below Q32.32 resolution for large t), scaled
        # by |P_r(t)|; the truncations of u, t and the products add a few 2^-32 each
        P = t * t - 6 * t + 3 if r == 4 else ((t - 15) * t + 45) * t - 15
        assert abs(got - ref) <= 2.0 ** -30 * (1 + abs(P)) + 1e-8, (d, got, ref)
    assert oracle_mod.q32_term(0, rg, r) == (3 if r == 4 else -15) * ONE  # P_r(0) e^0, exact


@pytest.mark.parametrize("r", [4, 6])
def test_term_of_far_and_extreme_pairs_is_zero(oracle_mod, r):
    # reading Q4: the term is 0 once u = |d| rg > 7 (t > 42), judged on the exact product: with
    # |d| rg >= 2^95 the Q32.32 value of u does not fit int64 and must not wrap into range
    big = (1 << 63) - 1
    for d, rg in ((1 << 40, 3 * ONE), (1 << 62, 1 << 51), (big, (1 << 52) - 1), (-big - 1, 1 << 33),
                  (8 * ONE, ONE), (7 * ONE + 1, ONE)):
        exact_u = Fraction(abs(d) * rg, ONE * ONE)
        assert exact_u > 7
        assert oracle_mod.q32_term(d, rg, r) == 0, (d, rg)
    # just inside: u = 6.5 gives t = 42.25 > 42 -> 0; u = 6 gives a tiny non-zero term
    assert oracle_mod.q32_term(6 * ONE, ONE, r) != 0


@pytest.mark.parametrize("r", [4, 6])
def test_halved_sum_of_extreme_values_drops_far_pairs(oracle_mod, r):
    # values near the int64 limits: every pair with an extreme member is far (term 0), so the
    # sum equals the sum over the ordinary values alone (no wrapped differences)
    zq = oracle_mod.q32_encode(inputs.normal(40, 8))
    ext = np.array([(1 << 62), -(1 << 62), (1 << 63) - 1], dtype=np.int64)
    rg = ONE
    both = oracle_mod.q32_psi_sum(np.concatenate([zq, ext]), rg, r)
    extp = oracle_mod.q32_psi_sum(ext, rg, r)
    assert both == oracle_mod.q32_psi_sum(zq, rg, r) + extp
    assert extp == 0


@pytest.mark.parametrize("r", [4, 6])
def test_halved_sum_equals_literal_double_sum_exactly(oracle_mod, r):
    # Eq. 5-7 in integers: sum_i sum_j term = 2 sum_{i<j} term + n term(0), bit for bit
    zq = oracle_mod.q32_encode(inputs.normal(60, 4))
    rg = int(oracle_mod.q32_encode([1 / 0.5])[0])
    full = sum(oracle_mod.q32_term(int(a) - int(b), rg, r) for a in zq for b in zq)
    half = oracle_mod.q32_psi_sum(zq, rg, r)
    assert full == 2 * half + len(zq) * oracle_mod.q32_term(0, rg, r)
    perm = np.random.default_rng(3).permutation(zq)
    assert oracle_mod.q32_psi_sum(perm, rg, r) == half                     # order-free
    assert oracle_mod.q32_psi_sum(zq, rg, r, threads=1) == half


def test_single_point_closed_form(oracle_mod):
    zq = oracle_mod.q32_encode([0.25])
    for r, k0 in ((6, -15), (4, 3)):
        res = oracle_mod.q32_psi(zq, 0.8, r)
        assert res["total"] == k0 * ONE
        assert res["psi"] == pytest.approx(k0 / math.sqrt(2 * math.pi) / 0.8 ** (r + 1), rel=1e-15)


@pytest.mark.parametrize("n", [128, 256, 512, 768, 1024])
def test_h_within_the_papers_fixed_point_accuracy(oracle_mod, n):
    # Table 4: the Q32.32 FPGA h is within 4.2e-6 relative of the fp64 h_ref
    x = inputs.normal(n, 100 + n // 128 - 1)
    a, b = oracle_mod.q32_plugin(x), oracle_mod.plugin(x)
    assert abs(a["h"] - b["h"]) / b["h"] <= 4.2e-6
    assert abs(a["psi4_z"] - b["psi4_z"]) / b["psi4_z"] <= 2.1e-5
    assert a["psi6_z"] < 0 < a["psi4_z"]


@pytest.mark.parametrize("r", [4, 6])
def test_term_is_zero_far_out(oracle_mod, r):
    # K^(r)(u) = 0 to all Q32.32 digits for |u| > 7 (reading Q4); u*u leaves int64 at
    # u >= 46341, which must not wrap into a non-zero term
    for u in (7.5, 100.0, 46340.0, 46341.0, 46342.0, 70000.0, 2.0 ** 18, 2.0 ** 30):
        d = int(u * ONE)
        assert oracle_mod.q32_term(d, ONE, r) == 0, u
        assert oracle_mod.q32_term(-d, ONE, r) == 0, u
    assert oracle_mod.q32_term(7 * ONE, ONE, r) == 0  # t = 49 > 42
