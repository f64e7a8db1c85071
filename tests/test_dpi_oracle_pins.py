"""Pins for the oracle's general even-r functionals and the l-stage direct plug-in
(Alg. 1 is the l = 2 member), each against something other
than the oracle's code: mpmath derivatives of phi, printed constants, textbook normal-scale
values, Gaussian quadrature of the normal density's derivatives, the normal reference rule,
the quadrature identity and a 50-digit brute force.  CPU only (-m "not gpu")."""
import math

import mpmath as mp
import numpy as np
import pytest
from scipy import integrate, special

from paper_1505_02100_b200 import inputs

SQ2PI = math.sqrt(2 * math.pi)


@pytest.mark.parametrize("r", [0, 2, 4, 6, 8, 10, 12])
@pytest.mark.parametrize("u", [0.0, 0.35, -1.2, 2.4, 5.5])
def test_K_hermite_is_rth_derivative_of_phi(oracle_mod, r, u):
    mp.mp.dps = 40
    phi = lambda v: mp.exp(-v * v / 2) / mp.sqrt(2 * mp.pi)
    ref = float(mp.diff(phi, mp.mpf(u), r))
    assert oracle_mod.K_hermite(r, u) == pytest.approx(ref, rel=1e-12, abs=1e-13)


@pytest.mark.parametrize("r", [4, 6])
def test_hermite_form_equals_printed_polynomials(oracle_mod, r):
    for u in np.linspace(-7, 7, 29):
        assert oracle_mod.K_hermite(r, u) == pytest.approx(oracle_mod.K(r, u), rel=1e-13, abs=1e-16)


@pytest.mark.parametrize("r", [2, 4, 6, 8, 10, 12])
def test_K_at_zero(oracle_mod, r):
    # scipy's Hermite He_r(0) (a library routine) times phi(0); r = 6, 4 are the printed values
    assert oracle_mod.K_at_zero(r) == pytest.approx(special.eval_hermitenorm(r, 0.0) / SQ2PI, rel=1e-14)
    assert oracle_mod.K_hermite(r, 0.0) == pytest.approx(oracle_mod.K_at_zero(r), rel=1e-14)


def test_psi_ns_printed_and_textbook_values(oracle_mod):
    assert oracle_mod.psi_ns(8, 1.7) == pytest.approx(105 / (32 * math.sqrt(math.pi) * 1.7 ** 9), rel=1e-14)
    assert oracle_mod.psi_ns(4, 1.0) == pytest.approx(0.2115710938304086, rel=1e-14)
    assert oracle_mod.psi_ns(6, 1.0) == pytest.approx(-0.5289277345760215, rel=1e-14)


@pytest.mark.parametrize("r", [2, 4, 6, 8, 10, 12])
def test_psi_ns_is_the_normal_functional(oracle_mod, r):
    # Psi_r(f) = int f^(r) f dx for f = N(0, sigma^2), by quadrature of scipy Hermite derivatives
    sig = 1.3

    def f(x):
        return math.exp(-0.5 * (x / sig) ** 2) / (sig * SQ2PI)

    def fr(x):
        return special.eval_hermitenorm(r, x / sig) * f(x) / sig ** r

    v, _ = integrate.quad(lambda x: fr(x) * f(x), -30, 30, limit=400, epsabs=1e-14, epsrel=1e-12)
    assert oracle_mod.psi_ns(r, sig) == pytest.approx(v, rel=1e-9)


def test_two_stage_member_is_algorithm_1(oracle_mod):
    x = inputs.mixture(800, 2)
    a, b = oracle_mod.plugin(x), oracle_mod.dpi(x, 2)
    assert b["h"] == a["h"] and b["psi_z"][2] == a["psi6_z"] and b["psi_z"][1] == a["psi4_z"]
    assert b["g_z"][2] == a["g1_z"] and b["g_z"][1] == a["g2_z"]


def test_zero_stage_member_is_the_normal_reference_rule(oracle_mod):
    x = inputs.normal(500, 3, mean=2.0, sd=0.7)
    s = oracle_mod.step1(x)["sigma"]
    assert oracle_mod.dpi(x, 0)["h"] == pytest.approx((4.0 / (3.0 * 500)) ** 0.2 * s, rel=1e-14)


@pytest.mark.parametrize("s", [1, 4, 5])
def test_quadrature_identity_higher_orders(oracle_mod, s):
    # psi_2s(g) = (-1)^s int (f_hat^(s)_{g/sqrt2})^2   (phi_a * phi_b = phi_sqrt(a^2+b^2))
    x = inputs.mixture(40, 7).astype(np.float64)
    g = 0.6
    hh = g / math.sqrt(2)
    grid = np.linspace(x.min() - 12 * hh, x.max() + 12 * hh, 40001)
    u = (grid[:, None] - x[None, :]) / hh
    fs = np.sum(special.eval_hermitenorm(s, u) * np.exp(-0.5 * u * u), axis=1) * ((-1) ** s) / (
        SQ2PI * x.size * hh ** (s + 1))
    rhs = (-1) ** s * integrate.simpson(fs * fs, x=grid)
    lhs = oracle_mod.psi(x, g, 2 * s)
    assert lhs == pytest.approx(rhs, rel=1e-9)
    assert (lhs > 0) == (s % 2 == 0)


@pytest.mark.parametrize("r", [8, 10])
def test_psi_general_r_mpmath_brute_force(oracle_mod, r):
    mp.mp.dps = 50
    x = inputs.normal(9, 77)
    g = 0.8
    phi = lambda v: mp.exp(-v * v / 2) / mp.sqrt(2 * mp.pi)
    tot = mp.mpf(0)
    for a in x:
        for b in x:
            tot += mp.diff(phi, (mp.mpf(float(a)) - mp.mpf(float(b))) / g, r)
    ref = tot / (len(x) ** 2 * mp.mpf(g) ** (r + 1))
    assert oracle_mod.psi(x.astype(np.float64), g, r) == pytest.approx(float(ref), rel=1e-12)


def test_single_point_and_signs(oracle_mod):
    for r in (2, 8, 10, 12):
        assert oracle_mod.psi(np.array([0.4]), 0.9, r) == pytest.approx(oracle_mod.K_at_zero(r) / 0.9 ** (r + 1),
                                                                          rel=1e-14)
    res = oracle_mod.dpi(inputs.mixture(600, 4), 5)
    for j, v in res["psi_z"].items():
        assert (v > 0) == (j % 2 == 1)   # Psi_{2j+2}: sign (-1)^(j+1)
