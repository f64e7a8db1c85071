"""Pins for the oracle's kernel density estimate (Eq. 1-2; SURVEY §8(f)
NEXT 1), each against something other than the oracle's own loop: printed/closed-form
values, exact symmetry, the moments of a Gaussian mixture, scipy's gaussian_kde (a library
routine), a 50-digit mpmath brute force, and the convolution identity
int f^2 = n^-2 sum_ij phi_{h sqrt 2}(X_i - X_j).  CPU only (-m "not gpu")."""
import math

import mpmath as mp
import numpy as np
import pytest
from scipy import stats

from paper_1505_02100_b200 import inputs

PHI0 = 0.3989422804014327      # phi(0) = 1/sqrt(2 pi)
PHI1 = 0.24197072451914337     # phi(1) = e^{-1/2}/sqrt(2 pi), textbook table value


def _trapz(f, x):
    return float(np.sum((f[1:] + f[:-1]) * np.diff(x)) / 2.0)


def test_single_point_is_the_kernel(oracle_mod):
    # X = {0}, h = 1, x = 0 -> 1/sqrt(2 pi)
    assert oracle_mod.kde(np.array([0.0], np.float32), 1.0, [0.0])[0] == pytest.approx(PHI0, rel=1e-15)
    # one sample at a, point at a + h: phi(1)/h
    f = oracle_mod.kde(np.array([1.5], np.float32), 0.25, [1.75, 1.25])
    assert f[0] == pytest.approx(PHI1 / 0.25, rel=1e-14)
    assert f[1] == f[0]


def test_mirror_symmetry_exact(oracle_mod):
    # X = {-1, 1} -> f(x) = f(-x) exactly, any h
    x = np.array([-1.0, 1.0], np.float32)
    for h in (0.3, 1.0, 2.7):
        pts = np.array([0.1, 0.77, 1.5, 3.0])
        assert np.array_equal(oracle_mod.kde(x, h, pts), oracle_mod.kde(x, h, -pts))


@pytest.mark.parametrize("seed", [0, 1])
def test_unit_mass_mean_and_variance(oracle_mod, seed):
    # f is an equal-weight mixture of N(X_i, h^2): mass 1, mean X-bar,
    # variance h^2 + (1/n) sum (X_i - X-bar)^2 (trapezoid is spectrally exact for Gaussians)
    x = inputs.mixture(300, seed)
    xd = x.astype(np.float64)
    h = 0.2
    grid = np.linspace(xd.min() - 12 * h, xd.max() + 12 * h, 6001)
    f = oracle_mod.kde(x, h, grid)
    mass = _trapz(f, grid)
    mean = _trapz(grid * f, grid)
    var = _trapz((grid - xd.mean()) ** 2 * f, grid)
    assert mass == pytest.approx(1.0, abs=1e-12)
    assert mean == pytest.approx(xd.mean(), abs=1e-10)
    assert var == pytest.approx(h * h + np.mean((xd - xd.mean()) ** 2), rel=1e-10)


def test_toy_data_curve_integrates_to_one(oracle_mod):
    # the toy data of P:51 with its PLUGIN h (0.96146759322923324)
    x = inputs.TOY.astype(np.float32)
    h = 0.96146759322923324
    grid = np.linspace(float(x.min()) - 5 * h, float(x.max()) + 5 * h, 4001)
    f = oracle_mod.kde(x, h, grid)
    assert np.all(f > 0)
    assert 0.99 <= _trapz(f, grid) <= 1.01


def test_matches_scipy_gaussian_kde(oracle_mod):
    # scipy's bandwidth is bw_method * std(X, ddof=1); pick it so that it equals h
    x = inputs.normal(500, 11, mean=3.0, sd=2.0)
    xd = x.astype(np.float64)
    h = 0.37
    ref = stats.gaussian_kde(xd, bw_method=h / np.std(xd, ddof=1))
    pts = np.linspace(-4, 10, 57)
    assert np.allclose(oracle_mod.kde(x, h, pts), ref(pts), rtol=1e-12, atol=0)


@pytest.mark.parametrize("n", [2, 5, 9])
def test_mpmath_brute_force(oracle_mod, n):
    mp.mp.dps = 50
    x = inputs.normal(n, 40 + n)
    h = 0.61
    pts = [-1.3, 0.0, 0.2, 2.9]
    got = oracle_mod.kde(x, h, pts)
    for p, g in zip(pts, got):
        ref = mp.fsum(mp.exp(-((mp.mpf(p) - mp.mpf(float(v))) / h) ** 2 / 2) for v in x)
        ref = ref / (mp.sqrt(2 * mp.pi) * n * h)
        assert g == pytest.approx(float(ref), rel=1e-14)


def test_convolution_identity(oracle_mod):
    # int f(x)^2 dx = n^-2 sum_i sum_j phi_{h sqrt2}(X_i - X_j)   (phi_a * phi_b = phi_sqrt(a^2+b^2))
    x = inputs.mixture(120, 5)
    xd = x.astype(np.float64)
    h = 0.3
    grid = np.linspace(xd.min() - 12 * h, xd.max() + 12 * h, 8001)
    f = oracle_mod.kde(x, h, grid)
    s = h * math.sqrt(2.0)
    d = xd[:, None] - xd[None, :]
    pair = np.sum(np.exp(-0.5 * (d / s) ** 2)) / (math.sqrt(2 * math.pi) * s) / xd.size ** 2
    assert _trapz(f * f, grid) == pytest.approx(pair, rel=1e-11)


def test_translation_and_power_of_two_scaling(oracle_mod):
    x = inputs.mixture(200, 8)
    pts = np.linspace(-6, 6, 31).astype(np.float32).astype(np.float64)
    f = oracle_mod.kde(x, 0.4, pts)
    # scaling samples, points and h by 2^k scales f by 2^-k exactly
    f2 = oracle_mod.kde(x * np.float32(8.0), 3.2, pts * 8.0)
    assert np.array_equal(f2 * 8.0, f)
    # shift: on dyadic data (X + 2 exact in float32) equal to fp64 rounding
    xq = (np.round(x.astype(np.float64) * 1024) / 1024).astype(np.float32)
    f = oracle_mod.kde(xq, 0.4, pts)
    f3 = oracle_mod.kde(xq + np.float32(2.0), 0.4, pts + 2.0)
    assert np.allclose(f3, f, rtol=1e-13, atol=0)


def test_rejects_bad_bandwidth(oracle_mod):
    with pytest.raises(ValueError):
        oracle_mod.kde(np.zeros(3, np.float32), 0.0, [0.0])
