"""GPU parity of kde_eval (Eq. 1-2) against the fp64 oracle.

Tolerance, derived from the fp32 term evaluation: with d = fl(x - X),
a = fl(fl(d k) d), k = fl(-log2(e)/(2h^2)), the exponent carries a relative error <= 5 * 2^-24,
so each term exp2(a) is off by <= ln2 * 3e-7 * |a| relatively, plus <= 2 ulp for ex2.approx and
<= 64 * 2^-24 for the fp32 chunk sums.  All terms are positive, so the bound per point is
5e-6 + 2.1e-7 * |a_min| (a_min: the exponent of the sample nearest the point).  Terms below
2^-126.5 are exactly zero on MUFU.EX2 and at most 2^-125.5 on the FMA-pipe exp of the hybrid
kernel (its exponent is clamped at -126): an absolute slack of 2^-124 phi(0)/h per point.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1505_02100_b200 import inputs  # noqa: E402

pytestmark = pytest.mark.gpu
LOG2E_2 = 0.5 * 1.4426950408889634


@pytest.fixture(scope="module")
def P():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1505_02100_b200 import plugin
    plugin.lib()
    return plugin


def _check(oracle_mod, P, x, h, pts, got=None):
    xs = np.sort(x.astype(np.float64))
    if got is None:
        got = P.kde_eval(torch.from_numpy(x).cuda(), h, torch.from_numpy(pts).cuda()).cpu().numpy()
    ref = oracle_mod.kde(x, h, pts.astype(np.float64))
    p = pts.astype(np.float64)
    k = np.clip(np.searchsorted(xs, p), 1, xs.size - 1) if xs.size > 1 else np.zeros(p.size, dtype=int)
    dmin = np.minimum(np.abs(p - xs[k]), np.abs(p - xs[k - 1])) if xs.size > 1 else np.abs(p - xs[0])
    amin = LOG2E_2 * (dmin / h) ** 2
    tol = (5e-6 + 2.1e-7 * amin) * ref + 2.0 ** -124 * 0.4 / h
    bad = ~(np.abs(got - ref) <= tol)
    assert not bad.any(), (int(bad.sum()), got[bad][:4], ref[bad][:4], p[bad][:4])
    return got, ref


@pytest.mark.parametrize("n", [1, 2, 31, 1025, 4097, 20000])
@pytest.mark.parametrize("m", [1, 7, 1023, 1025, 3000])
def test_kde_sweep_sorted_grid(P, oracle_mod, n, m):
    x = inputs.mixture(n, 100 + n) if n > 2 else inputs.normal(n, 7)
    h = 0.3
    lo, hi = float(x.min()) - 5 * h, float(x.max()) + 5 * h
    pts = np.linspace(lo, hi, m).astype(np.float32)
    _check(oracle_mod, P, x, h, pts)


@pytest.mark.parametrize("n", [33, 5000])
def test_kde_unsorted_points_and_far_tails(P, oracle_mod, n):
    x = inputs.normal(n, 3, mean=1.0, sd=2.0)
    rng = np.random.default_rng(5)
    pts = rng.uniform(-40, 40, 2500).astype(np.float32)   # many points where every term underflows
    got, ref = _check(oracle_mod, P, x, 0.5, pts)
    assert np.all(got >= 0)


@pytest.mark.parametrize("h", [1e-3, 0.05, 3.0, 1e3])
def test_kde_bandwidth_range(P, oracle_mod, h):
    x = inputs.mixture(3000, 21)
    pts = np.concatenate([x[:200], np.linspace(-8, 8, 301, dtype=np.float32)])  # points on samples too
    _check(oracle_mod, P, x, h, pts)


@pytest.mark.parametrize("case", ["ties", "offset"])
def test_kde_adversarial(P, oracle_mod, case):
    x = inputs.ties(6000, 2) if case == "ties" else inputs.offset(6000, 2)
    h = 0.2
    pts = np.linspace(float(x.min()) - 3, float(x.max()) + 3, 2001).astype(np.float32)
    _check(oracle_mod, P, x, h, pts)


def test_kde_single_sample_closed_form(P):
    # X = {0}, h = 1, x = 0 -> 1/sqrt(2 pi); X = {1.5}, h = 0.25, x = 1.75 -> phi(1)/h
    f = P.kde_eval(torch.tensor([0.0], device="cuda"), 1.0, torch.tensor([0.0], device="cuda")).item()
    assert f == pytest.approx(0.3989422804014327, rel=1e-7)
    f = P.kde_eval(torch.tensor([1.5], device="cuda"), 0.25, torch.tensor([1.75, 1.25], device="cuda")).cpu()
    assert f[0].item() == pytest.approx(0.24197072451914337 / 0.25, rel=2e-6)
    assert f[0].item() == f[1].item()


def test_kde_nonfinite_and_empty(P):
    x = torch.tensor([0.0, float("nan"), 1.0], device="cuda")
    f = P.kde_eval(x, 0.5, torch.tensor([0.0, 2.0], device="cuda")).cpu()
    assert torch.isnan(f).all()
    x = torch.tensor([0.0, 1.0], device="cuda")
    f = P.kde_eval(x, 0.5, torch.tensor([0.0, float("nan"), 1.0], device="cuda")).cpu()
    assert math.isnan(f[1].item()) and not math.isnan(f[0].item()) and f[0].item() == f[2].item()
    out = P.kde_eval(x, 0.5, torch.empty(0, device="cuda"))
    assert out.numel() == 0
    with pytest.raises(P.PluginError):
        P.kde_eval(x, 0.0, torch.tensor([0.0], device="cuda"))


def test_kde_mufu_only_variant_agrees(P, oracle_mod):
    # the MUFU-only kernel (PLUGIN_KDE_MUFU_ONLY=1, read once per process) in a subprocess
    import subprocess
    import sys
    code = ("import torch, numpy as np; from paper_1505_02100_b200 import plugin as P, inputs;"
            "x=torch.from_numpy(inputs.mixture(30000, 6)).cuda();"
            "f=P.kde_eval(x, 0.15, torch.linspace(-9, 9, 4000, device='cuda')).cpu().numpy();"
            "np.save('/tmp/kde_mufu.npy', f)")
    env = dict(__import__("os").environ, PLUGIN_KDE_MUFU_ONLY="1")
    subprocess.check_call([sys.executable, "-c", code], env=env)
    mufu = np.load("/tmp/kde_mufu.npy")
    x = inputs.mixture(30000, 6)
    pts = torch.linspace(-9, 9, 4000, device="cuda")
    hyb = P.kde_eval(torch.from_numpy(x).cuda(), 0.15, pts).cpu().numpy()
    _check(oracle_mod, P, x, 0.15, pts.cpu().numpy(), got=mufu)
    _check(oracle_mod, P, x, 0.15, pts.cpu().numpy(), got=hyb)


def test_kde_deterministic_and_permutation_invariant(P):
    x = inputs.mixture(50000, 4)
    pts = torch.linspace(-8, 8, 5000, device="cuda")
    a = P.kde_eval(torch.from_numpy(x).cuda(), 0.1, pts).cpu()
    b = P.kde_eval(torch.from_numpy(x).cuda(), 0.1, pts).cpu()
    c = P.kde_eval(torch.from_numpy(np.random.default_rng(1).permutation(x)).cuda(), 0.1, pts).cpu()
    assert torch.equal(a, b) and torch.equal(a, c)


@pytest.mark.parametrize("k", [4, 5])
def test_kde_full_size_sampled_points(P, oracle_mod, k):
    # BASELINE config k at full n, 65536-point curve over [min - 4h, max + 4h] as bench.py runs
    # it; the oracle checks 192 sampled points one by one (each an O(n) sum)
    x = inputs.config_data(k)
    h = 0.1326215 if k == 4 else 0.05  # fixed bandwidths (cfg4: its PLUGIN h rounded; not from the GPU)
    pts = np.linspace(float(x.min()) - 4 * h, float(x.max()) + 4 * h, 65536).astype(np.float32)
    got = P.kde_eval(torch.from_numpy(x).cuda(), h, torch.from_numpy(pts).cuda()).cpu().numpy()
    idx = np.unique(np.concatenate([np.arange(0, 65536, 347), [0, 1, 32767, 65534, 65535]]))
    _check(oracle_mod, P, x, h, pts[idx], got=got[idx])
    # unit mass of the whole curve (trapezoid)
    mass = float(np.sum((got[1:] + got[:-1]) * np.diff(pts.astype(np.float64))) / 2)
    assert mass == pytest.approx(1.0, abs=1e-4)


def test_kde_prepare_then_eval_equals_kde_eval(P):
    x = torch.from_numpy(inputs.mixture(40000, 9)).cuda()
    pts = torch.linspace(-7, 7, 3001, device="cuda")
    a = P.kde_eval(x, 0.12, pts).cpu()
    ws = P.kde_workspace(x.numel(), pts.numel(), x.device)
    P.kde_prepare(x, ws)
    b = P.kde_eval_prepared(x.numel(), 0.12, pts, ws).cpu()
    c = P.kde_eval_prepared(x.numel(), 0.12, pts[:1000].contiguous(), ws).cpu()   # re-use
    assert torch.equal(a, b)
    # another point set: other windows, segment splits and fp32 chunks -- equal within the
    # fp32 evaluation tolerance of this file
    assert torch.allclose(a[:1000], c, rtol=5e-6, atol=2.0 ** -124 * 0.4 / 0.12)
