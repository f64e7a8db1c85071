"""GPU parity of the grouped exact pass (group.cu): heavily tied samples (at most n/4 distinct
values, n >= 32768) are evaluated as sum_a sum_b c_a c_b K^(r)((v_a - v_b)/g) over distinct
values in fp64 -- an identity with the double sum of Eq. 6/7.  The result
must match the fp64 oracle (which evaluates the plain double sum, never grouping) to 1e-11
relative: both are binary64 evaluations of the same number."""
import json
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1505_02100_b200 import inputs  # noqa: E402

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
TOL_FP64 = 1e-11


@pytest.fixture(scope="module")
def P():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1505_02100_b200 import plugin
    plugin.lib()
    return plugin


def rel(a, b):
    return abs(a - b) / abs(b)


def _grid(n, q, seed, sd=1.0):
    return (np.round(np.random.default_rng(seed).normal(0, sd, n) / q) * q).astype(np.float32)


TIED = {
    "ties40k": lambda: inputs.ties(40000, 21),
    "integers": lambda: np.round(inputs.normal(50000, 22, sd=5)).astype(np.float32),
    "offset1e6": lambda: inputs.offset(40000, 23),
    "grid0.01": lambda: _grid(100000, 0.01, 24),
    "two_values": lambda: np.where(np.random.default_rng(25).random(60000) < 0.3, 1.5, -0.25).astype(np.float32),
}


@pytest.mark.parametrize("case", list(TIED))
def test_grouped_plugin_h_matches_oracle(P, oracle_mod, case):
    x = TIED[case]()
    assert np.unique(x).size * 4 <= x.size
    r = P.plugin_h_sync(torch.from_numpy(x).cuda())
    assert r["status"] == 0
    assert r["path"] & P.PLUGIN_PATH_GROUPED
    o = oracle_mod.plugin(x)
    for key in ("psi6_z", "psi4_z", "h", "g1", "g2", "sigma"):
        assert rel(r[key], o[key]) < TOL_FP64, (case, key, r[key], o[key], rel(r[key], o[key]))


def test_rounded_cfg4_takes_the_grouped_path_exactly(P):
    with open(os.path.join(HERE, "golden", "cfg4r.json")) as f:
        g = json.load(f)
    x = inputs.rounded_data("4r")
    r = P.plugin_h_sync(torch.from_numpy(x).cuda())
    assert r["status"] == 0 and r["path"] & P.PLUGIN_PATH_GROUPED
    for key in ("psi6_z", "psi4_z", "h", "g1", "g2"):
        assert rel(r[key], g[key]) < TOL_FP64, (key, r[key], g[key], rel(r[key], g[key]))


@pytest.mark.parametrize("extra", [0, 1])
def test_threshold_n_over_4_distinct(P, oracle_mod, extra):
    # exactly n/4 distinct values -> grouped; one more -> the fp32 tile pass (1e-5)
    n = 40000
    rng = np.random.default_rng(26)
    base = np.round(rng.normal(0, 1, n - n // 4) * 40) / 40       # ~300 grid values, many ties
    uniq = np.unique(base)
    need = n // 4 + extra - uniq.size
    fresh = np.setdiff1d(np.round(rng.normal(0, 1, 4 * need) * 1e4) / 1e4 + 1e-5, uniq)[:need]
    x = np.concatenate([base, fresh, np.full(n - base.size - need, uniq[0])]).astype(np.float32)
    rng.shuffle(x)
    assert x.size == n and np.unique(x).size == n // 4 + extra
    r = P.plugin_h_sync(torch.from_numpy(x).cuda())
    o = oracle_mod.plugin(x)
    grouped = bool(r["path"] & P.PLUGIN_PATH_GROUPED)
    assert grouped == (extra == 0)
    tol = TOL_FP64 if grouped else 1e-5
    for key in ("psi6_z", "psi4_z", "h"):
        assert rel(r[key], o[key]) < tol, (extra, key, r[key], o[key])


def test_not_grouped_below_min_n_or_continuous(P):
    a = P.plugin_h_sync(torch.from_numpy(inputs.ties(20000, 27)).cuda())      # n < 32768
    b = P.plugin_h_sync(torch.from_numpy(inputs.config_data(3)).cuda())       # continuous
    assert not (a["path"] & P.PLUGIN_PATH_GROUPED) and not (b["path"] & P.PLUGIN_PATH_GROUPED)


@pytest.mark.parametrize("r", [4, 6, 8, 12])
def test_grouped_psi_r(P, oracle_mod, r):
    x = TIED["integers"]()
    for g in (0.7, 2.5):
        got = P.psi_r(torch.from_numpy(x).cuda(), g, r).item()
        ref = oracle_mod.psi(oracle_mod.widen(x), g, r)
        # two binary64 evaluations of a sum whose cancellation grows like g^-r:
        # at r = 12 and an oversmoothing g both carry ~1e-11
        assert rel(got, ref) < (TOL_FP64 if r <= 8 else 1e-10), (r, g, got, ref)


@pytest.mark.parametrize("world", [2, 3, 7])
def test_grouped_shards_sum_to_single_gpu_bit_exact(P, world):
    xh = TIED["grid0.01"]()
    x = torch.from_numpy(xh).cuda()
    n = x.numel()
    ref = P.plugin_h_sync(x)
    assert ref["path"] & P.PLUGIN_PATH_GROUPED
    ws = P.workspace(n)
    out = P.new_result()
    P.plugin_step1(x, out, ws)
    for r, after in ((6, P.plugin_after_psi6), (4, P.plugin_after_psi4)):
        tot = torch.zeros(4, dtype=torch.int64, device="cuda")
        for rank in range(world):
            part = P.new_partial()
            P.psi_r_shard(n, r, rank, world, out, part, ws)
            tot += part
        after(tot, out)
    got = P.read_result(out)
    for k in ("psi6", "g2", "psi4", "h"):
        assert got[k] == ref[k], (k, got[k], ref[k])


def test_grouped_dpi_matches_oracle(P, oracle_mod):
    x = TIED["ties40k"]()
    got = P.read_dpi_result(P.plugin_dpi(torch.from_numpy(x).cuda(), 3))
    ref = oracle_mod.dpi(x, 3)
    assert got["status"] == 0
    assert rel(got["h"], ref["h"]) < TOL_FP64, (got["h"], ref["h"])


def test_grouped_permutation_and_graph(P):
    x = TIED["offset1e6"]()
    a = P.plugin_h_sync(torch.from_numpy(x).cuda())
    p = np.random.default_rng(28).permutation(x.size)
    b = P.plugin_h_sync(torch.from_numpy(np.ascontiguousarray(x[p])).cuda())
    xt = torch.from_numpy(x).cuda()
    g = P.PluginGraph(xt)
    c = P.read_result(g.launch())
    g.close()
    for k in ("psi6", "psi4", "h"):
        assert a[k] == b[k] == c[k]
    assert not math.isnan(a["h"])


@pytest.mark.parametrize("n", [32767, 32768])
def test_group_min_n_boundary(P, oracle_mod, n):
    # kGroupMinN = 32768: a heavily tied sample one below takes the fp32 pass (1e-5), at it the
    # grouped exact pass (fp64)
    x = inputs.ties(n, 41)
    r = P.plugin_h_sync(torch.from_numpy(x).cuda())
    o = oracle_mod.plugin(x)
    grouped = bool(r["path"] & P.PLUGIN_PATH_GROUPED)
    assert grouped == (n >= 32768)
    tol = TOL_FP64 if grouped else 1e-5
    for key in ("psi6_z", "psi4_z", "h"):
        assert rel(r[key], o[key]) < tol, (n, key, r[key], o[key])


def test_grouped_flags_and_statuses(P):
    x = TIED["integers"]()
    xt = torch.from_numpy(x).cuda()
    a = P.read_result(P.plugin_h(xt))
    b = P.read_result(P.plugin_h(xt, flags=P.PLUGIN_SKIP_UNDERFLOW))   # the grouped pass skips exactly too
    assert a["path"] & P.PLUGIN_PATH_GROUPED and all(a[k] == b[k] for k in a)
    # a non-finite value or zero variance: the data status wins, no grouped pass
    bad = x.copy()
    bad[123] = np.nan
    r = P.plugin_h_sync(torch.from_numpy(bad).cuda())
    assert r["status"] == P.PLUGIN_E_NONFINITE and not (r["path"] & P.PLUGIN_PATH_GROUPED) and math.isnan(r["h"])
    const = np.full(40000, 2.5, np.float32)
    r = P.plugin_h_sync(torch.from_numpy(const).cuda())
    assert r["status"] == P.PLUGIN_E_DEGENERATE and math.isnan(r["h"])
