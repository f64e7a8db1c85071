"""GPU parity of the Q32.32 datapath against the oracle:
bit-exact integer totals for the pair sums (integer work: bit-exact is the bar), and h of the
whole algorithm within the paper's fixed-point accuracy (Table 4, 4.2e-6 relative)."""
import json
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1505_02100_b200 import inputs  # noqa: E402

pytestmark = pytest.mark.gpu
ONE = 1 << 32


@pytest.fixture(scope="module")
def P():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1505_02100_b200 import plugin
    plugin.lib()
    return plugin


@pytest.mark.parametrize("n", [1, 2, 255, 1024, 1025, 3000])
@pytest.mark.parametrize("r", [4, 6])
def test_psi_q32_bit_exact(P, oracle_mod, n, r):
    x = inputs.mixture(n, 900 + n) if n > 2 else inputs.normal(n, 9)
    z = (x.astype(np.float64) - 0.3) / 1.7
    zq = oracle_mod.q32_encode(z)
    for g in (0.35, 0.9):
        rg = int(oracle_mod.q32_encode([1.0 / g])[0])
        got = P.psi_r_q32(torch.from_numpy(zq).cuda(), rg, r)
        half = oracle_mod.q32_psi_sum(zq, rg, r)
        assert got == 2 * half + n * oracle_mod.q32_term(0, rg, r), (n, r, g)


def test_psi_q32_order_free(P, oracle_mod):
    zq = oracle_mod.q32_encode(inputs.mixture(5000, 3).astype(np.float64))
    rg = int(oracle_mod.q32_encode([1 / 0.3])[0])
    a = P.psi_r_q32(torch.from_numpy(zq).cuda(), rg, 6)
    b = P.psi_r_q32(torch.from_numpy(np.random.default_rng(0).permutation(zq)).cuda(), rg, 6)
    assert a == b


@pytest.mark.parametrize("case", ["cfg1", "n512", "cfg2"])
def test_plugin_h_q32(P, oracle_mod, case):
    x = inputs.config_data(1) if case == "cfg1" else (inputs.normal(512, 103) if case == "n512"
                                                         else inputs.config_data(2))
    got = P.read_result(P.plugin_h_q32(torch.from_numpy(x).cuda()))
    q = oracle_mod.q32_plugin(x)
    f = oracle_mod.plugin(x)
    assert got["status"] == 0
    # vs the Q32.32 oracle: the same datapath (z may differ by an ulp through Step I rounding)
    for k in ("psi6_z", "psi4_z", "h"):
        assert abs(got[k] - q[k]) / abs(q[k]) < 1e-6, (k, got[k], q[k])
    # vs fp64: the paper's Table 4 bound on h
    assert abs(got["h"] - f["h"]) / f["h"] <= 4.2e-6


def test_q32_errors(P):
    zq = torch.zeros(10, dtype=torch.int64, device="cuda")
    with pytest.raises(P.PluginError):
        P.psi_r_q32(zq, 0, 4)
    with pytest.raises(P.PluginError):
        P.psi_r_q32(zq, ONE, 5)
    r = P.read_result(P.plugin_h_q32(torch.full((100,), 1.5, device="cuda")))
    assert r["status"] == P.PLUGIN_E_DEGENERATE and math.isnan(r["h"])


TABLE4 = {}


@pytest.fixture(scope="module", autouse=True)
def _dump_table4():
    # a Table 4-style accuracy table on the synthetic stand-in data, written next to
    # the GPU evidence when gpurun_out/ exists
    yield
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    if TABLE4 and os.path.isdir(out):
        with open(os.path.join(out, "table4.json"), "w") as f:
            json.dump(TABLE4, f, indent=1, sort_keys=True)


@pytest.mark.parametrize("n", list(range(128, 1025, 128)))
def test_table4_accuracy_at_the_papers_sizes(P, oracle_mod, n):
    # Table 4 reports |h - h_ref| / h_ref of the FPGA's Q32.32 designs against an fp64 C++ h_ref,
    # at most 4.2e-6.  Here: the fp32 GPU path and the Q32.32 GPU path against the fp64
    # oracle on N(0,1) samples of the paper's sizes (seeds 100..107)
    x = inputs.normal(n, 100 + n // 128 - 1)
    ref = oracle_mod.plugin(x)["h"]
    xt = torch.from_numpy(x).cuda()
    h32 = P.read_result(P.plugin_h(xt))["h"]
    hq = P.read_result(P.plugin_h_q32(xt))["h"]
    TABLE4[n] = {"h_ref": ref, "fp32_path": h32, "q32_path": hq, "rel_fp32": abs(h32 - ref) / ref,
                 "rel_q32": abs(hq - ref) / ref}
    assert TABLE4[n]["rel_fp32"] <= 4.2e-6 and TABLE4[n]["rel_q32"] <= 4.2e-6


def test_psi_q32_far_pairs_bit_exact(P, oracle_mod):
    # differences up to 1e5 bandwidths: the far terms are exactly 0 on both sides
    rng = np.random.default_rng(5)
    z = np.concatenate([rng.normal(0, 1, 3000), [5e4, -5e4, 2e4]])
    zq = oracle_mod.q32_encode(z)
    rg = ONE
    got = P.psi_r_q32(torch.from_numpy(zq).cuda(), rg, 4)
    assert got == 2 * oracle_mod.q32_psi_sum(zq, rg, 4) + zq.size * oracle_mod.q32_term(0, rg, 4)


def test_psi_q32_extreme_values_bit_exact(P, oracle_mod):
    # Q32.32 values near the int64 limits (|d| rg >= 2^95): their pairs are far (term 0) on
    # both sides, judged on the exact product (q32.cu q32_term), never on a wrapped one
    zq = oracle_mod.q32_encode(np.random.default_rng(6).normal(0, 1, 2000))
    zq = np.concatenate([zq, np.array([(1 << 62), -(1 << 62), (1 << 63) - 1, -(1 << 63)], dtype=np.int64)])
    for rg in (ONE, (1 << 51) + 12345):
        got = P.psi_r_q32(torch.from_numpy(zq).cuda(), rg, 6)
        assert got == 2 * oracle_mod.q32_psi_sum(zq, rg, 6) + zq.size * oracle_mod.q32_term(0, rg, 6)
