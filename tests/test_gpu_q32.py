"""GPU parity of the Q32.32 datapath against the oracle:
bit-exact integer totals for the pair sums (integer work: bit-exact is the bar), and h of the
whole algorithm within the paper's fixed-point accuracy (Table 4, 4.2e-6 relative)."""
import math

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
