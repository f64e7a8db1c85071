"""GPU parity of the general even-r passes and the l-stage direct plug-in
against the fp64 oracle (oracle.psi with the Hermite K^(r), oracle.dpi).  Tolerance: 1e-5
relative as for Alg. 1 (BASELINE.json north_star); l = 2 must equal plugin_h bit for bit."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1505_02100_b200 import inputs  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 1e-5


@pytest.fixture(scope="module")
def P():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1505_02100_b200 import plugin
    plugin.lib()
    return plugin


def rel(a, b):
    return abs(a - b) / abs(b)


@pytest.mark.parametrize("r", [0, 2, 8, 10, 12])
@pytest.mark.parametrize("n", [1, 33, 257, 1025, 5000])
def test_psi_r_general_order(P, oracle_mod, r, n):
    x = inputs.mixture(n, 500 + n) if n > 1 else np.array([0.7], np.float32)
    for g in (0.4, 1.1):
        got = P.psi_r(torch.from_numpy(x).cuda(), g, r).item()
        ref = oracle_mod.psi(oracle_mod.widen(x), g, r)
        assert rel(got, ref) < TOL, (n, r, g, got, ref)


@pytest.mark.parametrize("stages", [0, 1, 2, 3, 4, 5])
@pytest.mark.parametrize("case", ["mixture", "cfg1", "cfg2"])
def test_dpi_matches_oracle(P, oracle_mod, stages, case):
    x = inputs.mixture(20000, 8) if case == "mixture" else inputs.config_data(int(case[-1]))
    got = P.read_dpi_result(P.plugin_dpi(torch.from_numpy(x).cuda(), stages))
    ref = oracle_mod.dpi(x, stages)
    assert got["status"] == 0
    assert rel(got["h"], ref["h"]) < TOL
    for j in range(1, stages + 1):
        assert rel(got["g_z"][j], ref["g_z"][j]) < TOL, (j, got["g_z"][j], ref["g_z"][j])
        assert rel(got["psi_z"][j], ref["psi_z"][j]) < TOL, (j, got["psi_z"][j], ref["psi_z"][j])


@pytest.mark.parametrize("k", [2, 3])
def test_dpi_two_stage_is_plugin_h_bit_for_bit(P, k):
    x = torch.from_numpy(inputs.config_data(k)).cuda()
    a = P.read_result(P.plugin_h(x, flags=P.PLUGIN_MULTI_KERNEL))
    b = P.read_dpi_result(P.plugin_dpi(x, 2))
    assert b["h"] == a["h"] and b["h_z"] == a["h_z"]
    assert b["g_z"][2] == a["g1_z"] and b["psi_z"][2] == a["psi6_z"]
    assert b["g_z"][1] == a["g2_z"] and b["psi_z"][1] == a["psi4_z"]


def test_dpi_zero_stage_normal_reference(P):
    x = inputs.normal(4000, 2, mean=-1.0, sd=3.0)
    b = P.read_dpi_result(P.plugin_dpi(torch.from_numpy(x).cuda(), 0))
    assert rel(b["h"], (4.0 / (3.0 * 4000)) ** 0.2 * b["sigma"]) < 1e-14


def test_dpi_errors(P):
    x = torch.from_numpy(inputs.normal(100, 1)).cuda()
    with pytest.raises(P.PluginError):
        P.plugin_dpi(x, 6)
    with pytest.raises(P.PluginError):
        P.psi_r(x, 0.5, 3)
    c = torch.full((64,), 2.0, device="cuda")
    assert P.read_dpi_result(P.plugin_dpi(c, 3))["status"] == P.PLUGIN_E_DEGENERATE
    assert math.isnan(P.read_dpi_result(P.plugin_dpi(c, 3))["h"])


@pytest.mark.parametrize("stages", [3, 5])
def test_dpi_at_config3_size(P, oracle_mod, stages):
    # the higher-order passes (r = 8 .. 12) cancel more (C ~ g^-r): check them at n = 131072
    # (BASELINE config 3) against the oracle (its 3-5 passes take ~10-20 s on the GPU box)
    x = inputs.config_data(3)
    got = P.read_dpi_result(P.plugin_dpi(torch.from_numpy(x).cuda(), stages))
    ref = oracle_mod.dpi(x, stages)
    assert got["status"] == 0
    assert rel(got["h"], ref["h"]) < TOL
    for j in range(1, stages + 1):
        assert rel(got["psi_z"][j], ref["psi_z"][j]) < TOL, (j, got["psi_z"][j], ref["psi_z"][j])
