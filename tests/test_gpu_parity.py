"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Tolerance: relative 1e-5 on psi6, psi4 and h (BASELINE.json north_star).  Values of
the five BASELINE configurations come from tests/golden/cfg*.json, written by
`python -m oracle.make_golden` (oracle/ only).  Smaller cases call the oracle here.
"""
import json
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1505_02100_b200 import inputs  # noqa: E402

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
TOL = 1e-5


@pytest.fixture(scope="module")
def P():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1505_02100_b200 import plugin
    plugin.lib()
    return plugin


def rel(a, b):
    return abs(a - b) / abs(b)


def _golden(k):
    p = os.path.join(HERE, "golden", f"cfg{k}.json")
    if not os.path.exists(p):
        pytest.skip(f"golden cfg{k} not generated yet (python -m oracle.make_golden {k})")
    with open(p) as f:
        g = json.load(f)
    assert g["sha256"] == inputs.SHA256[k]
    return g


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_plugin_h_matches_oracle_on_baseline_configs(P, k):
    g = _golden(k)
    x = torch.from_numpy(inputs.config_data(k)).cuda()
    r = P.plugin_h_sync(x)
    assert r["status"] == 0
    for key in ("psi6_z", "psi4_z", "h_z", "psi6", "psi4", "h", "g1", "g2", "sigma"):
        assert rel(r[key], g[key]) < TOL, (key, r[key], g[key], rel(r[key], g[key]))


@pytest.mark.parametrize("name", list(inputs.ROUNDED))
def test_plugin_h_matches_oracle_on_rounded_configs(P, name):
    # BASELINE configs rounded to a grid (cfg4 to 0.01: n = 2^20 on 1631 distinct values,
    # cancellation ~2e4 on psi6): golden values written by oracle.make_golden (oracle/ only)
    p = os.path.join(HERE, "golden", f"cfg{name}.json")
    with open(p) as f:
        g = json.load(f)
    x = inputs.rounded_data(name)
    assert inputs.sha256_f32(x) == g["sha256"]
    r = P.plugin_h_sync(torch.from_numpy(x).cuda())
    assert r["status"] == 0
    for key in ("psi6_z", "psi4_z", "h_z", "psi6", "psi4", "h", "g1", "g2", "sigma"):
        assert rel(r[key], g[key]) < TOL, (key, r[key], g[key], rel(r[key], g[key]))


@pytest.mark.parametrize("n", [1, 2, 3, 31, 32, 33, 255, 256, 257, 1023, 1025, 4097, 9000])
@pytest.mark.parametrize("r", [4, 6])
def test_psi_r_small_sweep(P, oracle_mod, n, r):
    # tile edges (T = 256, 512, ...) and ragged tails; raw units, g given
    x = inputs.normal(n, 1000 + n, mean=0.5, sd=1.3)
    for gscale in (0.25, 1.0):
        g = gscale * 1.3
        got = P.psi_r(torch.from_numpy(x).cuda(), g, r).item()
        ref = oracle_mod.psi(oracle_mod.widen(x), g, r)
        assert rel(got, ref) < TOL, (n, r, g, got, ref)


def _grid(n, q, seed):
    return (np.round(np.random.default_rng(seed).standard_normal(n) / q) * q).astype(np.float32)


# Discretised samples (few distinct differences, so the fp32 rounding of each
# repeated difference must not be systematic): values on coarse grids, integers, 1e6 + N(0,1)
# quantised by float32 (0.0625 steps), 3e4 + N(0,1) (2^-9 steps), heavy ties
ADVERSARIAL = {
    "mixture": lambda: inputs.mixture(20000, 3),
    "ties": lambda: inputs.ties(12000, 4),
    "ties20": lambda: inputs.ties(20000, 7, levels=20),
    "ties60": lambda: inputs.ties(30000, 11, levels=60),
    "integers": lambda: np.round(inputs.normal(20000, 12, sd=5)).astype(np.float32),
    "offset": lambda: inputs.offset(12000, 5),
    "offset3e4": lambda: inputs.offset(20000, 8, base=3.0e4),
    "grid001": lambda: _grid(20000, 0.001, 31),
    "grid0001": lambda: _grid(20000, 0.0001, 31),
    "normal_small": lambda: inputs.normal(2, 6),
    "toy": lambda: inputs.TOY.astype(np.float32),
}


@pytest.mark.parametrize("case", list(ADVERSARIAL))
def test_plugin_h_adversarial(P, oracle_mod, case):
    x = ADVERSARIAL[case]()
    o = oracle_mod.plugin(x)
    r = P.plugin_h_sync(torch.from_numpy(x).cuda())
    assert r["status"] == 0
    for key in ("psi6_z", "psi4_z", "h", "g1", "g2", "sigma"):
        assert rel(r[key], o[key]) < TOL, (case, key, r[key], o[key], rel(r[key], o[key]))


@pytest.mark.parametrize("g", [1.0, 0.5, 2.0 ** -3, 0.999999])
@pytest.mark.parametrize("r", [4, 6, 8])
def test_psi_r_power_of_two_scale(P, oracle_mod, g, r):
    # s = 1/g a power of two: the per-row scale dither s + k ulp(s) must stay symmetric where
    # s - |k| ulp(s) falls into the binade below (psi_tile.cuh dithered_scale); an oversmoothing
    # g makes the sum cancel strongly, so a one-sided dilation would show
    x = inputs.normal(5000, 5040)
    got = P.psi_r(torch.from_numpy(x).cuda(), g, r).item()
    ref = oracle_mod.psi(oracle_mod.widen(x), g, r)
    assert rel(got, ref) < TOL, (g, r, got, ref)


def test_two_point_closed_form(P):
    # n = 2: h = 0.74338814253112600 |a - b| (pinned in test_oracle_pins.py)
    for a, b in ((0.0, 1.0), (-3.0, 2.5)):
        r = P.plugin_h_sync(torch.tensor([a, b], dtype=torch.float32, device="cuda"))
        assert rel(r["h"], 0.74338814253112600 * abs(b - a)) < TOL


def test_psi_single_point(P):
    for r, k0 in ((6, -15 / math.sqrt(2 * math.pi)), (4, 3 / math.sqrt(2 * math.pi))):
        got = P.psi_r(torch.tensor([0.3], dtype=torch.float32, device="cuda"), 0.7, r).item()
        assert rel(got, k0 / 0.7 ** (r + 1)) < 1e-12


def test_deterministic_and_host_path_identical(P):
    xh = inputs.config_data(2)
    x = torch.from_numpy(xh).cuda()
    a = P.plugin_h_sync(x)
    b = P.plugin_h_sync(x)
    c = P.plugin_h_host(torch.from_numpy(xh).pin_memory())
    d = P.read_result(P.plugin_h(x))
    for k in a:
        if k != "n":
            assert a[k] == b[k] == c[k] == d[k] or (math.isnan(a[k]) and math.isnan(c[k])), k


@pytest.mark.parametrize("k2", [5, -7])
def test_pow2_scale_equivariance_bit_exact(P, k2):
    x = inputs.mixture(30000, 9)
    a = P.plugin_h_sync(torch.from_numpy(x).cuda())
    b = P.plugin_h_sync(torch.from_numpy((x * np.float32(2.0 ** k2)).astype(np.float32)).cuda())
    assert b["h"] == a["h"] * 2.0 ** k2
    assert b["psi6_z"] == a["psi6_z"] and b["psi4_z"] == a["psi4_z"]


def test_permutation_invariance_bit_exact(P):
    # the device sorts X first, so any permutation gives the identical result
    x = inputs.mixture(25000, 10)
    p = np.random.default_rng(1).permutation(x.size)
    a = P.plugin_h_sync(torch.from_numpy(x).cuda())
    b = P.plugin_h_sync(torch.from_numpy(np.ascontiguousarray(x[p])).cuda())
    assert a["h"] == b["h"] and a["psi6"] == b["psi6"]


@pytest.mark.parametrize("world", [2, 3, 8])
def test_shards_sum_to_single_gpu_bit_exact(P, world):
    """Every rank's psi_r_shard on one GPU, limbs summed on the host (what the NCCL
    allreduce does), finalised: identical bits to plugin_h."""
    xh = inputs.config_data(2)
    x = torch.from_numpy(xh).cuda()
    n = x.numel()
    ref = P.plugin_h_sync(x)
    ws = P.workspace(n)
    out = P.new_result()
    P.plugin_step1(x, out, ws)
    tot = torch.zeros(4, dtype=torch.int64, device="cuda")
    for rank in range(world):
        part = P.new_partial()
        P.psi_r_shard(n, 6, rank, world, out, part, ws)
        tot += part
    P.plugin_after_psi6(tot, out)
    tot.zero_()
    for rank in range(world):
        part = P.new_partial()
        P.psi_r_shard(n, 4, rank, world, out, part, ws)
        tot += part
    P.plugin_after_psi4(tot, out)
    r = P.read_result(out)
    for k in ("psi6", "g2", "psi4", "h"):
        assert r[k] == ref[k], (k, r[k], ref[k])


@pytest.mark.parametrize("n", [4400, 16384, 40000, 70000])
def test_scheduler_modes_same_result_and_shards_bit_exact(P, n, monkeypatch):
    """The pass scheduler (psi.cu): whole tiles from one counter (PLUGIN_PSI_TAIL=0), the remainder
    tiles as 64-column slices (1), slices plus the per-SM quota of the whole tiles (2; the default
    with 2000 to 5000 tiles).  In every mode the result is reproducible bit for bit, the shards of 3 ranks sum
    to plugin_h's bits (the items depend on n only), and the modes agree to fp64 rounding (the same
    fp32 pair terms, grouped into different items)."""
    xh = inputs.mixture(n, 4100 + n)
    x = torch.from_numpy(xh).cuda()
    ws = P.workspace(n)
    res = {}
    for mode in ("0", "1", "2", None):
        if mode is None:
            monkeypatch.delenv("PLUGIN_PSI_TAIL", raising=False)
        else:
            monkeypatch.setenv("PLUGIN_PSI_TAIL", mode)
        a, b = P.plugin_h_sync(x), P.plugin_h_sync(x)
        assert a["status"] == 0 and _same(a, b), mode
        out = P.new_result()
        P.plugin_step1(x, out, ws)
        for r, after in ((6, P.plugin_after_psi6), (4, P.plugin_after_psi4)):
            tot = torch.zeros(4, dtype=torch.int64, device="cuda")
            covered = 0
            for rank in range(3):
                part = P.new_partial()
                P.psi_r_shard(n, r, rank, 3, out, part, ws)
                tot += part
                ib, ie = P.plugin_shard_tiles(n, r, rank, 3)
                covered += ie - ib
            assert covered == P.plugin_num_tiles(n, r)
            after(tot, out)
        sh = P.read_result(out)
        for k in ("psi6", "g2", "psi4", "h"):
            assert sh[k] == a[k], (mode, k, sh[k], a[k])
        res[mode] = a
    T, tiles = P.plugin_tile_edge(n, 6), P.plugin_num_tiles(n, 6)        # (default mode again)
    nb = -(-n // T)
    whole = nb * (nb + 1) // 2
    assert (tiles > whole) == (2000 <= whole <= 5000)                     # slices by default only there
    assert _same(res[None], res["2" if tiles > whole else "0"])
    for mode in ("1", "2"):
        for k in ("psi6", "psi4", "h"):
            assert rel(res[mode][k], res["0"][k]) < 1e-12, (mode, k)


def test_data_errors(P):
    r = P.plugin_h_sync(torch.tensor([1.0, float("nan"), 2.0], device="cuda"))
    assert r["status"] == P.PLUGIN_E_NONFINITE and math.isnan(r["h"])
    r = P.plugin_h_sync(torch.full((5000,), 3.25, device="cuda"))
    assert r["status"] == P.PLUGIN_E_DEGENERATE and math.isnan(r["h"])
    assert math.isnan(P.psi_r(torch.tensor([1.0, float("inf")], device="cuda"), 1.0, 4).item())


def test_argument_errors(P):
    x = torch.randn(100, device="cuda")
    with pytest.raises(P.PluginError) as e:
        P.plugin_h_sync(x[:1])
    assert e.value.status == P.PLUGIN_E_INVALID
    for bad in (dict(g=0.0, r=4), dict(g=float("nan"), r=4), dict(g=1.0, r=5)):
        with pytest.raises(P.PluginError):
            P.psi_r(x, bad["g"], bad["r"])
    with pytest.raises(P.PluginError, match="workspace too small"):
        P.plugin_h(x, ws=P.workspace(10))


def _tile_coords(t, nb):
    # row-major upper block triangle incl. the diagonal (the order psi_r_shard walks)
    b = 0
    lo, hi = 0, nb - 1
    while lo < hi:                       # largest b with off(b) <= t, off(b) = b*nb - b(b-1)/2
        mid = (lo + hi + 1) // 2
        if mid * nb - mid * (mid - 1) // 2 <= t:
            lo = mid
        else:
            hi = mid - 1
    b = lo
    return b, b + (t - (b * nb - b * (b - 1) // 2))


@pytest.mark.parametrize("k", [3, 4, 5])
def test_full_size_sampled_tile_shards(P, oracle_mod, k):
    """Full-size configs in the launch configuration bench.py times (cfg3: R = 4 tiles, cfg4/5:
    R = 8): sampled tile ranges of both passes (psi_r_shard, exact fixed-point partials) against the oracle's block sums of
    the same pairs.  Bandwidths come from the oracle: g1 (Steps I-III, closed form) for r=6
    and 0.2 sigma for r=4 (the identity checked holds at any g)."""
    from paper_1505_02100_b200.distributed import from_limbs
    x = inputs.config_data(k)
    n = x.size
    s1 = oracle_mod.step1(x)
    sigma = s1["sigma"]
    g1 = oracle_mod.g1_bandwidth(oracle_mod.psi8_ns(1.0), n) * sigma
    g4 = 0.2 * sigma
    xd = torch.from_numpy(x).cuda()
    ws = P.workspace(n)
    P.plugin_step1(xd, P.new_result(), ws)           # sorts X into the workspace
    res = P.plugin_result()
    res.status, res.n, res.g1, res.g2 = 0, n, g1, g4
    dres = torch.frombuffer(bytearray(bytes(res)), dtype=torch.uint8).cuda()
    zs = np.sort(oracle_mod.widen(x))
    world = 1024
    phi0 = 1 / math.sqrt(2 * math.pi)
    for r, g in ((6, g1), (4, g4)):
        for rank in (0, world // 2, world - 1):
            part = P.new_partial()
            P.psi_r_shard(n, r, rank, world, dres, part, ws)
            got = from_limbs(part.cpu().tolist()) / 2.0 ** 64 * phi0
            ib, ie = P.plugin_shard_tiles(n, r, rank, world)
            ref = 0.0
            for it in range(ib, ie):        # each work item: a tile or a column slice of a remainder tile
                rows, cols, w = P.plugin_work_item(n, r, it)
                if cols[1] > cols[0]:
                    ref += w * oracle_mod.psi_block_sum(zs, g, r, *rows, *cols)
            assert rel(got, ref) < TOL, (k, r, rank, got, ref, rel(got, ref))


@pytest.mark.parametrize("k", [2, 3, 5])
def test_skip_underflow_tiles_bit_identical(P, k):
    # tiles whose every term is exactly 0 in fp32 are skipped; the
    # result must be bit-identical to the full evaluation (every field, both passes)
    x = torch.from_numpy(inputs.config_data(k)).cuda()
    ws = P.workspace(x.numel(), x.device)
    a = P.read_result(P.plugin_h(x, ws=ws))
    b = P.read_result(P.plugin_h(x, ws=ws, flags=P.PLUGIN_SKIP_UNDERFLOW))
    for key in a:
        assert a[key] == b[key] or (math.isnan(a[key]) and math.isnan(b[key])), (key, a[key], b[key])


def test_skip_underflow_far_clusters_bit_identical(P):
    # two clusters 1e3 bandwidths apart: almost every off-diagonal tile is skipped
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.normal(0, 1, 30000), rng.normal(400, 1, 30000)]).astype(np.float32)
    xt = torch.from_numpy(x).cuda()
    a = P.read_result(P.plugin_h(xt))
    b = P.read_result(P.plugin_h(xt, flags=P.PLUGIN_SKIP_UNDERFLOW))
    assert a["status"] == 0 and all(a[k] == b[k] for k in a if not (isinstance(a[k], float) and math.isnan(a[k])))
    with pytest.raises(P.PluginError):
        P.plugin_h(xt, flags=8)


def _same(a, b):
    return all(a[k] == b[k] or (isinstance(a[k], float) and math.isnan(a[k]) and math.isnan(b[k])) for k in a)


@pytest.mark.parametrize("n", [2, 3, 31, 63, 64, 65, 255, 256, 257, 1000, 1024, 1025, 2047, 2048, 2049, 4096])
def test_fused_small_n_bit_identical_to_multi_kernel(P, oracle_mod, n):
    # n <= 2048: plugin_h runs one thread-block-cluster launch (fused.cu); it must reproduce the
    # multi-kernel sequence bit for bit, and both must match the oracle
    x = inputs.mixture(n, 300 + n) if n > 3 else inputs.normal(n, 300 + n)
    xt = torch.from_numpy(x).cuda()
    ws = P.workspace(n, xt.device)
    a = P.read_result(P.plugin_h(xt, ws=ws))
    b = P.read_result(P.plugin_h(xt, ws=ws, flags=P.PLUGIN_MULTI_KERNEL))
    c = P.read_result(P.plugin_h(xt, ws=ws, flags=P.PLUGIN_SKIP_UNDERFLOW))
    assert _same(a, b) and _same(a, c), (a, b)
    o = oracle_mod.plugin(x)
    for key in ("psi6_z", "psi4_z", "h", "g1", "g2", "sigma"):
        assert rel(a[key], o[key]) < TOL, (n, key, a[key], o[key])


def test_fused_cluster_of_8_bit_identical(P):
    # the single launch falls back to an 8-CTA cluster where 16 cannot be scheduled
    # (PLUGIN_FUSED_CLUSTER=8 forces it; read once per process, hence the subprocess): other
    # slices, other chunk-to-CTA deals, the same bits (integer chunk sums)
    import subprocess
    import sys
    sizes = [2, 65, 700, 1024, 1025, 1500, 2048]
    code = (
        "import json, sys, torch\n"
        "sys.path.insert(0, %r)\n"
        "from paper_1505_02100_b200 import inputs, plugin as P\n"
        "out = {}\n"
        "for n in %r:\n"
        "    x = inputs.mixture(n, 900 + n) if n > 3 else inputs.normal(n, 900 + n)\n"
        "    r = P.read_result(P.plugin_h(torch.from_numpy(x).cuda()))\n"
        "    out[n] = {k: float(r[k]).hex() for k in ('psi6', 'psi4', 'h', 'g1', 'g2', 'sigma')}\n"
        "print(json.dumps(out))\n" % (os.path.dirname(HERE), sizes))
    env = dict(os.environ, PLUGIN_FUSED_CLUSTER="8")
    res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    got = json.loads(res.stdout.strip().splitlines()[-1])
    for n in sizes:
        x = inputs.mixture(n, 900 + n) if n > 3 else inputs.normal(n, 900 + n)
        r = P.read_result(P.plugin_h(torch.from_numpy(x).cuda()))
        mk = P.read_result(P.plugin_h(torch.from_numpy(x).cuda(), flags=P.PLUGIN_MULTI_KERNEL))
        for k, v in got[str(n)].items():
            assert float.fromhex(v) == r[k] == mk[k], (n, k, v, r[k], mk[k])


@pytest.mark.parametrize("case", ["constant", "nan", "inf"])
def test_fused_error_status_matches_multi_kernel(P, case):
    x = np.full(700, 1.25, np.float32)
    if case != "constant":
        x = inputs.normal(700, 1)
        x[123] = np.nan if case == "nan" else np.inf
    xt = torch.from_numpy(x).cuda()
    a = P.read_result(P.plugin_h(xt))
    b = P.read_result(P.plugin_h(xt, flags=P.PLUGIN_MULTI_KERNEL))
    want = P.PLUGIN_E_DEGENERATE if case == "constant" else P.PLUGIN_E_NONFINITE
    assert a["status"] == b["status"] == want
    assert _same(a, b)


def test_fused_toy_data_bit_identical(P):
    x = torch.from_numpy(inputs.TOY.astype(np.float32)).cuda()
    a = P.read_result(P.plugin_h(x))
    b = P.read_result(P.plugin_h(x, flags=P.PLUGIN_MULTI_KERNEL))
    assert _same(a, b)
    assert rel(a["h"], 0.96146759322923324) < TOL   # SURVEY App. B.2 (50-digit value)


@pytest.mark.parametrize("n", [2049, 4096, 12020, 30001, 32768])
def test_small_sort_matches_radix_sort_bit_for_bit(P, n):
    # n <= 32768 sorts by blocks of 2048 + a rank merge (blocksort.cuh); PLUGIN_SORT_RADIX=1
    # forces the 4-pass radix sort: both give the same unique ascending array, hence identical
    # results (ties, +-0 and tiny values included)
    import subprocess
    import sys
    code = ("import json, numpy as np, torch; from paper_1505_02100_b200 import plugin as P, inputs;"
            f"n = {n};"
            "x = np.concatenate([inputs.mixture(n - 20 - n // 4, 12), np.array([0.0, -0.0, 1e-30, -1e-30] * 5, np.float32),"
            " inputs.ties(n // 4, 1)]).astype(np.float32);"
            "r = P.read_result(P.plugin_h(torch.from_numpy(x).cuda(), flags=P.PLUGIN_MULTI_KERNEL));"
            "print(json.dumps({k: float(v).hex() for k, v in r.items()}))")
    env = dict(__import__("os").environ)
    a = subprocess.check_output([sys.executable, "-c", code], env=env, text=True).strip().splitlines()[-1]
    env["PLUGIN_SORT_RADIX"] = "1"
    b = subprocess.check_output([sys.executable, "-c", code], env=env, text=True).strip().splitlines()[-1]
    assert a == b


def test_cli_bandwidth_and_compare(P, tmp_path):
    import json
    import subprocess
    import sys
    x = inputs.TOY.astype(np.float32)
    np.save(tmp_path / "toy.npy", x)
    out = subprocess.check_output([sys.executable, "-m", "paper_1505_02100_b200", "compare", str(tmp_path / "toy.npy"),
                                   "--h-ref", "0.96146759322923324"], text=True)
    r = json.loads(out.strip().splitlines()[-1])
    assert r["status"] == 0 and r["rel_diff"] < TOL
    out = subprocess.check_output([sys.executable, "-m", "paper_1505_02100_b200", "kde", str(tmp_path / "toy.npy"),
                                   "--h", str(r["h"]), "--grid", "-5", "8.5", "4001"], text=True)
    k = json.loads(out.strip().splitlines()[-1])
    assert abs(k["trapezoid_mass"] - 1.0) < 1e-3


def test_plain_c_example_uses_the_abi(P, tmp_path):
    # examples/plugin_h_example.c: the C ABI from plain C (no Python, no torch on its path)
    import json
    import subprocess
    exe = os.path.join(os.path.dirname(HERE), "examples", "plugin_h_example")
    assert os.path.exists(exe), "built by __graft_entry__.build()"
    r = json.loads(subprocess.check_output([exe], text=True))
    assert r["status"] == 0 and rel(r["h"], 0.96146759322923324) < TOL       # toy data, SURVEY App. B.2
    x = inputs.config_data(1)
    x.astype("<f4").tofile(tmp_path / "cfg1.f32")
    r = json.loads(subprocess.check_output([exe, str(tmp_path / "cfg1.f32")], text=True))
    g = _golden(1)
    for k in ("psi6", "psi4", "h"):
        assert rel(r[k], g[k]) < TOL


def _key_sorted(x):
    # ascending order of the IEEE-754 bits' total order (the radix key of sort.cu), numpy only
    b = x.astype(np.float32).view(np.uint32)
    key = np.where(b & 0x80000000, ~b, b | 0x80000000).astype(np.uint32)
    return x.astype(np.float32)[np.argsort(key, kind="stable")]


@pytest.mark.parametrize("n", [1, 2, 7, 255, 256, 257, 1000, 2047, 2048, 2049, 4095, 4097, 12020, 30001, 32768,
                               32769, 100003])
def test_sort_is_exact(P, n):
    # the block sort (n <= 32768) and the radix sort (above) against numpy, bit for bit:
    # ties, +-0, denormals and the extremes of every run included
    rng = np.random.default_rng(n)
    x = rng.normal(0, 1, n).astype(np.float32)
    x[::7] = np.round(x[::7], 1)                      # ties
    if n > 8:
        x[:4] = [0.0, -0.0, 1e-40, -1e-40]
        x[-3:] = [3e38, -3e38, 0.5]
    got = P.plugin_sort(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), _key_sorted(x).view(np.uint32))


@pytest.mark.parametrize("n", [15872, 15873, 20001, 64512, 64513, 70001, 130047])
def test_psi_r_at_every_tile_shape(P, oracle_mod, n):
    # the tile edge T = 256 R switches with n (psi_rows_per_thread: R = 1 up to 15872, 2 up to
    # 64512, 4 up to 260096, then 8): both sides of each switch and ragged R = 2 / R = 4 shapes
    # against the oracle (up to a few 1e9 pairs, seconds)
    x = inputs.mixture(n, 77)
    for r, g in ((6, 0.4), (4, 0.15)):
        got = P.psi_r(torch.from_numpy(x).cuda(), g, r).item()
        ref = oracle_mod.psi(oracle_mod.widen(x), g, r)
        assert rel(got, ref) < TOL, (n, r, got, ref)


def test_batch_matches_single_runs(P, oracle_mod):
    # plugin_h_batch: one CTA per sample with T = 1024 tiles; each result agrees with plugin_h on
    # the sample (T = 64 tiles) to fp32 evaluation rounding, and with the oracle at TOL
    rng = np.random.default_rng(11)
    sizes = [2, 3, 64, 65, 128, 300, 1000, 1024, 1500, 2048, 1, 2049, 700]
    samples = []
    for k, n in enumerate(sizes):
        x = inputs.mixture(n, 600 + k) if n > 3 else inputs.normal(n, 600 + k)
        samples.append(x.astype(np.float32))
    samples.append(np.full(500, 2.5, np.float32))                       # degenerate
    bad = inputs.normal(400, 3)
    bad[7] = np.nan
    samples.append(bad)                                                  # non-finite
    offs = np.cumsum([0] + [s.size for s in samples]).astype(np.int64)
    x = torch.from_numpy(np.concatenate(samples)).cuda()
    res = P.read_results(P.plugin_h_batch(x, torch.from_numpy(offs).cuda()), len(samples))
    for s, r in zip(samples, res):
        if s.size < 2 or s.size > 2048:
            assert r["status"] == P.PLUGIN_E_INVALID
            continue
        one = P.read_result(P.plugin_h(torch.from_numpy(s).cuda()))
        if one["status"] != 0:
            assert r["status"] == one["status"]
            continue
        assert r["status"] == 0 and r["sigma"] == one["sigma"] and r["g1"] == one["g1"]  # same Step I
        for key in ("psi6", "psi4", "h"):
            assert rel(r[key], one[key]) < TOL, (s.size, key, r[key], one[key])
        if s.size in (300, 2048):
            o = oracle_mod.plugin(s)
            for key in ("psi6_z", "psi4_z", "h"):
                assert rel(r[key], o[key]) < TOL, (s.size, key, r[key], o[key])
    assert res[-2]["status"] == P.PLUGIN_E_DEGENERATE and res[-1]["status"] == P.PLUGIN_E_NONFINITE
    empty = P.plugin_h_batch(x, torch.zeros(1, dtype=torch.int64, device="cuda"))
    assert empty.numel() == P.RESULT_BYTES


@pytest.mark.parametrize("n", [1000, 50000])
def test_graph_api_repeats_plugin_h(P, n):
    # plugin_graph_*: one capture (the cooperative launch for n <= 2048, the kernel sequence
    # above), many launches with the sample refilled in place: each result bit-identical to
    # plugin_h on the same data
    x = torch.empty(n, device="cuda")
    g = P.PluginGraph(x)
    for seed in (1, 2, 3):
        xs = inputs.mixture(n, 900 + seed)
        x.copy_(torch.from_numpy(xs))
        got = P.read_result(g.launch())
        ref = P.read_result(P.plugin_h(torch.from_numpy(xs).cuda()))
        assert _same(got, ref), (n, seed)
    g.close()


@pytest.mark.parametrize("n", [2, 1500, 5000])
@pytest.mark.parametrize("r", [4, 6, 8, 10, 12])
def test_psi_r_far_pairs_do_not_overflow(P, oracle_mod, n, r):
    # |u| = |x_i - x_j| / g far beyond the exp underflow: K^(r)(u) = 0, but the fp32 He_r(u^2)
    # overflows to inf (|u| > ~1600 at r = 12 ... ~4e9 at r = 4) and inf * 0 would be NaN;
    # the pair evaluation clamps u^2 (psi_tile.cuh kTClamp) on tiles that span that far
    if n == 2:
        x, g = np.array([0.0, 1e7], dtype=np.float32), (1e-3 if r == 4 else 1.0)
    else:
        rng = np.random.default_rng(40 + n)
        far = np.array([3e3, -5e3, 1e5, 1e7, -2e4], dtype=np.float32)
        x = np.concatenate([rng.normal(0, 1, n - far.size).astype(np.float32), far])
        x = x[rng.permutation(n)]
        g = 1.0
    got = P.psi_r(torch.from_numpy(x).cuda(), g, r).item()
    ref = oracle_mod.psi(oracle_mod.widen(x), g, r)
    assert math.isfinite(got) and rel(got, ref) < TOL, (n, r, got, ref)


@pytest.mark.parametrize("n", [1800, 50000])
def test_plugin_h_with_outliers(P, oracle_mod, n):
    # a few points 1e4 sigma out: the tiles holding them span > kCenterSpan bandwidths and take
    # the difference-first variant (psi_tile_wide); the batch kernel decides the same way
    rng = np.random.default_rng(77)
    x = np.concatenate([rng.normal(0, 1, n - 4), [1e4, -2e4, 3e4, 2.5]]).astype(np.float32)
    x = x[rng.permutation(n)]
    got = P.plugin_h_sync(torch.from_numpy(x).cuda())
    ref = oracle_mod.plugin(x)
    assert got["status"] == 0
    for key in ("psi6", "psi4", "h"):
        assert rel(got[key], ref[key]) < TOL, (key, got[key], ref[key])
    if n <= 2048:
        xt = torch.from_numpy(x).cuda()
        offs = torch.tensor([0, n], dtype=torch.int64, device="cuda")
        b = P.read_results(P.plugin_h_batch(xt, offs), 1)[0]
        for key in ("psi6", "psi4", "h"):
            assert rel(b[key], ref[key]) < TOL, (key, b[key], ref[key])


@pytest.mark.parametrize("n", [5000, 40000])
def test_data_errors_multi_kernel(P, n):
    # n > 2048: the multi-kernel sequence, where Step I's last block NaN-fills the record and each
    # pass finalises itself in its last CTA (or skips on a failed status)
    x = torch.from_numpy(inputs.normal(n, 5)).cuda()
    x[n // 3] = float("nan")
    r = P.plugin_h_sync(x)
    assert r["status"] == P.PLUGIN_E_NONFINITE
    assert all(math.isnan(r[k]) for k in ("sigma", "g1", "psi6", "g2", "psi4", "h"))
    x[n // 3] = float("inf")
    assert math.isnan(P.psi_r(x, 0.5, 6).item())
    g = P.PluginGraph(x)
    assert P.read_result(g.launch())["status"] == P.PLUGIN_E_NONFINITE
    x[n // 3] = 0.25  # the same buffers, now valid: the graph's next launch succeeds
    ok = P.read_result(g.launch())
    assert ok["status"] == 0 and ok["h"] == P.plugin_h_sync(x)["h"]
    g.close()


def test_plugin_h_concurrent_streams_distinct_workspaces(P):
    # the header's promise: calls on different streams with distinct workspaces may run
    # concurrently.  Two samples (n = 16384: block sort + rank merge with the dynamic-smem
    # opt-in; n = 40000: radix sort) interleaved on two streams, three rounds, against
    # sequential runs; temporaries of the binding are allocated on the call's stream
    xs = [inputs.config_data(2), inputs.mixture(40000, 77)]
    ref = [P.plugin_h_sync(torch.from_numpy(x).cuda()) for x in xs]
    streams = (torch.cuda.Stream(), torch.cuda.Stream())
    bufs = []
    for _ in range(3):
        for k, (x, s) in enumerate(zip(xs, streams)):
            with torch.cuda.stream(s):  # the input is produced on the stream that consumes it
                xt = torch.from_numpy(x).cuda()
            st = s if k == 0 else s.cuda_stream  # a torch stream and a raw cudaStream_t handle
            # the caller drops xt right away: the binding's record_stream keeps its memory alive
            bufs.append((k, P.plugin_h(xt, stream=st)))
            del xt
    torch.cuda.synchronize()
    for k, b in bufs:
        got = P.read_result(b)
        assert _same(got, ref[k]), (k, got["h"], ref[k]["h"])


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_plugin_h_on_a_second_device(P):
    # per-device launch caches (occupancy, the sort-merge smem opt-in, SM counts): the same
    # sample on cuda:1 after cuda:0 gives the same bits
    x = inputs.mixture(20000, 78)
    a = P.plugin_h_sync(torch.from_numpy(x).to("cuda:0"))
    b = P.plugin_h_sync(torch.from_numpy(x).to("cuda:1"))
    assert _same(a, b)


def _tile_sum_oracle(oracle_mod, P, zs, g, r, n, t):
    rows, cols, w = P.plugin_work_item(n, r, t)
    return w * oracle_mod.psi_block_sum(zs, g, r, *rows, *cols) if cols[1] > cols[0] else 0.0


def _one_tile(P, n, r, t, ntiles, dres, ws):
    """The exact fixed-point sum of work item t alone (psi_r_shard with one item per 'rank')."""
    from paper_1505_02100_b200.distributed import from_limbs
    part = P.new_partial()
    P.psi_r_shard(n, r, t, ntiles, dres, part, ws)
    assert P.plugin_shard_tiles(n, r, t, ntiles) == (t, t + 1)
    return from_limbs(part.cpu().tolist()) / 2.0 ** 64 / math.sqrt(2 * math.pi)


def _tile_of_item(P, n, r, item, ntiles):
    """All work items of the tile that holds `item`: the item itself when tiles are whole (the
    default), the tile's column slices under the scheduler A/B switch PLUGIN_PSI_TAIL."""
    T = P.plugin_tile_edge(n, r)

    def key(it):
        rows, cols, _ = P.plugin_work_item(n, r, it)
        return rows[0], cols[0] // T

    k, lo, hi = key(item), item, item + 1
    while lo > 0 and key(lo - 1) == k:
        lo -= 1
    while hi < ntiles and key(hi) == k:
        hi += 1
    return range(lo, hi)


def _tile_got_ref(P, oracle_mod, zs, g, r, n, item, ntiles, dres, ws):
    """GPU and oracle sums over the whole tile that holds `item` (one psi_r_shard call per item)."""
    items = _tile_of_item(P, n, r, item, ntiles)
    return (sum(_one_tile(P, n, r, t, ntiles, dres, ws) for t in items),
            sum(_tile_sum_oracle(oracle_mod, P, zs, g, r, n, t) for t in items))


def _bandwidth_record(P, n, g_a, g_b):
    res = P.plugin_result()
    res.status, res.n, res.g1, res.g2 = 0, n, g_a, g_b
    return torch.frombuffer(bytearray(bytes(res)), dtype=torch.uint8).cuda()


@pytest.mark.parametrize("n", [100000, 300000])
def test_wide_tiles_with_outliers_at_full_size(P, oracle_mod, n):
    """Outliers at the sizes that select R = 4 (n = 1e5, T = 1024) and R = 8 (n = 3e5, r = 4: T = 2048)
    tiles: the tiles that hold them span far more than 64 bandwidths and take the wide path
    (difference first, clamped u^2, psi_tile.cuh); those tiles, the diagonal tiles at both ends and
    a middle tile, one by one against the oracle's block sums of the same pairs."""
    rng = np.random.default_rng(50 + n)
    far = np.array([3e3, -5e3, 1e5, 1e7, -2e4, 40.0, -60.0], dtype=np.float32)
    x = np.concatenate([rng.normal(0, 1, n - far.size).astype(np.float32), far])
    x = x[rng.permutation(n)]
    xd = torch.from_numpy(x).cuda()
    ws = P.workspace(n)
    P.plugin_step1(xd, P.new_result(), ws)
    zs = np.sort(oracle_mod.widen(x))
    for r, g in ((6, 0.3), (4, 0.2)):
        ntiles, T = P.plugin_num_tiles(n, r), P.plugin_tile_edge(n, r)
        assert T == (2048 if (n == 300000 and r == 4) else 1024)   # R = 8 only for r <= 4
        nb = -(-n // T)
        picks = sorted({0, 1, nb - 1, nb // 2 * nb - (nb // 2) * (nb // 2 - 1) // 2,   # row 0 (outliers), mid diag
                        ntiles - 1, ntiles - 2,                                           # last tiles
                        (nb - 2) * nb - (nb - 2) * (nb - 3) // 2 + 1})                    # row nb-2, last column
        dres = _bandwidth_record(P, n, g, g)
        for t in picks:
            got, ref = _tile_got_ref(P, oracle_mod, zs, g, r, n, t, ntiles, dres, ws)
            assert math.isfinite(got)
            # relative 1e-5; terms below the fp32 range (e^(-u^2/2) < 2^-126: the far tiles) are
            # +0 on the GPU, so an absolute T^2 2^-100 is allowed on top
            assert abs(got - ref) <= TOL * abs(ref) + T * T * 2.0 ** -100, (n, r, t, P.plugin_work_item(n, r, t), got, ref)


@pytest.mark.parametrize("r", [8, 12])
def test_general_r_pass_at_cfg4_sampled_tiles(P, oracle_mod, r):
    """The general-r pass (He_r phi, the plugin_dpi family) at BASELINE config 4 (R = 4 tiles at
    this size, where test_gpu_dpi's full-oracle cases do not reach): sampled tiles against the oracle."""
    x = inputs.config_data(4)
    n = x.size
    xd = torch.from_numpy(x).cuda()
    ws = P.workspace(n)
    P.plugin_step1(xd, P.new_result(), ws)
    zs = np.sort(oracle_mod.widen(x))
    sigma = oracle_mod.step1(x)["sigma"]
    g = 0.35 * sigma
    ntiles, T = P.plugin_num_tiles(n, r), P.plugin_tile_edge(n, r)
    nb = -(-n // T)
    dres = _bandwidth_record(P, n, g, g)
    for t in (0, 5, nb + 3, ntiles // 2, ntiles // 2 + 1, ntiles - 3, ntiles - 1):
        got, ref = _tile_got_ref(P, oracle_mod, zs, g, r, n, t, ntiles, dres, ws)
        assert abs(got - ref) <= TOL * abs(ref) + T * T * 2.0 ** -100, (r, t, P.plugin_work_item(n, r, t), got, ref)


@pytest.mark.parametrize("case", ["cfg2", "ties_grouped", "small"])
@pytest.mark.parametrize("world", [1, 3, 8])
def test_psi_r_shard_g_sums_to_psi_r_bit_exact(P, case, world):
    # the explicit-bandwidth shard of SURVEY §8(b): every rank's partial at a host g, limbs
    # summed (what the NCCL allreduce does), finalised -> psi_r's bits, r = 6, 4 and 8
    x = {"cfg2": lambda: inputs.config_data(2), "ties_grouped": lambda: inputs.ties(40000, 31),
         "small": lambda: inputs.normal(777, 32)}[case]()
    xt = torch.from_numpy(x).cuda()
    n = x.size
    ws = P.workspace(n)
    P.plugin_prepare(xt, ws)
    for r, g in ((6, 0.4), (4, 0.3), (8, 0.55)):
        tot = torch.zeros(4, dtype=torch.int64, device="cuda")
        for rank in range(world):
            part = P.new_partial()
            P.psi_r_shard_g(n, g, r, rank, world, part, ws)
            tot += part
        got = P.plugin_psi_from_total(tot, n, g, r).item()
        ref = P.psi_r(xt, g, r).item()
        assert got == ref, (case, world, r, got, ref)


@pytest.mark.parametrize("n", [500, 1000, 2048])
@pytest.mark.parametrize("kind", ["ties", "integers", "offset"])
def test_small_n_discretised_single_launch_and_batch(P, oracle_mod, n, kind):
    # n <= 2048 (the paper's sizes): the single launch (small tiles, difference first) and the
    # batch kernel (T = 256 centred tiles, dither amplitude n/16) on discretised samples
    x = {"ties": lambda: inputs.ties(n, 60 + n), "integers": lambda: np.round(inputs.normal(n, 61 + n, sd=4)).astype(np.float32),
         "offset": lambda: inputs.offset(n, 62 + n)}[kind]()
    o = oracle_mod.plugin(x)
    xt = torch.from_numpy(x).cuda()
    a = P.plugin_h_sync(xt)
    off = torch.tensor([0, n], dtype=torch.int64, device="cuda")
    b = P.read_results(P.plugin_h_batch(xt, off), 1)[0]
    for r in (a, b):
        assert r["status"] == 0
        for key in ("psi6_z", "psi4_z", "h"):
            assert rel(r[key], o[key]) < TOL, (kind, n, key, r[key], o[key])
