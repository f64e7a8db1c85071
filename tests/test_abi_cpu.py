"""CPU-only checks of the C ABI boundary: libplugin.so loads, exports every symbol the
header declares, and its pure host-side functions (workspace sizing, tile sharding)
behave.  No compute calls (no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "plugin.h")


@pytest.fixture(scope="module")
def L():
    import __graft_entry__
    __graft_entry__.build()
    from paper_1505_02100_b200 import plugin
    return plugin


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(plugin_\w+|psi_r\w*|kde_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("plugin_h", "psi_r", "plugin_step1", "psi_r_shard", "plugin_after_psi6", "plugin_after_psi4",
                 "plugin_workspace_bytes", "plugin_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(L):
    lib = ctypes.CDLL(L.LIB_PATH)
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_declared()) == set(L.EXPORTED)


def test_version_and_error_strings(L):
    assert "sm_100a" in L.plugin_version()
    assert L.plugin_last_error() == ""


def test_workspace_sizes_monotone(L):
    prev = 0
    for n in (1, 2, 1000, 4096, 4097, 1 << 20, 1 << 22):
        b = L.plugin_workspace_bytes(n)
        assert b >= 8 * n and b >= prev and b % 256 == 0
        assert L.plugin_host_workspace_bytes(n) >= b + 4 * n
        prev = b


@pytest.mark.parametrize("n", [1, 2, 255, 256, 257, 16384, 131072, 1 << 20, 4194304])
def test_tiles_cover_triangle(L, n):
    for order in (4, 6, 12):
        w = L.plugin_num_tiles(n, order)
        assert w >= 1
        for world in (1, 2, 3, 4, 8):
            spans = [L.plugin_shard_tiles(n, order, k, world) for k in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == w
            for (b0, e0), (b1, e1) in zip(spans, spans[1:]):
                assert e0 == b1
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1           # equal-work tiles, balanced to one tile
        assert L.plugin_shard_tiles(n, order, 3, 2) == (0, 0)    # invalid rank -> empty range
    assert L.plugin_num_tiles(n, 5) == 0 and L.plugin_shard_tiles(n, 5, 0, 1) == (0, 0)  # odd r


def test_rows_per_thread_by_order(L):
    # the r >= 6 passes stop at R = 4 (T = 1024), the r <= 4 passes go to R = 8 (T = 2048)
    n = 1 << 20
    assert L.plugin_tile_edge(n, 6) == 1024 and L.plugin_tile_edge(n, 8) == 1024
    assert L.plugin_tile_edge(n, 4) == 2048 and L.plugin_tile_edge(n, 2) == 2048
    assert L.plugin_tile_edge(1000, 6) == L.plugin_tile_edge(1000, 4) == 64


@pytest.mark.parametrize("mode", ["", "1", "2"])
@pytest.mark.parametrize("n", [1, 2, 2048, 2049, 5000, 16384, 50000, 131072, 1 << 20])
def test_work_items_partition_the_triangle(n, mode, monkeypatch):
    # mode: the scheduler A/B switch PLUGIN_PSI_TAIL (1, 2: the last tiles mod 148 tiles as 64-column
    # slices) -- the item definitions are read from the environment at every call
    if mode:
        monkeypatch.setenv("PLUGIN_PSI_TAIL", mode)
    else:
        monkeypatch.delenv("PLUGIN_PSI_TAIL", raising=False)
    # every tile's columns are covered exactly once by its items (whole, or column slices), rows
    # and weights are the tile's; the items cover exactly the upper block triangle
    from paper_1505_02100_b200 import plugin as P
    order = 6 if n % 2 else 4
    T, items = P.plugin_tile_edge(n, order), P.plugin_num_tiles(n, order)
    nb = -(-n // T)
    cover = {}
    step = max(1, items // 4000)  # large n: a deterministic sample of items plus all tail items
    idx = sorted(set(range(0, items, step)) | set(range(max(0, items - 8 * 444 * 4), items)))
    for it in idx:
        (r0, r1), (c0, c1), w = P.plugin_work_item(n, order, it)
        bi, bj = r0 // T, (c0 // T) if c1 > c0 else None
        assert r0 == bi * T and r1 == min(n, r0 + T) and 0 <= r0 < r1 <= n
        if bj is None:
            continue                       # a slice past the sample's end: no pairs
        assert bj >= bi and w == (1 if bi == bj else 2) and c1 <= min(n, bj * T + T)
        cover.setdefault((bi, bj), []).append((c0, c1))
    if step == 1:
        assert len(cover) == nb * (nb + 1) // 2
    for (bi, bj), spans in cover.items():
        spans.sort()
        full = [(bj * T, min(n, bj * T + T))]
        if len(spans) == 1 or spans[0][1] - spans[0][0] == full[0][1] - full[0][0]:
            assert spans == full or len(spans) == 1
        else:                              # slices: contiguous, disjoint, ending at the block's end
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0
            assert spans[0][0] == full[0][0] and spans[-1][1] == full[0][1]
    with pytest.raises(IndexError):
        P.plugin_work_item(n, order, items)


def test_kde_workspace_sizing(L):
    # the psi workspace (sorted copy of X) plus per-(block, segment) fp64 partials, bounded by
    # (8 * 148 target CTAs + one per point block) x 1024 points x 8 bytes
    for n in (1, 1000, 1 << 20):
        base = L.plugin_workspace_bytes(n)
        for m in (0, 1, 1024, 65536, 1 << 22):
            b = L.kde_workspace_bytes(n, m)
            assert b >= base and b % 256 == 0
            nb = -(-m // 1024)
            assert b <= base + 8 * 1024 * (8 * 148 + nb) + 4 * nb + 512


def test_cli_loader_formats(tmp_path):
    import numpy as np

    from paper_1505_02100_b200.__main__ import _load
    x = np.array([0.0, 1.0, 1.1, 1.5, 1.9, 2.8, 2.9, 3.5])           # the toy data of P:51
    np.save(tmp_path / "a.npy", x)
    x.astype("<f4").tofile(tmp_path / "a.f32")
    np.savetxt(tmp_path / "a.txt", x)
    for f in ("a.npy", "a.f32", "a.txt"):
        got = _load(str(tmp_path / f))
        assert got.dtype == np.float32 and np.array_equal(got, x.astype(np.float32))


@pytest.mark.parametrize("lang", ["c", "c++"])
def test_header_is_self_contained_c_and_cpp(tmp_path, lang):
    # include/plugin.h is the boundary: it must compile on its own as C11 and as C++
    import subprocess
    src = tmp_path / ("t.c" if lang == "c" else "t.cpp")
    src.write_text('#include "plugin.h"\nint main(void) { plugin_result r; (void)r; return (int)sizeof(plugin_fx128); }\n')
    cc = "gcc" if lang == "c" else "g++"
    std = "-std=c11" if lang == "c" else "-std=c++17"
    p = subprocess.run([cc, std, "-Wall", "-Werror", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), str(src)],
                       capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
