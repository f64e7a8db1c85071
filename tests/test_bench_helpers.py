"""CPU checks of bench.py's host-side work counters (the algorithmic units its roofline
fractions divide by): the pairs the skip-underflow pass evaluates and the terms kde_eval
visits, against brute force on small samples."""
import numpy as np

import bench


def test_psi_pairs_evaluated_full_when_nothing_is_skipped():
    x = np.random.default_rng(0).normal(0, 1, 5000).astype(np.float32)
    n = x.size
    assert bench.psi_pairs_evaluated(x, g=100.0, tile=256) == n * (n - 1) / 2


def test_psi_pairs_evaluated_skips_only_far_tiles():
    rng = np.random.default_rng(1)
    x = np.concatenate([rng.normal(0, 1, 3000), rng.normal(500, 1, 3000)]).astype(np.float32)
    n, tile, g = x.size, 256, 0.3
    got = bench.psi_pairs_evaluated(x, g, tile)
    xs = np.sort(x).astype(np.float64)
    s = float(np.float32(1 / g))
    # brute force: a tile pair (bi < bj) may be skipped only if every pair in it is beyond the cutoff
    nb = -(-n // tile)
    ref = 0
    for bi in range(nb):
        ri = xs[bi * tile:(bi + 1) * tile]
        ref += ri.size * (ri.size - 1) // 2
        for bj in range(bi + 1, nb):
            rj = xs[bj * tile:(bj + 1) * tile]
            far = (rj.min() - ri.max()) * s * (1 - 1e-5) > 13.25
            if far:
                assert np.all(np.abs(rj[None, :] - ri[:, None]) * s > 13.2)
            else:
                ref += ri.size * rj.size
    assert got == ref
    assert got < n * (n - 1) / 2 * 0.6       # the two clusters never meet


def test_kde_terms_visited_counts_the_window():
    rng = np.random.default_rng(2)
    x = rng.normal(0, 1, 4000).astype(np.float32)
    h = 0.1
    pts = np.linspace(-6, 6, 3000).astype(np.float32)
    got = bench.kde_terms_visited(x, h, pts)
    kf = float(np.float32(-1.4426950408889634 / (2 * h * h)))
    cut = (126.5 / abs(kf)) ** 0.5 * (1 + 1e-6)
    xs = np.sort(x.astype(np.float64))
    ref = 0
    for b in range(0, pts.size, 1024):
        p = pts[b:b + 1024].astype(np.float64)
        inside = (xs >= p.min() - cut) & (xs <= p.max() + cut)
        ref += p.size * int(inside.sum())
        # every sample outside the window is beyond the cutoff for every point of the block
        d = np.abs(p[:, None] - xs[None, ~inside])
        assert d.size == 0 or d.min() > cut * (1 - 1e-9)
    assert got == ref


def test_launch_plan_never_runs_one_rank_labelled_n():
    # --gpus N outside torchrun: re-exec with N ranks, or refuse; inside: WORLD_SIZE must match
    assert bench.launch_plan(1, {}, 0) == ("run", "")
    assert bench.launch_plan(2, {}, 8)[0] == "reexec"
    assert bench.launch_plan(8, {}, 8)[0] == "reexec"
    assert bench.launch_plan(2, {}, 1)[0] == "error"
    assert bench.launch_plan(4, {"WORLD_SIZE": "4"}, 8) == ("run", "")
    assert bench.launch_plan(2, {"WORLD_SIZE": "1"}, 8)[0] == "error"
    assert bench.launch_plan(1, {"WORLD_SIZE": "1"}, 8) == ("run", "")


def test_bench_gpus_2_without_gpus_fails_loudly():
    # on this CPU-only box `bench.py --gpus 2` must exit non-zero with a reason, not measure
    # one process and label it 2 GPUs
    import subprocess
    import sys
    p = subprocess.run([sys.executable, bench.__file__, "--gpus", "2", "--steps", "2", "--warmup", "3"],
                       capture_output=True, text=True, timeout=600, env={k: v for k, v in __import__("os").environ.items()
                                                                         if k not in ("WORLD_SIZE", "RANK")})
    assert p.returncode != 0
    assert "needs 2 visible CUDA devices" in p.stderr
    assert p.stdout.strip() == ""
