"""Host logic of the multi-GPU path on CPU: two gloo ranks all-reduce the 4-limb
fixed-point partials exactly as the NCCL path does, and the result equals the exact
128-bit sum (the property that makes N-GPU results bit-identical)."""
import os
import random

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1505_02100_b200.distributed import from_limbs, to_limbs


def test_limbs_roundtrip():
    rng = random.Random(0)
    for _ in range(2000):
        v = rng.randrange(-(1 << 126), 1 << 126)
        assert from_limbs(to_limbs(v)) == v
    for v in (0, 1, -1, (1 << 127) - 1, -(1 << 127), 1 << 64, -(1 << 64)):
        assert from_limbs(to_limbs(v)) == v


def test_limb_sums_are_exact():
    rng = random.Random(1)
    for _ in range(200):
        vals = [rng.randrange(-(1 << 120), 1 << 120) for _ in range(rng.randint(1, 64))]
        summed = [sum(to_limbs(v)[k] for v in vals) for k in range(4)]
        assert from_limbs(summed) == sum(vals)


def _worker(rank, world, port, vals, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = torch.tensor(to_limbs(vals[rank]), dtype=torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    q.put((rank, from_limbs(t.tolist())))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_allreduce_of_limbs(world):
    rng = random.Random(5)
    vals = [rng.randrange(-(1 << 110), 1 << 110) for _ in range(world)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + random.Random().randrange(2000)
    procs = [ctx.Process(target=_worker, args=(r, world, port, vals, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(v == sum(vals) for v in got.values())


class _FakePlugin:
    """CPU stand-in for the CUDA calls plugin_h_distributed sequences: each psi shard 'computes'
    sum over its tiles of a per-tile integer (tile index * r + 1) with the REAL tile sharding of
    libplugin.so (a host-only function), as the 4-limb partial the device would export."""

    def __init__(self, real):
        self.real = real
        self.totals = {}

    class _On:  # the device / stream context of the binding: nothing to switch on CPU
        def __init__(self, device, stream=None):
            self.stream = stream

        def __enter__(self):
            return self

        def __exit__(self, *exc):
            return False

    def workspace(self, n, device=None):
        return torch.zeros(1, dtype=torch.uint8)

    def new_result(self, device=None):
        return torch.zeros(1, dtype=torch.uint8)

    def new_partial(self, device=None):
        return torch.zeros(4, dtype=torch.int64)

    def plugin_step1(self, x, out, ws, stream=None):
        return out

    def psi_r_shard(self, n, r, rank, world, out, partial, ws, stream=None):
        tb, te = self.real.plugin_shard_tiles(n, r, rank, world)
        v = sum(t * r + 1 for t in range(tb, te)) << 70      # exercise the upper limbs too
        partial.copy_(torch.tensor(to_limbs(v), dtype=torch.int64))
        return partial

    def plugin_after_psi6(self, total, out, stream=None):
        self.totals[6] = from_limbs(total.tolist())
        return out

    def plugin_after_psi4(self, total, out, stream=None):
        self.totals[4] = from_limbs(total.tolist())
        return out


def _worker_dist(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1505_02100_b200 import distributed as D
    from paper_1505_02100_b200 import plugin as real
    fake = _FakePlugin(real)
    D.P = fake                                   # the module's handle on the C ABI binding
    D.plugin_h_distributed(torch.zeros(n), out=fake.new_result(), ws=fake.workspace(n))
    q.put((rank, fake.totals))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 1 << 20), (3, 100003)])
def test_plugin_h_distributed_sequencing_with_gloo(world, n):
    # the N > 1 path of bench.py on CPU: every rank runs its shard of each pass, the limbs are
    # all-reduced (gloo here, NCCL on GPUs) and every rank finalises the same exact totals,
    # which equal the single-rank sums over all tiles (shards cover each tile exactly once)
    import __graft_entry__
    __graft_entry__.build()
    from paper_1505_02100_b200 import plugin as real
    want = {r: sum(t * r + 1 for t in range(real.plugin_num_tiles(n, r))) << 70 for r in (6, 4)}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + random.Random().randrange(2000)
    procs = [ctx.Process(target=_worker_dist, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(got[r] == want for r in range(world))
