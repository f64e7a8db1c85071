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
