"""Multi-GPU PLUGIN: one process per GPU (torchrun), the pair triangle split into
equal-work tile ranges, one 32-byte NCCL allreduce per psi pass.

Every rank holds the whole sample X (<= 16 MB) and runs Step I and the sort itself
(deterministic, identical on every rank), then its share of each psi pass.  The
per-rank partial is an exact 128-bit fixed-point integer exported as four 32-bit
limbs in int64, so the allreduce is integer addition: the result is bit-identical
for any number of GPUs.  Compute stays in libplugin.so; this module only sequences
the C-ABI calls and the collective.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import plugin as P

MASK32 = (1 << 32) - 1


def to_limbs(v: int) -> list[int]:
    """Python int (two's complement, 128-bit) -> the 4 limbs of plugin_fx128 (host-side helper)."""
    v &= (1 << 128) - 1
    lo, hi = v & ((1 << 64) - 1), v >> 64
    hi_signed = hi - (1 << 64) if hi >> 63 else hi
    return [lo & MASK32, lo >> 32, hi & MASK32, hi_signed >> 32]


def from_limbs(limbs) -> int:
    """Carry-propagate 4 summed limbs (as the device finalize does) -> signed 128-bit int."""
    c = 0
    w = []
    for k in range(4):
        v = int(limbs[k]) + c
        w.append(v & MASK32)
        c = v >> 32
    v = w[0] | (w[1] << 32) | (w[2] << 64) | (w[3] << 96)
    return v - (1 << 128) if v >> 127 else v


def plugin_h_distributed(x: torch.Tensor, group=None, out: torch.Tensor | None = None,
                         ws: torch.Tensor | None = None, stream=None, events: dict | None = None) -> torch.Tensor:
    """Algorithm 1 over all ranks of `group`; every rank ends with the same result buffer.

    ``events`` (optional) maps names to pairs of CUDA events recorded around the two psi
    shards (used by bench.py to time the hot kernel on its own stream)."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    n = x.numel()
    # everything (the library calls, the NCCL allreduce, the events, the temporaries) on ONE
    # stream, made current: the collective then reads each partial after its shard wrote it,
    # and the finalize reads the reduced total after the collective
    with P._On(x.device, stream) as on:
        s = on.stream
        ws = P.workspace(n, x.device) if ws is None else ws
        out = P.new_result(x.device) if out is None else out
        P.plugin_step1(x, out, ws, s)
        for r, after in ((6, P.plugin_after_psi6), (4, P.plugin_after_psi4)):
            part = P.new_partial(x.device)
            ev = events.get(f"psi{r}") if events else None
            if ev:
                ev[0].record(s)
            P.psi_r_shard(n, r, rank, world, out, part, ws, s)
            if ev:
                ev[1].record(s)
            if world > 1:
                dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)
            after(part, out, s)
    return out
