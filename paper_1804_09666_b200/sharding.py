"""System-index sharding over ranks: configs 1-4 are independent
systems, so a batch is cut into contiguous per-rank slices with no collective
on the solve path; the only collectives are the optional final gather of x
and the MAX reduction of per-system residuals / "still iterating" flags.
One process per GPU, ``torch.distributed`` (NCCL on the box, gloo in the CPU
tests)."""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_bounds(batch: int, rank: int, world: int):
    """[lo, hi) of this rank's contiguous slice; the first batch % world ranks
    take one extra system."""
    base, extra = divmod(batch, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_rows(arrays, rank: int, world: int):
    """Per-rank slices of (B, ...) host/device arrays (system index first)."""
    lo, hi = shard_bounds(arrays[0].shape[0], rank, world)
    return [a[lo:hi] for a in arrays], (lo, hi)


def gather_systems(local: torch.Tensor, batch: int, group=None):
    """All ranks' (b_r, ...) slices -> the full (batch, ...) tensor on every
    rank (uneven slices padded to the largest one for the collective)."""
    world = dist.get_world_size(group)
    sizes = [shard_bounds(batch, r, world) for r in range(world)]
    cap = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:hi - lo] for p, (lo, hi) in zip(parts, sizes)], dim=0)


def global_max(value: torch.Tensor, group=None):
    """MAX over ranks (max residual_inf, or "any system still iterating")."""
    out = value.clone()
    dist.all_reduce(out, op=dist.ReduceOp.MAX, group=group)
    return out
