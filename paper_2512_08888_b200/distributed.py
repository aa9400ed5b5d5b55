"""Batch-sharded multi-GPU driver: one process per GPU.

The layer shards naturally: every image is independent.  The batch is split into
contiguous shards (rc_shard_range: the first n % world ranks get one extra image),
each rank builds the same bank from identical weights (no broadcast), runs the fused
kernel on its shard, and outputs stay sharded.  NCCL over NVLink is used ONLY when the
caller asks to gather the outputs (``gather_shards``).  There is no data-path
collective on the forward itself.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist

from .rotconv import Desc, bank_precompute, ri_conv_forward, shard_range


def env_rank_world() -> tuple[int, int, int]:
    """(rank, world, local_rank) from the torchrun environment (1-process defaults)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def local_desc(desc: Desc, world: int, rank: int) -> tuple[Desc, int, int]:
    """Descriptor of this rank's shard of a global-batch descriptor."""
    b, e = shard_range(desc.n, world, rank)
    d = Desc(**{**desc.__dict__, "n": e - b})
    return d, b, e


def sharded_forward(desc: Desc, x_local: torch.Tensor, w0: torch.Tensor,
                    w1: torch.Tensor | None = None, bias: torch.Tensor | None = None,
                    world: int | None = None, rank: int | None = None, bank=None):
    """Run this rank's shard.  x_local holds only this rank's images."""
    if world is None or rank is None:
        rank, world, _ = env_rank_world()
    d, b, e = local_desc(desc, world, rank)
    if x_local.shape[0] != e - b:
        raise ValueError(f"sharded_forward: rank {rank} expects {e - b} images, got {x_local.shape[0]}")
    if bank is None:
        bank = bank_precompute(d, w0, w1)
    return ri_conv_forward(d, x_local, bank, bias)


def gather_shards(y_local: torch.Tensor, n_total: int, group=None, to_all: bool = True):
    """Concatenate every rank's contiguous batch shard along dim 0.

    Shards may be ragged (n % world != 0): they are padded to the largest shard for the
    collective (all_gather is NCCL's native primitive; NCCL has no gather) and trimmed.
    Returns the full batch on every rank (to_all) or on rank 0 only (None elsewhere).
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = [shard_range(n_total, world, r) for r in range(world)]
    counts = [e - b for b, e in sizes]
    if y_local.shape[0] != counts[rank]:
        raise ValueError("gather_shards: local shard size does not match shard_range")
    mx = max(counts)
    pad = torch.zeros((mx,) + tuple(y_local.shape[1:]), dtype=y_local.dtype, device=y_local.device)
    pad[: counts[rank]] = y_local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    if not to_all and rank != 0:
        return None
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)
