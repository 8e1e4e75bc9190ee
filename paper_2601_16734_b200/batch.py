"""Data-parallel sharding of independent chains over GPUs.

Config 5 compresses 1024 independent chains; rank r of N owns the contiguous
block [r*B/N, (r+1)*B/N).  There is no exchange while the chains are swept; the
only collective is one all-gather of the per-chain scalars (norm, error,
sweeps) at the end of each batch, over NCCL (NVLink) on the GPU box and gloo in
the CPU tests.
"""
from __future__ import annotations

from typing import Tuple

import torch
import torch.distributed as dist


def shard_range(total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced block of `total` units for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_chain_stats(local: torch.Tensor, total: int, world: int) -> torch.Tensor:
    """All-gather per-chain rows [norm, error, sweeps] from every rank into a
    (total, 3) tensor ordered by global chain index (one collective)."""
    if world == 1:
        return local
    sizes = [shard_range(total, world, r)[1] - shard_range(total, world, r)[0] for r in range(world)]
    width = max(sizes)
    pad = torch.zeros((width, local.shape[1]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = torch.empty((world * width, local.shape[1]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, pad)
    rows = [out[r * width: r * width + sizes[r]] for r in range(world)]
    return torch.cat(rows, 0)
