"""Data-parallel sharding of independent chains over GPUs.

Config 5 compresses 1024 independent chains; rank r of N owns the contiguous
block [r*B/N, (r+1)*B/N).  There is no exchange while the chains are swept; the
only collective is one all-gather of the per-chain scalars (norm, error,
sweeps) at the end of each batch.  On the GPU box it runs on the NCCL
communicator the library context owns (`ttg_comm_*`, `init_context_comm` +
`gather_chain_stats_ctx`); `gather_chain_stats` is the same collective through
torch.distributed (NCCL, or gloo in the CPU tests).
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


def init_context_comm(ctx, world: int, rank: int) -> None:
    """Give `ctx` (a ttlab.Context) its NCCL communicator: rank 0 draws the id, torch.distributed ships
    the 128 bytes (any host transport would do), every rank joins (ncclCommInitRank)."""
    if world == 1:
        return
    uid = [ctx.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    ctx.comm_init(world, rank, uid[0])


def gather_chain_stats_ctx(ctx, local, total: int, world: int):
    """`gather_chain_stats` on the context's own communicator: `local` is a (chains, 3) numpy array of
    this rank's [norm, error, sweeps] rows; returns the (total, 3) array in global chain order."""
    import numpy as np
    local = np.ascontiguousarray(local, dtype=np.float64)
    if world == 1:
        return local
    sizes = [shard_range(total, world, r)[1] - shard_range(total, world, r)[0] for r in range(world)]
    width = max(sizes)
    pad = np.zeros((width, local.shape[1]))
    pad[: local.shape[0]] = local
    out = ctx.allgather_f64(pad).reshape(world, width, local.shape[1])
    return np.concatenate([out[r, : sizes[r]] for r in range(world)], 0)
