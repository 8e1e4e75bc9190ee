"""Multi-rank path of the batched config on CPU (gloo, world size 2)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_16734_b200.batch import gather_chain_stats, gather_chain_stats_ctx, shard_range


def test_shard_range_covers_everything():
    for total in (1, 7, 1024, 1025):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                lo, hi = shard_range(total, world, r)
                seen.extend(range(lo, hi))
            assert seen == list(range(total))
            sizes = [shard_range(total, world, r)[1] - shard_range(total, world, r)[0] for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(total, world, rank)
    local = torch.tensor([[float(c), 0.5 * c, float(c % 4)] for c in range(lo, hi)], dtype=torch.float64)
    allst = gather_chain_stats(local, total, world)

    class GlooCtx:  # stands in for ttlab.Context.allgather_f64 (ncclAllGather on the GPU box)
        def allgather_f64(self, send):
            t = torch.from_numpy(send.ravel().copy())
            out = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(out, t)
            return torch.stack(out).numpy()

    native = gather_chain_stats_ctx(GlooCtx(), local.numpy(), total, world)  # padding / reordering of the ctx path
    q.put((rank, allst.tolist(), native.tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [10, 1024])
def test_gather_chain_stats_gloo_world2(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    res = {r: a for r, a, _ in got}
    nat = {r: b for r, _, b in got}
    for p in procs:
        p.join(timeout=60)
    expect = [[float(c), 0.5 * c, float(c % 4)] for c in range(total)]
    assert res[0] == expect and res[1] == expect  # bit-exact, identical on every rank
    assert nat[0] == expect and nat[1] == expect
