"""World-size-2 gloo test of the multi-GPU host logic (no GPU needed)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_11498_b200.sharding import gather_results, pack_results, shard_range


def test_shard_range_covers_exactly():
    for n in (0, 1, 7, 10, 1001):
        for w in (1, 2, 3, 8):
            got = [shard_range(n, r, w) for r in range(w)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(n, rank, world)
    idx = torch.arange(lo, hi)
    # stand-in for each rank's projection results over its shard
    block = pack_results(idx.double() * 0.5, idx.double() + 0.25, (idx % 7).int())
    full = gather_results(block, n, world, rank)
    if rank == 0:
        out.put(full.numpy().tolist())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [10, 1001])
def test_gather_world_size_2(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    full = torch.tensor(q.get(timeout=120))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    i = torch.arange(n).double()
    assert torch.equal(full[:, 0], i * 0.5)
    assert torch.equal(full[:, 1], i + 0.25)
    assert torch.equal(full[:, 2], (torch.arange(n) % 7).double())


def _chunk_worker(rank, world, port, n, chunks, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_11498_b200.sharding import gather_chunk, unchunk
    lo, hi = shard_range(n, rank, world)
    idx = torch.arange(lo, hi)
    bounds = [(hi - lo) * i // chunks for i in range(chunks + 1)]
    got = []
    for i in range(chunks):
        sl = idx[bounds[i]:bounds[i + 1]]
        blk = pack_results(sl.double() * 0.5, sl.double() + 0.25, (sl % 7).int())
        _, bufs = gather_chunk(blk, world, rank)
        got.append(bufs)
    if rank == 0:
        out.put(unchunk(got, world, hi - lo, bounds).numpy().tolist())
    dist.barrier()
    dist.destroy_process_group()


def test_chunked_gather_world_size_2():
    """bench.py's N > 1 step: each rank's shard in chunks, one gather per
    chunk; rank 0 reassembles the global order (rank-major, then chunk)."""
    n, chunks = 800, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chunk_worker, args=(r, 2, port, n, chunks, q))
             for r in range(2)]
    for p in procs:
        p.start()
    full = torch.tensor(q.get(timeout=120))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    i = torch.arange(n).double()
    assert torch.equal(full[:, 0], i * 0.5)
    assert torch.equal(full[:, 2], (torch.arange(n) % 7).double())
