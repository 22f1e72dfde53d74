"""Query sharding across ranks and the single result gather.

Each rank projects a contiguous query range against its own replica of the
segment table; the only exchange is gathering (t, distance, segment id) to
rank 0.  Works with NCCL on CUDA tensors (bench.py) and gloo on CPU tensors
(tests/test_sharding.py).
"""

import torch
import torch.distributed as dist


def shard_range(n_total: int, rank: int, world: int):
    """Contiguous [lo, hi) of the queries owned by `rank` (ceil-balanced)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    k = -(-n_total // world)
    lo = min(rank * k, n_total)
    return lo, min(lo + k, n_total)


def pack_results(t, dist_, seg):
    """(n,3) float64 block: t, distance, segment id (exact as float64)."""
    return torch.stack([t.to(torch.float64), dist_.to(torch.float64),
                        seg.to(torch.float64)], 1).contiguous()


def gather_results(block, n_total, world, rank, dst=0):
    """Gather every rank's (n_r, 3) block to `dst`; returns the concatenated
    (n_total, 3) tensor on dst, None elsewhere.  Uneven shards are padded to
    the common shard size for the collective and trimmed after."""
    k = -(-n_total // world)
    pad = torch.zeros((k, 3), dtype=block.dtype, device=block.device)
    pad[: block.shape[0]] = block
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    dist.gather(pad, bufs, dst=dst)
    if rank != dst:
        return None
    parts = []
    for r in range(world):
        lo, hi = shard_range(n_total, r, world)
        parts.append(bufs[r][: hi - lo])
    return torch.cat(parts, 0)


def gather_chunk(block, world, rank, dst=0, async_op=False):
    """Gather one equal-sized (k, 3) chunk block from every rank to `dst`.
    NCCL (CUDA tensors, async_op=True): the collective runs on NCCL's stream
    after the work already queued on the current stream, so the caller can
    queue the next chunk's projection at once; returns (work, bufs) -- wait on
    `work` before reading `bufs` (rank-ordered list on dst, None elsewhere).
    gloo: the block is staged through host memory and the call is blocking
    (work None)."""
    if block.is_cuda and dist.get_backend() == "gloo":
        block = block.cpu()
    bufs = [torch.empty_like(block) for _ in range(world)] if rank == dst else None
    work = dist.gather(block, bufs, dst=dst, async_op=async_op)
    return (work if async_op else None), bufs


def unchunk(chunk_bufs, world, n_per_rank, bounds):
    """Reassemble rank-0 gathered chunks (list over chunks of rank-ordered
    block lists) into the (world * n_per_rank, 3) result in global query
    order (rank-major, then chunk)."""
    out = []
    for r in range(world):
        for i in range(len(bounds) - 1):
            out.append(chunk_bufs[i][r].to("cpu"))
    return torch.cat(out, 0)
