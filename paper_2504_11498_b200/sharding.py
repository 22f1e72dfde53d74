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
