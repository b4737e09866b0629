"""Index-space sharding across GPUs and digest combination.

The sequence is partitioned by logical index exactly like the reference
partitions it over threads (make_plan, parallel.cpp:35-52): rank r of W owns
[r*ceil(N/W), min(N, (r+1)*ceil(N/W))) and fills it with base_offset = its
start. There is no collective on the data path; the only collective is the
optional verification exchange of 3 x u64 digests per rank.
"""
from __future__ import annotations

MASK = (1 << 64) - 1


def shard(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """(start, count) of `rank`'s contiguous shard of make_plan(n_total, world)."""
    if n_total <= 0 or world <= 0 or not 0 <= rank < world:
        raise ValueError("shard: need n_total > 0, world > 0, 0 <= rank < world")
    wpw = -(-n_total // world)
    start = min(n_total, rank * wpw)
    return start, max(0, min(wpw, n_total - start))


def chunks(start: int, count: int, max_chunk: int):
    """Split [start, start+count) into launches of at most max_chunk items."""
    off = 0
    while off < count:
        c = min(max_chunk, count - off)
        yield start + off, c
        off += c


def combine(parts) -> tuple[int, int, int]:
    """Combine per-shard digests (each computed with index_base = shard start)
    into the digest of the concatenation: sums mod 2^64 and xor."""
    s = ws = x = 0
    for d in parts:
        s = (s + int(d[0])) & MASK
        ws = (ws + int(d[1])) & MASK
        x ^= int(d[2])
    return s, ws, x


def _to_i64(v: int) -> int:
    v &= MASK
    return v - (1 << 64) if v >= 1 << 63 else v


def allgather_digest(d, device=None) -> tuple[int, int, int]:
    """All-gather every rank's digest (torch.distributed, any backend) and
    combine. 24 bytes per rank; used for verification only."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([_to_i64(x) for x in d], dtype=torch.int64, device=device)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return combine([[int(v) & MASK for v in o.tolist()] for o in out])


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank scalar (timings are reported as the max over ranks)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
