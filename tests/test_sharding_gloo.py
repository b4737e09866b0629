"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host path:
shard bounds, per-shard generation with base_offset, the verification
digest exchange and the max-over-ranks timing reduction. The per-shard data
comes from the CPU oracle here (no GPU); on the B200 the same code runs with
the device fill (bench.py)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1206_1187_b200 import sharding


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_total, q):
    import torch.distributed as dist

    import oracle as O

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = O.Oracle()
    start, count = sharding.shard(n_total, world, rank)
    parts = []
    for s, c in sharding.chunks(start, count, 40000):
        buf = o.fill(c, O.FMT_F64, base_offset=s, threads=2)
        parts.append(o.digest(buf.view(np.uint64), index_base=s))
    local = sharding.combine(parts)
    glob = sharding.allgather_digest(local)
    t = sharding.max_over_ranks(float(rank + 1))
    if rank == 0:
        q.put((glob, t))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_shards_concatenate_to_the_serial_stream(world, oracle):
    import oracle as O

    n_total = 250_003
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_total, q)) for r in range(world)]
    for p in procs:
        p.start()
    glob, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    whole = oracle.fill(n_total, O.FMT_F64)
    assert glob == oracle.digest(whole.view(np.uint64))
    assert tmax == float(world)


def test_shard_bounds_match_make_plan(oracle):
    for n, w in ((10, 3), (1 << 36, 8), (7, 16), (1, 1), (1000003, 7)):
        eff, wpw = oracle.make_plan(n, w)
        got = [sharding.shard(n, w, r) for r in range(w)]
        assert sum(c for _, c in got) == n
        for r in range(eff):
            assert got[r] == (r * wpw, min(wpw, n - r * wpw))
        assert all(c == 0 for _, c in got[eff:])
    assert list(sharding.chunks(5, 10, 4)) == [(5, 4), (9, 4), (13, 2)]
    with pytest.raises(ValueError):
        sharding.shard(0, 2, 0)
