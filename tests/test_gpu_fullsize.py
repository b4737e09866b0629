"""Full-size parity at the configurations `north_star` names (SURVEY §8d C2,
C3, C5): EVERY 2^24-element chunk of the device output is compared with the
digest the CPU oracle computed for it (`tests/golden/chunk_digests.json`,
`tests/golden/make_chunk_digests.py`; its u64/f64 rows are spot-checked against
the unmodified reference compiled in `oracle/_ref`), and the 2^36 C5 stream
with the oracle's digest of all of it (`tests/golden/c5_digest.json`).

Reference contract: `par::fill` / `par::fill_residues` over the whole window
(`/root/reference/proj/src/parallel.cpp:56-79`, `:101-111`). A digest is
(Σv, Σ(g+1)v, XOR v(2g+1)) mod 2^64 over the item bits at absolute index g.
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu

A0 = O.MIN_SEED
HERE = os.path.dirname(os.path.abspath(__file__))
CHUNK = 1 << 24
MASK = (1 << 64) - 1
FMT = {"u64": (O.FMT_U64, torch.int64), "f64": (O.FMT_F64, torch.float64),
       "f32": (O.FMT_F32, torch.float32)}


def _load(name):
    with open(os.path.join(HERE, "golden", name)) as f:
        return json.load(f)


GOLD = _load("chunk_digests.json")


def golden_chunks(fmt: str, c0: int, c1: int) -> list[tuple[int, int, int]]:
    return [tuple(int(x) for x in r) for r in GOLD["formats"][fmt][c0:c1]]


def combine(parts) -> tuple[int, int, int]:
    s = ws = x = 0
    for d in parts:
        s, ws, x = (s + d[0]) & MASK, (ws + d[1]) & MASK, x ^ d[2]
    return s, ws, x


def raw(buf: torch.Tensor) -> torch.Tensor:
    return buf.view(torch.int32 if buf.element_size() == 4 else torch.int64)


def device_chunks(bcn, buf: torch.Tensor, index_base: int) -> list[tuple[int, int, int]]:
    """Per-2^24 chunk digests of a device buffer whose element 0 sits at
    absolute index `index_base` (a multiple of 2^24)."""
    r = raw(buf)
    return [bcn.device.digest(r[o:o + CHUNK], index_base=index_base + o)
            for o in range(0, r.numel(), CHUNK)]


def fill(bcn, buf, fmt, base, engine="Auto"):
    bcn.par.fill_format(buf, bcn.par.make_plan(buf.numel(), 1), A0, bcn.Method.BarrettModified, base,
                        bcn.par.Format(FMT[fmt][0]), engine=bcn.par.Engine[engine], sync=True)


def first_bad(got, want):
    bad = [i for i, (g, w) in enumerate(zip(got, want)) if tuple(g) != tuple(w)]
    return bad[:8]


@pytest.fixture(autouse=True)
def _release():
    yield
    torch.cuda.empty_cache()


# ------------------------------------------------------------------- C2
@pytest.mark.parametrize("fmt", ["f64", "u64", "f32"])
def test_c2_every_chunk_vs_oracle(bcn, cuda, fmt):
    """C2: 2^30 variates from a0 on one B200 — all 64 chunks bit-exact (the
    bench headline's exact launch: default engine, paced kernel for u64/f64)."""
    n = 1 << 30
    buf = torch.empty(n, dtype=FMT[fmt][1], device=cuda)
    fill(bcn, buf, fmt, 0)
    got = device_chunks(bcn, buf, 0)
    want = golden_chunks(fmt, 0, n // CHUNK)
    assert first_bad(got, want) == []


@pytest.mark.parametrize("rank", [1, 7])
def test_c2_weak_scaling_shard_vs_oracle(bcn, cuda, rank):
    """Rank r of the weak-scaling bench fills [r 2^30, (r+1) 2^30) with
    base_offset r 2^30: every chunk of the shards of ranks 1 and 7 (of 8)."""
    n = 1 << 30
    buf = torch.empty(n, dtype=torch.float64, device=cuda)
    fill(bcn, buf, "f64", rank * n)
    got = device_chunks(bcn, buf, rank * n)
    want = golden_chunks("f64", rank * 64, (rank + 1) * 64)
    assert first_bad(got, want) == []


# ------------------------------------------------------------------- C3
@pytest.mark.parametrize("log2n", [31, 32])
@pytest.mark.parametrize("fmt", ["u64", "f64", "f32"])
def test_c3_full_window_every_engine(bcn, cuda, fmt, log2n):
    """C3 at 2^31 and 2^32 variates: the default engine chunk by chunk, then
    every other engine (Barrett and Montgomery included) over the whole window
    in the same buffer."""
    n = 1 << log2n
    buf = torch.empty(n, dtype=FMT[fmt][1], device=cuda)
    fill(bcn, buf, fmt, 0)
    want = golden_chunks(fmt, 0, n // CHUNK)
    assert first_bad(device_chunks(bcn, buf, 0), want) == []
    whole = combine(want)
    for engine in ("Barrett", "Montgomery", "FP64", "Mixed", "Bulk", "Staged"):
        raw(buf).fill_(-1)
        fill(bcn, buf, fmt, 0, engine)
        assert bcn.device.digest(raw(buf)) == whole, engine


def test_c3_ragged_misaligned_full_scale(bcn, cuda, oracle):
    """A 2^31 + 12345 item fill at base_offset 3 * 2^24 into a buffer one item
    past a 32-byte boundary (edge rows, partial last round of the paced grid):
    the 128 whole chunks against the goldens, the ragged tail against the oracle."""
    for fmt in ("f64", "f32"):
        n = (1 << 31) + 12345
        base = 3 * CHUNK
        store = torch.full((n + 1,), -1, dtype=torch.int64 if fmt == "f64" else torch.int32, device=cuda)
        buf = store[1:].view(FMT[fmt][1])
        fill(bcn, buf, fmt, base)
        whole = (n // CHUNK) * CHUNK
        got = device_chunks(bcn, buf[:whole], base)
        assert first_bad(got, golden_chunks(fmt, 3, 3 + whole // CHUNK)) == [], fmt
        tail = oracle.fill(n - whole, FMT[fmt][0], base_offset=base + whole)
        dev_tail = buf[whole:].cpu().numpy()
        assert np.array_equal(dev_tail.view(np.uint8), tail.view(np.uint8)), fmt
        assert int(store[0].item()) == -1  # nothing written before the buffer


# ------------------------------------------------------------------- C5
@pytest.mark.parametrize("shards", [1, 3, 8])
def test_c5_2e36_digest_one_gpu(bcn, cuda, shards):
    """C5: the 2^36-double stream (512 GiB) generated on one GPU as the index
    shards of make_plan(2^36, G) — G = 3 makes the shard boundaries
    non-chunk-aligned — each shard in launches of <= 2^32 items, digests
    combined: equal to the oracle's digest of all 2^36 doubles. The first 2^33
    doubles are also checked chunk by chunk."""
    from paper_1206_1187_b200 import sharding

    want = tuple(int(x) for x in _load("c5_digest.json")["digest"])
    total = 1 << 36
    buf = torch.empty(1 << 32, dtype=torch.float64, device=cuda)
    parts = []
    for r in range(shards):
        start, count = sharding.shard(total, shards, r)
        for b, c in sharding.chunks(start, count, 1 << 32):
            fill(bcn, buf[:c], "f64", b)
            parts.append(bcn.device.digest(raw(buf[:c]), index_base=b))
            if shards == 1 and b < (1 << 33):
                assert first_bad(device_chunks(bcn, buf[:c], b),
                                 golden_chunks("f64", b // CHUNK, (b + c) // CHUNK)) == []
    assert combine(parts) == want
