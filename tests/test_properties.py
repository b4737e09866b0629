"""Property-based checks (hypothesis) of the host side of the boundary on CPU:
the C-ABI scalar generator entry points and plan arithmetic against the
oracle, the closed form the seeding kernel uses, and the multi-GPU shard /
digest algebra. No kernel launches; these run in the `-m "not gpu"` suite."""
from __future__ import annotations

import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle as O
from paper_1206_1187_b200 import sharding

M = 5559060566555523
P = 3706040377703682
A0 = M + 100

seeds = st.integers(min_value=A0, max_value=1 << 53)
offsets = st.integers(min_value=0, max_value=(1 << 64) - 1)
ORACLE = O.Oracle()


@settings(max_examples=300, deadline=None)
@given(a=seeds, k=offsets)
def test_state_at_matches_oracle_and_closed_form(bcn, a, k):
    """generator.cpp:42-49 through the C ABI == the oracle == the closed form
    z_k = m - 2^((a - 3^33 - 1 + 53 k) mod P) mod m used by the seeding kernel."""
    z = bcn.gen.state_at(a, k).z
    assert z == ORACLE.state_at(a, k)
    assert z == M - pow(2, (a - M - 1 + 53 * k) % P, M)


@settings(max_examples=200, deadline=None)
@given(a=seeds, k=offsets, steps=st.integers(min_value=1, max_value=40))
def test_skip_ahead_composes_with_next(bcn, a, k, steps):
    """test_generator.cpp:85-114: state_at(a, k) followed by `steps` next()
    calls is the state k + steps steps in (as an exact integer: stepping past
    k = 2^64 - 1 does not wrap the exponent, unlike a u64 argument to
    state_at, since P does not divide 2^64)."""
    s = bcn.gen.state_at(a, k)
    for _ in range(steps):
        bcn.gen.next(s)
    assert s.z == M - pow(2, (a - M - 1 + 53 * (k + steps)) % P, M)
    if k + steps < 1 << 64:
        assert s.z == bcn.gen.state_at(a, k + steps).z


@settings(max_examples=200, deadline=None)
@given(z=st.integers(min_value=1, max_value=M - 1))
def test_to_unit_interval_is_one_rounded_multiply(bcn, z):
    """generator.hpp:74-78 / test_generator.cpp:131-132: RN(double(z) * RN(1/m))."""
    u = bcn.gen.to_unit_interval(z)
    assert u == float(np.float64(z) * np.float64(1.0 / M))
    assert 0.0 < u < 1.0


@settings(max_examples=150, deadline=None)
@given(n=st.integers(min_value=1, max_value=3000), workers=st.integers(min_value=1, max_value=70),
       layout=st.sampled_from([0, 1]))
def test_physical_index_is_a_bijection_matching_the_oracle(bcn, n, workers, layout):
    """parallel.cpp:24-52: the plan's physical_index covers [0, n) exactly once
    and agrees with the oracle's restatement for every (w, i)."""
    plan = bcn.par.make_plan(n, workers, bcn.Layout(layout))
    eff, wpw = ORACLE.make_plan(n, workers)
    assert (plan.workers, plan.work_per_worker) == (eff, wpw)
    seen = set()
    for w in range(plan.workers):
        for i in range(min(wpw, n - w * wpw)):
            q = plan.physical_index(w, i)
            assert q == ORACLE.physical_index(n, workers, layout, w, i)
            seen.add(q)
    assert seen == set(range(n))


@settings(max_examples=300, deadline=None)
@given(n=st.integers(min_value=1, max_value=1 << 40), world=st.integers(min_value=1, max_value=64))
def test_shards_partition_the_index_space(n, world):
    """make_plan(n, G) shards: contiguous, disjoint, covering [0, n)."""
    pos = 0
    for r in range(world):
        start, count = sharding.shard(n, world, r)
        if count:
            assert start == pos
            pos += count
    assert pos == n


@settings(max_examples=60, deadline=None)
@given(n=st.integers(min_value=2, max_value=20000), cuts=st.lists(st.floats(0, 1), max_size=6),
       base=st.integers(min_value=0, max_value=1 << 50))
def test_shard_digests_combine_to_the_whole(n, cuts, base):
    """The verification exchange: digests of contiguous pieces (each with its
    own index_base) combine to the digest of the concatenation."""
    buf = ORACLE.fill(n, O.FMT_U64, base_offset=base)
    edges = sorted({0, n, *[int(c * n) for c in cuts]})
    parts = [ORACLE.digest(buf[lo:hi], index_base=lo) for lo, hi in zip(edges, edges[1:]) if hi > lo]
    assert sharding.combine(parts) == ORACLE.digest(buf, index_base=0)
