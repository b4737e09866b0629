"""Pins the CPU oracle (oracle/bcn_oracle.c) before it is trusted as the GPU
checker: against the reference's own golden values (tests/test_modred.cpp,
test_generator.cpp, test_cli.cpp), the committed fixtures
made by running the reference (tests/golden/reference_vectors.json), and —
where it is built — the reference library itself (oracle/_ref)."""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.json")
U64 = (1 << 64) - 1
HALF_M = 2779530283277761


# ------------------------------------------------------------- modred goldens
def test_reduce_ref_goldens(oracle):
    """test_modred.cpp:13-16, :38-44"""
    assert oracle.reduce_ref(0) == 0
    assert oracle.reduce_ref(1) == 3448138688185469
    assert oracle.reduce_ref(HALF_M) == 1055460939185027
    assert oracle.reduce_ref(O.MODULUS - 1) == 2110921878370054
    with pytest.raises(O.DomainError):
        oracle.reduce_ref(O.MODULUS)


def test_modified_barrett_exhaustive_and_random(oracle):
    """test_modred.cpp:73-96 (exhaustive [1, 1e5) + random residues)."""
    for z in range(1, 100000, 7):
        assert oracle.barrett_modified_step(z) == oracle.reduce_ref(z)
    rng = np.random.Generator(np.random.MT19937(0xB0C1D2E3))
    for z in rng.integers(1, O.MODULUS, size=20000, dtype=np.uint64):
        assert oracle.barrett_modified_step(int(z)) == oracle.reduce_ref(int(z))
    with pytest.raises(O.DomainError):
        oracle.barrett_modified_step(0)


def test_modified_barrett_worst_case_quotient(oracle):
    """The q3 = Q-1 branch (SURVEY §7 hard part 3): residues whose 2^53 z mod m
    is tiny exercise the r >= m correction."""
    hits = 0
    for r in (1, 2, 4, 1000, 3 * 10**15):
        # z = r * 2^-53 mod m has 2^53 z mod m == r.
        z = r * pow(2, -53, O.MODULUS) % O.MODULUS
        if z:
            assert oracle.barrett_modified_step(z) == r
            hits += 1
    assert hits == 5


# ----------------------------------------------------------- generator goldens
def test_generator_goldens(oracle):
    """test_generator.cpp:13-17, :20-28, :85-101"""
    assert oracle.modpow2(0) == 1
    assert oracle.modpow2(53) == 3448138688185469
    assert oracle.modpow2(106) == 5239873117944745
    with pytest.raises(O.InvalidArgument):
        oracle.modpow2(10, 4)
    with pytest.raises(O.InvalidArgument):
        oracle.modpow2(10, (1 << 63) + 1)
    assert oracle.seed_from_index(O.MIN_SEED) == 4258649398211344
    assert oracle.seed_from_index(O.MAX_SEED) == 1895384862748766
    assert oracle.state_at(O.MIN_SEED, 1) == 2138759898642167
    assert oracle.state_at(O.MIN_SEED, 1000) == 5492007519572011
    with pytest.raises(O.OutOfRange):
        oracle.seed_from_index(O.MIN_SEED - 1)
    with pytest.raises(O.OutOfRange):
        oracle.seed_from_index(O.MAX_SEED + 1)
    assert oracle.state_at(O.MIN_SEED, 123456789) == oracle.state_at(O.MIN_SEED, 123456789 + O.PERIOD)


def test_closed_form_state(oracle):
    """The closed form every kernel relies on (bcn_math.cuh):
    z_k(a) = m - 2^((a - 3^33 - 1 + 53 k) mod P) mod m."""
    rng = np.random.Generator(np.random.MT19937(20000))
    for _ in range(2000):
        a = int(rng.integers(O.MIN_SEED, O.MAX_SEED + 1))
        k = int(rng.integers(0, U64, endpoint=True, dtype=np.uint64))
        e = (a - O.MODULUS - 1 + 53 * k) % O.PERIOD
        assert oracle.state_at(a, k) == O.MODULUS - pow(2, e, O.MODULUS)


def test_seed_doubling_and_units(oracle):
    """test_generator.cpp:44-52, :135-144"""
    for a in (O.MIN_SEED, O.MIN_SEED + 12345, O.MAX_SEED - 1):
        assert oracle.seed_from_index(a + 1) == 2 * oracle.seed_from_index(a) % O.MODULUS
    z = oracle.seed_from_index(O.MIN_SEED + 777)
    for _ in range(2000):
        z = oracle.next(z)
        assert z % 3 != 0
        assert 0.0 < oracle.to_unit_interval(z) < 1.0


def test_unit_interval_normative_and_f32(oracle):
    """test_generator.cpp:123-133 and the repo's f32 definition (RZ of f64)."""
    assert oracle.to_unit_interval(12345677) == 12345677.0 * (1.0 / 5559060566555523.0)
    with pytest.raises(O.DomainError):
        oracle.to_unit_interval(0)
    for z in (1, 2, HALF_M, O.MODULUS - 1, 12345677, O.MODULUS - 2):
        d = oracle.to_unit_interval(z)
        f = oracle.to_unit_float(z)
        assert 0.0 < float(f) <= d < 1.0  # RZ never rounds up, so never reaches 1.0f
        assert d - float(f) < 2.0 ** -24 * d * 2
        assert O.f32_rz(np.array([d]))[0] == f
    # the largest residue: RN would give 1.0f; RZ stays below 1
    assert float(oracle.to_unit_float(O.MODULUS - 1)) < 1.0


# ---------------------------------------------------------------- config 1
def test_config1_appendix_a(oracle):
    """SURVEY Appendix A / test_cli.cpp:76-86: n = 10^6 from a0."""
    u = oracle.fill(10**6, O.FMT_F64, threads=1)
    z = oracle.fill(10**6, O.FMT_U64)
    assert hashlib.sha256(u.tobytes()).hexdigest() == \
        "eb8dc6c55cbbf8dd7d64a7a08583401aecfcc89d22fa112aa6d83e12a3d8fa0f"
    assert hashlib.sha256(z.tobytes()).hexdigest() == \
        "05ad1e442fe2fe60371779e0b73add6454f16304f0375dd9f0a0b82bce2db223"
    assert oracle.digest(z)[0] == 11204447702781092184
    acc = 0
    for i, b in enumerate(u.view(np.uint64)):
        acc ^= (int(b) * (2 * i + 1)) & U64
    assert acc == 0xae3d99be5727a391
    assert [int(x) for x in z[:4]] == [2138759898642167, 906908310809773, 121054228244396,
                                       915076623799633]
    assert int(u.view(np.uint64)[999999]) == 0x3fd82ada9a711586


def test_period_wrap_and_far_offset(oracle):
    assert [int(x) for x in oracle.fill(6, O.FMT_U64, base_offset=O.PERIOD - 3)] == [
        1867496909077246, 5488691822377859, 4258649398211344, 2138759898642167,
        906908310809773, 121054228244396]
    assert [int(x) for x in oracle.fill(6, O.FMT_U64, seed_index=1 << 53, base_offset=1 << 40,
                                        workers=3, layout=O.INTERLEAVED)] == [
        1584414649962571, 4289752975226581, 752696664753940, 663488620216616,
        2266604546227133, 4919938457993333]


# ------------------------------------------------------------ plans & fills
def test_plan_and_physical_index(oracle):
    """test_parallel.cpp:22-71"""
    assert oracle.make_plan(8, 2) == (2, 4)
    assert oracle.make_plan(7, 2) == (2, 4)
    assert oracle.make_plan(3, 16) == (3, 1)
    with pytest.raises(O.InvalidArgument):
        oracle.make_plan(0, 2)
    with pytest.raises(O.InvalidArgument):
        oracle.make_plan(5, 0)
    rng = np.random.Generator(np.random.MT19937(5))
    for _ in range(60):
        n = int(rng.integers(1, 300))
        w = int(rng.integers(1, 10))
        for layout in (0, 1):
            eff, wpw = oracle.make_plan(n, w)
            seen = set()
            for ww in range(eff):
                for i in range(min(wpw, n - ww * wpw)):
                    p = oracle.physical_index(n, w, layout, ww, i)
                    assert 0 <= p < n and p not in seen
                    seen.add(p)
            assert len(seen) == n


def test_fill_thread_count_invariance(oracle):
    ref = oracle.fill(100003, O.FMT_F64, workers=7, layout=1, threads=1)
    for t in (2, 3, 8, 13):
        assert np.array_equal(oracle.fill(100003, O.FMT_F64, workers=7, layout=1, threads=t), ref)


def test_deinterleave_roundtrip(oracle):
    n, w = 10000, 6
    phys = oracle.fill(n, O.FMT_F64, workers=w, layout=1)
    assert np.array_equal(oracle.deinterleave(phys, w), oracle.fill(n, O.FMT_F64))


# ------------------------------------------------ committed reference fixtures
def _golden():
    with open(GOLDEN) as f:
        return json.load(f)


def test_oracle_matches_reference_fixtures(oracle):
    """Fixtures generated by running the reference (tests/golden/make_golden.py)."""
    g = _golden()
    sc = g["scalars"]
    for a, z in sc["seed_from_index"].items():
        assert oracle.seed_from_index(int(a)) == z
    for a, k, z in sc["state_at"]:
        assert oracle.state_at(a, k) == z
    for e, m, v in sc["modpow2"]:
        assert oracle.modpow2(e, m) == v
    for z, v in sc["step"]:
        assert oracle.next(z) == v
    for z, b in sc["to_unit_interval_bits"]:
        assert int(np.float64(oracle.to_unit_interval(z)).view(np.uint64)) == b
    for n, w, eff, wpw in sc["make_plan"]:
        assert oracle.make_plan(n, w) == (eff, wpw)
    assert len(g["fills"]) >= 30
    for c in g["fills"]:
        out = oracle.fill(c["n"], c["fmt"], seed_index=c["seed_index"], base_offset=c["base_offset"],
                          workers=c["workers"], layout=c["layout"])
        bits = out.view(np.uint64)
        assert [str(x) for x in oracle.digest(bits)] == c["digest"], c
        if "values" in c:
            assert [str(int(x)) for x in bits] == c["values"]
        else:
            assert [str(int(x)) for x in bits[:8]] == c["head"]
            assert [str(int(x)) for x in bits[-8:]] == c["tail"]


def test_oracle_matches_reference_library(oracle, reference):
    """Live comparison with the compiled reference (skipped where it is absent)."""
    rng = np.random.Generator(np.random.MT19937(77))
    for _ in range(40):
        n = int(rng.integers(1, 5000))
        w = int(rng.integers(1, 12))
        layout = int(rng.integers(0, 2))
        seed = int(rng.integers(O.MIN_SEED, O.MAX_SEED + 1))
        base = int(rng.integers(0, U64, endpoint=True, dtype=np.uint64))
        fmt = int(rng.integers(0, 2))
        a = oracle.fill(n, fmt, seed_index=seed, base_offset=base, workers=w, layout=layout)
        b = reference.fill(n, fmt, seed_index=seed, base_offset=base, workers=w, layout=layout,
                           method=int(rng.integers(0, 4)))
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    walk = reference.walk(O.MIN_SEED, 5, 100)
    z = oracle.state_at(O.MIN_SEED, 5)
    for v in walk:
        z = oracle.next(z)
        assert z == v


def test_c5_digest_fixture_consistent(oracle):
    """The committed 2^36 digest (tests/golden/c5_digest.json) is a pure function
    of the oracle; spot-check its generator on a 2^22 prefix."""
    path = os.path.join(os.path.dirname(__file__), "golden", "c5_digest.json")
    if not os.path.exists(path) or os.path.getsize(path) == 0:
        pytest.skip("c5 digest not generated yet")
    with open(path) as f:
        d = json.load(f)
    assert d["log2n"] == 36 and len(d["digest"]) == 3


def test_chunk_digest_goldens_pinned(oracle, reference):
    """tests/golden/chunk_digests.json (per-2^24-chunk digests of the first 2^33
    variates, every format) recomputed for sampled chunks: the oracle in all
    three formats, the unmodified reference (oracle/_ref) in u64 and f64."""
    path = os.path.join(os.path.dirname(__file__), "golden", "chunk_digests.json")
    with open(path) as f:
        g = json.load(f)
    chunk = 1 << g["chunk_log2"]
    assert g["seed_index"] == O.MIN_SEED and g["log2n"] == 33
    rng = np.random.default_rng(0x1206)
    picks = sorted({0, 63, 64, 255, 511, *rng.integers(0, 512, 2).tolist()})
    for name, fmt in (("u64", O.FMT_U64), ("f64", O.FMT_F64), ("f32", O.FMT_F32)):
        assert len(g["formats"][name]) == 512
        for c in picks:
            buf = oracle.fill(chunk, fmt, base_offset=c * chunk)
            view = buf.view(np.uint64 if buf.itemsize == 8 else np.uint32)
            assert [str(x) for x in oracle.digest(view, index_base=c * chunk)] == g["formats"][name][c]
            if fmt != O.FMT_F32 and c in (0, 255):
                rbuf = reference.fill(chunk, fmt, base_offset=c * chunk)
                assert [str(x) for x in oracle.digest(rbuf.view(np.uint64), index_base=c * chunk)] == \
                    g["formats"][name][c]
