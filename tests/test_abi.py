"""CPU-side checks of the C-ABI boundary (no kernel launches): the product
library loads, exports every symbol include/bcnrand_b200.h declares, its host
entry points agree with the oracle, errors map onto the reference's exception
types, and generating calls fail loudly — never silently on the CPU — when
there is no CUDA device."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bcnrand_b200.h")


def declared_symbols() -> list[str]:
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(bcn_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("bcn_fill", "bcn_seed_from_index", "bcn_state_at", "bcn_next", "bcn_make_plan",
              "bcn_physical_index", "bcn_deinterleave", "bcn_seed_states", "bcn_fill_multi",
              "bcn_digest", "bcn_fill_constant", "bcn_fill_noise", "bcn_engine_check", "bcn_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(bcn):
    from paper_1206_1187_b200 import _lib

    so = _lib.LIB_PATH
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True,
                         check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    # and the Python binding covers all of them
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert set(declared_symbols()) <= bound
    assert _lib.lib().bcn_abi_version() == 2


def test_library_is_sm100a_code(bcn):
    """The fatbin holds sm_100a SASS with 256-bit stores and TMA bulk copies."""
    from paper_1206_1187_b200 import _lib

    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True,
                          check=True).stdout
    assert "arch = sm_100a" in sass
    assert "STG.E.ENL2.256" in sass or "STG.E.256" in sass
    assert "UBLKCP" in sass


def test_host_generator_entry_points_match_oracle(bcn, oracle):
    g = bcn.gen
    rng = np.random.Generator(np.random.MT19937(3))
    for _ in range(300):
        a = int(rng.integers(O.MIN_SEED, O.MAX_SEED + 1))
        k = int(rng.integers(0, (1 << 64) - 1, endpoint=True, dtype=np.uint64))
        assert g.seed_from_index(a).z == oracle.seed_from_index(a)
        assert g.state_at(a, k).z == oracle.state_at(a, k)
        z = oracle.state_at(a, k)
        s = g.GeneratorState(a, z, k)
        assert g.next(s) == oracle.next(z) and s.k == k + 1
        assert g.to_unit_interval(s.z) == oracle.to_unit_interval(s.z)
    for e in (0, 53, 106, (1 << 64) - 1):
        assert g.modpow2(e, O.MODULUS) == oracle.modpow2(e)
    assert g.modpow2(12345, 1000003) == pow(2, 12345, 1000003)


def test_error_mapping(bcn):
    g, par = bcn.gen, bcn.par
    with pytest.raises(bcn.OutOfRange):
        g.seed_from_index(O.MIN_SEED - 1)
    with pytest.raises(bcn.OutOfRange):
        g.state_at(O.MAX_SEED + 1, 5)
    with pytest.raises(bcn.InvalidArgument):
        g.modpow2(10, 4)
    with pytest.raises(bcn.InvalidArgument):
        g.modpow2(10, (1 << 63) + 1)
    with pytest.raises(bcn.DomainError):
        g.to_unit_interval(0)
    with pytest.raises(bcn.DomainError):
        g.to_unit_interval(O.MODULUS)
    with pytest.raises(bcn.DomainError):
        g.next(g.GeneratorState(O.MIN_SEED, 0, 0))
    with pytest.raises(bcn.InvalidArgument):
        par.make_plan(0, 2)
    with pytest.raises(bcn.InvalidArgument):
        par.make_plan(5, 0)
    with pytest.raises(bcn.InvalidArgument):
        g.parse_method("mt19937")
    assert g.parse_method("barrettmodified") == g.Method.BarrettModified
    assert g.method_name(g.Method.Barrett) == "Barrett"
    # InvalidArgument is a ValueError, OutOfRange an IndexError (Python idiom)
    assert issubclass(bcn.InvalidArgument, ValueError) and issubclass(bcn.OutOfRange, IndexError)


def test_validation_precedes_device_work(bcn):
    """Size and seed errors are reported before any CUDA call, so they surface
    identically with or without a GPU (parallel.cpp:59-61, generator.cpp:33-35)."""
    par = bcn.par
    small = np.empty(99, dtype=np.float64)
    with pytest.raises(bcn.InvalidArgument):
        par.fill(small, par.make_plan(100, 2), O.MIN_SEED)
    buf = np.empty(100, dtype=np.float64)
    with pytest.raises(bcn.OutOfRange):
        par.fill(buf, par.make_plan(100, 8), O.MIN_SEED - 1)
    with pytest.raises(bcn.InvalidArgument):
        par.fill_residues(buf, par.make_plan(100, 1), O.MIN_SEED)


def test_no_cpu_fallback_without_gpu(bcn):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    buf = np.full(1000, -1.0)
    with pytest.raises(bcn.CudaError, match="no CUDA device"):
        bcn.par.fill(buf, bcn.par.make_plan(1000, 1), O.MIN_SEED)
    assert (buf == -1.0).all()  # nothing was computed on the host
    # the other device-only entry points fail the same way (no host compute)
    from paper_1206_1187_b200 import _lib

    assert _lib.lib().bcn_l2_bytes(0) == 0 and _lib.lib().bcn_device_count() == 0
    with pytest.raises(bcn.CudaError):
        bcn.device.engine_check(bcn.Engine.FP64, np.array([5], dtype=np.uint64), np.array([7], dtype=np.uint64))


def test_physical_index_and_plans_match_reference_semantics(bcn, oracle):
    par = bcn.par
    rng = np.random.Generator(np.random.MT19937(8))
    for _ in range(40):
        n = int(rng.integers(1, 400))
        w = int(rng.integers(1, 12))
        for layout in (par.Layout.Contiguous, par.Layout.Interleaved):
            plan = par.make_plan(n, w, layout)
            assert (plan.workers, plan.work_per_worker) == oracle.make_plan(n, w)
            assert plan.start_offsets == [i * plan.work_per_worker for i in range(plan.workers)]
            for ww in range(plan.workers):
                for i in range(plan.elements_for(ww)):
                    assert plan.physical_index(ww, i) == oracle.physical_index(n, w, int(layout), ww, i)
    with pytest.raises(bcn.InvalidArgument):
        par.make_plan(10, 3).physical_index(3, 0)
    p = par.make_plan(3, 16)
    assert p.workers == 3 and p.work_per_worker == 1  # test_parallel.cpp:36-40


def test_engine_names(bcn):
    from paper_1206_1187_b200 import _lib

    names = [_lib.lib().bcn_engine_name(i).decode() for i in range(8)]
    assert names == ["auto", "barrett", "montgomery", "fp64", "staged", "bulk", "mixed", "hybrid"]
    assert bcn.par.Engine(_lib.lib().bcn_auto_engine(1)) in (bcn.Engine.Barrett, bcn.Engine.FP64)
    assert _lib.lib().bcn_last_error() is not None
    assert isinstance(_lib.lib().bcn_launch_count(), int)


def test_oracle_is_not_linked_into_the_product(bcn):
    from paper_1206_1187_b200 import _lib

    out = subprocess.run(["nm", "-D", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "bcno_" not in out and "bref_" not in out
    ldd = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in ldd and "bcnref" not in ldd
    assert ctypes  # keep import


def test_pacing_and_multi_gpu_arguments_validated_without_device(bcn):
    """absurd pacing targets and short fill_multi shards are
    invalid_argument before any device work (no GPU needed to see it)."""
    import ctypes

    from paper_1206_1187_b200 import _lib

    h = _lib.lib()
    old = bcn.device.write_pacing_config()
    try:
        for bad in (1e-12, 50.0, 99.9, float("nan"), 2e5):
            assert h.bcn_set_write_pacing(bad, 1, 3) == 1, bad
        for good in (0.0, 100.0, 7200.0, -1.0):
            assert h.bcn_set_write_pacing(good, 1, 3) == 0, good
        assert h.bcn_write_pacing() == -1.0  # automatic
    finally:
        h.bcn_set_write_pacing(*old)
    out = np.empty(64, dtype=np.float64)
    ptrs = (ctypes.c_void_p * 2)(out.ctypes.data, out.ctypes.data)
    devs = (ctypes.c_int * 2)(0, 0)
    caps = (ctypes.c_uint64 * 2)(50, 49)  # make_plan(100, 2): 50 + 50
    assert h.bcn_fill_multi(ptrs, caps, devs, 2, 100, 1, O.MIN_SEED, 0, 0, None) == 1
    assert b"smaller than its shard" in h.bcn_last_error()
    assert h.bcn_fill_multi(ptrs, None, devs, 2, 100, 1, O.MIN_SEED, 0, 0, None) == 1


def test_python_mirror_matches_reference_scalar_semantics(bcn):
    """next() on z = 0 returns 0 for every method but
    BarrettModified (generator.hpp:52-70 with modred.hpp:150), and Python ints
    outside [0, 2^64) are rejected instead of truncated by ctypes."""
    g = bcn.gen
    for m in (g.Method.Ref128, g.Method.LEcuyer, g.Method.Barrett):
        s = g.GeneratorState(O.MIN_SEED, 0, 5, m)
        assert g.next(s) == 0 and s.k == 6
    with pytest.raises(bcn.DomainError):
        g.next(g.GeneratorState(O.MIN_SEED, 0, 0, g.Method.BarrettModified))
    with pytest.raises(bcn.OutOfRange):
        g.seed_from_index((1 << 64) + O.MIN_SEED)  # would truncate to a valid seed
    with pytest.raises(bcn.OutOfRange):
        g.state_at(-1, 0)
    with pytest.raises(bcn.DomainError):
        g.to_unit_interval((1 << 64) + 5)
    with pytest.raises(bcn.InvalidArgument):
        g.modpow2(1 << 64, 7)
    assert g.state_at(O.MIN_SEED, -1).z == g.state_at(O.MIN_SEED, (1 << 64) - 1).z  # k wraps like u64
    buf = np.empty(8, dtype=np.float64)
    with pytest.raises(bcn.OutOfRange):
        bcn.par.fill(buf, bcn.par.make_plan(8, 1), (1 << 64) + O.MIN_SEED)
