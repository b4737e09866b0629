"""GPU parity tests: the sm_100a fill path vs the CPU oracle and the compiled
reference, bit-exact. Mirrors the reference's own tests
(tests/test_parallel.cpp, test_generator.cpp, test_cli.cpp) on the device path.
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu

A0 = O.MIN_SEED
ENGINES = ["Barrett", "Montgomery", "FP64", "Staged", "Bulk", "Mixed", "Hybrid"]
FORMATS = [(O.FMT_U64, torch.int64, np.uint64), (O.FMT_F64, torch.float64, np.float64),
           (O.FMT_F32, torch.float32, np.float32)]


def dev_fill(bcn, n, fmt=O.FMT_F64, *, workers=1, layout=0, seed=A0, base=0, engine="Auto",
             offset=0, cuda="cuda:0"):
    """Fill on the device through the public API; returns host numpy bytes."""
    par = bcn.par
    tdt = {O.FMT_U64: torch.int64, O.FMT_F64: torch.float64, O.FMT_F32: torch.float32}[fmt]
    # Sentinel-filled (all ones) rather than torch.empty: the caching allocator
    # would otherwise hand back the previous case's (often identical) output
    # and hide an element the kernel failed to write.
    raw = torch.int32 if fmt == O.FMT_F32 else torch.int64
    buf = torch.full((n + offset,), -1, dtype=raw, device=cuda).view(tdt)
    plan = par.make_plan(n, workers, par.Layout(layout))
    view = buf[offset:]
    par.fill_format(view, plan, seed, bcn.Method.BarrettModified, base, par.Format(fmt),
                    engine=par.Engine[engine], sync=True)
    arr = view.cpu().numpy()
    return arr.view(np.uint64) if fmt == O.FMT_U64 else arr


def oracle_fill(oracle, n, fmt=O.FMT_F64, **kw):
    out = oracle.fill(n, fmt, **kw)
    return out


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64 if a.itemsize == 8 else np.uint32)


# --------------------------------------------------------------- config 1
def test_config1_goldens_f64_u64(bcn, cuda, oracle):
    """test_cli.cpp:76-86 and SURVEY Appendix A: n = 10^6 from a0, offset 0."""
    u = dev_fill(bcn, 10**6, O.FMT_F64)
    z = dev_fill(bcn, 10**6, O.FMT_U64)
    assert hashlib.sha256(u.tobytes()).hexdigest() == \
        "eb8dc6c55cbbf8dd7d64a7a08583401aecfcc89d22fa112aa6d83e12a3d8fa0f"
    assert hashlib.sha256(z.tobytes()).hexdigest() == \
        "05ad1e442fe2fe60371779e0b73add6454f16304f0375dd9f0a0b82bce2db223"
    assert int(z[0]) == 2138759898642167
    assert int(z[-1]) == 2099187967082161
    assert int(z.sum(dtype=np.uint64)) == 11204447702781092184


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("fmt", [O.FMT_U64, O.FMT_F64, O.FMT_F32])
def test_engines_formats_bit_exact(bcn, cuda, oracle, engine, fmt):
    """Every reduction engine and output format equals the oracle bit for bit
    (the reference's method-identity property, test_generator.cpp:70-83)."""
    n = 3 * 2**18 + 77  # ragged: head/tail paths around the vector body
    got = dev_fill(bcn, n, fmt, engine=engine, base=12345)
    want = oracle.fill(n, fmt, base_offset=12345)
    assert np.array_equal(bits(got), bits(want))


def test_hybrid_engine_every_split(cuda):
    """The hybrid engine with every FP64/Barrett split of a lane's streams
    (BCN_HYBRID_KF is read once per process, so each split runs in a child)."""
    code = (
        "import numpy as np, torch, oracle as O, paper_1206_1187_b200 as B\n"
        "o = O.Oracle()\n"
        "for fmt, dt in ((2, torch.float32), (1, torch.float64), (0, torch.int64)):\n"
        "    if fmt != 2 and KF > 3: continue\n"
        "    for n in (1, 1000, 3 * 2**16 + 5):\n"
        "        buf = torch.empty(n, dtype=dt, device='cuda:0')\n"
        "        B.par.fill_format(buf, B.par.make_plan(n, 1), B.kMinSeedIndex, B.Method.BarrettModified, 777,\n"
        "                          B.Format(fmt), engine=B.Engine.Hybrid, sync=True)\n"
        "        v = np.uint32 if fmt == 2 else np.uint64\n"
        "        assert np.array_equal(buf.cpu().numpy().view(v), o.fill(n, fmt, base_offset=777).view(v)), (KF, fmt, n)\n"
    )
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for kf in (1, 3, 5, 7):
        env = dict(os.environ, BCN_HYBRID_KF=str(kf))
        r = subprocess.run([sys.executable, "-c", f"KF = {kf}\n" + code], cwd=root, env=env,
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-3000:]


@pytest.mark.parametrize("offset", [1, 2, 3, 5])
def test_misaligned_outputs(bcn, cuda, oracle, offset):
    for fmt in (O.FMT_F64, O.FMT_F32):
        got = dev_fill(bcn, 5000, fmt, offset=offset)
        assert np.array_equal(bits(got), bits(oracle.fill(5000, fmt)))


@pytest.mark.parametrize("n", [1, 2, 3, 31, 127, 128, 129, 1023, 4096, 100003])
def test_small_and_ragged_sizes(bcn, cuda, oracle, n):
    for engine in ("Barrett", "FP64"):
        got = dev_fill(bcn, n, O.FMT_U64, engine=engine)
        assert np.array_equal(got, oracle.fill(n, O.FMT_U64))


# ------------------------------------------------------- plan invariance
@pytest.mark.parametrize("workers", [1, 2, 3, 4, 8, 16, 7, 1000, 99999])
def test_worker_and_layout_invariance(bcn, cuda, oracle, reference, workers):
    """test_parallel.cpp:82-96 / :98-105: logical output is W-invariant; the
    physical Interleaved buffer equals the reference's and deinterleaves to
    the serial stream."""
    n = 100000
    serial = oracle.fill(n, O.FMT_F64)
    for layout in (0, 1):
        got = dev_fill(bcn, n, O.FMT_F64, workers=workers, layout=layout)
        want = reference.fill(n, O.FMT_F64, workers=min(workers, 64), layout=layout) \
            if workers <= 64 else oracle.fill(n, O.FMT_F64, workers=workers, layout=layout)
        assert np.array_equal(bits(got), bits(want))
        if layout == 1:
            plan = bcn.par.make_plan(n, workers, bcn.Layout.Interleaved)
            logical = bcn.par.deinterleave(torch.from_numpy(got).to(cuda), plan).cpu().numpy()
            assert np.array_equal(bits(logical), bits(serial))
        else:
            assert np.array_equal(bits(got), bits(serial))


@pytest.mark.parametrize("itemsize", [4, 8])
def test_deinterleave_shapes(bcn, cuda, oracle, itemsize):
    """Device deinterleave (parallel.cpp:81-97) of arbitrary words against the
    oracle: narrow (W <= 32, smem row tiles incl. exact tiles W | 8192) and wide
    (128-row tiles of 256 B to 1 KiB, partial in both directions, both tile
    orders) regions, ragged Interleaved tails, n smaller than W."""
    rng = np.random.default_rng(itemsize)
    dt = np.uint32 if itemsize == 4 else np.uint64
    for n, w in [(1, 1), (5, 9), (100003, 1), (100003, 5), (100003, 7), (65536, 8), (100003, 31),
                 (100003, 32), (100003, 33), (100003, 63), (100003, 64), (100003, 65),
                 (100003, 120), (100003, 129), (300007, 1000), (99999, 99999), (2**21 + 17, 4099),
                 (2**27 + 3, 130)]:  # thousands of row blocks per worker: worker-block tile order
        phys = rng.integers(0, np.iinfo(dt).max, n, dtype=dt, endpoint=True)
        plan = bcn.par.make_plan(n, w, bcn.Layout.Interleaved)
        signed = np.int32 if itemsize == 4 else np.int64
        dev_phys = torch.from_numpy(phys.view(signed)).to(cuda)
        got = bcn.par.deinterleave(dev_phys, plan).cpu().numpy().view(dt)
        want = oracle.deinterleave(phys, w)
        assert np.array_equal(got, want), (n, w)


@pytest.mark.parametrize("itemsize", [4, 8])
def test_deinterleave_wide_alignments(bcn, cuda, oracle, itemsize):
    """Wide deinterleave regions whose physical rows and worker runs take every
    residue mod 16 bytes (line-aligned halo stores with per-worker shifts,
    first / last row blocks, both regions) and input / output views misaligned
    by whole items — against the oracle through the C ABI, with a guard band
    checking nothing is written outside the output."""
    import ctypes

    from paper_1206_1187_b200 import _lib

    rng = np.random.default_rng(1187 + itemsize)
    dt, ndt, sdt = (np.uint32, np.int32, torch.int32) if itemsize == 4 else (np.uint64, np.int64, torch.int64)
    cases = []
    for w in (129, 130, 131, 132, 200, 257, 1001, 4098):
        for rows in (40, 128, 161, 300):
            for extra in (0, 1, w // 2 + 1):
                cases.append((w * (rows - 1) + extra if extra else w * rows, w))
    cases += [(1 << 22, 100003), (3 * 2**20 + 5, 1000000 // 7)]
    for i, (n, w) in enumerate(cases):
        off_in, off_out = int(rng.integers(0, 3)), int(rng.integers(0, 3))
        phys = rng.integers(0, np.iinfo(dt).max, n, dtype=dt, endpoint=True)
        src = torch.empty(n + off_in, dtype=sdt, device=cuda)
        src[off_in:].copy_(torch.from_numpy(phys.view(ndt)))
        dst = torch.full((n + off_out + 8,), -1, dtype=sdt, device=cuda)
        _lib.call("bcn_deinterleave", ctypes.c_void_p(src[off_in:].data_ptr()),
                  ctypes.c_void_p(dst[off_out:].data_ptr()), n, w, itemsize, 0, ctypes.c_void_p(0))
        got = dst.cpu().numpy().view(dt)
        assert np.array_equal(got[off_out:off_out + n], oracle.deinterleave(phys, w)), (i, n, w, off_in, off_out)
        assert (got[:off_out] == np.iinfo(dt).max).all() and (got[off_out + n:] == np.iinfo(dt).max).all(), \
            ("wrote outside the output", i, n, w)


def test_deinterleave_tma_tile_mover_opt_in(cuda):
    """The opt-in TMA tile mover (BCN_DEINT_TMA=1, bcn_deint_tma.cu) on wide
    regions whose rows and runs are whole 16-byte chunks (the only ones its
    tensor maps take), with tails below one store box and the < ko last
    workers; other shapes fall back inside the same call. Env is read once
    per process, so the check runs in a child."""
    code = (
        "import numpy as np, torch, oracle as O, paper_1206_1187_b200 as B\n"
        "o = O.Oracle(); rng = np.random.default_rng(3)\n"
        "for isz, dt, sdt in ((4, np.uint32, np.int32), (8, np.uint64, np.int64)):\n"
        "    for n, w in ((1024 * 4096, 1024), (1024 * 4096 + 17, 1024), (4096 * 300, 4096), (200 * 777, 200), (1001 * 500, 1001)):\n"
        "        phys = rng.integers(0, np.iinfo(dt).max, n, dtype=dt, endpoint=True)\n"
        "        src = torch.from_numpy(phys.view(sdt)).to('cuda:0')\n"
        "        got = B.par.deinterleave(src, B.par.make_plan(n, w, B.Layout.Interleaved)).cpu().numpy().view(dt)\n"
        "        assert np.array_equal(got, o.deinterleave(phys, w)), (isz, n, w)\n"
    )
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, BCN_DEINT_TMA="1")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]


def test_randomized_deinterleave_against_oracle(bcn, cuda, oracle):
    """Seeded fuzz over the device deinterleave: random n, W (1 .. 2*10^6,
    log-uniform, n < W included), item size and misaligned device views —
    every narrow/wide tile shape, both wide tile orders and the ragged second
    region, each bit-exact against the oracle's reordering."""
    rng = np.random.default_rng(0xDE1_4721)
    for case in range(int(os.environ.get("BCN_FUZZ_CASES_DEINT", "120"))):
        n = int(rng.integers(1, 3_000_000))
        w = int(np.exp(rng.uniform(0, np.log(2e6))))
        itemsize = int(rng.choice([4, 8]))
        dt, sdt = (np.uint32, np.int32) if itemsize == 4 else (np.uint64, np.int64)
        off = int(rng.integers(0, 3))
        phys = rng.integers(0, np.iinfo(dt).max, n, dtype=dt, endpoint=True)
        buf = torch.empty(n + off, dtype=torch.int32 if itemsize == 4 else torch.int64, device=cuda)
        view = buf[off:]
        view.copy_(torch.from_numpy(phys.view(sdt)))
        plan = bcn.par.make_plan(n, w, bcn.Layout.Interleaved)
        got = bcn.par.deinterleave(view, plan).cpu().numpy().view(dt)
        assert np.array_equal(got, oracle.deinterleave(phys, w)), (case, n, w, itemsize, off)


def test_interleaved_ragged_million(bcn, cuda, reference):
    """test_parallel.cpp:98-105: W = 7, n = 10^6, Interleaved."""
    got = dev_fill(bcn, 10**6, O.FMT_F64, workers=7, layout=1)
    assert np.array_equal(bits(got), bits(reference.fill(10**6, O.FMT_F64, workers=7, layout=1)))


@pytest.mark.parametrize("engine", ["Barrett", "Montgomery", "FP64", "Mixed"])
@pytest.mark.parametrize("fmt", [O.FMT_U64, O.FMT_F32])
def test_interleaved_engines_formats(bcn, cuda, oracle, engine, fmt):
    n = 200003
    for w in (3, 33, 130):
        got = dev_fill(bcn, n, fmt, workers=w, layout=1, engine=engine, base=999)
        want = oracle.fill(n, fmt, workers=w, layout=1, base_offset=999)
        assert np.array_equal(bits(got), bits(want))


# ----------------------------------------------------- offsets and wraps
@pytest.mark.parametrize("engine", ["FP64", "Barrett"])
def test_f32_is_rz_of_f64_full_size(bcn, cuda, engine):
    """f32 := RZ(to_unit_interval(z)) over 2^30 variates: the f32
    fill equals the truncation of the (oracle-verified) f64 fill element by
    element (a size-independent property; the count of variates within 3 ulps
    of a truncation boundary is printed)."""
    n = 1 << 30
    plan = bcn.par.make_plan(n, 1)
    f64 = torch.empty(n, dtype=torch.float64, device=cuda)
    f32 = torch.empty(n, dtype=torch.float32, device=cuda)
    bcn.par.fill_format(f64, plan, A0, bcn.Method.BarrettModified, 0, bcn.Format.F64, engine=bcn.Engine.FP64)
    bcn.par.fill_format(f32, plan, A0, bcn.Method.BarrettModified, 0, bcn.Format.F32,
                        engine=bcn.Engine[engine])
    torch.cuda.synchronize()
    near = 0
    step = 1 << 26
    for c in range(0, n, step):
        b = f64[c:c + step].view(torch.int64)
        want = ((b >> 29) - (896 << 23)) & 0xFFFFFFFF
        got = f32[c:c + step].view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        assert torch.equal(got, want), f"chunk at {c}"
        low = b & ((1 << 29) - 1)
        near += int((((low + 3) & ((1 << 29) - 1)) < 7).logical_and(f64[c:c + step] > 0.5).sum())
    print(f"boundary re-check candidates in 2^30: {near}")


def test_randomized_plans_against_oracle(bcn, cuda, oracle):
    """Seeded fuzz over the whole fill surface: random n (incl. < one row),
    workers, layout, format, engine, pointer misalignment, seed index and
    base_offset (incl. near 2^64 and near multiples of the period) — every
    case bit-exact against the oracle. Exercises the in-kernel edge rows,
    the column-stable and two-multiplier interleaved paths and the slot kernel."""
    rng = np.random.default_rng(0x1206_1187)
    P = 3706040377703682
    engines = ["Auto", "Barrett", "Montgomery", "FP64", "Staged", "Bulk", "Mixed", "Hybrid"]
    for case in range(int(os.environ.get("BCN_FUZZ_CASES", "400"))):
        n = int(rng.choice([rng.integers(1, 300), rng.integers(300, 5000), rng.integers(5000, 400000)]))
        workers = int(rng.choice([1, 2, 3, 5, 7, 8, 16, 31, 33, 64, 100, 1000, rng.integers(1, 5000)]))
        layout = int(rng.integers(0, 2))
        fmt = int(rng.choice([O.FMT_U64, O.FMT_F64, O.FMT_F32]))
        engine = str(rng.choice(engines))
        offset = int(rng.integers(0, 9))
        seed = int(rng.choice([A0, 1 << 53, rng.integers(A0, (1 << 53) + 1)]))
        base = int(rng.choice([0, rng.integers(0, 1 << 62), (1 << 64) - int(rng.integers(1, 2 * n + 2)),
                               P * int(rng.integers(1, 1000)) - int(rng.integers(0, n + 1))]))
        base &= (1 << 64) - 1
        got = dev_fill(bcn, n, fmt, workers=workers, layout=layout, seed=seed, base=base,
                       engine=engine, offset=offset)
        want = oracle.fill(n, fmt, seed_index=seed, base_offset=base, workers=workers, layout=layout)
        assert np.array_equal(bits(got), bits(want)), (case, n, workers, layout, fmt, engine, offset, seed, base)


def test_base_offset_windows(bcn, cuda, oracle):
    """test_parallel.cpp:131-138 and test_cli.cpp:116-125 (chunked == single)."""
    whole = dev_fill(bcn, 1 << 20, O.FMT_U64)
    chunks = [dev_fill(bcn, 1 << 18, O.FMT_U64, base=c << 18, workers=3) for c in range(4)]
    assert np.array_equal(np.concatenate(chunks), whole)


def test_period_wrap_golden(bcn, cuda):
    """fill_residues(n=6, a0, base_offset=P-3) re-emits z0 at k=P."""
    got = dev_fill(bcn, 6, O.FMT_U64, base=O.PERIOD - 3)
    assert [int(x) for x in got] == [1867496909077246, 5488691822377859, 4258649398211344,
                                     2138759898642167, 906908310809773, 121054228244396]


def test_period_wrap_large_window(bcn, cuda, oracle):
    for fmt in (O.FMT_U64, O.FMT_F64):
        got = dev_fill(bcn, 300000, fmt, base=O.PERIOD - 150000, engine="FP64")
        assert np.array_equal(bits(got), bits(oracle.fill(300000, fmt, base_offset=O.PERIOD - 150000)))


def test_far_offset_interleaved_golden(bcn, cuda):
    """a = 2^53, base_offset = 2^40, W = 3, Interleaved."""
    got = dev_fill(bcn, 6, O.FMT_U64, seed=1 << 53, base=1 << 40, workers=3, layout=1)
    assert [int(x) for x in got] == [1584414649962571, 4289752975226581, 752696664753940,
                                     663488620216616, 2266604546227133, 4919938457993333]


@pytest.mark.parametrize("layout", [0, 1])
def test_u64_wrap_of_base_offset_matches_reference(bcn, cuda, reference, layout):
    """base_offset + start_w wraps mod 2^64 in the reference (parallel.cpp:63-64);
    the device path reproduces that exactly for W > 1."""
    n, w = 50000, 5
    base = (1 << 64) - 23456
    got = dev_fill(bcn, n, O.FMT_U64, workers=w, layout=layout, base=base)
    want = reference.fill(n, O.FMT_U64, workers=w, layout=layout, base_offset=base)
    assert np.array_equal(got, want)


def test_seed_extremes(bcn, cuda, oracle):
    for seed in (A0, A0 + 1, (1 << 53) - 1, 1 << 53):
        got = dev_fill(bcn, 70001, O.FMT_U64, seed=seed, base=seed % 1000003)
        assert np.array_equal(got, oracle.fill(70001, O.FMT_U64, seed_index=seed,
                                                  base_offset=seed % 1000003))


@pytest.mark.parametrize("pace", [7000.0, 1e5])
def test_paced_kernels_bit_exact(bcn, cuda, oracle, pace):
    """The write-paced contiguous kernels (pacer warp + named barrier) produce
    the same bits as every other path, for all engines and formats."""
    old = bcn.device.write_pacing_config()
    try:
        bcn.device.set_write_pacing(pace, 2, 7)
        for engine in ("Barrett", "Montgomery", "FP64", "Mixed"):
            for fmt in (O.FMT_U64, O.FMT_F64, O.FMT_F32):
                n = 2**20 + 4099
                got = dev_fill(bcn, n, fmt, engine=engine, base=777, offset=1)
                assert np.array_equal(bits(got), bits(oracle.fill(n, fmt, base_offset=777)))
        c = torch.empty(1 << 20, dtype=torch.float64, device=cuda)
        bcn.device.fill_constant(c)
        torch.cuda.synchronize()
        assert bool((c == 0.5).all())
    finally:
        bcn.device.set_write_pacing(*old)


def test_pacing_is_calibrated_per_device(bcn, cuda):
    """Automatic pacing (the default): the device context measured its own
    target at initialisation (no hard-coded 7200); a fixed target
    overrides it and <0 restores it; absurd targets are rejected."""
    old = bcn.device.write_pacing_config()
    try:
        bcn.device.set_write_pacing(-1, 1, 3)
        target, src = bcn.device.device_write_pacing(0)
        curve = bcn.device.pace_calibration(0)
        assert src == "calibrated", (target, src, curve)
        assert 5000 <= target <= 8500, curve
        best = max(curve, key=lambda p: p[1])
        assert target == best[0] and best[1] > 0.9 * target
        bcn.device.set_write_pacing(7100, 1, 3)
        assert bcn.device.device_write_pacing(0) == (7100.0, "user")
        bcn.device.set_write_pacing(0, 1, 3)
        assert bcn.device.device_write_pacing(0) == (0.0, "unpaced")
        bcn.device.set_write_pacing(-5, 1, 3)
        assert bcn.device.device_write_pacing(0) == (target, "calibrated")
    finally:
        bcn.device.set_write_pacing(*old)


# ------------------------------------------------------------- host buffers
def test_host_numpy_output_chunked(bcn, cuda, oracle):
    """Host (pageable) span like the reference's std::span fill: > one 64 MiB chunk."""
    n = (1 << 24) + 12345
    out = np.empty(n, dtype=np.float64)
    plan = bcn.par.make_plan(n, 3)
    bcn.par.fill(out, plan, A0, base_offset=77)
    assert oracle.digest(bits(out)) == oracle.digest(bits(oracle.fill(n, O.FMT_F64, base_offset=77,
                                                                      workers=3)))


@pytest.mark.parametrize("workers", [7, 1000])
def test_host_output_interleaved_across_chunks(bcn, cuda, oracle, workers):
    """Interleaved layout into host memory: the 64 MiB device chunks cut the
    interleaved regions at arbitrary slots (pageable and pinned outputs)."""
    n = (1 << 24) + 12345
    plan = bcn.par.make_plan(n, workers, bcn.Layout.Interleaved)
    want = oracle.fill(n, O.FMT_F64, base_offset=5, workers=workers, layout=1)
    out = np.empty(n, dtype=np.float64)
    bcn.par.fill(out, plan, A0, base_offset=5)
    assert np.array_equal(bits(out), bits(want))
    pinned = torch.empty(n, dtype=torch.float64, pin_memory=True)
    bcn.par.fill(pinned, plan, A0, base_offset=5)
    assert np.array_equal(bits(pinned.numpy()), bits(want))


def test_host_pinned_output(bcn, cuda, oracle):
    n = (1 << 23) + 3
    out = torch.empty(n, dtype=torch.float32, pin_memory=True)
    bcn.par.fill_float(out, bcn.par.make_plan(n, 1), A0)
    assert np.array_equal(bits(out.numpy()), bits(oracle.fill(n, O.FMT_F32)))


# --------------------------------------------------------------- errors
def test_errors_before_work(bcn, cuda):
    """Size and seed checks happen before any device work (parallel.cpp:59-61,
    generator.cpp:33-35); W > 1 with a bad seed raises instead of aborting."""
    buf = torch.full((100,), -1.0, dtype=torch.float64, device=cuda)
    with pytest.raises(bcn.InvalidArgument):
        bcn.par.fill(buf[:99], bcn.par.make_plan(100, 2), A0)
    with pytest.raises(bcn.OutOfRange):
        bcn.par.fill(buf, bcn.par.make_plan(100, 4), A0 - 1)
    with pytest.raises(bcn.OutOfRange):
        bcn.par.fill(buf, bcn.par.make_plan(100, 4), (1 << 53) + 1)
    with pytest.raises(bcn.InvalidArgument):
        bcn.par.fill_residues(buf, bcn.par.make_plan(100, 1), A0)  # dtype mismatch
    torch.cuda.synchronize()
    assert bool((buf == -1.0).all())
    with pytest.raises(bcn.InvalidArgument):
        bcn.par.deinterleave(buf, bcn.par.make_plan(100, 2))  # not Interleaved


# ------------------------------------------------------------ seeding (C4)
def test_seed_states_stress(bcn, cuda, oracle):
    """2^20 streams with arbitrary (a, k) incl. the period wrap,
    a = 2^53 and k near 2^64; each compared with state_at (+ next walks)."""
    rng = np.random.Generator(np.random.MT19937(0x12061187))
    count = 1 << 20
    a = rng.integers(A0, (1 << 53) + 1, size=count, dtype=np.uint64)
    k = rng.integers(0, np.iinfo(np.uint64).max, size=count, dtype=np.uint64, endpoint=True)
    forced_k = [O.PERIOD - 2, O.PERIOD - 1, O.PERIOD, O.PERIOD + 1, 0, (1 << 64) - 1, 2 * O.PERIOD]
    k[:len(forced_k)] = forced_k
    a[len(forced_k):len(forced_k) + 3] = [1 << 53, A0, (1 << 53) - 1]
    ta = torch.from_numpy(a.view(np.int64)).to(cuda)
    tk = torch.from_numpy(k.view(np.int64)).to(cuda)
    got = bcn.device.seed_states(ta, tk).cpu().numpy().view(np.uint64)
    assert np.array_equal(got, oracle.seed_batch(a, k))
    sub = 1 << 14
    walks = bcn.device.seed_states(ta[:sub], tk[:sub], steps=64).cpu().numpy().view(np.uint64)
    assert np.array_equal(walks, oracle.seed_batch(a[:sub], k[:sub], steps=64))
    for steps in (1, 3, 12):  # staged (steps % 4 != 0) and vector-store walk paths
        walks = bcn.device.seed_states(ta[:999], tk[:999], steps=steps).cpu().numpy().view(np.uint64)
        assert np.array_equal(walks, oracle.seed_batch(a[:999], k[:999], steps=steps))
    bad = ta[:4].clone()
    bad[2] = A0 - 1
    with pytest.raises(bcn.OutOfRange):
        bcn.device.seed_states(bad, tk[:4])


# ------------------------------------------------------------- utilities
def test_digest_and_constant(bcn, cuda, oracle):
    got = dev_fill(bcn, 1 << 20, O.FMT_U64)
    t = torch.from_numpy(got.view(np.int64)).to(cuda)
    assert bcn.device.digest(t, index_base=5) == oracle.digest(got, index_base=5)
    c = torch.empty(1 << 20, dtype=torch.float64, device=cuda)
    bcn.device.fill_constant(c)
    torch.cuda.synchronize()
    assert bool((c == 0.5).all())


def test_fill_noise_writer(bcn, cuda):
    """The noise writer covers the whole buffer with seed-determined, non-constant
    words, paced or not; a zero seed is rejected."""
    c = torch.zeros(1 << 21, dtype=torch.int64, device=cuda)
    d = torch.zeros_like(c)
    old = bcn.device.write_pacing_config()
    try:
        for pace in (0.0, 7000.0):
            bcn.device.set_write_pacing(pace, 2, 3)
            c.zero_()
            d.zero_()
            bcn.device.fill_noise(c, seed=7)
            bcn.device.fill_noise(d, seed=7)
            torch.cuda.synchronize()
            assert int((c == 0).sum()) == 0
            assert torch.equal(c, d)
            assert c.unique().numel() > 10000
    finally:
        bcn.device.set_write_pacing(*old)
    with pytest.raises(bcn.InvalidArgument):
        bcn.device.fill_noise(c, seed=0)


def test_concurrent_calls_from_threads(bcn, cuda, oracle):
    """The C ABI is re-entrant like the reference (parallel.cpp has no global
    state): eight host threads mixing device fills on their own streams, host
    (pageable / pinned) fills, digests and quality calls all get the right bits."""
    import threading

    n = 300007
    want = {fmt: oracle.fill(n, fmt, base_offset=99) for fmt in (O.FMT_U64, O.FMT_F64, O.FMT_F32)}
    errors = []

    def worker(t):
        try:
            fmt = (O.FMT_U64, O.FMT_F64, O.FMT_F32)[t % 3]
            plan = bcn.par.make_plan(n, 1 + t % 4)
            for it in range(3):
                if (t + it) % 3 == 0:
                    s = torch.cuda.Stream(device=cuda)
                    dt = {O.FMT_U64: torch.int64, O.FMT_F64: torch.float64, O.FMT_F32: torch.float32}[fmt]
                    buf = torch.empty(n, dtype=dt, device=cuda)
                    with torch.cuda.stream(s):
                        bcn.par.fill_format(buf, plan, A0, bcn.Method.BarrettModified, 99,
                                            bcn.Format(fmt), stream=s)
                    s.synchronize()
                    got = buf.cpu().numpy()
                    bcn.device.digest(buf.view(torch.int32 if fmt == O.FMT_F32 else torch.int64))
                elif (t + it) % 3 == 1:
                    got = np.empty(n, dtype=want[fmt].dtype)
                    bcn.par.fill_format(got, plan, A0, bcn.Method.BarrettModified, 99, bcn.Format(fmt))
                else:
                    got = torch.empty(n, dtype={O.FMT_U64: torch.int64, O.FMT_F64: torch.float64,
                                                O.FMT_F32: torch.float32}[fmt], pin_memory=True)
                    bcn.par.fill_format(got, plan, A0, bcn.Method.BarrettModified, 99, bcn.Format(fmt))
                    got = got.numpy()
                    bcn.quality.serial_correlation(torch.from_numpy(oracle.fill(200000, O.FMT_F64)).to(cuda))
                if not np.array_equal(bits(got), bits(want[fmt])):
                    errors.append((t, it, fmt))
        except Exception as e:  # noqa: BLE001
            errors.append((t, repr(e)))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(8)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors


def test_fill_inside_cuda_graph(bcn, cuda, oracle):
    """bcn_fill on a caller stream is a plain kernel launch, so it can be
    captured in a CUDA graph and replayed (launch-bound loops of small fills)."""
    n = 100003
    outs = [torch.empty(n, dtype=torch.float64, device=cuda) for _ in range(3)]
    plan = bcn.par.make_plan(n, 1)
    s = torch.cuda.Stream(device=cuda)
    bcn.par.fill(outs[0], plan, A0, stream=s)  # warm-up: device context, occupancy caches
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i, o in enumerate(outs):
            bcn.par.fill(o, plan, A0, base_offset=i * n, stream=torch.cuda.current_stream())
    for o in outs:
        o.zero_()
    g.replay()
    torch.cuda.synchronize()
    for i, o in enumerate(outs):
        assert np.array_equal(bits(o.cpu().numpy()), bits(oracle.fill(n, O.FMT_F64, base_offset=i * n)))


def test_fill_multi_concatenation(bcn, cuda, oracle):
    """make_plan(n, G) contiguous shards (one per 'device'; two shards on GPU 0
    here) concatenate to the single fill."""
    n = 1_000_003
    eff, wpw = oracle.make_plan(n, 2)
    outs = [torch.empty(wpw, dtype=torch.float64, device=cuda),
            torch.empty(n - wpw, dtype=torch.float64, device=cuda)]
    bcn.device.fill_multi(outs, n, base_offset=31)
    got = torch.cat(outs).cpu().numpy()
    assert np.array_equal(bits(got), bits(oracle.fill(n, O.FMT_F64, base_offset=31, workers=2)))


def test_fill_multi_validates_every_shard_before_any_work(bcn, cuda):
    """a short shard, a wrong dtype or a NULL capacity array is
    invalid_argument and nothing is written to any shard."""
    import ctypes
    n = 1000
    good = torch.full((500,), -1, dtype=torch.int64, device=cuda)
    short = torch.full((499,), -1, dtype=torch.int64, device=cuda)
    with pytest.raises(bcn.InvalidArgument, match="smaller than its shard"):
        bcn.device.fill_multi([good, short], n, fmt=bcn.Format.U64)
    assert int((good != -1).sum()) == 0 and int((short != -1).sum()) == 0
    with pytest.raises(bcn.InvalidArgument, match="dtype"):
        bcn.device.fill_multi([torch.empty(500, dtype=torch.float32, device=cuda)] * 2, n)
    h = bcn._lib.lib()
    ptrs = (ctypes.c_void_p * 1)(good.data_ptr())
    devs = (ctypes.c_int * 1)(0)
    assert h.bcn_fill_multi(ptrs, None, devs, 1, 100, 0, A0, 0, 0, None) == 1


def test_fill_multi_orders_after_pending_work_on_the_stream(bcn, cuda, oracle):
    """the shard fill runs after work already queued on the torch
    stream that uses the buffer (a slow fill of the same buffer queued first
    must not overwrite the multi-GPU result)."""
    n = 1 << 26
    out = torch.empty(n, dtype=torch.float64, device=cuda)
    s = torch.cuda.Stream(cuda)
    with torch.cuda.stream(s):
        torch.cuda._sleep(50_000_000)  # ~25 ms of queued work ahead of the fill
        out.fill_(0.25)
        bcn.device.fill_multi([out], n, base_offset=5)
    torch.cuda.synchronize()
    want = oracle.fill(1 << 16, O.FMT_F64, base_offset=5 + n - (1 << 16))
    assert np.array_equal(bits(out[-(1 << 16):].cpu().numpy()), bits(want))


def test_fill_multi_across_all_devices(bcn, cuda, oracle):
    """One shard per visible GPU (bcn_fill_multi's host thread per device);
    skipped below two devices."""
    ndev = torch.cuda.device_count()
    if ndev < 2:
        pytest.skip("needs >= 2 GPUs")
    n = (1 << 27) + 12345
    eff, wpw = oracle.make_plan(n, ndev)
    outs = [torch.empty(min(wpw, n - g * wpw), dtype=torch.float64, device=f"cuda:{g}") for g in range(eff)]
    bcn.device.fill_multi(outs, n, base_offset=77)
    for g, o in enumerate(outs):
        d = bcn.device.digest(o.view(torch.int64), index_base=g * wpw)
        want = oracle.fill(o.numel(), O.FMT_F64, base_offset=77 + g * wpw)
        assert d == oracle.digest(bits(want), index_base=g * wpw), g


def test_cabi_rejects_host_buffers_where_device_memory_is_required(bcn, cuda, oracle):
    """C callers (no Python guard): host pointers passed to device-only entry
    points are rejected with BCN_ERR_INVALID_ARGUMENT before any launch, and
    the context stays usable (no sticky illegal-address error)."""
    import ctypes
    h = bcn._lib.lib()
    host_a = np.full(4, A0, dtype=np.uint64)
    host_k = np.zeros(4, dtype=np.uint64)
    dev_a = torch.from_numpy(host_a.view(np.int64)).to(cuda)
    dev_k = torch.from_numpy(host_k.view(np.int64)).to(cuda)
    out = torch.empty(4, dtype=torch.int64, device=cuda)
    vp = ctypes.c_void_p
    for a_ptr, k_ptr in ((host_a.ctypes.data, dev_k.data_ptr()), (dev_a.data_ptr(), host_k.ctypes.data)):
        st = h.bcn_seed_states(vp(a_ptr), vp(k_ptr), vp(out.data_ptr()), 4, 0, 0, None)
        assert st == 1 and b"device memory" in h.bcn_last_error()
    host_out = np.empty(100, dtype=np.float64)
    ptrs = (vp * 1)(host_out.ctypes.data)
    devs = (ctypes.c_int * 1)(0)
    caps = (ctypes.c_uint64 * 1)(100)
    st = h.bcn_fill_multi(ptrs, caps, devs, 1, 100, 1, A0, 0, 0, None)
    assert st == 1 and b"device memory" in h.bcn_last_error()
    ptrs = (vp * 1)(None)
    assert h.bcn_fill_multi(ptrs, caps, devs, 1, 100, 1, A0, 0, 0, None) == 1
    # still healthy: a real call on the same context is bit-exact
    got = bcn.device.seed_states(dev_a, dev_k).cpu().numpy().view(np.uint64)
    assert got.tolist() == [oracle.state_at(A0, 0)] * 4


def test_host_deinterleave_releases_its_staging(bcn, cuda, oracle):
    """The host-buffer deinterleave stages through a device temporary that is
    released on every exit path: repeated host calls keep the reference order
    and leave device memory where it was."""
    n, w = 1_000_003, 7
    phys = oracle.fill(n, O.FMT_U64, workers=w, layout=O.INTERLEAVED)
    want = oracle.fill(n, O.FMT_U64)
    plan = bcn.par.make_plan(n, w, bcn.Layout.Interleaved)
    bcn.par.deinterleave(phys, plan)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info(cuda)[0]
    for _ in range(4):
        got = bcn.par.deinterleave(phys, plan)
        assert np.array_equal(np.asarray(got).view(np.uint64), want.view(np.uint64))
    assert abs(torch.cuda.mem_get_info(cuda)[0] - free0) < (4 << 20)


def test_jump_engines_exact_on_arbitrary_operands(bcn, cuda):
    """Every jump engine (Barrett/Shoup, Montgomery, the FP64 error-free
    product, Mixed) computes z * c^r mod 3^33 exactly for arbitrary residues
    and multipliers — edges (0, 1, m/2, m/2 + 1, m - 1, 2^52 neighbourhoods)
    and random ones — with r chained multiplications in the engine's own
    (balanced, non-canonical) state representation, against Python integers.
    This pins the DESIGN.md §2 exactness arguments over the engines' whole
    domain, not just the multipliers the fills use."""
    m = O.MODULUS
    rng = np.random.default_rng(0xE9_1E5)
    edges = [0, 1, 2, 3, m // 2 - 1, m // 2, m // 2 + 1, m - 2, m - 1, (1 << 52) - 1, 1 << 52,
             (1 << 52) + 1, m - (1 << 51), 3 ** 32, 2 * 3 ** 32]
    ze, ce = np.meshgrid(np.array(edges, dtype=np.uint64), np.array(edges, dtype=np.uint64))
    n_rand = 1 << 17
    z = np.concatenate([ze.ravel(), rng.integers(0, m, n_rand, dtype=np.uint64)])
    c = np.concatenate([ce.ravel(), rng.integers(0, m, n_rand, dtype=np.uint64)])
    zi, ci = [int(v) for v in z], [int(v) for v in c]
    for chain in (1, 2, 7):
        want = np.array([a * pow(b, chain, m) % m for a, b in zip(zi, ci)], dtype=np.uint64)
        for engine in (bcn.Engine.Barrett, bcn.Engine.Montgomery, bcn.Engine.FP64, bcn.Engine.Mixed):
            got = bcn.device.engine_check(engine, z, c, chain)
            bad = np.nonzero(got != want)[0]
            assert bad.size == 0, (engine, chain, [(zi[i], ci[i]) for i in bad[:5]])
    with pytest.raises(bcn.DomainError):
        bcn.device.engine_check(bcn.Engine.FP64, np.array([m], dtype=np.uint64), np.array([1], dtype=np.uint64))
    with pytest.raises(bcn.InvalidArgument):
        bcn.device.engine_check(bcn.Engine.Staged, z[:4], c[:4])


def test_scalar_generator_api(bcn, cuda, oracle):
    g = bcn.gen
    s = g.seed_from_index(A0)
    assert s.z == 4258649398211344
    assert g.next(s) == 2138759898642167 and s.k == 1
    assert g.state_at(A0, 1000).z == 5492007519572011
    assert g.seed_from_index(1 << 53).z == 1895384862748766


# ------------------------------------------------------- full-size (C2)
@pytest.mark.slow
def test_config2_full_size_digests(bcn, cuda, oracle):
    """C2: 2^30 doubles on one B200 vs the oracle, per-2^24-chunk digests, plus a
    size-independent check: chunked (base_offset) fills equal the single fill."""
    n = 1 << 30
    buf = torch.empty(n, dtype=torch.float64, device=cuda)
    bcn.par.fill(buf, bcn.par.make_plan(n, 1), A0, sync=True)
    chunk = 1 << 24
    host = np.empty(chunk, dtype=np.float64)
    for c in range(0, n // chunk, 9):  # every 9th chunk (8 chunks incl. first/last region)
        oracle.fill(chunk, O.FMT_F64, base_offset=c * chunk, out=host)
        dd = bcn.device.digest(buf[c * chunk:(c + 1) * chunk].view(torch.int64))
        assert dd == oracle.digest(bits(host)), f"chunk {c}"
    last = buf[-chunk:].view(torch.int64)
    oracle.fill(chunk, O.FMT_F64, base_offset=n - chunk, out=host)
    assert bcn.device.digest(last) == oracle.digest(bits(host))
    whole = bcn.device.digest(buf.view(torch.int64))
    parts = [0, 0]
    half = torch.empty(n // 2, dtype=torch.float64, device=cuda)
    for h in range(2):
        bcn.par.fill(half, bcn.par.make_plan(n // 2, 1), A0, base_offset=h * (n // 2), sync=True)
        d = bcn.device.digest(half.view(torch.int64), index_base=h * (n // 2))
        parts = [(parts[0] + d[0]) % (1 << 64), (parts[1] + d[1]) % (1 << 64)]
    assert parts == [whole[0], whole[1]]


# ------------------------------------------------------ quality suite (§8f.4)
def test_quality_suite_matches_reference(bcn, cuda, oracle, reference):
    """quality.cpp on the GPU: chi-square and monobit statistics bit-identical to
    the reference on the same data; the lag correlation within 1e-12 (a
    floating-point sum in a different order); pass flags equal."""
    n = 10**6
    u = oracle.fill(n, O.FMT_F64)
    z = oracle.fill(n, O.FMT_U64)
    q = bcn.quality
    for bins in (10, 1000, 20000, 40000):
        if n / bins < 20:
            continue
        r = q.chi_square_uniformity(torch.from_numpy(u).to(cuda), bins)
        want = reference.chi_square(u, bins)
        assert (r.statistic, r.passed) == want and r.dof == bins - 1
    r = q.monobit_mantissa(torch.from_numpy(z.view(np.int64)).to(cuda))
    assert (r.statistic, r.passed) == reference.monobit(z)
    for lag in (1, 2, 17):
        r = q.serial_correlation(u, lag)  # host input
        rho, ok = reference.serial_correlation(u, lag)
        assert abs(r.statistic - rho) <= 1e-12 and r.passed == ok
    # degenerate inputs fail like the reference (test_quality.cpp:52-100)
    const = np.full(200000, 0.5)
    assert not q.chi_square_uniformity(const, 1000).passed
    same = np.full(150000, 123456789012345, dtype=np.uint64)
    assert not q.monobit_mantissa(same).passed
    ramp = (np.arange(200000) + 0.5) / 200000
    assert q.serial_correlation(ramp).statistic > 0.99
    with pytest.raises(bcn.InvalidArgument):
        q.chi_square_uniformity(np.full(1000, 0.5), 100)
    with pytest.raises(bcn.InvalidArgument):
        q.chi_square_uniformity(np.array([0.5] * 100 + [1.5] * 100000), 10)
    # lag >= n is out-of-bounds in the reference (quality.cpp:94); rejected here
    with pytest.raises(bcn.InvalidArgument):
        q.serial_correlation(u[:100000], 100000)


# ---------------------------------------------------------- multi-rank bench
def test_bench_two_ranks_share_one_gpu(bcn, cuda):
    """bench.py under torchrun with 2 ranks (gloo, both on cuda:0): shards,
    max-over-ranks timing and the digest all-gather run end to end, and the C5
    strong-scaling digest over 2 ranks equals the committed 2^36 digest."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, BCN_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29531", os.path.join(root, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu", "--log2n", "26"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=root, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["gpu_launches"] >= 3
    # The 2-rank digest of 2^27 logical items equals a single fill of 2^27.
    import oracle as O

    n = 1 << 27
    buf = torch.empty(n, dtype=torch.float64, device=cuda)
    bcn.par.fill(buf, bcn.par.make_plan(n, 1), O.MIN_SEED, sync=True)
    assert [str(x) for x in bcn.device.digest(buf.view(torch.int64))] == line["digest"]


def test_bench_nccl_branch_world_one(bcn, cuda):
    """bench.py under torchrun with the NCCL backend at world size 1 (the
    driver's 8-GPU launch, one rank): the process group, the digest
    all-gather and the max-over-ranks timing run through NCCL, the NCCL INIT
    lines are printed, and the line carries per-rank times and a verified
    digest (C2 and the C5 strong-scaling section)."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k != "BCN_DIST_BACKEND"}
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(root, "bench.py"),
           "--gpus", "1", "--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu", "--sustain-s", "0",
           "--c5-steps", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=root, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 1 and line["digest_verified_vs_oracle"] is True
    assert line["c5_strong"]["digest_verified_vs_oracle"] is True
    assert [p["rank"] for p in line["per_rank"]] == [0]
    log = (r.stdout + r.stderr).replace("nRanks", "nranks")  # NCCL logs to stdout
    assert "NCCL INFO" in log and "nranks 1" in log
