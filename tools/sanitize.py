#!/usr/bin/env python
"""Exercise every library kernel at small sizes for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck), checking outputs against the
oracle so a sanitizer-clean run is also a correct one.

    compute-sanitizer --tool memcheck python tools/sanitize.py
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_1206_1187_b200 as B  # noqa: E402

A0 = B.kMinSeedIndex


def bits(x):
    return x.view(np.uint32 if x.dtype == np.float32 else np.uint64)


def main() -> None:
    dev = torch.device("cuda:0")
    o = O.Oracle()
    n = 70001  # ragged: heads, whole rows, tails
    for fmt, dt in ((B.Format.U64, torch.int64), (B.Format.F64, torch.float64), (B.Format.F32, torch.float32)):
        want = bits(o.fill(n, int(fmt), base_offset=12345))
        for eng in B.Engine:
            for layout in (B.Layout.Contiguous, B.Layout.Interleaved):
                if layout == B.Layout.Interleaved and eng in (B.Engine.Staged, B.Engine.Bulk):
                    continue
                for w in ((1,) if layout == B.Layout.Contiguous else (3, 40)):
                    buf = torch.empty(n + 1, dtype=dt, device=dev)[1:]  # misaligned start
                    plan = B.par.make_plan(n, w, layout)
                    B.par.fill_format(buf, plan, A0, B.Method.BarrettModified, 12345, fmt, engine=eng, sync=True)
                    got = buf.cpu().numpy()
                    if layout == B.Layout.Interleaved:
                        got = B.par.deinterleave(buf, plan).cpu().numpy()
                    assert np.array_equal(bits(got), want), (fmt, eng, layout, w)
    for pace in (0.0, 7200.0):
        B.device.set_write_pacing(pace, 1, 3)
        c = torch.empty(1 << 16, dtype=torch.int64, device=dev)
        B.device.fill_constant(c)
        B.device.fill_noise(c)
        buf = torch.empty(n, dtype=torch.float64, device=dev)
        B.par.fill(buf, B.par.make_plan(n, 1), A0, sync=True)
    a = torch.tensor([A0, 1 << 53, A0 + 7], dtype=torch.int64, device=dev)
    k = torch.tensor([0, 5, (1 << 62)], dtype=torch.int64, device=dev)
    B.device.seed_states(a, k, steps=3)
    B.device.digest(torch.empty(4096, dtype=torch.int64, device=dev).fill_(3))
    u = torch.from_numpy(o.fill(200000, O.FMT_F64)).to(dev)
    z = torch.from_numpy(o.fill(200000, O.FMT_U64).view(np.int64)).to(dev)
    B.quality.chi_square_uniformity(u, 1000)
    B.quality.chi_square_uniformity(u, 5000)
    B.quality.monobit_mantissa(z)
    B.quality.serial_correlation(u, 3)
    for w in (1, 5, 33, 130):
        p = B.par.make_plan(20000, w, B.Layout.Interleaved)
        for dt in (torch.float64, torch.float32):
            B.par.deinterleave(torch.empty(20000, dtype=dt, device=dev).fill_(1), p)
    # every transpose variant: 16-row narrow tiles (W = 100), 64-worker u32
    # tiles (W = 129), both wide tile orders (W = 300 / 5000 at 400003 items)
    rng = np.random.default_rng(5)
    # + sector-aligned halo tiles: narrow u64 (W = 65), wide u32 (W = 300), wide u64 (3_000_017 / 300)
    for n2, w in ((400003, 65), (400003, 100), (400003, 129), (400003, 300), (400003, 5000), (3_000_017, 300)):
        for npt, tdt in ((np.uint64, torch.int64), (np.uint32, torch.int32)):
            phys = rng.integers(0, np.iinfo(npt).max, n2, dtype=npt, endpoint=True)
            src = torch.from_numpy(phys.view(np.int64 if npt == np.uint64 else np.int32)).to(dev)
            got = B.par.deinterleave(src, B.par.make_plan(n2, w, B.Layout.Interleaved)).cpu().numpy()
            assert np.array_equal(got.view(npt), o.deinterleave(phys, w)), (n2, w, npt)
    zz = rng.integers(0, O.MODULUS, 4096, dtype=np.uint64)
    cc = rng.integers(0, O.MODULUS, 4096, dtype=np.uint64)
    for eng in (B.Engine.Barrett, B.Engine.Montgomery, B.Engine.FP64, B.Engine.Mixed):
        B.device.engine_check(eng, zz, cc, 3)
    torch.cuda.synchronize()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
