#!/usr/bin/env python
"""Launch every kernel of the library once (after one warm-up) so a single
`ncu --set full` run covers all of them (evidence tool).

    ncu --set full --clock-control none --import-source on -o gpurun_out/prof_all \
        python tools/profile_all.py
    python tools/ncu_summary.py gpurun_out/prof_all.ncu-rep -o profiles/r02/ncu_full_all_kernels.json
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1206_1187_b200 as B  # noqa: E402

A0 = B.kMinSeedIndex


def main() -> None:
    # `--pace X`: profile the paced kernels at a fixed target (e.g. the one the
    # bench's calibration chose on this box) instead of recalibrating under ncu.
    if "--pace" in sys.argv:
        B.device.set_write_pacing(float(sys.argv[sys.argv.index("--pace") + 1]), 1, 3)
    pace = B.device.write_pacing_config()
    dev = torch.device("cuda:0")
    n = 1 << 30
    f64 = torch.empty(n, dtype=torch.float64, device=dev)
    u64 = f64.view(torch.int64)
    f32 = torch.empty(n, dtype=torch.float32, device=dev)
    plan = B.par.make_plan(n, 1)
    sync = torch.cuda.synchronize

    def fill(buf, fmt, engine=B.Engine.Auto, p=plan, base=0):
        B.par.fill_format(buf, p, A0, B.Method.BarrettModified, base, fmt, engine=engine)

    runs = [
        ("paced f64 FP64 (default)", lambda: fill(f64, B.Format.F64)),
        ("paced u64 FP64", lambda: fill(u64, B.Format.U64)),
        ("contig f32 FP64 (default f32)", lambda: fill(f32, B.Format.F32)),
        ("paced f64 Barrett", lambda: fill(f64, B.Format.F64, B.Engine.Barrett)),
        ("bulk f64", lambda: fill(f64, B.Format.F64, B.Engine.Bulk)),
        ("staged f64 (paper T=1 + TMA)", lambda: fill(f64, B.Format.F64, B.Engine.Staged)),
        ("paced interleaved W=7 (column-stable)", lambda: fill(f64, B.Format.F64,
                                                               p=B.par.make_plan(n, 7, B.Layout.Interleaved))),
        ("paced interleaved W=1001 (super-rows)", lambda: fill(f64, B.Format.F64,
                                                                p=B.par.make_plan(n, 1001, B.Layout.Interleaved))),
        ("paced interleaved W=5003 (super-rows, 2 CTAs/SM)",
         lambda: fill(f64, B.Format.F64, p=B.par.make_plan(n, 5003, B.Layout.Interleaved))),
        ("paced interleaved W=100003 (two multipliers)",
         lambda: fill(f64, B.Format.F64, p=B.par.make_plan(n, 100003, B.Layout.Interleaved))),
        ("paced constant", lambda: B.device.fill_constant(u64)),
        ("paced noise writer", lambda: B.device.fill_noise(u64)),
    ]
    unpaced = [
        ("contig f64 FP64 unpaced", lambda: fill(f64, B.Format.F64, B.Engine.FP64)),
        ("contig f64 Barrett unpaced", lambda: fill(f64, B.Format.F64, B.Engine.Barrett)),
        ("contig f64 Montgomery unpaced", lambda: fill(f64, B.Format.F64, B.Engine.Montgomery)),
        ("contig f64 Mixed unpaced", lambda: fill(f64, B.Format.F64, B.Engine.Mixed)),
        ("interleaved W=7 unpaced", lambda: fill(f64, B.Format.F64,
                                                 p=B.par.make_plan(n, 7, B.Layout.Interleaved))),
        ("constant unpaced", lambda: B.device.fill_constant(u64)),
    ]
    for name, fn in runs:
        fn()
        sync()
        fn()
        sync()
    B.device.set_write_pacing(0, 1, 3)
    for name, fn in unpaced:
        fn()
        sync()
        fn()
        sync()
    B.device.set_write_pacing(*pace)
    # small / auxiliary kernels
    small = torch.empty(100003 + 1, dtype=torch.float64, device=dev)[1:]
    B.par.fill(small, B.par.make_plan(100003, 3), A0, base_offset=(1 << 64) - 50000)  # slots (wrap)
    rng = np.random.default_rng(7)
    cnt = 1 << 20
    a = torch.from_numpy(rng.integers(A0, (1 << 53) + 1, cnt, dtype=np.uint64).view(np.int64)).to(dev)
    k = torch.from_numpy(rng.integers(0, 1 << 62, cnt, dtype=np.uint64).view(np.int64)).to(dev)
    B.device.seed_states(a, k)
    B.device.seed_states(a, k, steps=64)
    B.device.digest(u64)
    m = 1 << 28
    B.par.deinterleave(f64[:m], B.par.make_plan(m, 1000, B.Layout.Interleaved))
    B.par.deinterleave(f64[:m], B.par.make_plan(m, 7, B.Layout.Interleaved))
    # sector-aligned halo tiles: u32 wide (W = 1000), u64 narrow (W = 65), u64 wide (odd runs)
    B.par.deinterleave(f32[:m], B.par.make_plan(m, 1000, B.Layout.Interleaved))
    B.par.deinterleave(f64[:m], B.par.make_plan(m, 65, B.Layout.Interleaved))
    B.par.deinterleave(f64[:m - 3 * 4096], B.par.make_plan(m - 3 * 4096, 4096, B.Layout.Interleaved))
    fill(f32, B.Format.F32, B.Engine.Hybrid)
    B.par.fill(f64[:m], B.par.make_plan(m, 1), A0, sync=True)
    B.quality.chi_square_uniformity(f64[:m], 1000)
    B.par.fill_residues(u64[:m], B.par.make_plan(m, 1), A0, sync=True)
    B.quality.monobit_mantissa(u64[:m])
    B.par.fill(f64[:m], B.par.make_plan(m, 1), A0, sync=True)
    B.quality.serial_correlation(f64[:m], 1)
    sync()
    print("profile_all: done")


if __name__ == "__main__":
    main()
