#!/usr/bin/env python
"""Quality-suite kernels on 2^28 device samples (evidence tool): run each
statistic a few times; per-kernel times come from an ncu launch list.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv \
        --log-file gpurun_out/quality_launches.csv python tools/quality_perf.py
"""
from __future__ import annotations

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1206_1187_b200 as B  # noqa: E402


def main() -> None:
    dev = torch.device("cuda:0")
    m = 1 << 28
    u = torch.empty(m, dtype=torch.float64, device=dev)
    z = torch.empty(m, dtype=torch.int64, device=dev)
    B.par.fill(u, B.par.make_plan(m, 1), B.kMinSeedIndex)
    B.par.fill_format(z, B.par.make_plan(m, 1), B.kMinSeedIndex, B.Method.BarrettModified, 0, B.Format.U64)
    torch.cuda.synchronize()
    for name, fn in (("chi_square_1000", lambda: B.quality.chi_square_uniformity(u, 1000)),
                     ("chi_square_20000", lambda: B.quality.chi_square_uniformity(u, 20000)),
                     ("monobit", lambda: B.quality.monobit_mantissa(z)),
                     ("lag1_correlation", lambda: B.quality.serial_correlation(u, 1))):
        for _ in range(3):
            t0 = time.perf_counter()
            r = fn()
            dt = time.perf_counter() - t0
        print(name, r.statistic, r.passed, f"{dt * 1e3:.3f} ms wall", flush=True)


if __name__ == "__main__":
    main()
