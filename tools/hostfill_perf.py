#!/usr/bin/env python
"""Host-output fill rate (pageable and pinned numpy/torch buffers), wall
clock of the synchronous call (exploration tool).

    BCN_COPY_THREADS=16 BCN_COPY_NT=1 python tools/hostfill_perf.py
"""
from __future__ import annotations

import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1206_1187_b200 as B  # noqa: E402


def main() -> None:
    h = 1 << 28
    plan = B.par.make_plan(h, 1)
    for kind in ("pageable", "pinned"):
        buf = np.ones(h) if kind == "pageable" else torch.empty(h, dtype=torch.float64, pin_memory=True)
        B.par.fill(buf, plan, B.kMinSeedIndex)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            B.par.fill(buf, plan, B.kMinSeedIndex)
            ts.append(time.perf_counter() - t0)
        s = statistics.median(ts)
        print(json.dumps({"memory": kind, "threads": os.environ.get("BCN_COPY_THREADS", "default"),
                          "nt": os.environ.get("BCN_COPY_NT", "0"), "gbs": h * 8 / s / 1e9,
                          "cpus": os.cpu_count()}), flush=True)


if __name__ == "__main__":
    main()
