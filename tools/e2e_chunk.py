#!/usr/bin/env python
"""e2e exploration (ran with a temporary BCN_HOST_CHUNK_MB knob, since removed): bcn_fill of 2^30 doubles into pinned host memory vs a plain
pinned D2H copy of the same bytes (CUDA-event / wall timing)."""
from __future__ import annotations

import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1206_1187_b200 as B  # noqa: E402


def main() -> None:
    n = 1 << 30
    host = torch.empty(n, dtype=torch.float64, pin_memory=True)
    plan = B.par.make_plan(n, 1)
    B.par.fill(host, plan, B.kMinSeedIndex)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        B.par.fill(host, plan, B.kMinSeedIndex)
        ts.append(time.perf_counter() - t0)
    dev = torch.empty(n, dtype=torch.float64, device="cuda")
    cs = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        host.copy_(dev, non_blocking=True)
        torch.cuda.synchronize()
        cs.append(time.perf_counter() - t0)
    print(json.dumps({"chunk_mb": os.environ.get("BCN_HOST_CHUNK_MB", "64"),
                      "fill_gbs": n * 8 / statistics.median(ts) / 1e9,
                      "copy_gbs": n * 8 / statistics.median(cs) / 1e9}), flush=True)


if __name__ == "__main__":
    main()
