#!/usr/bin/env python
"""Device deinterleave throughput (exploration / evidence tool): CUDA-event
median per call, GB/s counting read + write (2 x itemsize per item).

    python tools/deint_perf.py [W1,W2,...] >> gpurun_out/deint.jsonl
"""
from __future__ import annotations

import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1206_1187_b200 as B  # noqa: E402


def main() -> None:
    widths = (1, 2, 7, 16, 31, 33, 64, 100, 128, 129, 200, 1000, 100003)
    if len(sys.argv) > 1:
        widths = tuple(int(w) for w in sys.argv[1].split(","))
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream(dev)
    n = 1 << int(os.environ.get("BCN_DEINT_LOG2N", "28"))
    for dt, isz in ((torch.float64, 8), (torch.float32, 4)):
        buf = torch.empty(n, dtype=dt, device=dev)
        for w in widths:
            plan = B.par.make_plan(n, w, B.Layout.Interleaved)
            B.par.deinterleave(buf, plan)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
            ev[0].record(stream)
            for i in range(10):
                B.par.deinterleave(buf, plan)
                ev[i + 1].record(stream)
            torch.cuda.synchronize()
            ms = statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(10))
            print(json.dumps({"path": "deinterleave", "tma": os.environ.get("BCN_DEINT_TMA", "1"), "itemsize": isz, "workers": w, "items": n,
                              "ms": ms, "gbs_rw": 2 * n * isz / ms / 1e6}), flush=True)
        del buf


if __name__ == "__main__":
    main()
