#!/usr/bin/env python
"""Deinterleave throughput vs alignment of the physical rows (W * itemsize)
and of the per-worker output runs (wpw * itemsize) — exploration tool:
    python tools/deint_align.py >> gpurun_out/deint_align.jsonl"""
from __future__ import annotations

import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1206_1187_b200 as B  # noqa: E402


def run(n, w, dt, isz, st):
    buf = torch.empty(n, dtype=dt, device="cuda:0")
    plan = B.par.make_plan(n, w, B.Layout.Interleaved)
    B.par.deinterleave(buf, plan)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
    ev[0].record(st)
    for i in range(10):
        B.par.deinterleave(buf, plan)
        ev[i + 1].record(st)
    torch.cuda.synchronize()
    ms = statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(10))
    print(json.dumps({"itemsize": isz, "workers": w, "n": n, "wpw": plan.work_per_worker,
                      "row_bytes_mod128": w * isz % 128, "run_bytes_mod128": plan.work_per_worker * isz % 128,
                      "ms": ms, "gbs_rw": 2 * n * isz / ms / 1e6}), flush=True)
    del buf


def main() -> None:
    st = torch.cuda.current_stream()
    for dt, isz in ((torch.float64, 8), (torch.float32, 4)):
        for w in (1024, 1000, 1001, 4096, 4099):
            for wpw in (1 << 20, (1 << 20) - 3, (1 << 20) - 8, (1 << 20) - 32):
                run(w * wpw, w, dt, isz, st)


if __name__ == "__main__":
    main()
