#!/usr/bin/env python
"""Interleaved-layout fill throughput vs paced-grid CTAs per SM (exploration
tool). One JSON line per (workers, ctas_per_sm).

    python tools/inter_perf.py > gpurun_out/inter.jsonl
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
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", default="1,7,64,1000,100003")
    ap.add_argument("--cps", default="1,2,3")
    ap.add_argument("--rounds", type=int, default=2)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream(dev)
    n = 1 << 30
    buf = torch.empty(n, dtype=torch.float64, device=dev)
    for rnd in range(args.rounds):
        for w in [int(x) for x in args.workers.split(",")]:
            plan = B.par.make_plan(n, w, B.Layout.Interleaved)
            for cps in [int(x) for x in args.cps.split(",")]:
                B.device.set_write_pacing(7200, cps, 3)
                fn = lambda: B.par.fill(buf, plan, B.kMinSeedIndex, stream=stream)  # noqa: E731
                fn()
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
                ev[0].record(stream)
                for i in range(5):
                    fn()
                    ev[i + 1].record(stream)
                torch.cuda.synchronize()
                ms = statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(5))
                print(json.dumps({"round": rnd, "workers": w, "ctas_per_sm": cps, "ms": ms,
                                  "gbs": n * 8 / ms / 1e6}), flush=True)


if __name__ == "__main__":
    main()
