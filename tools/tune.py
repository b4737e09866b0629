#!/usr/bin/env python
"""Launch-configuration sweep of the contiguous fill (exploration tool):
format x engine x row order x CTAs/SM, interleaved rounds, median GB/s.

    python tools/tune.py [--log2n 30] [--rounds 3] > gpurun_out/tune.jsonl
"""
from __future__ import annotations

import argparse
import itertools
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1206_1187_b200 as B  # noqa: E402

A0 = B.kMinSeedIndex


def main() -> None:
    p = argparse.ArgumentParser()
    p.add_argument("--log2n", type=int, default=30)
    p.add_argument("--rounds", type=int, default=3)
    p.add_argument("--reps", type=int, default=4)
    p.add_argument("--fmts", default="f64,u64,f32")
    p.add_argument("--engines", default="Barrett,FP64")
    p.add_argument("--cps", default="1,2,3,4,6,8")
    p.add_argument("--pace", default="", help="comma list of pacing targets (GB/s); sweeps the paced kernels")
    a = p.parse_args()
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream(dev)
    n = 1 << a.log2n
    bufs = {"f64": torch.empty(n, dtype=torch.float64, device=dev)}
    bufs["u64"] = bufs["f64"].view(torch.int64)
    bufs["f32"] = torch.empty(n, dtype=torch.float32, device=dev)
    plan = B.par.make_plan(n, 1)
    if a.pace:
        # (fmt, engine, pace GB/s, ctas per SM)
        configs = list(itertools.product(a.fmts.split(","), a.engines.split(",") + ["Constant"],
                                         [float(x) for x in a.pace.split(",")],
                                         [int(c) for c in a.cps.split(",")]))
    else:
        configs = list(itertools.product(a.fmts.split(","), a.engines.split(",") + ["Constant"],
                                         (0, 1), [int(c) for c in a.cps.split(",")]))
    samples = {c: [] for c in configs}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.reps + 1)]
    for _ in range(a.rounds):
        for c in configs:
            fmt, eng, order, cps = c
            if a.pace:
                B.device.set_write_pacing(order, cps, 7)
            else:
                B.device.set_write_pacing(0, 1)
                B.device.set_launch_config(cps, order)
            buf = bufs[fmt]
            if eng == "Constant":
                raw = buf.view(torch.int32) if fmt == "f32" else buf.view(torch.int64)
                fn = lambda: B.device.fill_constant(raw, stream=stream)  # noqa: E731
            else:
                f, e = B.Format[fmt.upper()], B.Engine[eng]
                fn = lambda: B.par.fill_format(buf, plan, A0, B.Method.BarrettModified, 0, f,  # noqa: E731
                                               engine=e, stream=stream)
            fn()
            ev[0].record(stream)
            for i in range(a.reps):
                fn()
                ev[i + 1].record(stream)
            torch.cuda.synchronize()
            samples[c] += [ev[i].elapsed_time(ev[i + 1]) for i in range(a.reps)]
    for c, v in samples.items():
        fmt, eng, order, cps = c
        nbytes = n * (4 if fmt == "f32" else 8)
        med = statistics.median(v)
        print(json.dumps({"fmt": fmt, "engine": eng, "order": (f"pace{order:.0f}" if a.pace else
                                                             "stride" if order else "rows"),
                          "ctas_per_sm": cps, "median_ms": med, "gbs": nbytes / (med * 1e-3) / 1e9,
                          "best_gbs": nbytes / (min(v) * 1e-3) / 1e9, "samples": len(v)}), flush=True)


if __name__ == "__main__":
    main()
