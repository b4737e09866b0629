#!/usr/bin/env python
"""Sustained-load comparison (exploration tool): each configuration runs
back-to-back fills for `--seconds`, sampling SM clock, power and throttle
reasons with NVML; reports GB/s over the second half, median clock, mean power.

    python tools/sustain.py [--seconds 3] > gpurun_out/sustain.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import pynvml  # noqa: E402
import torch  # noqa: E402

import paper_1206_1187_b200 as B  # noqa: E402

A0 = B.kMinSeedIndex
CONFIGS = [
    # (name, fmt, engine, pace GB/s, pace cps)
    ("constant_paced7200", "f64", "Constant", 7200, 2),
    ("f64_fp64_paced7200", "f64", "FP64", 7200, 2),
    ("f64_mixed_paced7200", "f64", "Mixed", 7200, 2),
    ("f64_mixed_paced7200_cps3", "f64", "Mixed", 7200, 3),
    ("f64_mixed_unpaced", "f64", "Mixed", 0, 2),
    ("u64_fp64_paced7200", "u64", "FP64", 7200, 2),
    ("u64_mixed_paced7200", "u64", "Mixed", 7200, 2),
    ("u64_barrett_unpaced", "u64", "Barrett", 0, 2),
    ("f32_fp64_unpaced", "f32", "FP64", 0, 2),
    ("f32_mixed_unpaced", "f32", "Mixed", 0, 2),
    ("f32_mixed_paced7200", "f32", "Mixed", 7200, 2),
]


def main() -> None:
    p = argparse.ArgumentParser()
    p.add_argument("--seconds", type=float, default=3.0)
    p.add_argument("--only", default="")
    a = p.parse_args()
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream(dev)
    n = 1 << 30
    f64 = torch.empty(n, dtype=torch.float64, device=dev)
    f32 = torch.empty(n, dtype=torch.float32, device=dev)
    plan = B.par.make_plan(n, 1)
    for name, fmt, eng, pace, cps in CONFIGS:
        if a.only and a.only not in name:
            continue
        B.device.set_write_pacing(pace, cps, 7 if fmt == 'f32' else 3)
        buf = f32 if fmt == "f32" else (f64.view(torch.int64) if fmt == "u64" else f64)
        if eng == "Constant":
            fn = lambda: B.device.fill_constant(buf.view(torch.int64), stream=stream)  # noqa: E731
        else:
            F, E = B.Format[fmt.upper()], B.Engine[eng]
            fn = lambda: B.par.fill_format(buf, plan, A0, B.Method.BarrettModified, 0, F,  # noqa: E731
                                           engine=E, stream=stream)
        samples, stop = [], threading.Event()

        def sampler():
            while not stop.is_set():
                try:
                    samples.append((time.perf_counter(),
                                    pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                    pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                                    pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
                except pynvml.NVMLError:
                    pass
                time.sleep(0.01)

        th = threading.Thread(target=sampler, daemon=True)
        th.start()
        t_end = time.perf_counter() + a.seconds
        evs = []
        while time.perf_counter() < t_end:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(20):
                fn()
            e1.record(stream)
            evs.append((time.perf_counter(), e0, e1))
            e1.synchronize()
        stop.set()
        th.join()
        half = time.perf_counter() - a.seconds / 2
        ms = [e0.elapsed_time(e1) / 20 for (t, e0, e1) in evs if t >= half - a.seconds / 2 * 0 and t > evs[0][0] + a.seconds / 2]
        nbytes = n * (4 if fmt == "f32" else 8)
        late = [s for s in samples if s[0] > samples[0][0] + a.seconds / 2]
        reasons = 0
        for s in late:
            reasons |= s[3]
        print(json.dumps({"config": name, "gbs": nbytes / (statistics.mean(ms) * 1e-3) / 1e9,
                          "ms": statistics.mean(ms), "sm_mhz": statistics.median([s[1] for s in late]),
                          "power_w": statistics.mean([s[2] for s in late]),
                          "power_cap": bool(reasons & 0x4), "reasons_mask": reasons}), flush=True)
        time.sleep(1.0)
    B.device.set_write_pacing(7200, 2, 3)


if __name__ == "__main__":
    main()
