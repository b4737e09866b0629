#!/usr/bin/env python
"""Pacer-variant study (exploration tool): for this process's BCN_PACE_FLAGS
(kPaceConsumed = 1, kPaceSmClock = 2), each configuration runs a burst (20
launches after 1 s idle) and then back-to-back fills for `--seconds`
(sustained: the board power controller acts), with NVML SM clock / power.

    BCN_PACE_FLAGS=2 python tools/pace_modes.py --tag sm >> gpurun_out/pace_modes.jsonl
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
CONFIGS = [  # (fmt, pace GB/s (-1 = calibrated), ctas per SM)
    ("f64", -1, 1), ("f64", 7000, 1), ("f64", 7200, 1), ("f64", 7400, 1), ("f64", 7600, 1),
    ("u64", -1, 1), ("u64", 7200, 1),
    ("f32", 0, 1), ("f32", 6800, 2), ("f32", 7200, 2), ("f32", 7200, 1),
]


def main() -> None:
    p = argparse.ArgumentParser()
    p.add_argument("--seconds", type=float, default=2.0)
    p.add_argument("--tag", default="")
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
    cal = B.device.device_write_pacing(0)
    for fmt, pace, cps in CONFIGS:
        if a.only and a.only != fmt:
            continue
        B.device.set_write_pacing(pace, cps, 7)
        buf = f32 if fmt == "f32" else (f64.view(torch.int64) if fmt == "u64" else f64)
        F = B.Format[fmt.upper()]

        def fn():
            B.par.fill_format(buf, plan, A0, B.Method.BarrettModified, 0, F, stream=stream)

        nbytes = n * (4 if fmt == "f32" else 8)
        time.sleep(1.0)
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(20):
            fn()
        e1.record(stream)
        e1.synchronize()
        burst = nbytes * 20 / (e0.elapsed_time(e1) * 1e-3) / 1e9
        samples, stop = [], threading.Event()

        def sampler():
            while not stop.is_set():
                try:
                    samples.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                    pynvml.nvmlDeviceGetFieldValues(h, [pynvml.NVML_FI_DEV_POWER_INSTANT])[0].value.uiVal / 1000.0))
                except pynvml.NVMLError:
                    pass
                time.sleep(0.01)

        th = threading.Thread(target=sampler, daemon=True)
        th.start()
        t_start = time.perf_counter()
        evs = []
        while time.perf_counter() < t_start + a.seconds:
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            b0.record(stream)
            for _ in range(20):
                fn()
            b1.record(stream)
            evs.append((time.perf_counter(), b0, b1))
            b1.synchronize()
        stop.set()
        th.join()
        late_ms = [x.elapsed_time(y) / 20 for (t, x, y) in evs if t > t_start + a.seconds / 2]
        late = [s for s in samples if s[0] > t_start + a.seconds / 2]
        print(json.dumps({"tag": a.tag, "flags": os.environ.get("BCN_PACE_FLAGS", "0"), "fmt": fmt,
                          "pace": pace if pace >= 0 else cal[0], "cps": cps, "burst_gbs": round(burst, 1),
                          "sustained_gbs": round(nbytes / (statistics.mean(late_ms) * 1e-3) / 1e9, 1),
                          "sm_mhz": statistics.median([s[1] for s in late]) if late else None,
                          "power_w": round(statistics.mean([s[2] for s in late]), 1) if late else None}),
              flush=True)
    B.device.set_write_pacing(-1, 1, 3)


if __name__ == "__main__":
    main()
