#!/usr/bin/env python
"""Per-launch timeline of back-to-back fills (exploration tool): CUDA-event
time of every launch plus NVML power / SM clock samples, summarised in
buckets, for one configuration per line.

    python tools/timeline.py [--launches 600] [--pace 7200] [--fmt f64]
                             [--engine FP64] [--bucket 50] >> gpurun_out/timeline.jsonl
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


def main() -> None:
    p = argparse.ArgumentParser()
    p.add_argument("--launches", type=int, default=600)
    p.add_argument("--bucket", type=int, default=50)
    p.add_argument("--pace", type=float, default=7200.0)
    p.add_argument("--cps", type=int, default=2)
    p.add_argument("--fmt", default="f64")
    p.add_argument("--engine", default="FP64")
    p.add_argument("--log2n", type=int, default=30)
    p.add_argument("--idle", type=float, default=2.0, help="seconds of idle before the run")
    p.add_argument("--tag", default="")
    a = p.parse_args()
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream(dev)
    n = 1 << a.log2n
    dt = {"f64": torch.float64, "u64": torch.int64, "f32": torch.float32}[a.fmt]
    buf = torch.empty(n, dtype=dt, device=dev)
    plan = B.par.make_plan(n, 1)
    B.device.set_write_pacing(a.pace, a.cps, 7)
    if a.engine in ("Constant", "Noise"):
        raw = buf.view(torch.int32) if a.fmt == "f32" else buf.view(torch.int64)
        writer = B.device.fill_constant if a.engine == "Constant" else B.device.fill_noise
        fn = lambda: writer(raw, stream=stream)  # noqa: E731
    else:
        F, E = B.Format[a.fmt.upper()], B.Engine[a.engine]
        fn = lambda: B.par.fill_format(buf, plan, B.kMinSeedIndex, B.Method.BarrettModified, 0, F,  # noqa: E731
                                       engine=E, stream=stream)
    fn()
    torch.cuda.synchronize()
    time.sleep(a.idle)
    samples, stop = [], threading.Event()

    def instant_w():
        try:
            v = pynvml.nvmlDeviceGetFieldValues(h, [pynvml.NVML_FI_DEV_POWER_INSTANT])[0]
            return v.value.uiVal / 1000.0 if v.nvmlReturn == 0 else float("nan")
        except Exception:  # noqa: BLE001
            return float("nan")

    def sampler():
        while not stop.is_set():
            try:
                samples.append((time.perf_counter(),
                                pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                                pynvml.nvmlDeviceGetCurrentClocksEventReasons(h),
                                instant_w(),
                                pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM)))
            except pynvml.NVMLError:
                pass
            time.sleep(0.005)

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.launches + 1)]
    th = threading.Thread(target=sampler, daemon=True)
    th.start()
    t0 = time.perf_counter()
    ev[0].record(stream)
    for i in range(a.launches):
        fn()
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    stop.set()
    th.join()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(a.launches)]
    nbytes = n * buf.element_size()
    buckets = []
    for b in range(0, a.launches, a.bucket):
        chunk = per[b:b + a.bucket]
        buckets.append(round(nbytes / (statistics.mean(chunk) * 1e-3) / 1e9, 1))
    load = [s for s in samples if t0 <= s[0] <= t1]
    print(json.dumps({
        "tag": a.tag, "fmt": a.fmt, "engine": a.engine, "pace": a.pace, "cps": a.cps,
        "launches": a.launches,
        "gbs_all": round(nbytes * a.launches / (sum(per) * 1e-3) / 1e9, 1),
        "gbs_first": round(nbytes / (per[0] * 1e-3) / 1e9, 1),
        "gbs_buckets": buckets,
        "sm_mhz_median": statistics.median([s[1] for s in load]) if load else None,
        "sm_mhz_min": min([s[1] for s in load]) if load else None,
        "power_w_mean": round(statistics.mean([s[2] for s in load]), 1) if load else None,
        "power_w_max": round(max([s[2] for s in load]), 1) if load else None,
        "power_instant_w_mean": round(statistics.mean([s[4] for s in load]), 1) if load else None,
        "power_instant_w_max": round(max([s[4] for s in load]), 1) if load else None,
        "mem_mhz_min": min([s[5] for s in load]) if load else None,
        "power_limit_w": pynvml.nvmlDeviceGetEnforcedPowerLimit(h) / 1000.0,
        "power_cap_frac": round(sum(1 for s in load if s[3] & 0x4) / len(load), 2) if load else None,
    }), flush=True)


if __name__ == "__main__":
    main()
