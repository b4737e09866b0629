#!/usr/bin/env python
"""Throughput of the non-headline §8 paths (exploration/evidence tool):
interleaved fill, device deinterleave, seed-states (C4), quality suite, and
the host-output paths (pinned / pageable). One JSON line per measurement.

    python tools/secondary_perf.py > gpurun_out/secondary.jsonl
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

A0 = B.kMinSeedIndex
dev = torch.device("cuda:0")
stream = torch.cuda.current_stream(dev)


def cuda_ms(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record(stream)
    for i in range(reps):
        fn()
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    return statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(reps))


def wall_ms(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e3)
    return statistics.median(ts)


def emit(**kw):
    print(json.dumps(kw), flush=True)


def main() -> None:
    n = 1 << 30
    buf = torch.empty(n, dtype=torch.float64, device=dev)
    # Interleaved layout (reference Layout::Interleaved) at several worker counts.
    for w in (1, 7, 64, 1000, 100003):
        plan = B.par.make_plan(n, w, B.Layout.Interleaved)
        for eng in ("FP64", "Barrett"):
            ms = cuda_ms(lambda: B.par.fill(buf, plan, A0, engine=B.Engine[eng], stream=stream))
            emit(path="fill_interleaved", workers=w, engine=eng, items=n, ms=ms, gbs=n * 8 / ms / 1e6)
    # Device deinterleave (read + write, 16 B of traffic per item).
    out = torch.empty_like(buf)
    for w in (7, 1000):
        plan = B.par.make_plan(n, w, B.Layout.Interleaved)
        ms = cuda_ms(lambda: B.par.deinterleave(buf, plan), reps=5)
        emit(path="deinterleave", workers=w, items=n, ms=ms, gbs=n * 16 / ms / 1e6)
    del out
    # Seed states (C4): 2^20 arbitrary (a, k), plus 64-step walks.
    rng = np.random.default_rng(1)
    cnt = 1 << 20
    a = torch.from_numpy(rng.integers(A0, (1 << 53) + 1, cnt, dtype=np.uint64).view(np.int64)).to(dev)
    k = torch.from_numpy(rng.integers(0, 1 << 62, cnt, dtype=np.uint64).view(np.int64)).to(dev)
    ms = wall_ms(lambda: B.device.seed_states(a, k))
    emit(path="seed_states", streams=cnt, steps=0, ms_wall_sync=ms, mstates_s=cnt / ms / 1e3)
    ms = wall_ms(lambda: B.device.seed_states(a, k, steps=64))
    emit(path="seed_states", streams=cnt, steps=64, ms_wall_sync=ms, gvalues_s=cnt * 64 / ms / 1e6)
    # Quality suite on 2^28 samples (device inputs).
    m = 1 << 28
    u = buf[:m]
    B.par.fill(u, B.par.make_plan(m, 1), A0, sync=True)
    z = torch.empty(m, dtype=torch.int64, device=dev)
    B.par.fill_residues(z, B.par.make_plan(m, 1), A0, sync=True)
    for name, fn in (("chi_square_1000", lambda: B.quality.chi_square_uniformity(u, 1000)),
                     ("monobit", lambda: B.quality.monobit_mantissa(z)),
                     ("lag1_correlation", lambda: B.quality.serial_correlation(u, 1))):
        ms = wall_ms(fn)
        emit(path="quality", test=name, items=m, ms_wall_sync=ms, gitems_s=m / ms / 1e6)
    # Host outputs through bcn_fill (generation + D2H inside).
    h = 1 << 28
    pinned = torch.empty(h, dtype=torch.float64, pin_memory=True)
    pageable = np.empty(h, dtype=np.float64)
    plan = B.par.make_plan(h, 1)
    ms = wall_ms(lambda: B.par.fill(pinned, plan, A0))
    emit(path="host_fill", memory="pinned", items=h, ms=ms, gbs=h * 8 / ms / 1e6)
    ms = wall_ms(lambda: B.par.fill(pageable, plan, A0))
    emit(path="host_fill", memory="pageable", items=h, ms=ms, gbs=h * 8 / ms / 1e6)


if __name__ == "__main__":
    main()
