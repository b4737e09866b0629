"""A/B of two builds of the product library in one process (round-robin, so
clock / power drift hits both alike): each `--libs` entry is a .so exporting
the C ABI; every round times `--per` back-to-back bcn_fill launches of 2^log2n
items per library with CUDA events on one stream.

    python tools/ab_lib.py --libs abtest/r01.so,paper_1206_1187_b200/libbcnrand_b200.so \
        [--fmt f64] [--pace 7200] [--rounds 15] [--per 8] [--log2n 30] [--engine 0]

--pace: a fixed target for every library (r01 builds take any value >= 0);
omit it to keep each build's default (r01: 7200, r02: calibrated).
Prints one JSON line per library (median / min per-launch ms, GB/s)."""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys

import torch

A0 = 5559060566555523 + 100


def main() -> None:
    p = argparse.ArgumentParser()
    p.add_argument("--libs", required=True)
    p.add_argument("--fmt", default="f64", choices=["u64", "f64", "f32"])
    p.add_argument("--pace", type=float, default=None)
    p.add_argument("--rounds", type=int, default=15)
    p.add_argument("--per", type=int, default=8)
    p.add_argument("--log2n", type=int, default=30)
    p.add_argument("--engine", type=int, default=0)
    p.add_argument("--tag", default="")
    p.add_argument("--workers", type=int, default=1, help="plan workers (with --interleaved: the width W)")
    p.add_argument("--interleaved", action="store_true")
    p.add_argument("--cps", type=int, default=1, help="paced CTAs per SM (with --pace)")
    p.add_argument("--mask", type=int, default=3, help="paced format mask (with --pace; 7 = f32 too)")
    a = p.parse_args()
    fmt = {"u64": 0, "f64": 1, "f32": 2}[a.fmt]
    isz = 4 if a.fmt == "f32" else 8
    n = 1 << a.log2n
    dev = torch.device("cuda:0")
    buf = torch.empty(n * isz // 8, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    sp = ctypes.c_void_p(stream.cuda_stream)
    libs = []
    for path in a.libs.split(","):
        lib = ctypes.CDLL(os.path.abspath(path), mode=ctypes.RTLD_LOCAL)
        lib.bcn_fill.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32,
                                 ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64, ctypes.c_int,
                                 ctypes.c_int, ctypes.c_void_p]
        lib.bcn_set_write_pacing.argtypes = [ctypes.c_double, ctypes.c_int, ctypes.c_int]
        lib.bcn_last_error.restype = ctypes.c_char_p
        if a.pace is not None:
            assert lib.bcn_set_write_pacing(a.pace, a.cps, a.mask) == 0
        libs.append((path, lib))
    times = {path: [] for path, _ in libs}

    def launch(lib):
        st = lib.bcn_fill(ctypes.c_void_p(buf.data_ptr()), n, n, fmt, a.workers, int(a.interleaved), A0, 3, 0,
                          a.engine, 0, sp)
        if st:
            raise RuntimeError(lib.bcn_last_error())

    for _, lib in libs:  # warm (context init, calibration)
        for _ in range(3):
            launch(lib)
    torch.cuda.synchronize()
    for _ in range(a.rounds):
        for path, lib in libs:
            launch(lib)
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(a.per + 1)]
            evs[0].record(stream)
            for i in range(a.per):
                launch(lib)
                evs[i + 1].record(stream)
            torch.cuda.synchronize()
            times[path] += [evs[i].elapsed_time(evs[i + 1]) for i in range(a.per)]
    for path, v in times.items():
        med = statistics.median(v)
        print(json.dumps({"tag": a.tag, "lib": path, "fmt": a.fmt, "pace": a.pace, "cps": a.cps, "mask": a.mask, "log2n": a.log2n,
                          "workers": a.workers, "layout": "interleaved" if a.interleaved else "contiguous",
                          "median_ms": med, "min_ms": min(v), "gbs_median": n * isz / med / 1e6,
                          "gbs_best": n * isz / min(v) / 1e6, "samples": len(v)}), flush=True)


if __name__ == "__main__":
    sys.exit(main())
