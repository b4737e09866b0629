#!/usr/bin/env python
"""One device deinterleave configuration for an ncu capture (exploration tool):
3 warm-up calls, then `--reps` calls.

    ncu --set full -k regex:deint\\|transpose -c 1 python tools/deint_one.py --w 1000000 --isz 4
"""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1206_1187_b200 as B  # noqa: E402


def main() -> None:
    p = argparse.ArgumentParser()
    p.add_argument("--w", type=int, required=True)
    p.add_argument("--isz", type=int, default=8)
    p.add_argument("--log2n", type=int, default=28)
    p.add_argument("--reps", type=int, default=1)
    a = p.parse_args()
    n = 1 << a.log2n
    buf = torch.empty(n, dtype=torch.float64 if a.isz == 8 else torch.float32, device="cuda:0")
    plan = B.par.make_plan(n, a.w, B.Layout.Interleaved)
    for _ in range(3 + a.reps):
        B.par.deinterleave(buf, plan)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
