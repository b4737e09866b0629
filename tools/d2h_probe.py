#!/usr/bin/env python
"""Pinned D2H copy rate vs concurrent streams and chunk size (exploration):
the ceiling of the host-output (e2e) path."""
import json
import torch

dev = torch.device("cuda:0")
total = 8 << 30
src = torch.empty(total // 8, dtype=torch.int64, device=dev).fill_(3)
dst = torch.empty(total // 8, dtype=torch.int64, pin_memory=True)
for chunk_mb in (32, 64, 128):
    for ns in (1, 2, 3, 4):
        streams = [torch.cuda.Stream(dev) for _ in range(ns)]
        chunk = chunk_mb << 20
        n = total // chunk
        best = 0
        for rep in range(3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for s in streams:
                s.wait_event(e0)
            for k in range(n):
                s = streams[k % ns]
                with torch.cuda.stream(s):
                    a = k * (chunk // 8)
                    dst[a:a + chunk // 8].copy_(src[a:a + chunk // 8], non_blocking=True)
            for s in streams:
                e = torch.cuda.Event(); e.record(s); torch.cuda.current_stream().wait_event(e)
            e1.record(); torch.cuda.synchronize()
            best = max(best, total / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        print(json.dumps({"chunk_mb": chunk_mb, "streams": ns, "gbs": round(best, 1)}), flush=True)
