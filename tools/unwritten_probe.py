#!/usr/bin/env python
"""Every fill path must write every element: pre-fill the output with a
sentinel, fill, compare with the oracle (exploration / triage tool)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_1206_1187_b200 as B  # noqa: E402

o = O.Oracle()
dev = torch.device("cuda:0")
bad = 0
for n in (70001, 1000, 130, 100003):
    for fmt, dt in ((B.Format.U64, torch.int64), (B.Format.F64, torch.float64), (B.Format.F32, torch.float32)):
        want = o.fill(n, int(fmt), base_offset=12345)
        want = want.view(np.uint32 if want.itemsize == 4 else np.uint64)
        for eng in B.Engine:
            for layout in (B.Layout.Contiguous, B.Layout.Interleaved):
                if layout == B.Layout.Interleaved and eng in (B.Engine.Staged, B.Engine.Bulk):
                    continue
                for w in ((1,) if layout == B.Layout.Contiguous else (3, 40, 1000)):
                    for off in (0, 1, 3):
                        base = torch.full((n + off,), -1, dtype=torch.int32 if dt == torch.float32 else torch.int64,
                                          device=dev).view(dt)
                        buf = base[off:]
                        plan = B.par.make_plan(n, w, layout)
                        B.par.fill_format(buf, plan, B.kMinSeedIndex, B.Method.BarrettModified, 12345, fmt,
                                          engine=eng, sync=True)
                        got = buf.cpu().numpy()
                        if layout == B.Layout.Interleaved:
                            got = B.par.deinterleave(buf, plan).cpu().numpy()
                        got = got.view(np.uint32 if got.itemsize == 4 else np.uint64)
                        if not np.array_equal(got, want):
                            bad += 1
                            idx = np.nonzero(got != want)[0]
                            print("MISMATCH", n, fmt.name, eng.name, layout.name, w, off, len(idx), idx[:8], flush=True)
print("done, bad =", bad)
