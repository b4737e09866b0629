#!/usr/bin/env python
"""Every deinterleave must write every output element: sentinel-filled output,
compare with the oracle (triage tool)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from paper_1206_1187_b200 import _lib  # noqa: E402

o = O.Oracle()
dev = torch.device("cuda:0")
bad = 0
rng = np.random.default_rng(3)
for n in (70001, 20000, 1000, 130, 100003, 1 << 20):
    for w in (1, 2, 3, 5, 7, 31, 32, 33, 40, 64, 100, 127, 128, 129, 1000, 4099):
        for isz, dt, ndt in ((8, torch.int64, np.uint64), (4, torch.int32, np.uint32)):
            phys = rng.integers(0, 2**31, n).astype(ndt)
            din = torch.from_numpy(phys.view(np.int64 if isz == 8 else np.int32)).to(dev)
            out = torch.full((n,), -1, dtype=dt, device=dev)
            _lib.call("bcn_deinterleave", ctypes.c_void_p(din.data_ptr()), ctypes.c_void_p(out.data_ptr()), n, w,
                      isz, 0, None)
            got = out.cpu().numpy().view(ndt)
            want = o.deinterleave(phys, w)
            if not np.array_equal(got, want):
                bad += 1
                idx = np.nonzero(got != want)[0]
                print("MISMATCH", n, w, isz, len(idx), idx[:8], flush=True)
print("done, bad =", bad)
