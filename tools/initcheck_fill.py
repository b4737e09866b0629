#!/usr/bin/env python
"""initcheck triage: which fill paths' writes does compute-sanitizer initcheck
see? (exploration tool)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1206_1187_b200 as B  # noqa: E402

which = sys.argv[1]
n = 1 << 16
buf = torch.empty(n, dtype=torch.float64, device="cuda")
plan = B.par.make_plan(n, 1)
if which == "paced":
    B.par.fill(buf, plan, B.kMinSeedIndex, sync=True)
elif which == "contig":
    B.device.set_write_pacing(0.0, 1, 3)
    B.par.fill(buf, plan, B.kMinSeedIndex, sync=True)
elif which == "paced_stream":
    s = torch.cuda.Stream()
    B.par.fill(buf, plan, B.kMinSeedIndex, stream=s)
    s.synchronize()
elif which == "torch":
    buf.fill_(0.5)
elif which == "misaligned_torch":
    buf = torch.empty(n + 1, dtype=torch.float64, device="cuda")[1:]
    buf.fill_(0.5)
elif which == "misaligned_ours":
    buf = torch.empty(n + 1, dtype=torch.float64, device="cuda")[1:]
    B.par.fill(buf, plan, B.kMinSeedIndex, sync=True)
elif which == "ragged_ours":
    m = 70001
    buf = torch.empty(m, dtype=torch.float64, device="cuda")
    B.par.fill(buf, B.par.make_plan(m, 1), B.kMinSeedIndex, sync=True)
print(which, float(buf.cpu()[5]))
