import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sys, torch, numpy as np, paper_1206_1187_b200 as B
n, w, isz = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dt = torch.int32 if isz == 4 else torch.int64
x = torch.arange(n, dtype=dt, device="cuda:0")
plan = B.par.make_plan(n, w, B.Layout.Interleaved)
y = B.par.deinterleave(x, plan)
torch.cuda.synchronize()
print("ok", n, w, isz)
