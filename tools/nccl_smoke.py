#!/usr/bin/env python
"""The bench's NCCL calls on a single rank (the only NCCL setup a 1-GPU box
allows): init_process_group("nccl", device_id=...), barrier, the float64 MAX
all_reduce and the int64 digest all_gather on CUDA tensors.

    torchrun --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 tools/nccl_smoke.py
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1206_1187_b200 import sharding  # noqa: E402


def main() -> None:
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    dist.barrier()
    t = torch.tensor([1.25], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    d = (2**64 - 1, 12345, 2**63 + 7)
    g = sharding.allgather_digest(d, dev)
    assert g == d, g
    assert float(t.item()) == 1.25
    dist.destroy_process_group()
    print("nccl smoke ok", flush=True)


if __name__ == "__main__":
    main()
