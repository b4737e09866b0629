"""Digest of the full C5 stream (2^36 doubles from a0, offset 0), computed with
the CPU oracle in chunks (TEST INFRASTRUCTURE; ~2 min on 8 cores).

    python tests/golden/make_c5_digest.py [log2n=36] > tests/golden/c5_digest.json

The GPU bench (`bench.py --workload c5`) and tests compare the all-reduced
per-shard device digests against this value at every GPU count.
"""
from __future__ import annotations

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402


def main() -> None:
    log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 36
    n = 1 << log2n
    chunk = 1 << 26
    o = O.Oracle()
    buf = np.empty(chunk, dtype=np.float64)
    s = ws = x = 0
    t0 = time.time()
    for c in range(0, n, chunk):
        o.fill(chunk, O.FMT_F64, base_offset=c, out=buf)
        d = o.digest(buf.view(np.uint64), index_base=c)
        s = (s + d[0]) % (1 << 64)
        ws = (ws + d[1]) % (1 << 64)
        x ^= d[2]
    print(json.dumps({"workload": f"2^{log2n} f64 from seed index a0, base_offset 0",
                      "log2n": log2n, "digest": [str(s), str(ws), str(x)],
                      "seconds": round(time.time() - t0, 1),
                      "generator": "tests/golden/make_c5_digest.py (oracle/liboracle.so)"}))


if __name__ == "__main__":
    main()
