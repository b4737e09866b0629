"""Per-2^24-chunk digests of the first 2^33 variates of the a0 stream in every
output format, computed with the CPU oracle (TEST INFRASTRUCTURE).

    python tests/golden/make_chunk_digests.py [log2n=33] > tests/golden/chunk_digests.json

Chunk c covers logical elements [c*2^24, (c+1)*2^24) of
`par::fill(…, a0, BarrettModified, base_offset=0)` (reference
`/root/reference/proj/src/parallel.cpp:101-111`) in format u64
(`fill_residues`), f64 (`fill`) or f32 (RZ of the f64); its digest
is (Σ v, Σ (g+1)·v, XOR v·(2g+1)) mod 2^64 over the item bits v at absolute
index g (`oracle/bcn_oracle.c:bcno_digest`, the device's `k_digest`). Sums and
weighted sums of consecutive chunks add and the xor terms xor, so any
chunk-aligned window of the stream has a digest derived from this table:
C2 = chunks [0, 64) (one GPU) or [64 r, 64 (r+1)) (rank r of the weak-scaling
run), C3 = the first 2^28 … 2^32 (chunks [0, 16) … [0, 256)).

The u64 and f64 digests of chunks 0, 1 and the last chunk are recomputed from the
reference itself (`oracle/_ref`, the unmodified sources compiled here) when it
is available; the script refuses to write a table that disagrees.
"""
from __future__ import annotations

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402

CHUNK_LOG2 = 24
FORMATS = {"u64": O.FMT_U64, "f64": O.FMT_F64, "f32": O.FMT_F32}


def bits(a: np.ndarray) -> np.ndarray:
    return a.view(np.uint64 if a.itemsize == 8 else np.uint32)


def main() -> None:
    log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 33
    chunk = 1 << CHUNK_LOG2
    nchunks = 1 << (log2n - CHUNK_LOG2)
    o = O.Oracle()
    t0 = time.time()
    table: dict[str, list[list[str]]] = {}
    for name, fmt in FORMATS.items():
        buf = np.empty(chunk, dtype=O._dtype(fmt))
        rows = []
        for c in range(nchunks):
            o.fill(chunk, fmt, base_offset=c * chunk, out=buf)
            rows.append([str(x) for x in o.digest(bits(buf), index_base=c * chunk)])
        table[name] = rows
        print(f"{name}: {nchunks} chunks, {time.time() - t0:.1f} s", file=sys.stderr)
    checked = []
    if os.path.exists(O.REF_SO) or os.path.isdir(O.REFERENCE_ROOT):
        ref = O.Reference()
        for name in ("u64", "f64"):
            buf = np.empty(chunk, dtype=O._dtype(FORMATS[name]))
            for c in (0, 1, nchunks - 1):
                ref.fill(chunk, FORMATS[name], base_offset=c * chunk, out=buf)
                got = [str(x) for x in o.digest(bits(buf), index_base=c * chunk)]
                if got != table[name][c]:
                    raise SystemExit(f"oracle and reference disagree on {name} chunk {c}")
                checked.append(f"{name}:{c}")
    print(json.dumps({
        "workload": f"first 2^{log2n} variates from seed index a0 = 3^33+100, base_offset 0, "
                    "contiguous plan, W=1",
        "seed_index": O.MIN_SEED, "log2n": log2n, "chunk_log2": CHUNK_LOG2,
        "digest": "[sum, weighted sum (g+1)*v, xor v*(2g+1)] mod 2^64 of the item bits, g absolute",
        "formats": table,
        "checked_vs_reference": checked,
        "seconds": round(time.time() - t0, 1),
        "generator": "tests/golden/make_chunk_digests.py (oracle/liboracle.so)",
    }))


if __name__ == "__main__":
    main()
