"""`bcnrand gen` / `seed-info` on the B200 path (reference cli.cpp:79-147,
:207-224): the byte formats of the reference CLI — raw-u64 and raw-f64 little
endian, or text lines "%.17g" — written in chunks, each chunk a GPU fill at
base_offset = items done (make_plan(chunk, workers, layout), de-interleaved
unless --keep-physical). Exit codes follow cli.cpp:24-27: 0 ok, 2 usage, 3 I/O.

    python -m paper_1206_1187_b200.cli gen --n 1000000 --format raw-f64 --out u.f64
"""
from __future__ import annotations

import argparse
import ctypes
import os
import sys

import numpy as np

EXIT_OK, EXIT_USAGE, EXIT_IO = 0, 2, 3


def default_workers() -> int:
    """bench.cpp:192-199: BCN_THREADS if set and positive, else hardware concurrency."""
    try:
        v = int(os.environ.get("BCN_THREADS", "0"))
    except ValueError:
        v = 0
    return v if v > 0 else (os.cpu_count() or 1)


def format_text(values: np.ndarray) -> bytes:
    from . import _lib

    values = np.ascontiguousarray(values, dtype=np.float64)
    out = np.empty(values.size * 24, dtype=np.uint8)
    written = ctypes.c_uint64()
    _lib.call("bcn_format_text", ctypes.c_void_p(values.ctypes.data), values.size,
              ctypes.c_void_p(out.ctypes.data), out.size, ctypes.byref(written))
    return out[: written.value].tobytes()


def run_gen(a) -> int:
    from . import generator as gen
    from . import parallel as par
    from .errors import CudaError, InvalidArgument, OutOfRange

    try:
        method = gen.parse_method(a.method)
        layout = par.parse_layout(a.layout)
    except InvalidArgument as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE
    if a.format not in ("text", "raw-f64", "raw-u64"):
        print(f"gen: unknown format {a.format}", file=sys.stderr)
        return EXIT_USAGE
    if not gen.kMinSeedIndex <= a.seed <= gen.kMaxSeedIndex:
        print(f"gen: seed outside [{gen.kMinSeedIndex}, {gen.kMaxSeedIndex}]", file=sys.stderr)
        return EXIT_USAGE
    if a.n == 0 or a.chunk == 0:
        print("gen: --n and --chunk must be at least 1", file=sys.stderr)
        return EXIT_USAGE
    workers = a.workers or default_workers()
    try:
        sink = open(a.out, "wb") if a.out else sys.stdout.buffer
    except OSError as e:
        print(f"gen: cannot open output file: {a.out} ({e})", file=sys.stderr)
        return EXIT_IO
    ok = False
    try:
        done = 0
        dtype = np.uint64 if a.format == "raw-u64" else np.float64
        chunk_buf = np.empty(min(a.chunk, a.n), dtype=dtype)  # reused: pages touched once
        while done < a.n:
            cn = min(a.chunk, a.n - done)
            plan = par.make_plan(cn, workers, layout)
            buf = chunk_buf[:cn]
            if a.format == "raw-u64":
                par.fill_residues(buf, plan, a.seed, method, done)
            else:
                par.fill(buf, plan, a.seed, method, done)
            if layout == par.Layout.Interleaved and not a.keep_physical:
                buf = par.deinterleave(buf, plan)
            if a.format == "text":
                sink.write(format_text(buf))
            elif sys.byteorder == "little":  # raw formats are little-endian (cli.cpp:93-135)
                sink.write(memoryview(np.ascontiguousarray(buf)).cast("B"))
            else:  # pragma: no cover - big-endian hosts
                sink.write(buf.astype(buf.dtype.newbyteorder("<")).tobytes())
            done += cn
        sink.flush()
        ok = True
    except (InvalidArgument, OutOfRange) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except CudaError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    except OSError as e:
        print(f"gen: write failed: {e}", file=sys.stderr)
        return EXIT_IO
    finally:
        if a.out:
            sink.close()
            if not ok:
                try:  # OutputFile removes a partial file on failure (cli.cpp:53-58)
                    os.remove(a.out)
                except OSError:
                    pass
    return EXIT_OK


def run_seed_info(a) -> int:
    from . import generator as gen
    from .errors import OutOfRange

    try:
        s = gen.seed_from_index(a.index)
    except OutOfRange as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE
    print(f"seed index a  = {a.index}")
    print(f"z0            = {s.z}")
    print(f"first variate = {gen.to_unit_interval(gen.next(s)):.17g}")
    return EXIT_OK


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage errors exit 2, like CLI11's parse errors
        self.print_usage(sys.stderr)
        print(f"error: {message}", file=sys.stderr)
        raise SystemExit(EXIT_USAGE)


def main(argv=None) -> int:
    p = _Parser(prog="bcnrand", description="alpha_{2,3} variates on B200")
    sub = p.add_subparsers(dest="cmd", required=True, parser_class=_Parser)
    g = sub.add_parser("gen", help="generate variates")
    g.add_argument("--n", type=int, required=True)
    g.add_argument("--seed", type=int, default=5559060566555623)
    g.add_argument("--method", default="BarrettModified")
    g.add_argument("--workers", type=int, default=0)
    g.add_argument("--layout", default="contiguous")
    g.add_argument("--format", default="text")
    g.add_argument("--out", default="")
    g.add_argument("--keep-physical", action="store_true")
    g.add_argument("--chunk", type=int, default=1 << 22)
    si = sub.add_parser("seed-info", help="describe a starting index")
    si.add_argument("index", type=int)
    try:
        a = p.parse_args(argv)
    except SystemExit as e:
        return int(e.code) if isinstance(e.code, int) else EXIT_USAGE
    return run_gen(a) if a.cmd == "gen" else run_seed_info(a)


if __name__ == "__main__":
    sys.exit(main())
