"""CPU oracle for the alpha_{2,3} fill path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package. It is the checker for the
CUDA product path, never the thing measured as the product or shipped: the
product library ``paper_1206_1187_b200`` does not import it.

Two back ends, both driven through ctypes:

* :class:`Oracle` — ``oracle/liboracle.so``, the plain-C restatement of the
  reference algorithm (``oracle/bcn_oracle.c``; every function cites the
  reference file:line it follows).
* :class:`Reference` — ``oracle/_ref/libbcnref.so``, the UNMODIFIED reference
  sources (``/root/reference/proj/src/{modred,generator,parallel}.cpp``)
  compiled in place by ``oracle/Makefile`` behind a tiny extern "C" shim. It is
  built in the development container and shipped pre-built to the GPU box.

Status codes from either library map onto the reference's exception types via
:data:`ERRORS`.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libbcnref.so")
REFERENCE_ROOT = "/root/reference/proj"

MODULUS = 5559060566555523
PERIOD = 3706040377703682
MIN_SEED = MODULUS + 100
MAX_SEED = 1 << 53

FMT_U64, FMT_F64, FMT_F32 = 0, 1, 2
CONTIGUOUS, INTERLEAVED = 0, 1
# include/bcnrand/generator.hpp:17
REF128, LECUYER, BARRETT, BARRETT_MODIFIED = 0, 1, 2, 3


class InvalidArgument(ValueError):
    """std::invalid_argument"""


class OutOfRange(IndexError):
    """std::out_of_range"""


class DomainError(ArithmeticError):
    """std::domain_error"""


ERRORS = {1: InvalidArgument, 2: OutOfRange, 3: DomainError}


def _check(status: int, what: str) -> None:
    if status:
        raise ERRORS.get(status, RuntimeError)(f"{what}: status {status}")


def build(reference: bool = True) -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference is present)."""
    targets = ["oracle"]
    if reference and os.path.isdir(REFERENCE_ROOT):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


_u64 = ctypes.c_uint64
_pu64 = ctypes.POINTER(ctypes.c_uint64)


def _dtype(fmt: int):
    return {FMT_U64: np.uint64, FMT_F64: np.float64, FMT_F32: np.float32}[fmt]


class Oracle:
    """ctypes view of the plain-C restatement (oracle/bcn_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(reference=False)
        lib = ctypes.CDLL(path)
        self.lib = lib
        lib.bcno_reduce_ref.argtypes = [_u64, _pu64]
        lib.bcno_barrett_modified_step.argtypes = [_u64, _pu64]
        lib.bcno_modpow2.argtypes = [_u64, _u64, _pu64]
        lib.bcno_seed_from_index.argtypes = [_u64, _pu64]
        lib.bcno_state_at.argtypes = [_u64, _u64, _pu64]
        lib.bcno_to_unit_interval.argtypes = [_u64, ctypes.POINTER(ctypes.c_double)]
        lib.bcno_to_unit_float.argtypes = [_u64, ctypes.POINTER(ctypes.c_float)]
        lib.bcno_make_plan.argtypes = [_u64, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32), _pu64]
        lib.bcno_elements_for.argtypes = [_u64, _u64, ctypes.c_uint32]
        lib.bcno_elements_for.restype = _u64
        lib.bcno_physical_index.argtypes = [_u64, ctypes.c_uint32, _u64, ctypes.c_int,
                                            ctypes.c_uint32, _u64]
        lib.bcno_physical_index.restype = _u64
        lib.bcno_fill.argtypes = [ctypes.c_void_p, _u64, ctypes.c_int, ctypes.c_uint32,
                                  ctypes.c_int, _u64, _u64, ctypes.c_uint32]
        lib.bcno_deinterleave.argtypes = [ctypes.c_void_p, ctypes.c_void_p, _u64,
                                          ctypes.c_uint32, ctypes.c_uint32]
        lib.bcno_digest.argtypes = [ctypes.c_void_p, _u64, ctypes.c_uint32, _u64, _pu64]
        lib.bcno_next.argtypes = [_pu64]
        lib.bcno_seed_batch.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, _u64,
                                        ctypes.c_uint32]

    def _u64_call(self, fn, *args) -> int:
        out = _u64()
        _check(fn(*args, ctypes.byref(out)), fn.__name__)
        return out.value

    def reduce_ref(self, z: int) -> int:
        return self._u64_call(self.lib.bcno_reduce_ref, z)

    def barrett_modified_step(self, z: int) -> int:
        return self._u64_call(self.lib.bcno_barrett_modified_step, z)

    def modpow2(self, e: int, modulus: int = MODULUS) -> int:
        return self._u64_call(self.lib.bcno_modpow2, e, modulus)

    def seed_from_index(self, a: int) -> int:
        return self._u64_call(self.lib.bcno_seed_from_index, a)

    def state_at(self, a: int, k: int) -> int:
        return self._u64_call(self.lib.bcno_state_at, a, k)

    def next(self, z: int) -> int:
        v = _u64(z)
        _check(self.lib.bcno_next(ctypes.byref(v)), "next")
        return v.value

    def seed_batch(self, a: np.ndarray, k: np.ndarray, steps: int = 0) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint64)
        k = np.ascontiguousarray(k, dtype=np.uint64)
        out = np.empty(a.size * max(steps, 1), dtype=np.uint64)
        _check(self.lib.bcno_seed_batch(a.ctypes.data, k.ctypes.data, out.ctypes.data, a.size,
                                        steps), "seed_batch")
        return out if steps == 0 else out.reshape(a.size, steps)

    def to_unit_interval(self, z: int) -> float:
        out = ctypes.c_double()
        _check(self.lib.bcno_to_unit_interval(z, ctypes.byref(out)), "to_unit_interval")
        return out.value

    def to_unit_float(self, z: int) -> np.float32:
        out = ctypes.c_float()
        _check(self.lib.bcno_to_unit_float(z, ctypes.byref(out)), "to_unit_float")
        return np.float32(out.value)

    def make_plan(self, n: int, workers: int) -> tuple[int, int]:
        eff = ctypes.c_uint32()
        wpw = _u64()
        _check(self.lib.bcno_make_plan(n, workers, ctypes.byref(eff), ctypes.byref(wpw)),
               "make_plan")
        return eff.value, wpw.value

    def physical_index(self, n: int, workers: int, layout: int, w: int, i: int) -> int:
        eff, wpw = self.make_plan(n, workers)
        return self.lib.bcno_physical_index(n, eff, wpw, layout, w, i)

    def fill(self, n: int, fmt: int = FMT_F64, *, seed_index: int = MIN_SEED,
             base_offset: int = 0, workers: int = 1, layout: int = CONTIGUOUS,
             threads: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty(n, dtype=_dtype(fmt))
        if threads is None:
            threads = os.cpu_count() or 1
        _check(self.lib.bcno_fill(out.ctypes.data, n, fmt, workers, layout, seed_index,
                                  base_offset, threads), "fill")
        return out

    def deinterleave(self, buf: np.ndarray, workers: int) -> np.ndarray:
        out = np.empty_like(buf)
        _check(self.lib.bcno_deinterleave(buf.ctypes.data, out.ctypes.data, buf.size,
                                          workers, buf.itemsize), "deinterleave")
        return out

    def digest(self, buf: np.ndarray, index_base: int = 0) -> tuple[int, int, int]:
        d = (_u64 * 3)()
        buf = np.ascontiguousarray(buf)
        self.lib.bcno_digest(buf.ctypes.data, buf.size, buf.itemsize, index_base, d)
        return d[0], d[1], d[2]


class Reference:
    """ctypes view of the reference library compiled in place (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            if os.path.isdir(REFERENCE_ROOT):
                build(reference=True)
            else:
                raise FileNotFoundError(f"{path} missing and {REFERENCE_ROOT} absent")
        lib = ctypes.CDLL(path)
        self.lib = lib
        lib.bref_modpow2.argtypes = [_u64, _u64, _pu64]
        lib.bref_seed_from_index.argtypes = [_u64, ctypes.c_int, _pu64]
        lib.bref_state_at.argtypes = [_u64, _u64, ctypes.c_int, _pu64]
        lib.bref_walk.argtypes = [_u64, _u64, ctypes.c_int, _u64, ctypes.c_void_p]
        lib.bref_step.argtypes = [_u64, ctypes.c_int, _pu64]
        lib.bref_to_unit_interval.argtypes = [_u64, ctypes.POINTER(ctypes.c_double)]
        lib.bref_make_plan.argtypes = [_u64, ctypes.c_uint, ctypes.POINTER(ctypes.c_uint), _pu64]
        lib.bref_physical_index.argtypes = [_u64, ctypes.c_uint, ctypes.c_int, ctypes.c_uint,
                                            _u64, _pu64]
        lib.bref_fill.argtypes = [ctypes.c_void_p, _u64, ctypes.c_int, _u64, ctypes.c_uint,
                                  ctypes.c_int, _u64, ctypes.c_int, _u64]
        lib.bref_deinterleave.argtypes = [ctypes.c_void_p, _u64, ctypes.c_void_p, ctypes.c_int,
                                          _u64, ctypes.c_uint, ctypes.c_int]
        pd, pi = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)
        lib.bref_chi_square.argtypes = [ctypes.c_void_p, _u64, ctypes.c_int, pd, pi]
        lib.bref_monobit.argtypes = [ctypes.c_void_p, _u64, pd, pi]
        lib.bref_serial_correlation.argtypes = [ctypes.c_void_p, _u64, ctypes.c_int, pd, pi]

    def modpow2(self, e: int, modulus: int = MODULUS) -> int:
        out = _u64()
        _check(self.lib.bref_modpow2(e, modulus, ctypes.byref(out)), "modpow2")
        return out.value

    def seed_from_index(self, a: int, method: int = BARRETT_MODIFIED) -> int:
        out = _u64()
        _check(self.lib.bref_seed_from_index(a, method, ctypes.byref(out)), "seed_from_index")
        return out.value

    def state_at(self, a: int, k: int, method: int = BARRETT_MODIFIED) -> int:
        out = _u64()
        _check(self.lib.bref_state_at(a, k, method, ctypes.byref(out)), "state_at")
        return out.value

    def walk(self, a: int, k: int, count: int, method: int = BARRETT_MODIFIED) -> np.ndarray:
        out = np.empty(count, dtype=np.uint64)
        _check(self.lib.bref_walk(a, k, method, count, out.ctypes.data), "walk")
        return out

    def step(self, z: int, method: int = BARRETT_MODIFIED) -> int:
        out = _u64()
        _check(self.lib.bref_step(z, method, ctypes.byref(out)), "step")
        return out.value

    def to_unit_interval(self, z: int) -> float:
        out = ctypes.c_double()
        _check(self.lib.bref_to_unit_interval(z, ctypes.byref(out)), "to_unit_interval")
        return out.value

    def make_plan(self, n: int, workers: int) -> tuple[int, int]:
        eff = ctypes.c_uint()
        wpw = _u64()
        _check(self.lib.bref_make_plan(n, workers, ctypes.byref(eff), ctypes.byref(wpw)),
               "make_plan")
        return eff.value, wpw.value

    def physical_index(self, n: int, workers: int, layout: int, w: int, i: int) -> int:
        out = _u64()
        _check(self.lib.bref_physical_index(n, workers, layout, w, i, ctypes.byref(out)),
               "physical_index")
        return out.value

    def fill(self, n: int, fmt: int = FMT_F64, *, seed_index: int = MIN_SEED,
             base_offset: int = 0, workers: int = 1, layout: int = CONTIGUOUS,
             method: int = BARRETT_MODIFIED, out: np.ndarray | None = None) -> np.ndarray:
        """par::fill (fmt=FMT_F64) or par::fill_residues (fmt=FMT_U64)."""
        if fmt not in (FMT_U64, FMT_F64):
            raise InvalidArgument("the reference has no f32 format")
        if out is None:
            out = np.empty(n, dtype=_dtype(fmt))
        _check(self.lib.bref_fill(out.ctypes.data, out.size, fmt, n, workers, layout,
                                  seed_index, method, base_offset), "fill")
        return out

    def chi_square(self, x: np.ndarray, bins: int) -> tuple[float, bool]:
        st, ok = ctypes.c_double(), ctypes.c_int()
        x = np.ascontiguousarray(x, dtype=np.float64)
        _check(self.lib.bref_chi_square(x.ctypes.data, x.size, bins, ctypes.byref(st), ctypes.byref(ok)),
               "chi_square")
        return st.value, bool(ok.value)

    def monobit(self, z: np.ndarray) -> tuple[float, bool]:
        st, ok = ctypes.c_double(), ctypes.c_int()
        z = np.ascontiguousarray(z, dtype=np.uint64)
        _check(self.lib.bref_monobit(z.ctypes.data, z.size, ctypes.byref(st), ctypes.byref(ok)), "monobit")
        return st.value, bool(ok.value)

    def serial_correlation(self, x: np.ndarray, lag: int = 1) -> tuple[float, bool]:
        st, ok = ctypes.c_double(), ctypes.c_int()
        x = np.ascontiguousarray(x, dtype=np.float64)
        _check(self.lib.bref_serial_correlation(x.ctypes.data, x.size, lag, ctypes.byref(st),
                                                ctypes.byref(ok)), "serial_correlation")
        return st.value, bool(ok.value)

    def deinterleave(self, buf: np.ndarray, workers: int, layout: int = INTERLEAVED) -> np.ndarray:
        fmt = FMT_U64 if buf.dtype == np.uint64 else FMT_F64
        out = np.empty_like(buf)
        _check(self.lib.bref_deinterleave(buf.ctypes.data, buf.size, out.ctypes.data, fmt,
                                          buf.size, workers, layout), "deinterleave")
        return out


def f32_rz(u: np.ndarray) -> np.ndarray:
    """RZ(double -> float) for positive normal doubles: the f32 format's
    definition. Equivalent to truncating the significand."""
    bits = np.ascontiguousarray(u, dtype=np.float64).view(np.uint64)
    exp = (bits >> np.uint64(52)) & np.uint64(0x7FF)
    f = ((exp - np.uint64(1023 - 127)) << np.uint64(23)) | ((bits >> np.uint64(29)) & np.uint64(0x7FFFFF))
    return f.astype(np.uint32).view(np.float32)
