"""Host mirror of the reference generator API (include/bcnrand/generator.hpp).

Same names, argument meaning and error behaviour as ``bcn::gen``; every call
goes through the C ABI (libbcnrand_b200.so). These are the scalar host
entry points (seed-by-index, skip-ahead, next, conversion); the array fill is
:func:`paper_1206_1187_b200.parallel.fill`, which runs on the GPU.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass

from . import _lib
from .errors import DomainError, InvalidArgument, OutOfRange

kModulus = 5559060566555523           # modred.hpp:22
kMinSeedIndex = kModulus + 100         # generator.hpp:19
kMaxSeedIndex = 1 << 53                # generator.hpp:20
kPeriod = 3706040377703682             # generator.hpp:21 (2 * 3^32)
kInvModulus = 1.0 / 5559060566555523.0 # generator.hpp:22


class Method(enum.IntEnum):
    """generator.hpp:17 — all methods produce identical bits."""

    Ref128 = 0
    LEcuyer = 1
    Barrett = 2
    BarrettModified = 3


def method_name(m: Method) -> str:
    """generator.cpp:51-59"""
    return Method(m).name


def parse_method(name: str) -> Method:
    """generator.cpp:61-70 (case-insensitive; unknown -> InvalidArgument)."""
    for m in Method:
        if m.name.lower() == name.lower():
            return m
    raise InvalidArgument(f"unknown method: {name}")


@dataclass
class GeneratorState:
    """generator.hpp:24-29"""

    seed_index: int = 0
    z: int = 0
    k: int = 0
    method: Method = Method.BarrettModified


_U64 = 1 << 64


def check_u64(x: int, what: str, exc=InvalidArgument) -> int:
    """The reference takes std::uint64_t here: a Python int outside [0, 2^64)
    raises `exc` instead of being truncated by ctypes."""
    if not 0 <= int(x) < _U64:
        raise exc(f"{what}: {x} is not a 64-bit unsigned value")
    return int(x)


def modpow2(exponent: int, modulus: int) -> int:
    """generator.hpp:33 — 2^e mod modulus (odd, < 2^63)."""
    check_u64(exponent, "modpow2")
    check_u64(modulus, "modpow2")
    out = ctypes.c_uint64()
    _lib.call("bcn_modpow2", exponent, modulus, ctypes.byref(out))
    return out.value


def seed_from_index(a: int, method: Method = Method.BarrettModified) -> GeneratorState:
    """generator.hpp:37 — rejects a outside [3^33+100, 2^53] with OutOfRange."""
    check_u64(a, "seed_from_index", OutOfRange)
    out = ctypes.c_uint64()
    _lib.call("bcn_seed_from_index", a, ctypes.byref(out))
    return GeneratorState(a, out.value, 0, Method(method))


def state_at(a: int, k: int, method: Method = Method.BarrettModified) -> GeneratorState:
    """generator.hpp:42-43 — state after k steps, O(log k). k is taken mod 2^64
    like the reference's std::uint64_t."""
    check_u64(a, "state_at", OutOfRange)
    out = ctypes.c_uint64()
    _lib.call("bcn_state_at", a, k & 0xFFFFFFFFFFFFFFFF, ctypes.byref(out))
    return GeneratorState(a, out.value, k, Method(method))


def next(state: GeneratorState) -> int:  # noqa: A001 - mirrors bcn::gen::next
    """generator.hpp:52-70 — advance one step, return the new residue. Every
    method gives the same residue; z = 0 is rejected (DomainError) by the
    modified Barrett step alone (modred.hpp:150) and maps to 0 otherwise."""
    check_u64(state.z, "next", DomainError)
    if state.z == 0 and Method(state.method) != Method.BarrettModified:
        state.k += 1
        return 0
    z = ctypes.c_uint64(state.z)
    _lib.call("bcn_next", ctypes.byref(z))
    state.z = z.value
    state.k += 1
    return state.z


def to_unit_interval(z: int) -> float:
    """generator.hpp:74-78 — double(z) * kInvModulus; z = 0 -> DomainError."""
    check_u64(z, "to_unit_interval", DomainError)
    out = ctypes.c_double()
    _lib.call("bcn_to_unit_interval", z, ctypes.byref(out))
    return out.value
