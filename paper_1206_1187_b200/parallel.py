"""Host mirror of the reference parallel API (include/bcnrand/parallel.hpp).

``make_plan`` / ``PartitionPlan`` / ``fill`` / ``fill_residues`` /
``deinterleave`` keep the reference names, argument meaning and exceptions.
The difference is where the work runs: ``fill`` launches the sm_100a kernels
through the C ABI. ``out`` may be

* a CUDA ``torch.Tensor`` — filled in place, asynchronously on the tensor
  device's current torch stream (pass ``stream=`` to override, or
  ``sync=True`` to block like the reference);
* a host ``numpy.ndarray`` or CPU tensor — generated on the GPU and copied
  back in chunks; synchronous, like the reference's ``std::span`` fill.

The plan's worker count only matters for the Interleaved layout and for the
reference's exact u64 wrap of ``base_offset + start_w``; the GPU's own
parallelism is independent of it.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import InvalidArgument
from .generator import Method


class Layout(enum.IntEnum):
    """parallel.hpp:15"""

    Contiguous = 0
    Interleaved = 1


class Format(enum.IntEnum):
    """Output item formats of the C ABI (bcn_format)."""

    U64 = 0
    F64 = 1
    F32 = 2


class Engine(enum.IntEnum):
    """Device reduction engine (bcn_engine). Auto = the measured best."""

    Auto = 0
    Barrett = 1
    Montgomery = 2
    FP64 = 3
    Staged = 4
    Bulk = 5
    Mixed = 6
    Hybrid = 7


def layout_name(layout: Layout) -> str:
    return "contiguous" if layout == Layout.Contiguous else "interleaved"


def parse_layout(name: str) -> Layout:
    if name == "contiguous":
        return Layout.Contiguous
    if name == "interleaved":
        return Layout.Interleaved
    raise InvalidArgument(f"unknown layout: {name}")


@dataclass
class PartitionPlan:
    """parallel.hpp:17-38"""

    n: int = 0
    workers: int = 1
    work_per_worker: int = 0
    start_offsets: list[int] = field(default_factory=list)
    layout: Layout = Layout.Contiguous
    step: int = 1

    def elements_for(self, w: int) -> int:
        """parallel.cpp:19-22"""
        return min(self.work_per_worker, self.n - self.start_offsets[w])

    def physical_index(self, w: int, i: int) -> int:
        """parallel.cpp:24-33 (through the C ABI)."""
        out = ctypes.c_uint64()
        _lib.call("bcn_physical_index", self.n, self.workers, int(self.layout), w, i,
                  ctypes.byref(out))
        return out.value


def make_plan(n: int, workers: int, layout: Layout = Layout.Contiguous) -> PartitionPlan:
    """parallel.hpp:42 — n = 0 or workers = 0 -> InvalidArgument."""
    if n < 0 or workers < 0 or workers >= 1 << 32:
        raise InvalidArgument("make_plan: n and workers must be non-negative")
    eff = ctypes.c_uint32()
    wpw = ctypes.c_uint64()
    _lib.call("bcn_make_plan", n, workers, ctypes.byref(eff), ctypes.byref(wpw))
    return PartitionPlan(n, eff.value, wpw.value, [w * wpw.value for w in range(eff.value)],
                         Layout(layout), eff.value)


_FMT_DTYPES = {
    Format.U64: ("uint64", "int64"),
    Format.F64: ("float64",),
    Format.F32: ("float32",),
}


def _buffer(out):
    """(pointer, capacity in items, dtype name, is_cuda, device, torch tensor or None)."""
    try:
        import torch
    except ImportError:  # pragma: no cover - torch is part of the image
        torch = None
    if torch is not None and isinstance(out, torch.Tensor):
        if not out.is_contiguous():
            raise InvalidArgument("fill: output tensor must be contiguous")
        dt = str(out.dtype).replace("torch.", "")
        dev = out.device.index if out.is_cuda else -1
        return out.data_ptr(), out.numel(), dt, out.is_cuda, dev, out
    if isinstance(out, np.ndarray):
        if not out.flags.c_contiguous:
            raise InvalidArgument("fill: output array must be C-contiguous")
        return out.ctypes.data, out.size, str(out.dtype), False, -1, None
    raise InvalidArgument("fill: out must be a torch.Tensor or numpy.ndarray")


def _stream_for(tensor, stream):
    if stream is not None:
        return ctypes.c_void_p(int(getattr(stream, "cuda_stream", stream)))
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream(tensor.device).cuda_stream)


def fill_format(out, plan: PartitionPlan, seed_index: int, method: Method, base_offset: int,
                fmt: Format, *, engine: Engine = Engine.Auto, stream=None,
                sync: bool = False) -> None:
    """Common body of fill / fill_residues / fill_float (parallel.cpp:56-79)."""
    from .generator import OutOfRange, check_u64

    check_u64(plan.n, "fill")
    check_u64(seed_index, "seed_from_index", OutOfRange)
    ptr, cap, dt, is_cuda, dev, tensor = _buffer(out)
    if dt not in _FMT_DTYPES[Format(fmt)]:
        raise InvalidArgument(f"fill: {Format(fmt).name} output needs dtype {_FMT_DTYPES[Format(fmt)][0]}, got {dt}")
    s = _stream_for(tensor, stream) if is_cuda else ctypes.c_void_p(0)
    _lib.call("bcn_fill", ctypes.c_void_p(ptr), cap, plan.n, int(fmt), plan.workers,
              int(plan.layout), seed_index, int(method), base_offset & 0xFFFFFFFFFFFFFFFF,
              int(engine), dev, s)
    if is_cuda and sync:
        import torch

        torch.cuda.synchronize(tensor.device)


def fill(out, plan: PartitionPlan, seed_index: int, method: Method = Method.BarrettModified,
         base_offset: int = 0, **kw) -> None:
    """parallel.hpp:48-49 — plan.n unit-interval doubles (float64 buffer)."""
    fill_format(out, plan, seed_index, method, base_offset, Format.F64, **kw)


def fill_residues(out, plan: PartitionPlan, seed_index: int,
                  method: Method = Method.BarrettModified, base_offset: int = 0, **kw) -> None:
    """parallel.hpp:52-54 — raw residues z_k (uint64/int64 buffer)."""
    fill_format(out, plan, seed_index, method, base_offset, Format.U64, **kw)


def fill_float(out, plan: PartitionPlan, seed_index: int,
               method: Method = Method.BarrettModified, base_offset: int = 0, **kw) -> None:
    """Extension: float32 variates, RZ(to_unit_interval(z))."""
    fill_format(out, plan, seed_index, method, base_offset, Format.F32, **kw)


def deinterleave(buffer, plan: PartitionPlan, *, stream=None):
    """parallel.hpp:58-60 — logical order of an Interleaved buffer (new array)."""
    if plan.layout != Layout.Interleaved:
        raise InvalidArgument("deinterleave: plan layout is not Interleaved")
    ptr, cap, dt, is_cuda, dev, tensor = _buffer(buffer)
    if cap < plan.n:
        raise InvalidArgument("deinterleave: buffer smaller than plan.n")
    itemsize = 4 if dt in ("float32", "int32", "uint32") else 8
    if is_cuda:
        import torch

        out = torch.empty(plan.n, dtype=tensor.dtype, device=tensor.device)
        s = _stream_for(tensor, stream)
        optr = out.data_ptr()
    elif tensor is not None:
        import torch

        out = torch.empty(plan.n, dtype=tensor.dtype)
        s, optr = ctypes.c_void_p(0), out.data_ptr()
    else:
        out = np.empty(plan.n, dtype=buffer.dtype)
        s, optr = ctypes.c_void_p(0), out.ctypes.data
    _lib.call("bcn_deinterleave", ctypes.c_void_p(ptr), ctypes.c_void_p(optr), plan.n,
              plan.workers, itemsize, dev, s)
    return out
