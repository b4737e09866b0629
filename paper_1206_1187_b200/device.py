"""Device-side entry points beyond the reference API (all via the C ABI).

* :func:`seed_states` — batched skip-ahead seeding kernel.
* :func:`digest` — order-sensitive checksums of a device buffer.
* :func:`fill_constant` — the Constant writer, the write-roofline denominator.
* :func:`fill_noise` — the Constant writer with random data (power-realistic ceiling).
* :func:`fill_multi` — one-process multi-GPU fill over contiguous shards.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from .errors import InvalidArgument
from .generator import kMinSeedIndex
from .parallel import Engine, Format


def _cuda(t: torch.Tensor, what: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda or not t.is_contiguous():
        raise InvalidArgument(f"{what}: expects a contiguous CUDA tensor")
    return t


def _stream(t: torch.Tensor, stream=None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream(t.device)
    return ctypes.c_void_p(int(getattr(s, "cuda_stream", s)))


def seed_states(a: torch.Tensor, k: torch.Tensor, steps: int = 0, stream=None) -> torch.Tensor:
    """state_at(a[t], k[t]) for every t (steps = 0), or the `steps` next()
    residues after it (shape [count, steps]). a, k: int64/uint64 CUDA tensors
    holding u64 values. Synchronous (reports out-of-range seeds)."""
    _cuda(a, "seed_states")
    _cuda(k, "seed_states")
    if a.numel() != k.numel() or a.element_size() != 8 or k.element_size() != 8:
        raise InvalidArgument("seed_states: a and k must be equal-length 64-bit tensors")
    count = a.numel()
    shape = (count,) if steps == 0 else (count, steps)
    out = torch.empty(shape, dtype=torch.int64, device=a.device)
    _lib.call("bcn_seed_states", ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(k.data_ptr()),
              ctypes.c_void_p(out.data_ptr()), count, steps, a.device.index, _stream(a, stream))
    return out


def engine_check(engine: Engine, z, c, chain: int = 1, device: int = 0):
    """z[i] * c[i]^chain mod 3^33 through one jump engine on the GPU
    (bcn_engine_check): a self-check of the engine arithmetic over arbitrary
    residues and multipliers. z, c: uint64 numpy arrays; returns uint64."""
    import numpy as np

    z = np.ascontiguousarray(z, dtype=np.uint64)
    c = np.ascontiguousarray(c, dtype=np.uint64)
    if z.shape != c.shape:
        raise InvalidArgument("engine_check: z and c must have the same shape")
    out = np.empty_like(z)
    _lib.call("bcn_engine_check", int(engine), ctypes.c_void_p(z.ctypes.data), ctypes.c_void_p(c.ctypes.data),
              ctypes.c_void_p(out.ctypes.data), z.size, chain, device)
    return out


def digest(buf: torch.Tensor, index_base: int = 0, stream=None) -> tuple[int, int, int]:
    """(sum x, sum (index_base+i+1) x, xor x (2(index_base+i)+1)) mod 2^64 over
    the raw 4- or 8-byte items of a CUDA tensor."""
    _cuda(buf, "digest")
    d = (ctypes.c_uint64 * 3)()
    _lib.call("bcn_digest", ctypes.c_void_p(buf.data_ptr()), buf.numel(), buf.element_size(),
              index_base, d, buf.device.index, _stream(buf, stream))
    return d[0], d[1], d[2]


def fill_constant(buf: torch.Tensor, pattern: int = 0x3FE0000000000000, stream=None) -> None:
    """Write a fixed 8-byte pattern (default 0.5) with the fill's access pattern.
    Asynchronous on the current torch stream."""
    _cuda(buf, "fill_constant")
    _lib.call("bcn_fill_constant", ctypes.c_void_p(buf.data_ptr()), buf.numel() * buf.element_size(),
              pattern, buf.device.index, _stream(buf, stream))


def fill_noise(buf: torch.Tensor, seed: int = 0x1206_1187, stream=None) -> None:
    """The Constant writer writing fixed per-thread pseudo-random words (the
    power-realistic write ceiling). Asynchronous on the current torch stream."""
    _cuda(buf, "fill_noise")
    _lib.call("bcn_fill_noise", ctypes.c_void_p(buf.data_ptr()), buf.numel() * buf.element_size(),
              seed, buf.device.index, _stream(buf, stream))


def fill_multi(outs: list[torch.Tensor], n: int, seed_index: int = kMinSeedIndex,
               base_offset: int = 0, fmt: Format = Format.F64,
               engine: Engine = Engine.Auto, streams=None) -> None:
    """Contiguous shards of make_plan(n, len(outs)) on each tensor's device; the
    concatenation equals a single fill of n items. Each shard is ordered after
    the work already queued on its device's current torch stream (or on
    `streams[g]`). Synchronous."""
    from .parallel import _FMT_DTYPES

    ndev = len(outs)
    if ndev == 0:
        raise InvalidArgument("fill_multi: no devices")
    for t in outs:
        _cuda(t, "fill_multi")
        dt = str(t.dtype).replace("torch.", "")
        if dt not in _FMT_DTYPES[Format(fmt)]:
            raise InvalidArgument(f"fill_multi: {Format(fmt).name} shards need dtype "
                                  f"{_FMT_DTYPES[Format(fmt)][0]}, got {dt}")
    ptrs = (ctypes.c_void_p * ndev)(*[t.data_ptr() for t in outs])
    caps = (ctypes.c_uint64 * ndev)(*[t.numel() for t in outs])
    devs = (ctypes.c_int * ndev)(*[t.device.index for t in outs])
    if streams is None:
        streams = [torch.cuda.current_stream(t.device) for t in outs]
    strs = (ctypes.c_void_p * ndev)(*[int(getattr(s, "cuda_stream", s)) for s in streams])
    _lib.call("bcn_fill_multi", ptrs, caps, devs, ndev, n, int(fmt), seed_index,
              base_offset & 0xFFFFFFFFFFFFFFFF, int(engine), strs)


def set_launch_config(ctas_per_sm: int = 0, row_order: int = 1) -> None:
    """Process-wide CTAs-per-SM / row-order tuning of the contiguous kernels
    (bits never change; see bcn_set_launch_config)."""
    _lib.call("bcn_set_launch_config", ctas_per_sm, row_order)


def set_write_pacing(target_gbs: float, ctas_per_sm: int = 1, format_mask: int = 3) -> None:
    """Meter the contiguous fill / Constant stores to `target_gbs` per device:
    < 0 automatic (each device's calibrated target, the default), 0 unpaced,
    else a fixed target >= 100, for the formats in `format_mask` (bit = Format
    value); see bcn_set_write_pacing."""
    _lib.call("bcn_set_write_pacing", float(target_gbs), ctas_per_sm, format_mask)


def write_pacing() -> float:
    """The pacing setting (< 0 automatic, 0 unpaced, else GB/s)."""
    return float(_lib.lib().bcn_write_pacing())


PACE_SOURCES = {0: "unpaced", 1: "user", 2: "calibrated", 3: "default"}


def device_write_pacing(device: int = 0) -> tuple[float, str]:
    """(effective target GB/s, source) of `device`: 'calibrated' by this
    process's sweep at context init, 'user' (set_write_pacing), 'default'
    (BCN_PACE_CALIBRATE=0) or 'unpaced'."""
    g, src = ctypes.c_double(), ctypes.c_int()
    _lib.call("bcn_device_write_pacing", device, ctypes.byref(g), ctypes.byref(src))
    return g.value, PACE_SOURCES.get(src.value, "?")


def pacing_source(device: int = 0) -> str:
    return device_write_pacing(device)[1]


def pace_calibration(device: int = 0) -> list[tuple[float, float]]:
    """(target, achieved) GB/s points of `device`'s calibration sweep."""
    t, a, n = (ctypes.c_double * 64)(), (ctypes.c_double * 64)(), ctypes.c_int()
    _lib.call("bcn_pace_calibration", device, t, a, 64, ctypes.byref(n))
    return [(t[i], a[i]) for i in range(min(n.value, 64))]


def write_pacing_config() -> tuple[float, int, int]:
    """(target GB/s, CTAs per SM, format mask) of the current write pacing."""
    g, c, m = ctypes.c_double(), ctypes.c_int(), ctypes.c_int()
    _lib.lib().bcn_get_write_pacing(ctypes.byref(g), ctypes.byref(c), ctypes.byref(m))
    return g.value, c.value, m.value


def auto_engine(fmt: Format = Format.F64) -> Engine:
    return Engine(_lib.lib().bcn_auto_engine(int(fmt)))


def device_count() -> int:
    return _lib.lib().bcn_device_count()
