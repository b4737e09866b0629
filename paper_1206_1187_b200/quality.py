"""Host mirror of the reference quality API (include/bcnrand/quality.hpp),
computed on the GPU through the C ABI (bcn_chi_square_uniformity,
bcn_monobit_mantissa, bcn_serial_correlation). Inputs: numpy arrays or torch
tensors (CUDA tensors are read in place)."""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import InvalidArgument


@dataclass
class QualityReport:
    """quality.hpp:16-22 (`pass` is spelled `passed`: a Python keyword)."""

    name: str
    statistic: float
    dof: int
    passed: bool
    threshold: str


def _ptr(x, dtypes):
    """(pointer, count, device, stream): CUDA tensors are read in place on the
    current torch stream (so earlier torch work on them is ordered first)."""
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(x, torch.Tensor):
        if not x.is_contiguous() or str(x.dtype).replace("torch.", "") not in dtypes:
            raise InvalidArgument(f"expects a contiguous {dtypes[0]} tensor")
        if x.is_cuda:
            stream = ctypes.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)
            return x.data_ptr(), x.numel(), x.device.index, stream
        return x.data_ptr(), x.numel(), -1, None
    x = np.ascontiguousarray(x)
    if str(x.dtype) not in dtypes:
        raise InvalidArgument(f"expects {dtypes[0]} samples, got {x.dtype}")
    return x.ctypes.data, x.size, -1, None


def chi_square_uniformity(samples, bins: int) -> QualityReport:
    """quality.hpp:27 — two-sided chi-square over `bins` bins of (0,1)."""
    keep = samples if not isinstance(samples, np.ndarray) else np.ascontiguousarray(samples)
    ptr, n, dev, stream = _ptr(keep, ("float64",))
    st, dof, ok = ctypes.c_double(), ctypes.c_int(), ctypes.c_int()
    _lib.call("bcn_chi_square_uniformity", ctypes.c_void_p(ptr), n, bins, ctypes.byref(st),
              ctypes.byref(dof), ctypes.byref(ok), dev, stream)
    band = 4.5 * math.sqrt(2.0 * dof.value)
    return QualityReport("chi_square_uniformity", st.value, dof.value, bool(ok.value),
                         f"|stat - {dof.value}| <= {band:.1f}")


def monobit_mantissa(residues) -> QualityReport:
    """quality.hpp:33 — bits 5..52 of floor(z 2^53 / m)."""
    keep = residues if not isinstance(residues, np.ndarray) else np.ascontiguousarray(residues)
    ptr, n, dev, stream = _ptr(keep, ("uint64", "int64"))
    st, wb, ok = ctypes.c_double(), ctypes.c_int(), ctypes.c_int()
    _lib.call("bcn_monobit_mantissa", ctypes.c_void_p(ptr), n, ctypes.byref(st), ctypes.byref(wb),
              ctypes.byref(ok), dev, stream)
    tol = 4.5 / (2.0 * math.sqrt(n))
    return QualityReport("monobit_mantissa", st.value, 48, bool(ok.value),
                         f"max|freq-0.5| <= {tol:.3g} (worst bit {wb.value})")


def serial_correlation(samples, lag: int = 1) -> QualityReport:
    """quality.hpp:37 — Pearson correlation between samples `lag` apart."""
    keep = samples if not isinstance(samples, np.ndarray) else np.ascontiguousarray(samples)
    ptr, n, dev, stream = _ptr(keep, ("float64",))
    rho, ok = ctypes.c_double(), ctypes.c_int()
    _lib.call("bcn_serial_correlation", ctypes.c_void_p(ptr), n, lag, ctypes.byref(rho),
              ctypes.byref(ok), dev, stream)
    name = "lag1_correlation" if lag == 1 else f"lag{lag}_correlation"
    return QualityReport(name, rho.value, min(n - lag, 1 << 30), bool(ok.value),
                         f"|rho| <= {4.5 / math.sqrt(n):.3g}")


def write_table(reports) -> str:
    """quality.hpp:40 — aligned table, one row per report."""
    lines = [f"{'test':<24} {'statistic':>14} {'dof':>8} {'pass':>6}  threshold"]
    for r in reports:
        lines.append(f"{r.name:<24} {r.statistic:>14.6g} {r.dof:>8} {'yes' if r.passed else 'NO':>6}  "
                     f"{r.threshold}")
    return "\n".join(lines) + "\n"


def write_kv(reports) -> str:
    """quality.hpp:44 — name=<n> statistic=<v> dof=<d> pass=<true|false> per line."""
    return "".join(f"name={r.name} statistic={r.statistic:.17g} dof={r.dof} "
                   f"pass={'true' if r.passed else 'false'}\n" for r in reports)
