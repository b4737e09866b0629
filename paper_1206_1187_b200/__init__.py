"""B200-native alpha_{2,3} normal-number generator (arXiv 1206.1187).

A drop-in for the reference's generator fill path (``bcn::gen`` /
``bcn::par``): seed-by-index, O(log k) skip-ahead and fill-array of raw u64
residues, doubles or floats, computed by sm_100a kernels behind the C ABI in
``include/bcnrand_b200.h``. Modules mirror the reference headers:

* :mod:`.generator` — generator.hpp (``seed_from_index``, ``state_at``, ``next`` …)
* :mod:`.parallel`  — parallel.hpp (``make_plan``, ``fill``, ``fill_residues`` …)
* :mod:`.device`    — device-only extras (seeding kernel, digests, Constant writer,
  multi-GPU fill)
"""
from . import device
from . import generator as gen
from . import parallel as par
from . import quality
from .errors import CudaError, DomainError, InvalidArgument, OutOfRange
from .generator import (GeneratorState, Method, kInvModulus, kMaxSeedIndex, kMinSeedIndex,
                        kModulus, kPeriod)
from .parallel import Engine, Format, Layout, PartitionPlan

__all__ = [
    "gen", "par", "device", "quality", "CudaError", "DomainError", "InvalidArgument", "OutOfRange",
    "GeneratorState", "Method", "Layout", "Format", "Engine", "PartitionPlan",
    "kModulus", "kMinSeedIndex", "kMaxSeedIndex", "kPeriod", "kInvModulus",
]
