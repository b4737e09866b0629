"""Exception types mirroring the reference's C++ exceptions.

    std::invalid_argument -> InvalidArgument (a ValueError)
    std::out_of_range     -> OutOfRange      (an IndexError)
    std::domain_error     -> DomainError     (an ArithmeticError)
    CUDA / driver failure -> CudaError       (a RuntimeError; no reference analogue)
"""


class InvalidArgument(ValueError):
    """std::invalid_argument (parallel.cpp:36-37, :59-61, generator.cpp:18-21)."""


class OutOfRange(IndexError):
    """std::out_of_range (generator.cpp:33-35)."""


class DomainError(ArithmeticError):
    """std::domain_error (modred.hpp:71-73, :150, generator.hpp:75)."""


class CudaError(RuntimeError):
    """The device path failed (no device, launch or copy error)."""


_BY_STATUS = {1: InvalidArgument, 2: OutOfRange, 3: DomainError, 4: CudaError}


def raise_for_status(status: int, message: str) -> None:
    if status:
        raise _BY_STATUS.get(status, CudaError)(message or f"bcnrand status {status}")
