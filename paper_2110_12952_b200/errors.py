"""The reference's four error types (proj/include/nbb/errors.hpp:10-27) plus the
CUDA failure class, and the C-ABI status-code mapping (include/nbbgpu.h)."""


class NbbError(RuntimeError):
    """Base of every error raised by this package (std::runtime_error analogue)."""


class ParseError(NbbError):
    """Malformed descriptor / rule text or a descriptor invariant violation."""


class NotInFractal(NbbError):
    """An embedded coordinate inside the box that is not a fractal cell."""


class OutOfDomain(NbbError):
    """A coordinate or parameter outside its domain."""


class CapacityError(NbbError):
    """Integer overflow or a memory-cap violation (device OOM included)."""


class CudaError(NbbError):
    """A CUDA runtime / driver failure inside the engine (std::runtime_error)."""


# NBBGPU_* status codes (include/nbbgpu.h) -> exception class
STATUS_TO_ERROR = {
    1: ParseError,
    2: NotInFractal,
    3: OutOfDomain,
    4: CapacityError,
    5: CudaError,
    6: NbbError,  # NBBGPU_ERR_INVALID (bad handle / argument)
}
