"""Error hierarchy mirroring qblock's (errors.hpp:24-81); raised from C-ABI return codes."""


class Error(RuntimeError):
    """Base class of every error raised by this library (qblock::Error)."""


class ValidationError(Error):
    """Bad argument values (overlapping qubits, wrong vector length, ...)."""


class ShapeError(Error):
    """Mismatched matrix/register dimensions."""


class RangeError(Error):
    """Index outside its documented range."""


class DispatchError(Error):
    """Unknown gate tag or unregistered gate name."""


class ResourceError(Error):
    """Request exceeds the configured qubit/memory cap."""


class UnsupportedError(Error):
    """Operation not defined for this node kind."""


class UndecidableError(Error):
    """A property query that cannot be decided at this size."""


class RenormalizationError(Error):
    """Projection onto a numerically zero-probability subspace."""


class SerializationError(Error):
    """Bad state file / no text form."""


class ParseError(Error):
    """Script syntax failure."""


class CudaError(Error):
    """CUDA runtime failure (no reference counterpart; the engine has no CPU fallback)."""


class NcclError(Error):
    """NCCL failure."""
