"""Exception taxonomy of the hot path.

Same class names and meanings as the reference (reference
pkg/src/voxpar/errors.py:4-77) so callers catching e.g. NonDivisible keep
working; the C ABI's negative status codes map 1:1 onto these
(include/vpx.h, `_lib._STATUS`).  Two additions cover failure modes the
CPU reference cannot have: Unsupported (a shape the sm_100a kernels do not
implement) and DeviceError (a CUDA / NCCL failure).
"""


class VoxparError(Exception):
    """Base class for all errors raised by this package."""


class NonDivisible(VoxparError):
    """A spatial extent does not divide evenly over its partition count."""


class BatchIndivisible(VoxparError):
    """Mini-batch size N is not divisible by the group count G."""


class OutOfBounds(VoxparError):
    """A region, rank or index lies outside its domain."""


class ShapeMismatch(VoxparError):
    """Array/buffer shapes are inconsistent with the operation's contract."""


class LengthMismatch(VoxparError):
    """Collective participants disagree on vector length."""


class UnsupportedWidth(VoxparError):
    """Requested network input width is outside the supported set."""


class ConfigError(VoxparError):
    """Run configuration failed validation."""


class Unsupported(VoxparError):
    """The requested shape is outside what the sm_100a kernels implement."""


class DeviceError(VoxparError):
    """A CUDA runtime/driver or NCCL call failed."""


class IoError(VoxparError):
    """Sample file / manifest could not be read or is malformed."""


class BadMagic(IoError):
    """HSB1 magic mismatch."""


class BadVersion(IoError):
    """Unsupported HSB1 version."""


class CacheNotEmpty(VoxparError):
    """ingest_epoch0 on an already populated cache."""


class MissingSample(VoxparError):
    """A scheduled sample has no owner / cached slab."""


class BadBatch(VoxparError):
    """Batch / group / dataset sizes that cannot form a schedule."""


class InsufficientData(VoxparError):
    """Too few samples for a performance-model fit."""


class DegenerateFit(VoxparError):
    """A performance-model fit has no spread in its inputs (or a negative slope)."""


class NoComparableEntry(VoxparError):
    """The kernel-time table has no row of the requested kind/phase."""
