"""Exception types of the drop-in API.

Names and meanings mirror the reference package's error hierarchy
(``corridor/errors.py:4-64``) so callers catching the reference's exceptions
catch ours. The native library never throws across the C ABI; it returns an
``EZ_*`` status code (``include/corridor_b200.h``) which
:func:`raise_for_status` maps back onto these classes.
"""

from __future__ import annotations


class CorridorError(Exception):
    """Root of every error raised by this package."""


class DimensionMismatch(CorridorError):
    """Vectors or matrices of incompatible dimension were combined."""


class EmptyChord(CorridorError):
    """A hit-and-run step found an empty feasible chord (degenerate polytope)."""


class SeedOutside(CorridorError):
    """A hit-and-run walk was started outside its polytope."""


class GradientUndefined(CorridorError):
    """The distance-to-segment gradient was requested on the segment itself."""


class SegmentInCollision(CorridorError):
    """The seed segment collides, or lies within ``t_col`` of an obstacle."""


class SeedOutsideDomain(CorridorError):
    """The seed segment is not strictly inside the domain polytope."""


class SamplingExhausted(CorridorError):
    """Rejection sampling ran out of budget."""


class GridMismatch(CorridorError):
    """A voxel map cannot be used with the roadmap's grid."""


class NativeError(CorridorError):
    """CUDA / driver failure inside the native library, or the library is missing."""


# Status codes returned by every ``ez_*`` entry point (include/corridor_b200.h).
EZ_OK = 0
EZ_DIMENSION_MISMATCH = 1
EZ_EMPTY_CHORD = 2
EZ_SEED_OUTSIDE = 3
EZ_GRADIENT_UNDEFINED = 4
EZ_SEGMENT_IN_COLLISION = 5
EZ_SEED_OUTSIDE_DOMAIN = 6
EZ_GRID_MISMATCH = 7
EZ_INVALID_ARGUMENT = 8
EZ_CUDA_ERROR = 9
EZ_UNSUPPORTED = 10
EZ_CAPACITY = 11

_STATUS_TO_EXC = {
    EZ_DIMENSION_MISMATCH: DimensionMismatch,
    EZ_EMPTY_CHORD: EmptyChord,
    EZ_SEED_OUTSIDE: SeedOutside,
    EZ_GRADIENT_UNDEFINED: GradientUndefined,
    EZ_SEGMENT_IN_COLLISION: SegmentInCollision,
    EZ_SEED_OUTSIDE_DOMAIN: SeedOutsideDomain,
    EZ_GRID_MISMATCH: GridMismatch,
    EZ_INVALID_ARGUMENT: ValueError,
    EZ_CUDA_ERROR: NativeError,
    EZ_UNSUPPORTED: NotImplementedError,
    EZ_CAPACITY: NativeError,
}


def raise_for_status(status: int, message: str = "") -> None:
    """Raise the exception class bound to a native status code (no-op for EZ_OK)."""
    if status == EZ_OK:
        return
    exc = _STATUS_TO_EXC.get(status, NativeError)
    raise exc(message or f"native status {status}")
