"""Exception taxonomy, mirroring the names in rfoam/errors.py:1-53 that the hot
path raises (trace() status mapping, shape validation)."""


class FoamError(Exception):
    """Base class for all package errors."""


class CycleDetected(FoamError):
    """Ray walk revisited a cell without advancing (status 3)."""


class StepLimit(FoamError):
    """Ray walk exceeded the hard per-ray cell cap (status 2)."""


class ShapeMismatch(FoamError):
    """Array arguments with inconsistent shapes."""


class OutOfBounds(FoamError):
    """Pixel outside the camera resolution."""


class DeviceError(FoamError):
    """A C-ABI call returned a non-zero (CUDA or argument) error code."""


class ExtensionMissing(FoamError):
    """The sm_100a extension (librfb.so) is not built or cannot be loaded."""


class DegenerateInput(FoamError):
    """Point set the Delaunay builder cannot triangulate (rfoam/errors.py:8)."""


class DuplicatePoints(FoamError):
    """Two sites within the duplicate tolerance (rfoam/errors.py:12)."""
