"""B200-native Radiant Foam hot path (arXiv 2502.01157).

Per-ray Voronoi-foam traversal with differentiable volume rendering, forward
and backward, as hand-written sm_100a CUDA kernels behind a C ABI
(include/rfb.h, librfb.so), with Python entry points that mirror the
reference's (rfoam.diffrender.render / rfoam.tracer.kernels).

Heavy modules (torch, the CUDA library) are imported lazily so the CPU-only
pieces (scene containers, camera math, fixtures) work without a GPU.
"""

from .camera import FISHEYE, PINHOLE, CameraModel, camera_rays, look_at, orbit_poses
from .errors import (CycleDetected, DeviceError, ExtensionMissing, FoamError, OutOfBounds,
                     ShapeMismatch, StepLimit)
from .scene import AdjacencyGraph, FoamScene, GradientBuffer, softplus, softplus_grad

__all__ = [
    "AdjacencyGraph", "CameraModel", "CycleDetected", "DeviceError", "ExtensionMissing",
    "FISHEYE", "FoamError", "FoamScene", "GradientBuffer", "OutOfBounds", "PINHOLE",
    "ShapeMismatch", "StepLimit", "camera_rays", "look_at", "orbit_poses", "softplus",
    "softplus_grad",
]

__version__ = "0.1.0"
