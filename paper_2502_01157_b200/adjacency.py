"""Delaunay adjacency rebuilt on the GPU.

Mirrors the reference's ``rfoam.geometry.build`` (delaunay.py:445-520) +
``AdjacencyGraph.from_triangulation`` (adjacency.py:46-64): the same
validation and errors, and the same product -- a symmetric CSR with
ascending neighbour ids plus hull flags.  The construction is
``rfb_build_adjacency`` in librfb.so (per-site Voronoi cell clipping, one
warp per site; see csrc/rfb_adjacency.cu and DESIGN.md §4.4).

  build_device(positions)  device fp64 [n,3] -> device CSR (int64), hull, stats
  build(points)            host numpy in, scene.AdjacencyGraph out
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import DegenerateInput, DeviceError, DuplicatePoints
from .scene import AdjacencyGraph

MAX_DEGREE = 128


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def build_device(positions: torch.Tensor, max_degree: int = MAX_DEGREE, stream=None):
    """Device Delaunay CSR of `positions` (CUDA fp64 [n, 3]).

    Returns (offsets int64 [n+1], neighbors int64 [E], hull bool [n], stats)
    on the positions' device.  Raises DuplicatePoints / DegenerateInput like
    delaunay.build."""
    lib = _lib.load()
    pos = positions.to(torch.float64).contiguous()
    if pos.dim() != 2 or pos.shape[1] != 3:
        raise DegenerateInput("expected an (n, 3) point array")
    n = pos.shape[0]
    if n < 4:
        raise DegenerateInput("need at least 4 points")
    dev = pos.device
    st = ctypes.c_void_p((stream or torch.cuda.current_stream(dev)).cuda_stream)
    with torch.cuda.device(dev):
        ws = torch.empty(int(lib.rfb_adjacency_workspace_bytes(n, max_degree)), dtype=torch.uint8,
                         device=dev)
        offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
        stats = (ctypes.c_int64 * 8)()
        code = lib.rfb_build_adjacency(_ptr(pos), n, max_degree, _ptr(offsets), None, 0, None,
                                       stats, _ptr(ws), ws.numel(), st)
        if code == -3:  # RFB_EDEGENERATE
            if not torch.isfinite(pos).all():
                raise DegenerateInput("non-finite coordinates")
            if int(stats[7]) & 2:
                raise DuplicatePoints("sites within duplicate tolerance "
                                      f"{1e-7 * _diag(pos):g}")
            raise DegenerateInput("degenerate configuration (coplanar cell faces)")
        if code == -2:
            raise DeviceError(f"rfb_build_adjacency: capacity exceeded (flags {int(stats[7])}, "
                              f"max vertices {int(stats[3])}, max planes {int(stats[4])})")
        _lib.check(code, "rfb_build_adjacency")
        E = int(stats[0])
        neighbors = torch.empty(max(E, 1), dtype=torch.int64, device=dev)
        hull = torch.empty(n, dtype=torch.uint8, device=dev)
        _lib.check(lib.rfb_adjacency_emit(n, max_degree, _ptr(offsets), _ptr(neighbors),
                                          _ptr(hull), _ptr(ws), ws.numel(), st),
                   "rfb_adjacency_emit")
    if bool(hull.all()) and _coplanar(pos):
        raise DegenerateInput("all points collinear or coplanar")  # delaunay.py:494-495
    info = {"edges": E, "reverse_edges_added": int(stats[1]), "pass2_sites": int(stats[2]),
            "max_cell_vertices": int(stats[3]), "max_cell_planes": int(stats[4]),
            "clip_tests_spiral": int(stats[5]), "clip_tests_rings": int(stats[6])}
    return offsets, neighbors[:E], hull.bool(), info


def _coplanar(pos: torch.Tensor) -> bool:
    """Every site on one plane (checked only when every cell is unbounded):
    fp64 orientation of all sites against three spread-out ones is exactly 0."""
    p = pos - pos[0]
    a = p[int(torch.argmax((p * p).sum(1)))]
    c = torch.linalg.cross(p, a.expand_as(p))
    b = p[int(torch.argmax((c * c).sum(1)))]
    normal = torch.linalg.cross(a, b)
    if not bool(torch.any(normal != 0)):
        return True  # collinear
    return not bool(torch.any(p @ normal != 0))


def _diag(pos: torch.Tensor) -> float:
    return float(torch.linalg.norm(pos.max(0).values - pos.min(0).values))


def build(points, ids=None, dup_tol=None) -> AdjacencyGraph:
    """delaunay.build + AdjacencyGraph.from_triangulation with the
    construction on the current CUDA device.  ``ids`` must be 0..n-1 here
    (from_triangulation's contiguous-id rule); dup_tol other than the default
    1e-7 x diagonal is not supported by the device builder."""
    pts = np.ascontiguousarray(np.asarray(points, dtype=np.float64))
    if pts.ndim != 2 or pts.shape[1] != 3:
        raise DegenerateInput("expected an (n, 3) point array")
    if not np.isfinite(pts).all():
        raise DegenerateInput("non-finite coordinates")
    n = len(pts)
    if ids is not None and not np.array_equal(np.asarray(ids), np.arange(n)):
        raise ValueError("adjacency extraction needs contiguous site ids")
    if dup_tol is not None:
        raise ValueError("the device builder uses the reference's default duplicate tolerance")
    if n < 4:
        raise DegenerateInput("need at least 4 points")
    if not torch.cuda.is_available():
        raise DeviceError("build_device needs a CUDA device")
    off, nbr, hull, _ = build_device(torch.from_numpy(pts).cuda())
    return AdjacencyGraph(pts, off.cpu().numpy(), nbr.cpu().numpy(), hull.cpu().numpy())
