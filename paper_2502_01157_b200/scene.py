"""Scene data model mirroring the reference's ``rfoam.foam`` / ``rfoam.geometry``.

Host-side containers only (numpy, fp64, int64 -- the reference's dtypes):

* ``FoamScene``     -- rfoam/foam.py:34-124 (positions, raw_density, sh_coeffs,
                       background, adjacency).
* ``AdjacencyGraph`` -- rfoam/geometry/adjacency.py:15-100 (CSR offsets /
                       neighbors ascending per site, bbox, diagonal,
                       ``nearest_site`` with the lowest-id tie rule).
* ``GradientBuffer`` -- rfoam/foam.py:127-150.
* ``softplus`` / ``softplus_grad`` -- rfoam/foam.py:22-31 (beta = 10).

Any object with the same attribute names (including the reference's own
classes) is accepted by the render entry points; see ``render.py``.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .errors import ShapeMismatch

SOFTPLUS_BETA = 10.0
N_SH = 16


def softplus(x, beta=SOFTPLUS_BETA):
    """(1/beta) ln(1 + exp(beta x)); same expression as foam.py:22-25."""
    x = np.asarray(x, dtype=np.float64)
    return np.maximum(x, 0.0) + np.log1p(np.exp(-np.abs(beta * x))) / beta


def softplus_grad(x, beta=SOFTPLUS_BETA):
    """logistic(beta x); foam.py:28-31."""
    x = np.asarray(x, dtype=np.float64)
    return 1.0 / (1.0 + np.exp(-beta * x))


class AdjacencyGraph:
    """Symmetric CSR site adjacency (adjacency.py:15-34).

    ``nearest_site`` is an exact brute-force query with the same squared
    distance expression and lowest-id tie rule as the reference grid query
    (adjacency.py:140-203); the device path locates start cells with a greedy
    walk on the CSR instead (``rfb_locate``).
    """

    def __init__(self, positions, offsets, neighbors, hull=None):
        self.positions = np.ascontiguousarray(positions, dtype=np.float64)
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        self.neighbors = np.ascontiguousarray(neighbors, dtype=np.int64)
        n = len(self.positions)
        if hull is None:
            hull = np.zeros(n, dtype=bool)
        self.hull = np.ascontiguousarray(hull, dtype=bool)
        if self.offsets.shape != (n + 1,) or self.offsets[-1] != len(self.neighbors):
            raise ShapeMismatch("offsets must be (n+1,) ending at len(neighbors)")
        self.bbox_lo = self.positions.min(axis=0)
        self.bbox_hi = self.positions.max(axis=0)
        self.diagonal = float(np.linalg.norm(self.bbox_hi - self.bbox_lo))

    @property
    def n_sites(self):
        return len(self.positions)

    def neighbor_list(self, i):
        return self.neighbors[self.offsets[i]: self.offsets[i + 1]]

    def degree(self, i):
        return int(self.offsets[i + 1] - self.offsets[i])

    @classmethod
    def from_lists(cls, positions, neighbor_lists, hull=None):
        """Hand-built graph, symmetrised and sorted (adjacency.py:66-83)."""
        positions = np.asarray(positions, dtype=np.float64)
        n = len(positions)
        pairs = set()
        for i, lst in enumerate(neighbor_lists):
            for j in lst:
                if i != j:
                    pairs.add((i, j))
                    pairs.add((j, i))
        arr = np.array(sorted(pairs), dtype=np.int64).reshape(-1, 2)
        offsets = np.zeros(n + 1, dtype=np.int64)
        np.add.at(offsets, arr[:, 0] + 1, 1)
        offsets = np.cumsum(offsets)
        if hull is None:
            hull = np.ones(n, dtype=bool)
        return cls(positions, offsets, arr[:, 1], hull)

    def nearest_site(self, query):
        q = np.asarray(query, dtype=np.float64)
        p = self.positions
        dx = p[:, 0] - q[0]
        dy = p[:, 1] - q[1]
        dz = p[:, 2] - q[2]
        d = dx * dx + dy * dy + dz * dz
        return int(np.argmin(d))  # first minimum == lowest id on ties


@dataclass
class FoamScene:
    positions: np.ndarray
    raw_density: np.ndarray
    sh_coeffs: np.ndarray
    background: np.ndarray = field(default_factory=lambda: np.zeros(3))
    adjacency: Optional[AdjacencyGraph] = None

    def __post_init__(self):
        self.positions = np.ascontiguousarray(self.positions, dtype=np.float64)
        self.raw_density = np.ascontiguousarray(self.raw_density, dtype=np.float64)
        self.sh_coeffs = np.ascontiguousarray(self.sh_coeffs, dtype=np.float64)
        self.background = np.asarray(self.background, dtype=np.float64)
        n = len(self.positions)
        if self.positions.shape != (n, 3):
            raise ShapeMismatch("positions must be (n, 3)")
        if self.raw_density.shape != (n,):
            raise ShapeMismatch("raw_density must be (n,)")
        if self.sh_coeffs.shape != (n, N_SH, 3):
            raise ShapeMismatch("sh_coeffs must be (n, 16, 3)")
        if self.background.shape != (3,):
            raise ShapeMismatch("background must be (3,)")

    @property
    def n_sites(self):
        return len(self.positions)

    def densities(self):
        return softplus(self.raw_density)

    def require_adjacency(self):
        if self.adjacency is None:
            raise ValueError("scene has no adjacency; Delaunay rebuild is out of scope "
                             "(build one with paper_2502_01157_b200.synthetic.delaunay_csr)")
        return self.adjacency


class GradientBuffer:
    """d(loss)/d(position, raw_density, sh) aligned to the scene (foam.py:127-150)."""

    def __init__(self, n_sites):
        self.d_position = np.zeros((n_sites, 3))
        self.d_raw_density = np.zeros(n_sites)
        self.d_sh = np.zeros((n_sites, N_SH, 3))

    def zero(self):
        self.d_position[:] = 0.0
        self.d_raw_density[:] = 0.0
        self.d_sh[:] = 0.0

    def all_finite(self):
        return bool(np.isfinite(self.d_position).all() and np.isfinite(self.d_raw_density).all()
                    and np.isfinite(self.d_sh).all())

    def add(self, other):
        self.d_position += other.d_position
        self.d_raw_density += other.d_raw_density
        self.d_sh += other.d_sh
