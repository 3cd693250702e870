"""Device-resident scene and the torch-level calls into librfb.so.

PyTorch is plumbing here: it owns device memory and streams; all compute is
in the sm_100a kernels behind the C ABI (include/rfb.h).  Layout in HBM
(DESIGN.md §3):

* ``site4``    float64 [n, 4]  x, y, z, sigma  -- one 32-byte record per site,
                                the only per-neighbour gather of the walk;
* ``offsets``  int32 [n+1], ``neighbors`` int32 [E]  -- the reference CSR
                                (ascending per site), narrowed from int64;
* ``sh``       float64 [n, 48] -- index k*3+ch as render.py:53;
* gradients    float32 [n, 52] -- ``[n,4]`` (dpos xyz, dsigma) then ``[n,48]``
                                (dSH); one flat buffer so a single NCCL
                                all-reduce covers it.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .scene import softplus

DEFAULT_EPSILON = 1e-3     # tracer/rays.py:12
DEFAULT_STEP_LIMIT = 4096  # tracer/rays.py:13
WIDTH_FLOOR_SCALE = 1e-12  # tracer/rays.py:14
DEFAULT_LANES = 0  # auto (rfb.h: rfb_params.lanes_per_ray)
# forward workspace: 256 bytes + room for the per-SM work counters (rfb.h rfb_render_rays)
FWD_WORKSPACE_BYTES = 4096


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class _Uploader:
    """Host -> device copies of large numpy arrays through a reusable pinned staging
    ring: the host side fills one chunk with several threads (numpy releases the GIL)
    while the previous chunk's DMA runs, instead of torch's single-threaded pageable
    copy (~10 GB/s for the 548 MB of a 1M-site scene)."""

    CHUNK = int(os.environ.get("RFB_UPLOAD_CHUNK_MB", "32")) << 20
    RING = 3
    THREADS = int(os.environ.get("RFB_UPLOAD_THREADS", "8"))

    def __init__(self):
        self.bufs = None
        self.events = None
        self.pool = None

    def _setup(self):
        from concurrent.futures import ThreadPoolExecutor

        self.bufs = [torch.empty(self.CHUNK, dtype=torch.uint8, pin_memory=True)
                     for _ in range(self.RING)]
        self.views = [b.numpy() for b in self.bufs]
        self.events = [None] * self.RING
        self.pool = ThreadPoolExecutor(self.THREADS)

    def _fill(self, dst: np.ndarray, src: np.ndarray):
        n = len(src)
        step = max(1, -(-n // self.THREADS))
        futs = [self.pool.submit(np.copyto, dst[i:i + step], src[i:i + step])
                for i in range(0, n, step)]
        for f in futs:
            f.result()

    def __call__(self, arr: np.ndarray, device) -> torch.Tensor:
        arr = np.ascontiguousarray(arr)
        out = torch.empty(arr.shape, dtype=torch.from_numpy(arr[:0]).dtype, device=device)
        if arr.nbytes < 2 * self.CHUNK:
            out.copy_(torch.from_numpy(arr))
            return out
        if self.bufs is None:
            self._setup()
        src = arr.reshape(-1).view(np.uint8)
        dst = out.view(-1).view(torch.uint8)
        stream = torch.cuda.current_stream(device)
        for k, off in enumerate(range(0, src.nbytes, self.CHUNK)):
            b = k % self.RING
            if self.events[b] is not None:
                self.events[b].synchronize()  # the DMA that last read this buffer is done
            n = min(self.CHUNK, src.nbytes - off)
            self._fill(self.views[b][:n], src[off:off + n])
            dst[off:off + n].copy_(self.bufs[b][:n], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            self.events[b] = ev
        return out


_upload = _Uploader()


def sh_degree_of(sh_coeffs: np.ndarray) -> int:
    """0 when bands 1..15 are all exactly zero (the DC-only kernel is then
    bit-identical), else 3."""
    return 0 if not np.any(sh_coeffs.reshape(len(sh_coeffs), 16, 3)[:, 1:, :]) else 3


class DeviceScene:
    """Kernel-ready copy of a scene on one GPU (render.py:49-54 scene_arrays).

    sigma is activated on the host with the reference's numpy softplus
    (foam.py:22-25) so it is bit-identical; ``set_raw_density`` activates on
    device instead (device-resident training).
    """

    def __init__(self, scene, device=None, sh_degree=None, packed=None, positions_f64=None):
        adj = scene.require_adjacency()
        sh = np.asarray(scene.sh_coeffs, dtype=np.float64).reshape(len(adj.positions), 48)
        self._init(adj.positions, adj.offsets, adj.neighbors, softplus(scene.raw_density), sh,
                   scene.background, adj.bbox_lo, adj.bbox_hi, device, sh_degree, packed,
                   positions_f64)

    @classmethod
    def from_arrays(cls, positions, offsets, neighbors, sigma, sh_flat, background, device=None,
                    sh_degree=None, packed=None, positions_f64=None, keep_csr64=False):
        """Flat kernel arrays as passed to kernels.render_rays (kernels.py:199-209).
        ``keep_csr64`` keeps the int64 device CSR for ``update_params``."""
        self = cls.__new__(cls)
        pos = np.asarray(positions, dtype=np.float64)
        self._init(pos, offsets, neighbors, sigma, sh_flat, background, pos.min(axis=0),
                   pos.max(axis=0), device, sh_degree, packed, positions_f64, keep_csr64)
        return self

    def _init(self, positions, offsets, neighbors, sigma, sh_flat, background, bbox_lo, bbox_hi,
              device, sh_degree, packed, positions_f64=None, keep_csr64=False):
        self._sh_degree_arg = sh_degree
        self.lib = _lib.load()
        self.device = torch.device(device or "cuda")
        pos = np.ascontiguousarray(positions, dtype=np.float64)
        n = len(pos)
        self.n_sites = n
        self.n_edges = int(len(neighbors))
        self.bbox_lo = np.asarray(bbox_lo, dtype=np.float64)
        self.bbox_hi = np.asarray(bbox_hi, dtype=np.float64)
        self.diagonal = float(np.linalg.norm(self.bbox_hi - self.bbox_lo))
        self.center = 0.5 * (self.bbox_lo + self.bbox_hi)
        self.width_floor = WIDTH_FLOOR_SCALE * self.diagonal
        self.background = np.asarray(background, dtype=np.float64).copy()
        sh = np.ascontiguousarray(np.asarray(sh_flat, dtype=np.float64).reshape(n, 48))
        sigma = np.ascontiguousarray(sigma, dtype=np.float64)
        self.packed = True if packed is None else bool(packed)
        dev = self.device
        with torch.cuda.device(dev):
            # upload first; the scene statistics the layout needs are reductions on
            # the device (one sync) instead of host passes over the 384 MB SH table
            self.sh = _upload(sh, dev)
            pos_d = _upload(pos, dev)
            sig_d = _upload(sigma, dev)
            off_d = _upload(np.ascontiguousarray(offsets, dtype=np.int64), dev)
            nbr_d = _upload(np.ascontiguousarray(neighbors, dtype=np.int64), dev)
            if n:
                st = torch.stack([self.sh.abs().max(),
                                  (self.sh.view(n, 16, 3)[:, 1:, :] != 0).any().double(),
                                  (pos_d.float().double() != pos_d).any().double()]).cpu()
                absmax, any_hi, not_exact32 = float(st[0]), bool(st[1] > 0), bool(st[2] > 0)
            else:
                absmax, any_hi, not_exact32 = 0.0, False, False
            # SH degree 0 when bands 1..15 are all zero (sh_degree_of), else 3
            self.sh_degree = (3 if any_hi else 0) if sh_degree is None else int(sh_degree)
            # fp32 upper bound of max |coefficient| (colour rounding bound, packed layout)
            self.sh_absmax = float(np.float32(absmax) * np.float32(1.0001))
            # packed layout by default; positions that do not survive an fp32 round trip
            # (or that will move, positions_f64=True) use the widened pre-filter bound
            # and exact phase from site4 (rfb_scene.positions_f64)
            self.positions_f64 = not_exact32 if positions_f64 is None else bool(positions_f64)
            self.site4 = torch.empty((n, 4), dtype=torch.float64, device=dev)
            self.offsets = torch.empty(n + 1, dtype=torch.int32, device=dev)
            self.neighbors = torch.empty(max(self.n_edges, 1), dtype=torch.int32, device=dev)
            # device copy of the colour bound: rfb_post_grad_adam raises it when a
            # training step grows a coefficient (the kernels read this copy)
            self.sh_absmax_dev = torch.tensor([self.sh_absmax], dtype=torch.float32, device=dev)
            if self.packed:
                self.cells = torch.empty((n, 8), dtype=torch.int32, device=dev)      # 32 B headers
                self._alloc_edges(n, self.n_edges, dev)
                self.sh32 = torch.empty((n, 48), dtype=torch.float32, device=dev)
            else:
                self.cells = self.edges = self.edge_nbr = self.sh32 = None
                self.pk_of = self.pk_id = None
            _lib.check(self.lib.rfb_pack_scene(
                _ptr(pos_d), _ptr(sig_d), _ptr(self.sh), _ptr(off_d), _ptr(nbr_d), n,
                self.n_edges, _ptr(self.site4), _ptr(self.offsets), _ptr(self.neighbors),
                _ptr(self.cells), _ptr(self.edges), _ptr(self.edge_nbr), _ptr(self.sh32),
                _ptr(self.pk_of), _ptr(self.pk_id), 1 if self.positions_f64 else 0, _stream()),
                "rfb_pack_scene")
            torch.cuda.current_stream().synchronize()
            self._csr64 = (off_d, nbr_d) if keep_csr64 else None
        self._c = _lib.rfb_scene()
        self._refresh_struct()
        self._build_locate_grid()

    def update_params(self, positions, sigma, sh_flat, background=None):
        """Re-derive the kernel arrays for new parameter values on the SAME
        adjacency (the reference re-reads scene_arrays on every call and its
        training loop moves sites / updates sigma and SH in place between
        rebuilds, foam.py:70-80): upload positions, sigma and SH and re-pack
        on the device, reusing the device CSR (needs ``keep_csr64``)."""
        if self._csr64 is None:
            raise RuntimeError("update_params needs a DeviceScene built with keep_csr64=True")
        off_d, nbr_d = self._csr64
        pos = np.ascontiguousarray(positions, dtype=np.float64)
        n = self.n_sites
        if pos.shape != (n, 3):
            raise ValueError("positions shape changed: build a new DeviceScene")
        sh = None if sh_flat is None else \
            np.ascontiguousarray(np.asarray(sh_flat, dtype=np.float64).reshape(n, 48))
        sigma = np.ascontiguousarray(sigma, dtype=np.float64)
        self.bbox_lo, self.bbox_hi = pos.min(axis=0), pos.max(axis=0)
        self.diagonal = float(np.linalg.norm(self.bbox_hi - self.bbox_lo))
        self.center = 0.5 * (self.bbox_lo + self.bbox_hi)
        self.width_floor = WIDTH_FLOOR_SCALE * self.diagonal
        if background is not None:
            self.background = np.asarray(background, dtype=np.float64).copy()
        if sh is not None:  # None: colours unused by the caller (walk only)
            if self._sh_degree_arg is None:
                self.sh_degree = sh_degree_of(sh)
            self.sh_absmax = float(np.float32(np.abs(sh).max() if sh.size else 0.0)
                                   * np.float32(1.0001))
        if not self.positions_f64:
            self.positions_f64 = not bool(np.array_equal(pos.astype(np.float32).astype(np.float64),
                                                         pos))
        dev = self.device
        with torch.cuda.device(dev):
            if sh is not None:
                self.sh.copy_(torch.from_numpy(sh))
                self.sh_absmax_dev.fill_(self.sh_absmax)
            pos_d = torch.from_numpy(pos).to(dev)
            sig_d = torch.from_numpy(sigma).to(dev)
            _lib.check(self.lib.rfb_pack_scene(
                _ptr(pos_d), _ptr(sig_d), _ptr(self.sh), _ptr(off_d), _ptr(nbr_d), n,
                self.n_edges, _ptr(self.site4), _ptr(self.offsets), _ptr(self.neighbors),
                _ptr(self.cells), _ptr(self.edges), _ptr(self.edge_nbr), _ptr(self.sh32),
                _ptr(self.pk_of), _ptr(self.pk_id), 1 if self.positions_f64 else 0, _stream()),
                "rfb_pack_scene")
        self._refresh_struct()
        self._build_locate_grid()

    # the packed arrays in a Morton order of the sites (rfb_pack_scene pk_of/pk_id):
    # cells a ray visits in turn sit near each other; ids outside stay site ids
    PACKED_ORDER = os.environ.get("RFB_PACKED_ORDER", "1") != "0"

    def _alloc_edges(self, n, n_edges, dev):
        """Packed records (16 B, rows padded to even length), the neighbour of
        every slot (RFB_PACKED_EDGE_SLOTS(n, E) = E + n + 2) and the packed order."""
        slots = n_edges + n + 2
        self.edges = torch.zeros((slots, 4), dtype=torch.float32, device=dev)
        self.edge_nbr = torch.full((slots,), -1, dtype=torch.int32, device=dev)
        if self.PACKED_ORDER:
            self.pk_of = torch.empty(n, dtype=torch.int32, device=dev)
            self.pk_id = torch.empty(n, dtype=torch.int32, device=dev)
        else:
            self.pk_of = self.pk_id = None

    LOCATE_GRID_RES = 64  # cells along the longest bounding-box axis

    def _build_locate_grid(self, stream=None):
        """Seed grid for point location (rfb_build_locate_grid)."""
        ext = np.maximum(self.bbox_hi - self.bbox_lo, 1e-12)
        cell = float(ext.max()) / self.LOCATE_GRID_RES
        dims = [max(1, int(np.ceil(e / cell))) for e in ext]
        self._hint = torch.empty(int(np.prod(dims)), dtype=torch.int32, device=self.device)
        g = _lib.rfb_locate_grid()
        for k in range(3):
            g.lo[k] = float(self.bbox_lo[k])
            g.dims[k] = dims[k]
        g.cell = cell
        g.hint = self._hint.data_ptr()
        self._grid = g
        _lib.check(self.lib.rfb_build_locate_grid(self.c, ctypes.byref(g), _stream(stream)),
                   "rfb_build_locate_grid")

    def _refresh_struct(self):
        c = self._c
        c.n_sites = self.n_sites
        c.n_edges = self.n_edges
        c.site4 = self.site4.data_ptr()
        c.offsets = self.offsets.data_ptr()
        c.neighbors = self.neighbors.data_ptr()
        c.sh = self.sh.data_ptr()
        c.cells = self.cells.data_ptr() if self.packed else None
        c.edges = self.edges.data_ptr() if self.packed else None
        c.edge_nbr = self.edge_nbr.data_ptr() if self.packed else None
        c.pk_of = self.pk_of.data_ptr() if (self.packed and self.pk_of is not None) else None
        c.pk_id = self.pk_id.data_ptr() if (self.packed and self.pk_id is not None) else None
        c.sh32 = self.sh32.data_ptr() if self.packed else None
        c.packed = 1 if self.packed else 0
        c.positions_f64 = 1 if (self.packed and self.positions_f64) else 0
        c.sh_absmax = self.sh_absmax
        c.sh_absmax_dev = self.sh_absmax_dev.data_ptr()
        c.sh_degree = self.sh_degree
        for k in range(3):
            c.background[k] = float(self.background[k])

    @property
    def c(self):
        return ctypes.byref(self._c)

    # -- view culling (rfb_cull_scene) -------------------------------------
    VIEW_CULL = os.environ.get("RFB_VIEW_CULL", "1") != "0"

    def view(self, dirs, stream=None):
        """The scene as walked by rays whose directions lie in the cone generated
        by ``dirs`` ([k][3], k <= 8; see ``view_cone``): a copy of the packed rows
        without the neighbours that are back-facing for every such ray (the
        reference skips them for every ray, kernels.py:118-119), re-derived on
        every call (the rows change when the scene does).  Returns a ctypes
        reference to the derived rfb_scene, or ``self.c`` when culling does not
        apply (generic layout, no cone, RFB_VIEW_CULL=0)."""
        if dirs is None or not self.packed or not self.VIEW_CULL or self.n_sites == 0:
            return self.c
        d = np.ascontiguousarray(np.asarray(dirs, dtype=np.float64).reshape(-1, 3))
        self._view_alloc(1)
        _lib.check(self.lib.rfb_cull_scene(
            self.c, d.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), int(len(d)),
            _ptr(self._view_cells), _ptr(self._view_edges), ctypes.byref(self._view_c),
            _stream(stream)), "rfb_cull_scene")
        return ctypes.byref(self._view_c)

    # image regions culled separately by render_image_device (rfb_cull_view): smaller
    # cones drop more faces; "RX"x"RY" from RFB_VIEW_REGIONS (e.g. "4x4"), "1x1" = one cone
    VIEW_REGIONS = tuple(int(v) for v in os.environ.get("RFB_VIEW_REGIONS", "4x2").split("x"))

    def _view_alloc(self, regions: int):
        if getattr(self, "_view_regions", 0) < regions:
            self._view_cells = self._view_edges = None
            stride = (self.n_edges + self.n_sites + 3) & ~1  # RFB_VIEW_STRIDE
            self._view_cells = torch.empty((regions * self.n_sites, 8), dtype=torch.int32,
                                           device=self.device)
            self._view_edges = torch.empty((regions * stride, 4), dtype=torch.float32,
                                           device=self.device)
            self._view_regions = regions
            self._view_c = _lib.rfb_scene()

    # the cull pass touches every row of every region (~0.07 ms per region per 1M sites),
    # the walk saves per ray: frames with fewer rays than this share of the sites walk the
    # full rows (1M sites, 4 x 2 regions: 480x270 1.93 vs 1.82 ms, 960x540 4.07 vs 5.27 ms;
    # break-even ~0.15 rays per site)
    VIEW_CULL_MIN_RAYS_PER_SITE = 0.2
    # and a fixed floor: small frames are launch-bound (config 1, 10k sites, 128x128:
    # 157 us without the cull launch, 171 us with it)
    VIEW_CULL_MIN_RAYS = 100_000

    def can_cull(self, camera, rays=None) -> bool:
        """Whether ``view_camera`` culls for this camera (packed layout, pinhole, culling
        enabled, and -- given the ray count -- a frame large enough to pay for the pass)."""
        if (not self.packed or not self.VIEW_CULL or self.n_sites == 0
                or getattr(camera, "kind", "pinhole") == "fisheye"):
            return False
        return rays is None or (rays >= self.VIEW_CULL_MIN_RAYS and
                                rays >= self.VIEW_CULL_MIN_RAYS_PER_SITE * self.n_sites)

    def view_camera(self, camera, regions=None, stream=None):
        """``view`` per image region of a pinhole camera (rfb_cull_view): an RX x RY
        grid of pixel rectangles, each culled against its own corner cone; the
        walk picks each pixel's region (rfb_render_image) or takes it from
        ``region_ids`` (ray batches).  Falls back like ``view``."""
        rx, ry = regions or self.VIEW_REGIONS
        rx, ry = max(1, min(int(rx), int(camera.width))), max(1, min(int(ry), int(camera.height)))
        if not self.can_cull(camera):
            return self.c
        self._view_alloc(rx * ry)
        cam = camera_struct(camera)
        _lib.check(self.lib.rfb_cull_view(self.c, ctypes.byref(cam), rx, ry,
                                          _ptr(self._view_cells), _ptr(self._view_edges),
                                          ctypes.byref(self._view_c), _stream(stream)),
                   "rfb_cull_view")
        return ctypes.byref(self._view_c)

    def region_ids(self, camera, pixels: torch.Tensor, regions=None) -> torch.Tensor:
        """uint8 region of each row-major pixel index for ``view_camera(camera,
        regions)`` (rfb.h: (py * ry / H) * rx + px * rx / W)."""
        rx, ry = regions or self.VIEW_REGIONS
        W, H = int(camera.width), int(camera.height)
        rx, ry = max(1, min(int(rx), W)), max(1, min(int(ry), H))
        p = pixels.to(self.device, torch.int64)
        py, px = p // W, p % W
        return ((py * ry // H) * rx + px * rx // W).to(torch.uint8)

    # -- device-resident updates (training) ------------------------------
    def rebuild_adjacency(self, positions: torch.Tensor | None = None, packed=None,
                          stream=None) -> dict:
        """Re-triangulate on the device after the sites moved (train.py:247-256
        rebuilds with delaunay.build; here rfb_build_adjacency) and re-pack the
        scene in place: CSR, packed headers/edges, bounding box and width floor.
        `positions` (device fp64 [n,3]) defaults to the current site4 xyz."""
        from . import adjacency

        pos = (self.site4[:, :3] if positions is None else positions).to(
            self.device, torch.float64).contiguous()
        off, nbr, hull, info = adjacency.build_device(pos, stream=stream)
        n = self.n_sites
        sig = self.site4[:, 3].contiguous()
        self.n_edges = int(nbr.numel())
        lo = pos.min(0).values.cpu().numpy()
        hi = pos.max(0).values.cpu().numpy()
        self.bbox_lo, self.bbox_hi = lo, hi
        self.diagonal = float(np.linalg.norm(hi - lo))
        self.center = 0.5 * (lo + hi)
        self.width_floor = WIDTH_FLOOR_SCALE * self.diagonal
        if packed is not None:
            self.packed = bool(packed)
        if not self.positions_f64:  # a scene built as fp32-exact stays so only if it still is
            self.positions_f64 = not bool(torch.equal(pos.float().double(), pos))
        dev = self.device
        with torch.cuda.device(dev):
            site4 = torch.empty((n, 4), dtype=torch.float64, device=dev)
            self.offsets = torch.empty(n + 1, dtype=torch.int32, device=dev)
            self.neighbors = torch.empty(max(self.n_edges, 1), dtype=torch.int32, device=dev)
            if self.packed:
                self.cells = torch.empty((n, 8), dtype=torch.int32, device=dev)
                self._alloc_edges(n, self.n_edges, dev)
                self.sh32 = torch.empty((n, 48), dtype=torch.float32, device=dev)
            else:
                self.cells = self.edges = self.edge_nbr = self.sh32 = None
                self.pk_of = self.pk_id = None
            _lib.check(self.lib.rfb_pack_scene(
                _ptr(pos), _ptr(sig), _ptr(self.sh), _ptr(off), _ptr(nbr), n, self.n_edges,
                _ptr(site4), _ptr(self.offsets), _ptr(self.neighbors), _ptr(self.cells),
                _ptr(self.edges), _ptr(self.edge_nbr), _ptr(self.sh32), _ptr(self.pk_of),
                _ptr(self.pk_id), 1 if self.positions_f64 else 0,
                _stream(stream)), "rfb_pack_scene")
            self.site4 = site4
        self.hull = hull
        self._refresh_struct()
        self._build_locate_grid(stream)
        return info


    def set_raw_density(self, raw: torch.Tensor, stream=None):
        raw = raw.to(self.device, torch.float64).contiguous()
        _lib.check(self.lib.rfb_softplus(_ptr(raw), self.n_sites, None, _ptr(self.site4),
                                         _ptr(self.cells), _ptr(self.pk_of), _stream(stream)),
                   "rfb_softplus")

    def default_t_max(self, origins: np.ndarray) -> float:
        """Batch fallback t_max (render.py:72-76)."""
        o = np.asarray(origins, dtype=np.float64).reshape(-1, 3)
        if len(o) == 1:  # one camera origin per frame: memoised on the inputs' bits
            key = (o.tobytes(), np.asarray(self.center).tobytes(), self.diagonal)
            memo = self.__dict__.setdefault("_t_max_memo", {})
            t = memo.get(key)
            if t is None:
                if len(memo) > 64:
                    memo.clear()
                t = memo[key] = DeviceScene.default_t_max(self, np.concatenate([o, o]))
            return t
        return float(np.linalg.norm(o - self.center, axis=1).max() + 2.0 * self.diagonal + 1.0)

    def locate(self, queries: torch.Tensor, seed: int = 0, stream=None) -> torch.Tensor:
        q = queries.to(self.device, torch.float64).contiguous()
        m = q.shape[0]
        out = torch.empty(m, dtype=torch.int32, device=self.device)
        _lib.check(self.lib.rfb_locate_seeded(self.c, _ptr(q), m, ctypes.byref(self._grid),
                                              int(seed), _ptr(out), _stream(stream)),
                   "rfb_locate_seeded")
        return out


EFFECT_KINDS = {"mirror": 0, "reflect": 0, "refract": 1}


def effect_rays_device(origins, directions, t_at, normal, effect="mirror", eta=1.5, stream=None):
    """Batched apply_effect (rays.py:166-176) on the device: every ray
    continues from origin + t_at * direction across one effect plane with
    normal `normal`.  Returns (origins', directions') fp64 [m, 3]; the new rays
    start at t_min = 0 with the old t_max."""
    if effect not in EFFECT_KINDS:
        raise ValueError(f"unknown effect {effect!r}")
    lib = _lib.load()
    o = origins.to(torch.float64).contiguous()
    d = directions.to(o.device, torch.float64).contiguous()
    m = o.shape[0]
    t = torch.as_tensor(t_at, dtype=torch.float64, device=o.device).expand(m).contiguous()
    n = (ctypes.c_double * 3)(*[float(v) for v in np.asarray(normal, dtype=np.float64)])
    oo = torch.empty_like(o)
    od = torch.empty_like(d)
    _lib.check(lib.rfb_effect_rays(_ptr(o), _ptr(d), _ptr(t), m, n, EFFECT_KINDS[effect],
                                   float(eta), _ptr(oo), _ptr(od), _stream(stream)),
               "rfb_effect_rays")
    return oo, od


def forward_schedule(origins: torch.Tensor, directions: torch.Tensor):
    """(order, lanes_per_ray) for a forward batch of arbitrary rays -- scheduling
    only, results stay per ray: batches too small to fill the resident threads
    walk each ray with several lanes (lanes_per_ray 0 = the library's auto rule),
    large ones are sorted coherently.  Measured on random training pixels
    (tools/train_batch_probe.py --forward --lanes L): 16k rays 2.85 / 1.93 / 1.54 /
    1.35 ms with 1 / 2 / 4 / 8 lanes, 65k rays 3.52 / 2.53 / 3.07 / 4.46 ms (the
    auto rule picks 8 and 2); 262k rays 8.8 -> 7.0 ms sorted."""
    m = origins.shape[0]
    order = coherent_order(origins, directions) if m >= 200_000 else None
    return order, 0


def make_params(epsilon=DEFAULT_EPSILON, width_floor=0.0, step_limit=DEFAULT_STEP_LIMIT,
                lanes_per_ray=DEFAULT_LANES):
    p = _lib.rfb_params()
    p.epsilon = float(epsilon)
    p.width_floor = float(width_floor)
    p.step_limit = int(step_limit)
    p.lanes_per_ray = int(lanes_per_ray)
    return p


@dataclass
class ForwardResult:
    rgb: torch.Tensor
    residual: torch.Tensor
    wsum: torch.Tensor
    status: torch.Tensor
    nseg: torch.Tensor | None = None
    ray_counters: torch.Tensor | None = None
    counters: torch.Tensor | None = None
    seg_cells: torch.Tensor | None = None
    seg_t0: torch.Tensor | None = None
    seg_t1: torch.Tensor | None = None
    seg_first: int = 0


class Workspace:
    """Grow-only device scratch (no allocation on the steady-state path)."""

    def __init__(self, device):
        self.device = device
        self.buf = None

    def get(self, nbytes: int) -> torch.Tensor:
        nbytes = max(int(nbytes), 256)
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        return self.buf


def alloc_forward(m: int, device, f64=False, per_ray=True, seg_capacity=0,
                  seg_rays=None) -> ForwardResult:
    """``seg_rays``: (first, count) -- dump the segments of rays first ..
    first + count - 1 only (rfb_fwd_out.seg_first / seg_count); default all m."""
    fdt = torch.float64 if f64 else torch.float32
    r = ForwardResult(
        rgb=torch.empty((m, 3), dtype=fdt, device=device),
        residual=torch.empty(m, dtype=fdt, device=device),
        wsum=torch.empty(m, dtype=fdt, device=device),
        status=torch.empty(m, dtype=torch.int8, device=device),
        counters=torch.zeros(2, dtype=torch.int64, device=device),
    )
    if per_ray:
        r.nseg = torch.empty(m, dtype=torch.int32, device=device)
        r.ray_counters = torch.empty((m, 2), dtype=torch.int32, device=device)
    if seg_capacity > 0:
        rows = m if seg_rays is None else int(seg_rays[1])
        r.seg_cells = torch.full((rows, seg_capacity), -1, dtype=torch.int32, device=device)
        r.seg_t0 = torch.zeros((rows, seg_capacity), dtype=torch.float64, device=device)
        r.seg_t1 = torch.zeros((rows, seg_capacity), dtype=torch.float64, device=device)
        r.seg_first = 0 if seg_rays is None else int(seg_rays[0])
    return r


def fwd_struct(r: ForwardResult) -> _lib.rfb_fwd_out:
    o = _lib.rfb_fwd_out()
    o.rgb = r.rgb.data_ptr()
    o.residual = r.residual.data_ptr() if r.residual is not None else None
    o.wsum = r.wsum.data_ptr() if r.wsum is not None else None
    o.status = r.status.data_ptr() if r.status is not None else None
    o.nseg = r.nseg.data_ptr() if r.nseg is not None else None
    o.ray_counters = r.ray_counters.data_ptr() if r.ray_counters is not None else None
    o.counters = r.counters.data_ptr() if r.counters is not None else None
    o.f64_outputs = 1 if r.rgb.dtype == torch.float64 else 0
    if r.seg_cells is not None:
        o.seg_capacity = r.seg_cells.shape[1]
        o.seg_cells = r.seg_cells.data_ptr()
        o.seg_t0 = r.seg_t0.data_ptr()
        o.seg_t1 = r.seg_t1.data_ptr()
        o.seg_first = int(r.seg_first)
        o.seg_count = r.seg_cells.shape[0]
    else:
        o.seg_capacity = 0
    return o


def _view_for(ds: DeviceScene, view_dirs, view, stream):
    """(scene struct, region ids) for a ray batch: ``view`` = (camera, pixels) walks
    the camera's region-culled rows with each ray's region from its row-major pixel
    index; ``view_dirs`` = a cone holding every direction (one region)."""
    if view is not None:
        cam, pixels = view
        if not ds.can_cull(cam, len(pixels)):
            return ds.c, None
        sc = ds.view_camera(cam, stream=stream)
        return sc, ds.region_ids(cam, pixels).contiguous()
    return ds.view(view_dirs, stream), None


def rays_struct(origins, directions, t_min, t_max, start, order=None) -> _lib.rfb_rays:
    r = _lib.rfb_rays()
    r.m = origins.shape[0]
    r.origins = origins.data_ptr()
    r.directions = directions.data_ptr()
    r.t_min = t_min.data_ptr()
    r.t_max = t_max.data_ptr()
    r.start_sites = start.data_ptr()
    r.order = order.data_ptr() if order is not None else None
    return r


AUTO_ORDER_MIN_RAYS = 500_000


def _order32(order, m, device, origins=None, directions=None):
    """None: the given order; "auto": coherent_order for batches of >= 500k
    rays (random training pixels: 1.5x at 1M rays; at 262k neutral, at 65k the
    per-lane reverse pass of incoherent warps is faster unsorted --
    tools/train_batch_probe.py); else an explicit permutation."""
    if isinstance(order, str):
        if order != "auto":
            raise ValueError(f"unknown order {order!r}")
        if m < AUTO_ORDER_MIN_RAYS:
            return None
        order = coherent_order(origins.to(device), directions.to(device))
    if order is None:
        return None
    o = order.to(device=device, dtype=torch.int32).contiguous()
    assert o.numel() == m, "order must be a permutation of the m rays"
    return o


def camera_struct(camera) -> _lib.rfb_camera:
    c = _lib.rfb_camera()
    c.pose[:] = np.asarray(camera.pose, dtype=np.float64).reshape(16).tolist()
    c.width = int(camera.width)
    c.height = int(camera.height)
    c.focal = float(camera.focal)
    c.cx = float(camera.cx)
    c.cy = float(camera.cy)
    c.kind = 1 if getattr(camera, "kind", "pinhole") == "fisheye" else 0
    return c


def render_rays_device(ds: DeviceScene, origins, directions, t_min, t_max, start, *,
                       epsilon=DEFAULT_EPSILON, step_limit=DEFAULT_STEP_LIMIT, f64=False,
                       per_ray=True, seg_capacity=0, lanes_per_ray=DEFAULT_LANES,
                       workspace: Workspace | None = None, out: ForwardResult | None = None,
                       order=None, stream=None, view_dirs=None, view=None) -> ForwardResult:
    """rfb_render_rays on device tensors (kernels.py:199-247).  ``order``: an
    optional processing permutation (e.g. coherent_order) -- outputs stay
    indexed by ray.  ``view_dirs``: generators of a cone holding every ray
    direction (``view_cone(camera)`` for a camera's pixels): the walk then
    uses the view-culled rows (``DeviceScene.view``; same output).  ``view``:
    (camera, pixels) -- the rays are those pixels (row-major indices) of a
    pinhole camera: the walk uses the camera's region-culled rows
    (``DeviceScene.view_camera``), a smaller cone per ray."""
    m = origins.shape[0]
    res = out or alloc_forward(m, ds.device, f64=f64, per_ray=per_ray, seg_capacity=seg_capacity)
    ws = (workspace or Workspace(ds.device)).get(FWD_WORKSPACE_BYTES)
    p = make_params(epsilon, ds.width_floor, step_limit, lanes_per_ray)
    order = _order32(order, m, ds.device)
    rays = rays_struct(origins, directions, t_min, t_max, start, order)
    o = fwd_struct(res)
    sc, reg = _view_for(ds, view_dirs, view, stream)
    if reg is not None:
        rays.region = reg.data_ptr()
    _lib.check(ds.lib.rfb_render_rays(sc, ctypes.byref(rays), ctypes.byref(p), ctypes.byref(o),
                                      _ptr(ws), ws.numel(), _stream(stream)), "rfb_render_rays")
    return res


def tile_grid(width: int, height: int, tile_w: int = 32, tile_h: int = 32):
    tiles_x = (width + tile_w - 1) // tile_w
    tiles_y = (height + tile_h - 1) // tile_h
    return tiles_x, tiles_y


def host_device_pointer(lib, host: torch.Tensor) -> int | None:
    """Device address of a pinned host tensor (rfb_host_device_pointer), or
    None when the memory is not mapped into the device address space."""
    dev = ctypes.c_void_p()
    if lib.rfb_host_device_pointer(ctypes.c_void_p(host.data_ptr()), ctypes.byref(dev)) != 0:
        return None
    return dev.value


def view_cone(camera):
    """Generators of the cone holding every pixel ray direction of a pinhole
    camera: its four corner-pixel directions R (u, v, -1) (camera.py:78-92 is
    linear in the pixel centre (u, v), so every pixel direction is a positive
    combination of them).  None for a fisheye camera."""
    if getattr(camera, "kind", "pinhole") == "fisheye":
        return None
    W, H = int(camera.width), int(camera.height)
    cols = np.array([0.0, W - 1.0, 0.0, W - 1.0])
    rows = np.array([0.0, 0.0, H - 1.0, H - 1.0])
    u = (cols + 0.5 - float(camera.cx)) / float(camera.focal)
    v = -(rows + 0.5 - float(camera.cy)) / float(camera.focal)
    d_cam = np.stack([u, v, -np.ones(4)], axis=1)
    return d_cam @ np.asarray(camera.pose, dtype=np.float64)[:3, :3].T


def render_image_device(ds: DeviceScene, camera, *, epsilon=DEFAULT_EPSILON,
                        step_limit=DEFAULT_STEP_LIMIT, t_max=None, start_site=-1, tile_ids=None,
                        tile_w=32, tile_h=32, f64=False, per_ray=False,
                        lanes_per_ray=DEFAULT_LANES, workspace: Workspace | None = None,
                        out: ForwardResult | None = None, stream=None,
                        rgb_ptr: int | None = None, cull: bool = True) -> ForwardResult:
    """Fused ray generation + render over a tile list (render.py:128-149).

    ``rgb_ptr``: optional device address (``host_device_pointer``) of a mapped
    page-locked (W*H, 3) host frame of ``out.rgb``'s dtype; the kernel then
    stores each ray's colour straight into host memory and ``out.rgb`` is
    left untouched.  ``cull``: walk a copy of the rows without the faces that
    are back-facing for the whole frame (``DeviceScene.view``, re-derived per
    call; bit-identical output)."""
    W, H = int(camera.width), int(camera.height)
    m = W * H
    if tile_ids is None:
        tx, ty = tile_grid(W, H, tile_w, tile_h)
        tile_ids = torch.arange(tx * ty, dtype=torch.int32, device=ds.device)
    res = out or alloc_forward(m, ds.device, f64=f64, per_ray=per_ray)
    ws = (workspace or Workspace(ds.device)).get(FWD_WORKSPACE_BYTES)
    if t_max is None:
        t_max = ds.default_t_max(np.asarray(camera.pose)[:3, 3][None, :])
    p = make_params(epsilon, ds.width_floor, step_limit, lanes_per_ray)
    cam = camera_struct(camera)
    o = fwd_struct(res)
    if rgb_ptr is not None:
        o.rgb = int(rgb_ptr)
    if cull == "last":  # diagnostics: the view the previous call derived, as it is now
        sc = ctypes.byref(ds._view_c)
    else:
        rays = min(m, int(tile_ids.numel()) * tile_w * tile_h)  # (a rank's tile subset)
        sc = ds.view_camera(camera, stream=stream) if cull and ds.can_cull(camera, rays) else ds.c
    _lib.check(ds.lib.rfb_render_image(sc, ctypes.byref(cam), ctypes.byref(p), 0.0, float(t_max),
                                       int(start_site), _ptr(tile_ids), int(tile_ids.numel()),
                                       int(tile_w), int(tile_h), ctypes.byref(o), _ptr(ws),
                                       ws.numel(), _stream(stream)), "rfb_render_image")
    return res


class GradBuffers:
    """Flat float32 [n, 52] gradient accumulator: view ``g4`` [n,4]
    (dpos xyz, dsigma) and ``sh`` [n,48] (rfb_grads)."""

    def __init__(self, n: int, device):
        self.n = n
        self.flat = torch.zeros(n * 52, dtype=torch.float32, device=device)
        self.g4 = self.flat[: 4 * n].view(n, 4)
        self.sh = self.flat[4 * n:].view(n, 48)

    def zero_(self):
        self.flat.zero_()

    def struct(self):
        g = _lib.rfb_grads()
        g.site4g = self.g4.data_ptr()
        g.sh = self.sh.data_ptr()
        return g

    @property
    def d_position(self):
        return self.g4[:, :3]

    @property
    def d_sigma(self):
        return self.g4[:, 3]


def backward_workspace_bytes(ds: DeviceScene, m: int, step_limit: int, quantile=True) -> int:
    """rfb_workspace_bytes: kind 1 (any loss) or 2 (no quantile term: compact records)."""
    return int(ds.lib.rfb_workspace_bytes(int(m), int(step_limit), 1 if quantile else 2))


def backward_rays_device(ds: DeviceScene, origins, directions, t_min, t_max, start, adjoints,
                         grads: GradBuffers, *, epsilon=DEFAULT_EPSILON,
                         step_limit=DEFAULT_STEP_LIMIT, f64=False,
                         workspace: Workspace | None = None, out: ForwardResult | None = None,
                         order="auto", lanes_per_ray=0, stream=None, view_dirs=None, view=None) -> ForwardResult:
    """rfb_backward_rays (render.py:152-221 generic adjoint).  ``order``: see _order32;
    ``lanes_per_ray``: 1 or 2 forces the kernel variant, 0 = the library's rule;
    ``view_dirs``, ``view``: see render_rays_device."""
    m = origins.shape[0]
    res = out or alloc_forward(m, ds.device, f64=f64, per_ray=True)
    ws = (workspace or Workspace(ds.device)).get(
        backward_workspace_bytes(ds, m, step_limit, quantile=False))
    p = make_params(epsilon, ds.width_floor, step_limit, lanes_per_ray)
    order = _order32(order, m, ds.device, origins, directions)
    rays = rays_struct(origins, directions, t_min, t_max, start, order)
    o = fwd_struct(res)
    g = grads.struct()
    adj = adjoints.to(ds.device, torch.float64).contiguous()
    sc, reg = _view_for(ds, view_dirs, view, stream)
    if reg is not None:
        rays.region = reg.data_ptr()
    _lib.check(ds.lib.rfb_backward_rays(sc, ctypes.byref(rays), ctypes.byref(p), _ptr(adj),
                                        ctypes.byref(o), ctypes.byref(g), _ptr(ws), ws.numel(),
                                        _stream(stream)), "rfb_backward_rays")
    return res


def train_batch_device(ds: DeviceScene, origins, directions, t_min, t_max, start, targets,
                       grads: GradBuffers, loss: torch.Tensor, *, rgb_scale: float,
                       quantile_scale: float = 0.0, u_pairs=None, weight_floor: float = 1e-4,
                       epsilon=DEFAULT_EPSILON, step_limit=DEFAULT_STEP_LIMIT, f64=False,
                       workspace: Workspace | None = None, out: ForwardResult | None = None,
                       order="auto", lanes_per_ray=0, stream=None, view_dirs=None, view=None) -> ForwardResult:
    """rfb_train_batch (kernels.py:372-453).  ``loss`` float64 [2] accumulates.
    ``order``: "auto" sorts batches of >= 500k rays coherently (see _order32);
    ``lanes_per_ray``: 1 or 2 forces the kernel variant, 0 = the library's rule;
    ``view_dirs``, ``view``: see render_rays_device."""
    m = origins.shape[0]
    res = out or alloc_forward(m, ds.device, f64=f64, per_ray=True)
    ws = (workspace or Workspace(ds.device)).get(
        backward_workspace_bytes(ds, m, step_limit, quantile=quantile_scale > 0.0))
    p = make_params(epsilon, ds.width_floor, step_limit, lanes_per_ray)
    order = _order32(order, m, ds.device, origins, directions)
    rays = rays_struct(origins, directions, t_min, t_max, start, order)
    o = fwd_struct(res)
    g = grads.struct()
    n_pairs = 0
    up = None
    if quantile_scale > 0.0:
        up = u_pairs.to(ds.device, torch.float64).contiguous()
        n_pairs = up.shape[1]
    sc, reg = _view_for(ds, view_dirs, view, stream)
    if reg is not None:
        rays.region = reg.data_ptr()
    _lib.check(ds.lib.rfb_train_batch(sc, ctypes.byref(rays), ctypes.byref(p), _ptr(targets),
                                      float(rgb_scale), float(quantile_scale), _ptr(up), n_pairs,
                                      float(weight_floor), ctypes.byref(o), ctypes.byref(g),
                                      _ptr(loss), _ptr(ws), ws.numel(), _stream(stream)),
               "rfb_train_batch")
    return res


def tile_order(width: int, height: int, tile_w: int = 32, tile_h: int = 32, sub_w: int = 4):
    """Permutation of row-major pixel indices into the order rfb_render_image
    walks them (32x32 tiles, each split into sub_w x (32/sub_w) warp patches),
    so a batch of rays covering a view hands each warp a compact pixel patch
    (coherent cells: L1 reuse in the walk, large cell groups in the reverse
    pass).  Returns int64 numpy indices; losses/gradients are order-free."""
    sub_h = 32 // sub_w
    tx = (width + tile_w - 1) // tile_w
    ty = (height + tile_h - 1) // tile_h
    out = []
    for t in range(tx * ty):
        x0, y0 = (t % tx) * tile_w, (t // tx) * tile_h
        for s in range((tile_w // sub_w) * (tile_h // sub_h)):
            sx = x0 + (s % (tile_w // sub_w)) * sub_w
            sy = y0 + (s // (tile_w // sub_w)) * sub_h
            yy, xx = np.meshgrid(np.arange(sy, sy + sub_h), np.arange(sx, sx + sub_w), indexing="ij")
            keep = (xx < width) & (yy < height)
            out.append((yy * width + xx)[keep])
    return np.concatenate(out).astype(np.int64)


def _spread10(x: torch.Tensor) -> torch.Tensor:
    """Interleave zeros between the low 16 bits (Morton helper)."""
    x = x & 0xFFFF
    x = (x | (x << 8)) & 0x00FF00FF
    x = (x | (x << 4)) & 0x0F0F0F0F
    x = (x | (x << 2)) & 0x33333333
    x = (x | (x << 1)) & 0x55555555
    return x


def coherent_order(origins: torch.Tensor, directions: torch.Tensor, bits: int = 10):
    """Device-side ray sort for large or incoherent batches (e.g. random
    training pixels, train.py:135-140): key = (origin id, Morton code of the
    octahedral direction cell), so 32 consecutive rays share a compact patch
    of directions.  Returns an int32 permutation for the ``order`` argument;
    it changes only scheduling (outputs stay indexed by ray; gradient sums
    are order-free up to fp32 summation order)."""
    d = directions
    n1 = d.abs().sum(dim=1, keepdim=True)
    p = d[:, :2] / n1
    neg = d[:, 2] < 0
    px = torch.where(neg, (1 - p[:, 1].abs()) * torch.sign(p[:, 0]), p[:, 0])
    py = torch.where(neg, (1 - p[:, 0].abs()) * torch.sign(p[:, 1]), p[:, 1])
    q = (1 << bits) - 1
    ix = ((px * 0.5 + 0.5) * q).clamp(0, q).long()
    iy = ((py * 0.5 + 0.5) * q).clamp(0, q).long()
    _, oid = torch.unique(origins, dim=0, return_inverse=True)
    key = (oid << (2 * bits)) | _spread10(ix) | (_spread10(iy) << 1)
    return torch.argsort(key).to(torch.int32)


# ---------------------------------------------------------------------------
# The reference's per-ray building blocks over caller-held segment lists
# (rfb_segments.cu; kernels.py:38-73, 165-196, 250-369, 456-567).  Segments
# are CSR per ray: seg_offsets [m+1] int64, seg_cells int32, t0/t1 fp64.
# ---------------------------------------------------------------------------
def _f64(a, dev):
    return torch.as_tensor(a).to(dev, torch.float64).contiguous()


def _segs_args(seg_offsets, seg_cells, seg_t0, seg_t1, dev):
    """Coerce a segment CSR to the ABI dtypes (int64 offsets, int32 cells, f64 depths)."""
    return (torch.as_tensor(seg_offsets).to(dev, torch.int64).contiguous(),
            torch.as_tensor(seg_cells).to(dev, torch.int32).contiguous(),
            _f64(seg_t0, dev), _f64(seg_t1, dev))


def sh_basis_device(dirs: torch.Tensor, stream=None) -> torch.Tensor:
    lib = _lib.load()
    d = dirs.to(torch.float64).reshape(-1, 3).contiguous()
    out = torch.empty((d.shape[0], 16), dtype=torch.float64, device=d.device)
    _lib.check(lib.rfb_sh_basis(_ptr(d), d.shape[0], _ptr(out), _stream(stream)), "rfb_sh_basis")
    return out


def cell_colors_device(sh: torch.Tensor, cells: torch.Tensor, basis: torch.Tensor, stream=None):
    lib = _lib.load()
    c = cells.to(torch.int32).contiguous()
    b = basis.to(torch.float64).reshape(-1, 16).contiguous()
    out = torch.empty((c.shape[0], 3), dtype=torch.float64, device=c.device)
    masks = torch.empty(c.shape[0], dtype=torch.int32, device=c.device)
    _lib.check(lib.rfb_cell_colors(_ptr(sh), _ptr(c), _ptr(b), c.shape[0], _ptr(out),
                                   _ptr(masks), _stream(stream)), "rfb_cell_colors")
    return out, masks


def composite_segments_device(sigma, sh, basis, seg_offsets, seg_cells, seg_t0, seg_t1,
                              background, stream=None):
    """kernels.py:165-196 per ray -> (rgb [m,3], T [m], wsum [m])."""
    lib = _lib.load()
    dev = sigma.device
    seg_offsets, seg_cells, seg_t0, seg_t1 = _segs_args(seg_offsets, seg_cells, seg_t0, seg_t1,
                                                        dev)
    m = seg_offsets.shape[0] - 1
    rgb = torch.empty((m, 3), dtype=torch.float64, device=dev)
    T = torch.empty(m, dtype=torch.float64, device=dev)
    ws = torch.empty(m, dtype=torch.float64, device=dev)
    bg = (ctypes.c_double * 3)(*[float(v) for v in background])
    _lib.check(lib.rfb_composite_segments(
        _ptr(sigma), _ptr(sh), _ptr(basis.contiguous()), m, _ptr(seg_offsets), _ptr(seg_cells),
        _ptr(seg_t0), _ptr(seg_t1), bg, _ptr(rgb), _ptr(T), _ptr(ws), _stream(stream)),
        "rfb_composite_segments")
    return rgb, T, ws


def backward_segments_device(positions, sigma, sh, background, origins, dirs, basis, adjoints,
                             seg_offsets, seg_cells, seg_t0, seg_t1, d_sigma, d_sh, d_pos,
                             stream=None):
    """kernels.py:250-337 (+ face_t_gradient) per ray; accumulates (fp64)."""
    lib = _lib.load()
    seg_offsets, seg_cells, seg_t0, seg_t1 = _segs_args(seg_offsets, seg_cells, seg_t0, seg_t1,
                                                        sigma.device)
    m = seg_offsets.shape[0] - 1
    S = int(seg_cells.shape[0])
    ws = torch.empty(max(int(lib.rfb_segments_workspace_bytes(m, S)) // 8, 1),
                     dtype=torch.float64, device=sigma.device)
    bg = (ctypes.c_double * 3)(*[float(v) for v in background])
    _lib.check(lib.rfb_backward_segments(
        _ptr(positions), _ptr(sigma), _ptr(sh), bg, _ptr(origins), _ptr(dirs),
        _ptr(basis.contiguous()), _ptr(adjoints), m, _ptr(seg_offsets), _ptr(seg_cells),
        _ptr(seg_t0), _ptr(seg_t1), _ptr(d_sigma), _ptr(d_sh), _ptr(d_pos), _ptr(ws),
        ws.numel() * 8, _stream(stream)), "rfb_backward_segments")


def quantile_segments_device(positions, sigma, origins, dirs, seg_offsets, seg_cells, seg_t0,
                             seg_t1, u_pairs, weight_floor, scale, d_sigma, d_pos, stream=None):
    """kernels.py:456-567 for every pair of every ray; accumulates, returns the
    per-ray loss (sum over its pairs)."""
    lib = _lib.load()
    seg_offsets, seg_cells, seg_t0, seg_t1 = _segs_args(seg_offsets, seg_cells, seg_t0, seg_t1,
                                                        sigma.device)
    m = seg_offsets.shape[0] - 1
    S = int(seg_cells.shape[0])
    up = u_pairs.to(torch.float64).reshape(m, -1, 2).contiguous()
    ws = torch.empty(max(int(lib.rfb_segments_workspace_bytes(m, S)) // 8, 1),
                     dtype=torch.float64, device=sigma.device)
    loss = torch.empty(m, dtype=torch.float64, device=sigma.device)
    _lib.check(lib.rfb_quantile_segments(
        _ptr(positions), _ptr(sigma), _ptr(origins), _ptr(dirs), m, _ptr(seg_offsets),
        _ptr(seg_cells), _ptr(seg_t0), _ptr(seg_t1), _ptr(up), up.shape[1], float(weight_floor),
        float(scale), _ptr(d_sigma), _ptr(d_pos), _ptr(loss), _ptr(ws), ws.numel() * 8,
        _stream(stream)), "rfb_quantile_segments")
    return loss


def face_t_gradients_device(positions, ij, origins, dirs, t, dt, d_pos, stream=None):
    lib = _lib.load()
    m = ij.shape[0]
    _lib.check(lib.rfb_face_t_gradients(_ptr(positions), _ptr(ij.to(torch.int32).contiguous()),
                                        _ptr(origins), _ptr(dirs), _ptr(t), _ptr(dt), m,
                                        _ptr(d_pos), _stream(stream)), "rfb_face_t_gradients")
