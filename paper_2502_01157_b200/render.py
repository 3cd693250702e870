"""Drop-in replacements for the reference's Python render entry points.

Same names, argument meaning, defaults, return types and error behaviour as
rfoam/diffrender/render.py and rfoam/tracer/rays.py; the arithmetic runs in
librfb.so on the current CUDA device.  Host numpy arrays go in and come out
(fp64, like the reference); pass ``device_scene=`` to reuse a resident
scene instead of uploading it on every call (the reference re-derives its
kernel arrays on every call too, render.py:49-54).

  render_ray_batch            render.py:57-125
  render_image                render.py:128-149
  render_rays_with_gradients  render.py:152-221
  trace                       rays.py:81-115
  intersect_face              rays.py:60-78
  EffectPlane, reflect, refract, apply_effect   rays.py:123-176 (single ray,
                              host; effect_rays() is the batched device form)
  RenderStats                 render.py:27-46
"""

from __future__ import annotations

import math
import os
import time
import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from . import device as dv
from .errors import CycleDetected, ShapeMismatch, StepLimit
from .scene import GradientBuffer, softplus, softplus_grad

DEFAULT_EPSILON = dv.DEFAULT_EPSILON
DEFAULT_STEP_LIMIT = dv.DEFAULT_STEP_LIMIT
WIDTH_FLOOR_SCALE = dv.WIDTH_FLOOR_SCALE

STATUS_OK = 0
STATUS_STEP_LIMIT = 2
STATUS_CYCLE = 3

# render_image returns frames that live in pinned host buffers (no host-side
# copy); at most this many per resolution, further frames a caller still holds
# go to pageable memory
PINNED_FRAMES = 2
# the walk kernel stores the frame straight into the mapped pinned buffer (the
# D2H overlaps the walk instead of following it); off: render to HBM + copy
ZERO_COPY_FRAMES = os.environ.get("RFB_ZERO_COPY", "1") != "0"


@dataclass
class RenderStats:
    rays: int = 0
    cells_stepped: int = 0
    neighbor_visits: int = 0
    grid_queries: int = 0
    failed_rays: int = 0
    seconds: float = 0.0

    @property
    def rays_per_sec(self):
        return self.rays / self.seconds if self.seconds > 0 else 0.0

    def merge(self, other):
        self.rays += other.rays
        self.cells_stepped += other.cells_stepped
        self.neighbor_visits += other.neighbor_visits
        self.grid_queries += other.grid_queries
        self.failed_rays += other.failed_rays
        self.seconds += other.seconds


@dataclass
class Ray:
    """rays.py:17-36 (validated single ray)."""
    origin: np.ndarray
    direction: np.ndarray
    t_min: float = 0.0
    t_max: float = np.inf

    def __post_init__(self):
        self.origin = np.asarray(self.origin, dtype=np.float64)
        self.direction = np.asarray(self.direction, dtype=np.float64)
        if self.origin.shape != (3,) or self.direction.shape != (3,):
            raise ShapeMismatch("ray origin/direction must be 3-vectors")
        norm = float(np.linalg.norm(self.direction))
        if abs(norm - 1.0) > 1e-6:
            raise ValueError(f"ray direction not unit length (|d| = {norm:g})")
        if not (0.0 <= self.t_min < self.t_max):
            raise ValueError("require 0 <= t_min < t_max")

    def at(self, t):
        return self.origin + t * self.direction


@dataclass
class RaySegments:
    """rays.py:39-57."""
    cells: np.ndarray
    t_entry: np.ndarray
    t_exit: np.ndarray
    residual_transmittance: float
    status: int = STATUS_OK

    def __len__(self):
        return len(self.cells)

    def widths(self):
        return self.t_exit - self.t_entry

    def midpoints(self, ray):
        mid = 0.5 * (self.t_entry + self.t_exit)
        return ray.origin[None, :] + mid[:, None] * ray.direction[None, :]


def intersect_face(ray, x, x_prime):
    """rays.py:60-78: depth of the bisector-plane crossing between sites x and
    x' and whether the face is a candidate exit of x's cell."""
    x = np.asarray(x, dtype=np.float64)
    xp = np.asarray(x_prime, dtype=np.float64)
    if np.array_equal(x, xp):
        raise ValueError("sites coincide; no bisector plane")
    n = xp - x
    denom = float(ray.direction @ n)
    if denom == 0.0:
        return np.inf, False
    return float((0.5 * (x + xp) - ray.origin) @ n) / denom, denom > 0.0


@dataclass
class EffectPlane:
    """rays.py:123-136: a tagged interface for mirror / refraction effects."""
    point: np.ndarray
    normal: np.ndarray
    kind: str = "mirror"
    eta: float = 1.5

    def __post_init__(self):
        self.point = np.asarray(self.point, dtype=np.float64)
        self.normal = np.asarray(self.normal, dtype=np.float64)
        self.normal = self.normal / np.linalg.norm(self.normal)
        if self.kind not in ("mirror", "refract"):
            raise ValueError(f"unknown effect kind {self.kind!r}")


def reflect(direction, normal):
    """rays.py:139-142."""
    d = np.asarray(direction, dtype=np.float64)
    n = np.asarray(normal, dtype=np.float64)
    return d - 2.0 * float(d @ n) * n


def refract(direction, normal, eta):
    """rays.py:145-163: Snell refraction into a medium of relative index eta;
    the back side flips the normal and inverts the ratio, total internal
    reflection falls back to the mirror direction."""
    d = np.asarray(direction, dtype=np.float64)
    n = np.asarray(normal, dtype=np.float64)
    cos_i = float(-d @ n)
    if cos_i < 0.0:
        n, eta = -n, 1.0 / eta
        cos_i = float(-d @ n)
    ratio = 1.0 / eta
    sin2_t = ratio * ratio * (1.0 - cos_i * cos_i)
    if sin2_t > 1.0:
        return reflect(d, n)
    out = ratio * d + (ratio * cos_i - np.sqrt(1.0 - sin2_t)) * n
    return out / np.linalg.norm(out)


def apply_effect(ray, normal, effect, eta=1.5, at_t=0.0):
    """rays.py:166-176: continue `ray` across an effect interface at depth at_t."""
    if effect in ("reflect", "mirror"):
        d = reflect(ray.direction, normal)
    elif effect == "refract":
        d = refract(ray.direction, normal, eta)
    else:
        raise ValueError(f"unknown effect {effect!r}")
    return Ray(ray.at(at_t), d / np.linalg.norm(d), 0.0, ray.t_max)


def effect_rays(origins, directions, t_at, normal, effect="mirror", eta=1.5):
    """Batched apply_effect for host arrays through librfb (rfb_effect_rays):
    (m,3) origins/directions, (m,) or scalar t_at -> new (origins, directions)."""
    o = torch.from_numpy(np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)).cuda()
    d = torch.from_numpy(np.ascontiguousarray(directions, dtype=np.float64).reshape(-1, 3)).cuda()
    oo, od = dv.effect_rays_device(o, d, torch.as_tensor(t_at, dtype=torch.float64).cuda(),
                                   normal, effect, eta)
    return oo.cpu().numpy(), od.cpu().numpy()


def _default_t_max(adj, ray):
    """rays.py:118-120."""
    to_center = 0.5 * (adj.bbox_lo + adj.bbox_hi) - ray.origin
    return float(np.linalg.norm(to_center) + 2.0 * adj.diagonal + 1.0)


def _default_t_max_batch(adj, origins, directions):
    """render.py:170-173 (``_default_t_max(adj, Ray(o_k, d_k))`` per ray) without the
    per-ray Python loop: the same unit-direction validation as Ray (rays.py:29-31),
    and the scalar expression evaluated once per distinct origin, so every value
    has the reference's bits."""
    m = len(origins)
    if m == 0:
        return np.zeros(0)
    norms = np.linalg.norm(directions, axis=1)
    bad = np.flatnonzero(np.abs(norms - 1.0) > 1e-6)
    if len(bad):
        raise ValueError(f"ray direction not unit length (|d| = {norms[bad[0]]:g})")
    center = 0.5 * (adj.bbox_lo + adj.bbox_hi)

    def one(o):
        return float(np.linalg.norm(center - o) + 2.0 * adj.diagonal + 1.0)

    if np.ptp(origins, axis=0).max() == 0.0:
        return np.full(m, one(origins[0]))
    uniq, inv = np.unique(origins, axis=0, return_inverse=True)
    return np.array([one(u) for u in uniq])[inv.reshape(-1)]


def _device_scene(scene, device_scene):
    if device_scene is not None:
        return device_scene
    return dv.DeviceScene(scene)


def _to_dev(a, dtype, device):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).to(device, non_blocking=False)


def render_ray_batch(scene, origins, directions, t_min=None, t_max=None, start_sites=None,
                     epsilon=DEFAULT_EPSILON, step_limit=DEFAULT_STEP_LIMIT, workers=None,
                     stats=None, return_wsum=False, device_scene=None, lanes_per_ray=None):
    """Forward-render arbitrary rays; returns (rgb, residual, status[, wsum]).

    ``workers`` is accepted for signature compatibility (the GPU has no
    worker pool).  Start cells: one device point location when all origins
    coincide, else one per ray (render.py:78-90).
    """
    ds = _device_scene(scene, device_scene)
    dev = ds.device
    origins = np.ascontiguousarray(origins, dtype=np.float64)
    directions = np.ascontiguousarray(directions, dtype=np.float64)
    m = len(origins)
    if t_min is None:
        t_min = np.zeros(m)
    if t_max is None:
        t_max = np.full(m, np.nan)
    t_min = np.ascontiguousarray(t_min, dtype=np.float64)
    t_max = np.ascontiguousarray(t_max, dtype=np.float64)
    if m > 0:
        fallback = ds.default_t_max(origins)
        t_max = np.where(np.isfinite(t_max), t_max, fallback)
    o_d = _to_dev(origins.reshape(m, 3), np.float64, dev)
    d_d = _to_dev(directions.reshape(m, 3), np.float64, dev)
    tmin_d = _to_dev(t_min, np.float64, dev)
    tmax_d = _to_dev(t_max, np.float64, dev)
    if start_sites is None:
        if m > 0 and np.ptp(origins, axis=0).max() == 0.0:
            s0 = ds.locate(o_d[:1])
            start_d = s0.expand(m).contiguous()
            grid_queries = 1
        elif m > 0:
            seed = int(ds.locate(o_d[:1]).item())
            start_d = ds.locate(o_d, seed=seed)
            grid_queries = m
        else:
            start_d = torch.empty(0, dtype=torch.int32, device=dev)
            grid_queries = 0
    else:
        start_d = _to_dev(start_sites, np.int32, dev)
        grid_queries = 0
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    order, auto_lanes = dv.forward_schedule(o_d, d_d)  # scheduling only
    if lanes_per_ray is None:
        lanes_per_ray = auto_lanes
    res = dv.render_rays_device(ds, o_d, d_d, tmin_d, tmax_d, start_d, epsilon=epsilon,
                                step_limit=step_limit, f64=True, per_ray=False,
                                lanes_per_ray=lanes_per_ray, order=order)
    torch.cuda.synchronize(dev)
    dt = time.perf_counter() - t0
    rgb = res.rgb.cpu().numpy()
    residual = res.residual.cpu().numpy()
    status = res.status.cpu().numpy()
    if stats is not None:
        cnt = res.counters.cpu().numpy()
        stats.merge(RenderStats(rays=m, cells_stepped=int(cnt[0]), neighbor_visits=int(cnt[1]),
                                grid_queries=grid_queries,
                                failed_rays=int((status != STATUS_OK).sum()), seconds=dt))
    if return_wsum:
        return rgb, residual, status, res.wsum.cpu().numpy()
    return rgb, residual, status


def render_image(scene, camera, epsilon=DEFAULT_EPSILON, step_limit=DEFAULT_STEP_LIMIT,
                 workers=None, stats=None, weight_check=False, device_scene=None,
                 lanes_per_ray=dv.DEFAULT_LANES):
    """Render a full frame; returns (H, W, 3) float64 image [, wsum, residual].

    Ray generation, the shared-origin start cell and the walk all run on the
    device in one pass (rfb_render_image).
    """
    ds = _device_scene(scene, device_scene)
    H, W = camera.height, camera.width
    fc = _frame_cache(ds, W, H, weight_check)
    # The frame goes to a free pinned buffer of this resolution and the caller
    # gets a view of it (no host-side copy); a buffer is free once the caller
    # dropped the image it holds.  With ZERO_COPY_FRAMES the kernel writes the
    # buffer directly through its mapped device address, otherwise it renders
    # to HBM and one D2H follows.  With PINNED_FRAMES buffers in use the frame
    # goes to fresh pageable memory instead (slower, but callers that keep
    # every frame never accumulate pinned memory).
    # [pinned tensor, weakref to the array handed out, mapped address]; shared by
    # every scene on this device at this resolution (a fresh DeviceScene per call
    # does not pay the page-locked allocation again)
    pool = _PINNED_POOLS.setdefault((str(ds.device), W, H, ZERO_COPY_FRAMES), [])
    free = next((e for e in pool if e[1] is None or e[1]() is None), None)
    if free is None and len(pool) < PINNED_FRAMES:
        h = torch.empty((W * H, 3), dtype=torch.float64, pin_memory=True)
        free = [h, None, dv.host_device_pointer(ds.lib, h) if ZERO_COPY_FRAMES else None]
        pool.append(free)
    direct = free is not None and free[2] is not None
    if stats is not None:  # counters and the timer only matter for stats
        fc["out"].counters.zero_()
        torch.cuda.synchronize(ds.device)
    t0 = time.perf_counter()
    res = dv.render_image_device(ds, camera, epsilon=epsilon, step_limit=step_limit, f64=True,
                                 tile_ids=fc["tiles"], lanes_per_ray=lanes_per_ray,
                                 workspace=fc["ws"], out=fc["out"],
                                 rgb_ptr=free[2] if direct else None)
    if free is not None:
        if not direct:
            free[0].copy_(res.rgb, non_blocking=True)
        root = free[0].numpy()
        free[1] = weakref.ref(root)
    else:
        root = np.empty((W * H, 3), dtype=np.float64)
        torch.from_numpy(root).copy_(res.rgb)
    if weight_check:
        fc["h_wsum"].copy_(res.wsum, non_blocking=True)
        fc["h_resid"].copy_(res.residual, non_blocking=True)
    torch.cuda.current_stream(ds.device).synchronize()
    dt = time.perf_counter() - t0
    img = root.reshape(H, W, 3)
    if stats is not None:
        cnt = res.counters.cpu().numpy()
        status = res.status.cpu().numpy()
        stats.merge(RenderStats(rays=H * W, cells_stepped=int(cnt[0]),
                                neighbor_visits=int(cnt[1]), grid_queries=1,
                                failed_rays=int((status != STATUS_OK).sum()), seconds=dt))
    if weight_check:
        return (img, fc["h_wsum"].numpy().reshape(H, W).copy(),
                fc["h_resid"].numpy().reshape(H, W).copy())
    return img


_PINNED_POOLS: dict = {}


def _frame_cache(ds, W, H, weight_check):
    """Per-(scene, resolution) device outputs, workspace and pinned host
    buffers, so the public render_image call does no allocation after the
    first frame."""
    cache = ds.__dict__.setdefault("_frame_cache", {})
    key = (W, H)
    fc = cache.get(key)
    if fc is None:
        tx, ty = dv.tile_grid(W, H)
        fc = {"ws": dv.Workspace(ds.device),
              "out": dv.alloc_forward(W * H, ds.device, f64=True, per_ray=False),
              "tiles": torch.arange(tx * ty, dtype=torch.int32, device=ds.device)}
        cache[key] = fc
    if weight_check and "h_wsum" not in fc:
        fc["h_wsum"] = torch.empty(W * H, dtype=torch.float64, pin_memory=True)
        fc["h_resid"] = torch.empty(W * H, dtype=torch.float64, pin_memory=True)
    return fc


def render_rays_with_gradients(scene, origins, directions, adjoints, t_min=None, t_max=None,
                               start_sites=None, epsilon=DEFAULT_EPSILON,
                               step_limit=DEFAULT_STEP_LIMIT, grad=None, device_scene=None):
    """Forward+backward for arbitrary per-ray colour adjoints; returns
    (rgb (m,3) f64, GradientBuffer).  Gradients accumulate into ``grad``."""
    ds = _device_scene(scene, device_scene)
    adj = scene.require_adjacency()
    dev = ds.device
    origins = np.ascontiguousarray(origins, dtype=np.float64)
    directions = np.ascontiguousarray(directions, dtype=np.float64)
    adjoints = np.ascontiguousarray(adjoints, dtype=np.float64)
    m = len(origins)
    if t_min is None:
        t_min = np.zeros(m)
    t_min = np.ascontiguousarray(t_min, dtype=np.float64)
    if t_max is None:
        t_max = _default_t_max_batch(adj, origins, directions)
    t_max = np.ascontiguousarray(t_max, dtype=np.float64)
    o_d = _to_dev(origins.reshape(m, 3), np.float64, dev)
    d_d = _to_dev(directions.reshape(m, 3), np.float64, dev)
    if start_sites is None:
        # host expression o + t_min*d (render.py:175-176), evaluated in numpy
        # for bit-identical query points, then located on device
        q = _to_dev(origins + t_min[:, None] * directions, np.float64, dev)
        seed = int(ds.locate(q[:1]).item()) if m else 0
        start_d = ds.locate(q, seed=seed)
    else:
        start_d = _to_dev(start_sites, np.int32, dev)
    n = ds.n_sites
    if grad is None:
        grad = GradientBuffer(n)
    gb = dv.GradBuffers(n, dev)
    res = dv.backward_rays_device(ds, o_d, d_d, _to_dev(t_min, np.float64, dev),
                                  _to_dev(t_max, np.float64, dev), start_d,
                                  _to_dev(adjoints.reshape(m, 3), np.float64, dev), gb,
                                  epsilon=epsilon, step_limit=step_limit, f64=True)
    torch.cuda.synchronize(dev)
    # fp32 accumulators come back as fp32 (half the bytes) and are widened by the +=
    g4 = gb.g4.cpu().numpy()
    grad.d_position += g4[:, :3]
    grad.d_sh += gb.sh.cpu().numpy().reshape(n, 16, 3)
    grad.d_raw_density += g4[:, 3] * softplus_grad(scene.raw_density)
    return res.rgb.cpu().numpy(), grad


def trace(scene, ray, epsilon=DEFAULT_EPSILON, step_limit=DEFAULT_STEP_LIMIT, start_site=None,
          counters=None, device_scene=None):
    """Walk one ray (rays.py:81-115); raises StepLimit / CycleDetected."""
    ds = _device_scene(scene, device_scene)
    adj = scene.require_adjacency()
    dev = ds.device
    t_max = ray.t_max
    if not np.isfinite(t_max):
        t_max = _default_t_max(adj, ray)
    o_d = _to_dev(ray.origin[None, :], np.float64, dev)
    d_d = _to_dev(ray.direction[None, :], np.float64, dev)
    if start_site is None:
        start_d = ds.locate(_to_dev(ray.at(ray.t_min)[None, :], np.float64, dev))
    else:
        start_d = torch.tensor([int(start_site)], dtype=torch.int32, device=dev)
    res = dv.render_rays_device(ds, o_d, d_d, _to_dev([ray.t_min], np.float64, dev),
                                _to_dev([t_max], np.float64, dev), start_d, epsilon=epsilon,
                                step_limit=step_limit, f64=True, per_ray=True,
                                seg_capacity=step_limit)
    torch.cuda.synchronize(dev)
    status = int(res.status.item())
    nseg = int(res.nseg.item())
    if counters is not None:
        rc = res.ray_counters.cpu().numpy()[0]
        counters[0, 0] += int(rc[0])
        counters[0, 1] += int(rc[1])
    if status == STATUS_STEP_LIMIT:
        raise StepLimit(f"ray exceeded {step_limit} cells")
    if status == STATUS_CYCLE:
        raise CycleDetected("walk stalled; same cell revisited without advancing")
    cells = res.seg_cells[0, :nseg].cpu().numpy().astype(np.int64)
    t0 = res.seg_t0[0, :nseg].cpu().numpy()
    t1 = res.seg_t1[0, :nseg].cpu().numpy()
    # walk_ray's residual is exp(log_T) (kernels.py:142); recompute it on the
    # host from the recorded segments with the same accumulation order (and
    # libm's exp, like numba's, rather than numpy's vectorised one)
    sig = softplus(scene.raw_density)
    log_T = 0.0
    for c, a, b in zip(cells.tolist(), t0.tolist(), t1.tolist()):
        log_T -= float(sig[c]) * (b - a)
    return RaySegments(cells, t0, t1, math.exp(log_T), status)
