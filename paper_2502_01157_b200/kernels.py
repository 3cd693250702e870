"""Flat-array drop-ins for ``rfoam.tracer.kernels``.

Same positional signatures, dtypes and in-place output semantics as the
reference's numba functions, so a caller (``render.py:103``,
``train.py:174``) can swap the module:

  render_rays   tracer/kernels.py:199-247
  train_batch   tracer/kernels.py:372-453
  walk_ray      tracer/kernels.py:76-162   (single ray, returns (nseg, status, residual))
  sh_basis_into, cell_color, composite_segments, backward_ray,
  face_t_gradient, quantile_backward_ray     kernels.py:38-73, 165-196, 250-369, 456-567
                (single ray over given segments, via rfb_segments.cu)

The GPU has no worker pool: ``n_workers`` is accepted, every ray's
contribution lands in worker 0's slice of the per-worker buffers
(``d_*_w[0]``, ``loss_w[0]``, ``counters[0]``), so the caller's reduction in
worker order (train.py:189-193) yields the full sum.  ``scratch_*`` arguments
are accepted and ignored (device scratch is internal).  Gradients accumulate
(+=) like the reference; the device sums them in fp32.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import device as dv

STATUS_OK = 0
STATUS_STEP_LIMIT = 2
STATUS_CYCLE = 3


def _dev(a, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


# One cached device scene per adjacency: the reference's callers pass the same
# CSR arrays on every call between rebuilds (train.py:174-188 reads
# adj.offsets / adj.neighbors) while positions, sigma and SH change, so the
# CSR stays on the device and only the parameters are re-uploaded and
# re-packed (DeviceScene.update_params).  Keyed on the CSR arrays' identity,
# address and shape, with references held so an id cannot be reused.
_SCENE_CACHE: dict = {}


def _scene(positions, offsets, neighbors, sigma, sh, background, slot="shade"):
    """slot "shade": full scene; "walk": geometry only (SH never uploaded again)."""
    n = len(positions)
    offsets = np.asarray(offsets)
    neighbors = np.asarray(neighbors)
    key = (id(offsets), id(neighbors), n, len(neighbors), offsets.ctypes.data,
           neighbors.ctypes.data, int(offsets[-1]) if n else 0)
    hit = _SCENE_CACHE.get(slot)
    if hit is not None and hit[0] == key and hit[1] is offsets and hit[2] is neighbors:
        ds = hit[3]
        ds.update_params(positions, sigma,
                         None if slot == "walk" else np.asarray(sh).reshape(n, 48), background)
        return ds
    sh = np.zeros((n, 48)) if slot == "walk" else np.asarray(sh).reshape(n, 48)
    ds = dv.DeviceScene.from_arrays(positions, offsets, neighbors, sigma, sh, background,
                                    keep_csr64=True)
    _SCENE_CACHE[slot] = (key, offsets, neighbors, ds)
    return ds


def render_rays(positions, offsets, neighbors, sigma, sh, background, origins, directions,
                t_min, t_max, start_sites, epsilon, step_limit, width_floor, n_workers, out_rgb,
                out_residual, out_status, out_wsum, counters, scratch_cells=None,
                scratch_t0=None, scratch_t1=None):
    """kernels.py:199-247 on the GPU; fills out_* in place, counters[0] +=."""
    ds = _scene(positions, offsets, neighbors, sigma, sh, background)
    ds.width_floor = float(width_floor)
    m = len(origins)
    if m == 0:
        return
    o, d = _dev(origins).view(m, 3), _dev(directions).view(m, 3)
    order, lanes = dv.forward_schedule(o, d)
    res = dv.render_rays_device(ds, o, d, _dev(t_min), _dev(t_max), _dev(start_sites, torch.int32),
                                epsilon=epsilon, step_limit=int(step_limit), f64=True,
                                per_ray=False, order=order, lanes_per_ray=lanes)
    torch.cuda.synchronize()
    out_rgb[...] = res.rgb.cpu().numpy().reshape(out_rgb.shape)
    out_residual[...] = res.residual.cpu().numpy()
    out_status[...] = res.status.cpu().numpy()
    out_wsum[...] = res.wsum.cpu().numpy()
    counters[0, :] += res.counters.cpu().numpy().astype(counters.dtype)


def walk_ray(positions, offsets, neighbors, sigma, ox, oy, oz, dx, dy, dz, t_min, t_max,
             start_site, epsilon, step_limit, width_floor, seg_cells, seg_t0, seg_t1, counters,
             worker):
    """kernels.py:76-162 for one ray: fills seg_* and returns (nseg, status, residual)."""
    ds = _scene(positions, offsets, neighbors, sigma, None, np.zeros(3), slot="walk")
    ds.width_floor = float(width_floor)
    cap = int(step_limit)
    res = dv.render_rays_device(ds, _dev([[ox, oy, oz]]), _dev([[dx, dy, dz]]), _dev([t_min]),
                                _dev([t_max]), _dev([start_site], torch.int32), epsilon=epsilon,
                                step_limit=cap, f64=True, per_ray=True, seg_capacity=cap)
    torch.cuda.synchronize()
    nseg = int(res.nseg.item())
    seg_cells[:nseg] = res.seg_cells[0, :nseg].cpu().numpy()
    seg_t0[:nseg] = res.seg_t0[0, :nseg].cpu().numpy()
    seg_t1[:nseg] = res.seg_t1[0, :nseg].cpu().numpy()
    rc = res.ray_counters.cpu().numpy()[0]
    counters[worker, 0] += int(rc[0])
    counters[worker, 1] += int(rc[1])
    log_t = 0.0  # kernels.py:142 (libm exp, like numba's)
    for c, a, b in zip(seg_cells[:nseg].tolist(), seg_t0[:nseg].tolist(), seg_t1[:nseg].tolist()):
        log_t -= float(sigma[c]) * (b - a)
    return nseg, int(res.status.item()), math.exp(log_t)


def train_batch(positions, offsets, neighbors, sigma, sh, background, origins, directions, t_min,
                t_max, start_sites, targets, epsilon, step_limit, width_floor, rgb_scale,
                quantile_scale, u_pairs, weight_floor, n_workers, out_rgb, out_status, d_sigma_w,
                d_sh_w, d_pos_w, loss_w, counters, scratch_cells=None, scratch_t0=None,
                scratch_t1=None):
    """kernels.py:372-453 on the GPU: accumulates into worker 0's buffers."""
    ds = _scene(positions, offsets, neighbors, sigma, sh, background)
    ds.width_floor = float(width_floor)
    m = len(origins)
    if m == 0:
        return
    gb = dv.GradBuffers(ds.n_sites, ds.device)
    loss = torch.zeros(2, dtype=torch.float64, device=ds.device)
    up = _dev(u_pairs) if quantile_scale > 0.0 else None
    res = dv.train_batch_device(ds, _dev(origins).view(m, 3), _dev(directions).view(m, 3),
                                _dev(t_min), _dev(t_max), _dev(start_sites, torch.int32),
                                _dev(targets).view(m, 3), gb, loss, rgb_scale=float(rgb_scale),
                                quantile_scale=float(quantile_scale), u_pairs=up,
                                weight_floor=float(weight_floor), epsilon=epsilon,
                                step_limit=int(step_limit), f64=True)
    torch.cuda.synchronize()
    out_rgb[...] = res.rgb.cpu().numpy().reshape(out_rgb.shape)
    out_status[...] = res.status.cpu().numpy()
    g4 = gb.g4.cpu().numpy()  # fp32 over the bus, widened by the +=
    d_pos_w[0] += g4[:, :3]
    d_sigma_w[0] += g4[:, 3]
    d_sh_w[0] += gb.sh.cpu().numpy().reshape(d_sh_w[0].shape)
    loss_w[0] += loss.cpu().numpy()
    counters[0, :] += res.counters.cpu().numpy().astype(counters.dtype)


# ---------------------------------------------------------------------------
# Per-ray building blocks (tracer/kernels.py:38-73, 165-196, 250-369, 456-567)
# with the reference's signatures; the arithmetic runs in rfb_segments.cu
# (fp64, reference operation order).  Outputs are written / accumulated in
# place like the numba originals.
# ---------------------------------------------------------------------------
def _one_ray_segments(seg_cells, seg_t0, seg_t1, nseg):
    n = int(nseg)
    off = torch.tensor([0, n], dtype=torch.int64, device="cuda")
    cells = _dev(np.asarray(seg_cells[:n]), torch.int32)
    return off, cells, _dev(np.asarray(seg_t0[:n])), _dev(np.asarray(seg_t1[:n]))


def sh_basis_into(dx, dy, dz, out):
    """kernels.py:38-58."""
    b = dv.sh_basis_device(torch.tensor([[dx, dy, dz]], dtype=torch.float64, device="cuda"))
    out[:16] = b.cpu().numpy()[0]


def cell_color(sh, i, basis, out):
    """kernels.py:61-73: clamped colour of cell i; returns the clamp mask."""
    row = _dev(np.asarray(sh).reshape(-1, 48)[int(i)][None, :])
    col, mask = dv.cell_colors_device(row, torch.zeros(1, dtype=torch.int32, device="cuda"),
                                      _dev(np.asarray(basis, dtype=np.float64)[None, :16]))
    out[:3] = col.cpu().numpy()[0]
    return int(mask.item())


def composite_segments(seg_cells, seg_t0, seg_t1, nseg, sigma, sh, basis, bg_r, bg_g, bg_b,
                       out_rgb):
    """kernels.py:165-196: returns (residual transmittance, weight sum)."""
    off, cells, t0, t1 = _one_ray_segments(seg_cells, seg_t0, seg_t1, nseg)
    rgb, T, ws = dv.composite_segments_device(
        _dev(sigma), _dev(np.asarray(sh).reshape(-1, 48)),
        _dev(np.asarray(basis, dtype=np.float64)[None, :16]), off, cells, t0, t1,
        (bg_r, bg_g, bg_b))
    out_rgb[:3] = rgb.cpu().numpy()[0]
    return float(T.item()), float(ws.item())


def backward_ray(positions, offsets, neighbors, sigma, sh, background, ox, oy, oz, dx, dy, dz,
                 adj_r, adj_g, adj_b, seg_cells, seg_t0, seg_t1, nseg, t_min_q, basis, d_sigma,
                 d_sh, d_pos):
    """kernels.py:250-337: accumulates into d_sigma (n), d_sh (n, 48), d_pos (n, 3)."""
    if int(nseg) == 0:
        return
    off, cells, t0, t1 = _one_ray_segments(seg_cells, seg_t0, seg_t1, nseg)
    n = len(sigma)
    gs = torch.zeros(n, dtype=torch.float64, device="cuda")
    gsh = torch.zeros((n, 48), dtype=torch.float64, device="cuda")
    gp = torch.zeros((n, 3), dtype=torch.float64, device="cuda")
    dv.backward_segments_device(
        _dev(positions), _dev(sigma), _dev(np.asarray(sh).reshape(-1, 48)), background,
        _dev(np.array([[ox, oy, oz]])), _dev(np.array([[dx, dy, dz]])),
        _dev(np.asarray(basis, dtype=np.float64)[None, :16]),
        _dev(np.array([[adj_r, adj_g, adj_b]])), off, cells, t0, t1, gs, gsh, gp)
    d_sigma += gs.cpu().numpy()
    d_sh.reshape(n, 48)[...] += gsh.cpu().numpy()
    d_pos += gp.cpu().numpy()


def face_t_gradient(positions, i, j, ox, oy, oz, dx, dy, dz, t, dt, d_pos):
    """kernels.py:340-369: accumulates dt * dt/d(x_i, x_j) into d_pos (n, 3)."""
    gp = torch.zeros((len(positions), 3), dtype=torch.float64, device="cuda")
    dv.face_t_gradients_device(
        _dev(positions), torch.tensor([[int(i), int(j)]], dtype=torch.int32, device="cuda"),
        _dev(np.array([[ox, oy, oz]])), _dev(np.array([[dx, dy, dz]])), _dev(np.array([t])),
        _dev(np.array([dt])), gp)
    d_pos += gp.cpu().numpy()


def quantile_backward_ray(seg_cells, seg_t0, seg_t1, nseg, sigma, u_pair, weight_floor,
                          positions, ox, oy, oz, dx, dy, dz, scale, d_sigma, d_pos):
    """kernels.py:456-567: one (u1, u2) pair; returns the loss term."""
    if int(nseg) == 0:
        return 0.0
    off, cells, t0, t1 = _one_ray_segments(seg_cells, seg_t0, seg_t1, nseg)
    n = len(sigma)
    gs = torch.zeros(n, dtype=torch.float64, device="cuda")
    gp = torch.zeros((n, 3), dtype=torch.float64, device="cuda")
    loss = dv.quantile_segments_device(
        _dev(positions), _dev(sigma), _dev(np.array([[ox, oy, oz]])),
        _dev(np.array([[dx, dy, dz]])), off, cells, t0, t1,
        _dev(np.asarray(u_pair, dtype=np.float64).reshape(1, 1, 2)), weight_floor, scale, gs, gp)
    d_sigma += gs.cpu().numpy()
    d_pos += gp.cpu().numpy()
    return float(loss.item())
