"""Flat-array drop-ins for ``rfoam.tracer.kernels``.

Same positional signatures, dtypes and in-place output semantics as the
reference's numba functions, so a caller (``render.py:103``,
``train.py:174``) can swap the module:

  render_rays   tracer/kernels.py:199-247
  train_batch   tracer/kernels.py:372-453
  walk_ray      tracer/kernels.py:76-162   (single ray, returns (nseg, status, residual))

The GPU has no worker pool: ``n_workers`` is accepted, every ray's
contribution lands in worker 0's slice of the per-worker buffers
(``d_*_w[0]``, ``loss_w[0]``, ``counters[0]``), so the caller's reduction in
worker order (train.py:189-193) yields the full sum.  ``scratch_*`` arguments
are accepted and ignored (device scratch is internal).  Gradients accumulate
(+=) like the reference; the device sums them in fp32.
"""

from __future__ import annotations

import numpy as np
import torch

from . import device as dv

STATUS_OK = 0
STATUS_STEP_LIMIT = 2
STATUS_CYCLE = 3


def _dev(a, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)


def _scene(positions, offsets, neighbors, sigma, sh, background):
    return dv.DeviceScene.from_arrays(positions, offsets, neighbors, sigma,
                                      np.asarray(sh).reshape(len(positions), 48), background)


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
    res = dv.render_rays_device(ds, _dev(origins).view(m, 3), _dev(directions).view(m, 3),
                                _dev(t_min), _dev(t_max), _dev(start_sites, torch.int32),
                                epsilon=epsilon, step_limit=int(step_limit), f64=True,
                                per_ray=False)
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
    n = len(positions)
    ds = _scene(positions, offsets, neighbors, sigma, np.zeros((n, 48)), np.zeros(3))
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
    log_t = 0.0
    for c, a, b in zip(seg_cells[:nseg], seg_t0[:nseg], seg_t1[:nseg]):
        log_t -= sigma[c] * (b - a)
    return nseg, int(res.status.item()), float(np.exp(log_t))


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
    g4 = gb.g4.double().cpu().numpy()
    d_pos_w[0] += g4[:, :3]
    d_sigma_w[0] += g4[:, 3]
    d_sh_w[0] += gb.sh.double().cpu().numpy().reshape(d_sh_w[0].shape)
    loss_w[0] += loss.cpu().numpy()
    counters[0, :] += res.counters.cpu().numpy().astype(counters.dtype)
