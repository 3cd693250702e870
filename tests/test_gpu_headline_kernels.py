"""Parity of the exact kernel instantiations the benchmark numbers come from.

bench.py's headline lines run one lane per ray: k_render<1, 3, 1, TileRays>
(config 2, rfb_render_image over 32x32 tiles) and k_train<3, 1, *, *, 1>
(config 3, a full view in tile order).  The library's auto rules pick one
lane only for batches larger than about half the resident threads
(rfb.cu launch_render / train_lanes), so the small golden frames never
reach them; here the frames are large enough for the auto rule AND the
lane count is forced, on a 100k-site foam (Qhull CSR):

* every ray's visited-cell sequence and segment depths bit-exact (per-ray
  walk_digest of the device's segment dump == the C oracle's), counters,
  nseg and status bit-exact, image / wsum / residual within 1e-4 abs;
* training (L2 loss, quantile off and on) and the generic adjoint backward:
  per-tensor gradients within 1e-3 relative (max|d - ref| / max|ref|), loss
  within 1e-6 relative (reference: tracer/kernels.py:199-247, 250-453).
"""

import os

import numpy as np
import pytest
import torch

from oracle import oracle as orc
from oracle.walk_digest import digests

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-4
GRAD_RTOL = 1e-3


@pytest.fixture(scope="module")
def scene100k():
    from paper_2502_01157_b200.synthetic import make_foam

    return make_foam(100_000, 21, 3)


@pytest.fixture(scope="module")
def sa100k(scene100k):
    from paper_2502_01157_b200.scene import softplus

    adj = scene100k.adjacency
    return orc.SceneArrays(adj.positions, adj.offsets, adj.neighbors,
                           softplus(scene100k.raw_density), scene100k.sh_coeffs.reshape(-1, 48),
                           scene100k.background)


@pytest.fixture(scope="module")
def ds100k(scene100k):
    from paper_2502_01157_b200 import device as dv

    return dv.DeviceScene(scene100k)


def _cam(W, H, k=0):
    from bench import make_views

    return make_views(k + 1, W, H)[k]


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / np.abs(b).max())


@pytest.mark.parametrize("view,eps,cull", [(0, 1e-3, True), (2, 0.0, True), (0, 1e-3, False)])
def test_render_image_one_lane_per_ray(cuda_ok, scene100k, sa100k, ds100k, view, eps, cull):
    """k_render<1, 3, 1, TileRays> (the config-2 kernel) on a 480x270 frame, over the
    view-culled rows (the default, rfb_cull_scene) and over the full rows."""
    from paper_2502_01157_b200 import device as dv

    W, H = 480, 270
    m = W * H
    assert 2 * m > 148 * 4 * 256, "frame must be large enough for the auto rule to pick 1 lane"
    cam = _cam(W, H, view)
    first = dv.render_image_device(ds100k, cam, epsilon=eps, f64=True, per_ray=True,
                                   lanes_per_ray=1, cull=cull)
    torch.cuda.synchronize()
    cap = int(first.nseg.max().item())
    out = dv.alloc_forward(m, ds100k.device, f64=True, per_ray=True, seg_capacity=cap)
    res = dv.render_image_device(ds100k, cam, epsilon=eps, lanes_per_ray=1, out=out, cull=cull)
    auto = dv.render_image_device(ds100k, cam, epsilon=eps, f64=True, per_ray=True, cull=cull)
    torch.cuda.synchronize()
    assert torch.equal(auto.rgb, res.rgb) and torch.equal(auto.ray_counters, res.ray_counters)

    dirs = cam.ray_directions()
    o = cam.position
    start = int(orc.nearest_sites(sa100k.positions, o[None, :])[0])
    t_max = float(np.linalg.norm(o - sa100k.center) + 2.0 * sa100k.diagonal + 1.0)
    ref = orc.render_rays(sa100k, np.broadcast_to(o, (m, 3)), dirs, 0.0, t_max, start,
                          epsilon=eps, threads=os.cpu_count() or 8, digest=True)
    np.testing.assert_array_equal(res.status.cpu().numpy(), ref["status"])
    np.testing.assert_array_equal(res.nseg.cpu().numpy(), ref["nseg"])
    np.testing.assert_array_equal(res.ray_counters.cpu().numpy(), ref["counters"])
    np.testing.assert_array_equal(res.counters.cpu().numpy(), ref["counters"].sum(axis=0))
    dig = digests(res.seg_cells, res.seg_t0, res.seg_t1, res.nseg)
    bad = np.flatnonzero(dig != ref["digest"])
    assert len(bad) == 0, f"{len(bad)} rays differ in cells/t0/t1, first {bad[:5]}"
    assert np.abs(res.rgb.cpu().numpy() - ref["rgb"]).max() <= IMG_TOL
    assert np.abs(res.wsum.cpu().numpy() - ref["wsum"]).max() <= IMG_TOL
    assert np.abs(res.residual.cpu().numpy() - ref["residual"]).max() <= IMG_TOL


def _view_batch(cam, ds, order_tiles=True):
    from paper_2502_01157_b200 import device as dv

    W, H = cam.width, cam.height
    dirs = cam.ray_directions()
    m = len(dirs)
    if order_tiles:  # the bench's config-3 schedule: rays in rfb_render_image's tile order
        perm = dv.tile_order(W, H)
        dirs = dirs[perm]
    o = np.broadcast_to(cam.position, (m, 3)).copy()
    start = int(ds.locate(torch.from_numpy(o[:1]).cuda()).item())
    t_max = np.full(m, ds.default_t_max(cam.position[None, :]))
    return o, dirs, start, t_max


def _d(a, dt=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)


@pytest.mark.parametrize("quantile,cull", [(False, "regions"), (True, "regions"),
                                           (False, "cone"), (False, None)])
def test_train_batch_one_lane_full_view(cuda_ok, sa100k, ds100k, quantile, cull):
    """k_train<3, 1, true, Q, 1> (the config-3 kernel) on an 81,920-ray view in tile
    order, against the oracle's train_batch (kernels.py:372-453); the bench walks
    the camera's region-culled rows (view = (camera, pixels), rfb_cull_view)."""
    from paper_2502_01157_b200 import device as dv

    W, H = 320, 256
    cam = _cam(W, H, 1)
    o, dirs, start, t_max = _view_batch(cam, ds100k)
    m = len(dirs)
    assert 2 * m > 148 * 7 * 128, "batch must be large enough for the auto rule to pick 1 lane"
    rng = np.random.default_rng(11)
    targets = rng.uniform(0.0, 1.0, (m, 3))
    u = rng.uniform(0.0, 1.0, (m, 2, 2)) if quantile else None
    qs = 0.01 / (m * 2) if quantile else 0.0
    ref = orc.train_batch(sa100k, o, dirs, np.zeros(m), t_max, np.full(m, start), targets,
                          1.0 / (3 * m), qs, u, 1e-4, n_workers=4,
                          threads=os.cpu_count() or 8)
    gb = dv.GradBuffers(ds100k.n_sites, ds100k.device)
    loss = torch.zeros(2, dtype=torch.float64, device="cuda")
    res = dv.train_batch_device(ds100k, _d(o), _d(dirs), _d(np.zeros(m)), _d(t_max),
                                _d(np.full(m, start), torch.int32), _d(targets), gb, loss,
                                rgb_scale=1.0 / (3 * m), quantile_scale=qs,
                                u_pairs=_d(u) if quantile else None, f64=True, order=None,
                                lanes_per_ray=1,
                                view_dirs=dv.view_cone(cam) if cull == "cone" else None,
                                view=(cam, torch.from_numpy(dv.tile_order(W, H)))
                                if cull == "regions" else None)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(res.status.cpu().numpy(), ref["status"])
    np.testing.assert_array_equal(res.counters.cpu().numpy(), ref["counters"].sum(axis=0))
    assert np.abs(res.rgb.cpu().numpy() - ref["rgb"]).max() <= IMG_TOL
    g4 = gb.g4.double().cpu().numpy()
    assert rel(g4[:, 3], ref["d_sigma_w"].sum(0)) <= GRAD_RTOL
    assert rel(g4[:, :3], ref["d_pos_w"].sum(0)) <= GRAD_RTOL
    assert rel(gb.sh.double().cpu().numpy(), ref["d_sh_w"].sum(0)) <= GRAD_RTOL
    np.testing.assert_allclose(loss.cpu().numpy(), ref["loss_w"].sum(0), rtol=1e-6)


def test_backward_rays_one_lane_full_view(cuda_ok, sa100k, ds100k):
    """k_train<3, 1, false, false, 1> (generic adjoint, render.py:152-221) on an
    81,920-ray view against the oracle's sequential render_rays_with_gradients."""
    from paper_2502_01157_b200 import device as dv

    W, H = 320, 256
    cam = _cam(W, H, 3)
    o, dirs, start, t_max = _view_batch(cam, ds100k)
    m = len(dirs)
    adj = np.random.default_rng(5).normal(0.0, 1.0 / m, (m, 3))
    rgb, status, ds_ref, dsh_ref, dp_ref, _ = orc.render_rays_with_gradients(
        sa100k, o, dirs, adj, np.zeros(m), t_max, np.full(m, start))
    gb = dv.GradBuffers(ds100k.n_sites, ds100k.device)
    res = dv.backward_rays_device(ds100k, _d(o), _d(dirs), _d(np.zeros(m)), _d(t_max),
                                  _d(np.full(m, start), torch.int32), _d(adj), gb, f64=True,
                                  order=None, lanes_per_ray=1, view_dirs=dv.view_cone(cam))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(res.status.cpu().numpy(), status)
    assert np.abs(res.rgb.cpu().numpy() - rgb).max() <= IMG_TOL
    g4 = gb.g4.double().cpu().numpy()
    assert rel(g4[:, 3], ds_ref) <= GRAD_RTOL
    assert rel(g4[:, :3], dp_ref) <= GRAD_RTOL
    assert rel(gb.sh.double().cpu().numpy(), dsh_ref) <= GRAD_RTOL


def _check_culled(full_h, full_e, view_h, view_e, cones, n, stride, rows):
    """Region r of a culled view: headers offset by r*stride, every row a CSR-ordered
    subset of the full row, dropped records back-facing with margin for the region's
    generators (kernel: fp32, 2^-18 |n|_1; checked here in fp64 with slack), kept ones
    not back-facing with a clear margin, n1max's low 5 bits = number dropped."""
    k0, k1 = full_h[:, 3], full_h[:, 6]
    n1f = full_h[:, 7].view(np.uint32)
    assert np.all(n1f & 31 == 0)
    tot_drop = tot = 0
    for r, cone in enumerate(cones):
        vh = view_h[r * n:(r + 1) * n]
        assert np.array_equal(vh[:, 3], k0 + r * stride)
        n1v = vh[:, 7].view(np.uint32)
        assert np.array_equal(n1v & ~np.uint32(31), n1f)
        dropped = (n1v & 31).astype(np.int64)
        kept = (vh[:, 6] - vh[:, 3]).astype(np.int64)
        assert np.array_equal(kept + dropped, k1 - k0)
        tot_drop += dropped.sum()
        tot += (k1 - k0).sum()
        c = cone / np.linalg.norm(cone, axis=1, keepdims=True)
        for u in rows:
            row = full_e[k0[u]:k1[u]]
            vrow = view_e[vh[u, 3]:vh[u, 3] + kept[u]]
            ids = row[:, 3].view(np.int32)
            vids = vrow[:, 3].view(np.int32)
            keep = np.isin(ids, vids)
            assert np.array_equal(ids[keep], vids), "CSR order kept"
            nn = row[:, :3].astype(np.float64) - full_h[u, :3].view(np.float32).astype(np.float64)
            dots = nn @ c.T
            l1 = np.abs(nn).sum(1)[:, None]
            assert np.all(dots[~keep] < -2.0 ** -19 * l1[~keep]), "dropped a face not back-facing"
            back = np.all(dots < -2.0 ** -17 * l1, axis=1)
            if keep.all() and back.sum() > 31:
                continue  # would drop more than the 5-bit count holds: copied whole
            assert not np.any(back[keep]), "kept a back face"
            if kept[u] & 1:
                assert np.all(np.isnan(view_e[vh[u, 3] + kept[u]]))
    return tot_drop / tot


def test_view_culled_rows(cuda_ok, ds100k):
    """rfb_cull_scene (one cone: the 4 corner-pixel directions) and rfb_cull_view (a
    4 x 2 grid of image regions, each with its own pixel-edge corner cone): the copies
    of the packed rows hold exactly the faces that are not back-facing for the cone."""
    from paper_2502_01157_b200 import device as dv

    cam = _cam(480, 270, 0)
    n = ds100k.n_sites
    full_h = ds100k.cells.cpu().numpy()
    full_e = ds100k.edges.cpu().numpy()
    rows = np.random.default_rng(0).choice(n, 200, replace=False)
    ds100k.view(dv.view_cone(cam))
    torch.cuda.synchronize()
    frac1 = _check_culled(full_h, full_e, ds100k._view_cells.cpu().numpy(),
                          ds100k._view_edges.cpu().numpy(), [dv.view_cone(cam)], n, 0, rows)
    assert 0.15 < frac1 < 0.4, frac1
    rx, ry = 4, 2
    ds100k.view_camera(cam, regions=(rx, ry))
    torch.cuda.synchronize()
    W, H = cam.width, cam.height
    R = np.asarray(cam.pose)[:3, :3]
    edges_c = [-(-ix * W // rx) for ix in range(rx + 1)]
    edges_r = [-(-iy * H // ry) for iy in range(ry + 1)]
    cones = []
    for iy in range(ry):
        for ix in range(rx):
            pts = [(edges_c[ix + a], edges_r[iy + b]) for b in (0, 1) for a in (0, 1)]
            d = np.array([[(c - cam.cx) / cam.focal, -(r - cam.cy) / cam.focal, -1.0]
                          for c, r in pts])
            cones.append(d @ R.T)
    stride = (ds100k.n_edges + n + 3) & ~1
    deg = full_h[:, 6] - full_h[:, 3]
    long_rows = np.flatnonzero(deg > 31)  # k_cull_rows' chunked path (and its 31-drop cap)
    frac8 = _check_culled(full_h, full_e, ds100k._view_cells.cpu().numpy(),
                          ds100k._view_edges.cpu().numpy(), cones, n, stride,
                          np.concatenate([rows, long_rows[:50]]))
    assert frac8 > frac1


def test_render_image_per_sm_queues_960x540(cuda_ok, sa100k, ds100k):
    """A 960x540 frame (510 tiles): large enough that the per-SM work queues deal tiles
    statically (fetch_unit: 80% of the 32-patch groups round-robin over 148 virtual SMs, the
    rest dynamically) -- every pixel rendered exactly once, each 9th row against the oracle
    (per-ray cells / depths bit-exact via digests, counters, image 1e-4)."""
    from paper_2502_01157_b200 import device as dv

    W, H = 960, 540
    cam = _cam(W, H, 1)
    first = dv.render_image_device(ds100k, cam, f64=True, per_ray=True, lanes_per_ray=1)
    torch.cuda.synchronize()
    cap = int(first.nseg.max().item())
    rows = np.arange(0, H, 9)
    pix = (rows[:, None] * W + np.arange(W)[None, :]).reshape(-1)
    out = dv.alloc_forward(W * H, ds100k.device, f64=True, per_ray=True, seg_capacity=cap)
    res = dv.render_image_device(ds100k, cam, lanes_per_ray=1, out=out)
    torch.cuda.synchronize()
    assert torch.equal(res.rgb, first.rgb) and torch.equal(res.ray_counters, first.ray_counters)
    dirs = cam.ray_directions()[pix]
    o = cam.position
    start = int(orc.nearest_sites(sa100k.positions, o[None, :])[0])
    t_max = float(np.linalg.norm(o - sa100k.center) + 2.0 * sa100k.diagonal + 1.0)
    ref = orc.render_rays(sa100k, np.broadcast_to(o, (len(pix), 3)), dirs, 0.0, t_max, start,
                          threads=os.cpu_count() or 8, digest=True)
    idx = torch.from_numpy(pix).cuda()
    np.testing.assert_array_equal(res.ray_counters[idx].cpu().numpy(), ref["counters"])
    np.testing.assert_array_equal(res.status[idx].cpu().numpy(), ref["status"])
    dig = digests(res.seg_cells[idx], res.seg_t0[idx], res.seg_t1[idx], res.nseg[idx])
    assert int((dig != ref["digest"]).sum()) == 0
    assert np.abs(res.rgb[idx].cpu().numpy() - ref["rgb"]).max() <= IMG_TOL
    # every pixel written by exactly one ray: the frame's counters add up to the per-ray sums
    np.testing.assert_array_equal(res.counters.cpu().numpy(),
                                  res.ray_counters.to(torch.int64).sum(0).cpu().numpy())


def test_view_batch_without_culling(cuda_ok, sa100k, ds100k, monkeypatch):
    """A ray batch passed with view=(camera, pixels) when culling does not apply (culling
    off, or a batch too small to pay for the pass) walks the full rows: same outputs."""
    from paper_2502_01157_b200 import device as dv

    W, H = 160, 96
    cam = _cam(W, H, 1)
    o, dirs, start, t_max = _view_batch(cam, ds100k)
    m = len(dirs)
    perm = torch.from_numpy(dv.tile_order(W, H))
    args = (_d(o), _d(dirs), _d(np.zeros(m)), _d(t_max), _d(np.full(m, start), torch.int32))
    assert not ds100k.can_cull(cam, m)  # 15,360 rays: below the floor
    a = dv.render_rays_device(ds100k, *args, f64=True, view=(cam, perm))
    monkeypatch.setattr(ds100k, "VIEW_CULL", False)
    b = dv.render_rays_device(ds100k, *args, f64=True, view=(cam, perm))
    c = dv.render_rays_device(ds100k, *args, f64=True)
    torch.cuda.synchronize()
    assert torch.equal(a.rgb, c.rgb) and torch.equal(b.rgb, c.rgb)
    assert torch.equal(a.ray_counters, c.ray_counters)
