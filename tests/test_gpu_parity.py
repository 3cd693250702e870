"""CUDA path (librfb.so through the C ABI) vs the CPU oracle and the
reference's golden vectors.

Bars (BASELINE.json north_star): per-ray visited-cell sequences, segment
depths, counters and status bit-exact; images within 1e-4 abs (the kernels
composite in fp64, so the observed gap is ~1e-15); gradients within 1e-3
relative per tensor, measured as max|d - ref| / max|ref| (the device
accumulates in fp32 with unordered atomics).
"""

import numpy as np
import pytest
import torch

from conftest import golden_scene, golden_scene_arrays, load_golden
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

FRAMES = ["frame_2k_deg3", "frame_2k_deg3_eps0_orbit", "frame_10k_deg0", "frame_3k_surface"]
ALL_FRAMES = FRAMES + ["frame_2k_deg3_fisheye"]
IMG_TOL = 1e-4
GRAD_RTOL = 1e-3


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.abs(b).max()
    return float(np.abs(a - b).max() / den) if den > 0 else float(np.abs(a).max())


def _dev(a, dt=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)


def frame_rays(g):
    sa = golden_scene_arrays(g)
    dirs = g["dirs"]
    m = len(dirs)
    origin = g["pose"][:3, 3]
    start = int(orc.nearest_sites(sa.positions, origin[None, :])[0])
    t_max = float(np.linalg.norm(origin - sa.center) + 2.0 * sa.diagonal + 1.0)
    return sa, np.broadcast_to(origin, (m, 3)).copy(), dirs, start, t_max


@pytest.mark.parametrize("lanes,packed", [(1, True), (1, False), (2, True), (4, False),
                                          (8, True), (16, False), (32, True)])
@pytest.mark.parametrize("name", FRAMES)
def test_render_rays_bit_exact_walk(cuda_ok, name, lanes, packed):
    from paper_2502_01157_b200 import device as dv

    g = load_golden(name)
    sa, origins, dirs, start, t_max = frame_rays(g)
    m = len(dirs)
    eps = float(g["epsilon"])
    ds = dv.DeviceScene(golden_scene(g), packed=packed)
    assert ds.packed == packed
    cap = 512
    res = dv.render_rays_device(ds, _dev(origins), _dev(dirs), _dev(np.zeros(m)),
                                _dev(np.full(m, t_max)), _dev(np.full(m, start), torch.int32),
                                epsilon=eps, f64=True, per_ray=True, seg_capacity=cap,
                                lanes_per_ray=lanes)
    torch.cuda.synchronize()
    ref = orc.render_rays(sa, origins, dirs, 0.0, t_max, start, epsilon=eps)
    np.testing.assert_array_equal(res.status.cpu().numpy(), ref["status"])
    np.testing.assert_array_equal(res.nseg.cpu().numpy(), ref["nseg"])
    np.testing.assert_array_equal(res.ray_counters.cpu().numpy(), ref["counters"])
    np.testing.assert_array_equal(res.counters.cpu().numpy(), ref["counters"].sum(axis=0))
    H, W = int(g["height"]), int(g["width"])
    rgb = res.rgb.cpu().numpy()
    assert np.abs(rgb - ref["rgb"]).max() <= IMG_TOL
    assert np.abs(rgb.reshape(H, W, 3) - g["img"]).max() <= IMG_TOL
    assert np.abs(res.wsum.cpu().numpy() - ref["wsum"]).max() <= IMG_TOL
    assert np.abs(res.residual.cpu().numpy() - ref["residual"]).max() <= IMG_TOL
    # every ray's visited-cell sequence and segment depths, bit for bit
    cells = res.seg_cells.cpu().numpy()
    t0 = res.seg_t0.cpu().numpy()
    t1 = res.seg_t1.cpu().numpy()
    for q in range(m):
        c, a, b, st, _, _ = orc.walk_ray(sa, origins[q], dirs[q], 0.0, t_max, start, epsilon=eps)
        L = min(len(c), cap)
        np.testing.assert_array_equal(cells[q, :L], c[:L])
        np.testing.assert_array_equal(t0[q, :L], a[:L])
        np.testing.assert_array_equal(t1[q, :L], b[:L])


@pytest.mark.parametrize("name", ALL_FRAMES)
def test_render_image_matches_reference(cuda_ok, name):
    from paper_2502_01157_b200 import render
    from paper_2502_01157_b200.camera import PINHOLE, CameraModel
    from paper_2502_01157_b200.render import RenderStats

    g = load_golden(name)
    cam = CameraModel(str(g["kind"]), int(g["width"]), int(g["height"]), float(g["focal"]),
                      g["pose"])
    stats = RenderStats()
    img, wsum, resid = render.render_image(golden_scene(g), cam, epsilon=float(g["epsilon"]),
                                           stats=stats, weight_check=True)
    assert np.abs(img - g["img"]).max() <= IMG_TOL
    assert np.abs(wsum - g["wsum"]).max() <= IMG_TOL
    assert np.abs(resid - g["residual"]).max() <= IMG_TOL
    st = g["stats"]
    assert (stats.rays, stats.cells_stepped, stats.neighbor_visits, stats.failed_rays) == tuple(st)


@pytest.mark.parametrize("name", FRAMES)
def test_render_ray_batch_api(cuda_ok, name):
    from paper_2502_01157_b200 import render

    g = load_golden(name)
    origin = g["pose"][:3, 3]
    m = len(g["dirs"])
    rgb, residual, status, wsum = render.render_ray_batch(
        golden_scene(g), np.broadcast_to(origin, (m, 3)), g["dirs"], epsilon=float(g["epsilon"]),
        return_wsum=True)
    H, W = int(g["height"]), int(g["width"])
    assert rgb.dtype == np.float64 and status.dtype == np.int8
    assert np.abs(rgb.reshape(H, W, 3) - g["img"]).max() <= IMG_TOL
    np.testing.assert_array_equal(status, g["status"])


def test_camera_rays_device_bit_exact(cuda_ok):
    g = load_golden("frame_2k_deg3")
    from paper_2502_01157_b200.camera import PINHOLE, CameraModel

    cam = CameraModel(PINHOLE, int(g["width"]), int(g["height"]), float(g["focal"]), g["pose"])
    d = cam.ray_directions_device().cpu().numpy()
    np.testing.assert_array_equal(d, g["dirs"])
    # fisheye: device sin/cos/hypot, so ~1 ulp instead of bits
    f = load_golden("frame_2k_deg3_fisheye")
    cam = CameraModel("fisheye", int(f["width"]), int(f["height"]), float(f["focal"]), f["pose"])
    d = cam.ray_directions_device().cpu().numpy()
    assert np.abs(d - f["dirs"]).max() <= 4e-16


def test_locate_matches_exact_nearest(cuda_ok):
    from paper_2502_01157_b200 import device as dv

    g = load_golden("frame_2k_deg3")
    ds = dv.DeviceScene(golden_scene(g))
    pos = g["positions"]
    rng = np.random.default_rng(5)
    nbr = g["neighbors"]
    off = g["offsets"]
    i = rng.integers(0, len(pos), 200)
    j = nbr[off[i]]  # a Delaunay neighbour: the midpoint is an exact tie
    q = np.concatenate([rng.uniform(-1.2, 1.2, (2000, 3)), rng.uniform(-6, 6, (500, 3)),
                        pos[rng.integers(0, len(pos), 200)], 0.5 * (pos[i] + pos[j])])
    got = ds.locate(_dev(q)).cpu().numpy()
    ref = orc.nearest_sites(pos, q)
    np.testing.assert_array_equal(got, ref)


@pytest.mark.parametrize("name", ["grad_2k_deg3", "grad_2k_deg3_inside_eps0", "grad_10k_deg0"])
def test_backward_matches_reference(cuda_ok, name):
    from paper_2502_01157_b200 import render

    g = load_golden(name)
    rgb, grad = render.render_rays_with_gradients(golden_scene(g), g["origins"], g["dirs"],
                                                  g["adjoints"], epsilon=float(g["epsilon"]))
    assert np.abs(rgb - g["rgb"]).max() <= IMG_TOL
    assert rel_err(grad.d_sh.reshape(-1, 48), g["d_sh"]) <= GRAD_RTOL
    assert rel_err(grad.d_position, g["d_position"]) <= GRAD_RTOL
    assert rel_err(grad.d_raw_density, g["d_raw_density"]) <= GRAD_RTOL


@pytest.mark.parametrize("packed", [True, False])
@pytest.mark.parametrize("name", ["train_2k_deg3_q", "train_3k_surface_q"])
def test_train_batch_matches_reference(cuda_ok, name, packed):
    from paper_2502_01157_b200 import device as dv

    g = load_golden(name)
    ds = dv.DeviceScene(golden_scene(g), packed=packed)
    m = len(g["origins"])
    gb = dv.GradBuffers(ds.n_sites, ds.device)
    loss = torch.zeros(2, dtype=torch.float64, device="cuda")
    res = dv.train_batch_device(ds, _dev(g["origins"]), _dev(g["dirs"]), _dev(np.zeros(m)),
                                _dev(g["t_max"]), _dev(g["start"], torch.int32),
                                _dev(g["targets"]), gb, loss, rgb_scale=float(g["rgb_scale"]),
                                quantile_scale=float(g["quantile_scale"]),
                                u_pairs=_dev(g["u_pairs"]), weight_floor=1e-4,
                                epsilon=float(g["epsilon"]), f64=True)
    torch.cuda.synchronize()
    assert np.abs(res.rgb.cpu().numpy() - g["out_rgb"]).max() <= IMG_TOL
    np.testing.assert_array_equal(res.status.cpu().numpy(), g["out_status"])
    np.testing.assert_array_equal(res.counters.cpu().numpy(), g["counters"].sum(axis=0))
    lw = g["loss_w"].sum(axis=0)
    np.testing.assert_allclose(loss.cpu().numpy(), lw, rtol=1e-6)  # fp32 colour inputs (packed)
    g4 = gb.g4.double().cpu().numpy()
    assert rel_err(g4[:, 3], g["d_sigma_w"].sum(axis=0)) <= GRAD_RTOL
    assert rel_err(g4[:, :3], g["d_pos_w"].sum(axis=0)) <= GRAD_RTOL
    assert rel_err(gb.sh.double().cpu().numpy(), g["d_sh_w"].sum(axis=0)) <= GRAD_RTOL


def test_empty_and_step_limit(cuda_ok):
    from paper_2502_01157_b200 import device as dv

    g = load_golden("frame_2k_deg3")
    sa, origins, dirs, start, t_max = frame_rays(g)
    ds = dv.DeviceScene(golden_scene(g))
    e = torch.empty((0, 3), dtype=torch.float64, device="cuda")
    z = torch.empty(0, dtype=torch.float64, device="cuda")
    res = dv.render_rays_device(ds, e, e, z, z, torch.empty(0, dtype=torch.int32, device="cuda"))
    assert res.rgb.shape == (0, 3)
    # step_limit 5: most rays fail with status 2 and render the background
    m = 256
    res = dv.render_rays_device(ds, _dev(origins[:m]), _dev(dirs[:m]), _dev(np.zeros(m)),
                                _dev(np.full(m, t_max)), _dev(np.full(m, start), torch.int32),
                                step_limit=5, f64=True)
    torch.cuda.synchronize()
    ref = orc.render_rays(sa, origins[:m], dirs[:m], 0.0, t_max, start, step_limit=5)
    np.testing.assert_array_equal(res.status.cpu().numpy(), ref["status"])
    assert (ref["status"] == 2).any()
    np.testing.assert_array_equal(res.rgb.cpu().numpy()[ref["status"] == 2],
                                  np.broadcast_to(g["background"], ((ref["status"] == 2).sum(), 3)))
    np.testing.assert_array_equal(res.ray_counters.cpu().numpy(), ref["counters"])


def test_flat_kernels_drop_in(cuda_ok):
    """paper_2502_01157_b200.kernels.train_batch with the reference's exact
    positional signature and per-worker buffers (kernels.py:372-385)."""
    from paper_2502_01157_b200 import kernels as K
    from paper_2502_01157_b200.scene import softplus

    g = load_golden("train_2k_deg3_q")
    n = len(g["positions"])
    m = len(g["origins"])
    W = int(g["workers"])
    out_rgb = np.empty((m, 3))
    out_status = np.empty(m, dtype=np.int8)
    d_sigma_w, d_sh_w, d_pos_w = np.zeros((W, n)), np.zeros((W, n, 48)), np.zeros((W, n, 3))
    loss_w = np.zeros((W, 2))
    counters = np.zeros((W, 2), dtype=np.int64)
    sc = np.empty((W, 4096), dtype=np.int64)
    K.train_batch(g["positions"], g["offsets"].astype(np.int64), g["neighbors"].astype(np.int64),
                  softplus(g["raw_density"]), g["sh"], g["background"], g["origins"], g["dirs"],
                  np.zeros(m), g["t_max"], g["start"], g["targets"], float(g["epsilon"]), 4096,
                  1e-12 * float(np.linalg.norm(g["positions"].max(0) - g["positions"].min(0))),
                  float(g["rgb_scale"]), float(g["quantile_scale"]), g["u_pairs"], 1e-4, W,
                  out_rgb, out_status, d_sigma_w, d_sh_w, d_pos_w, loss_w, counters, sc, sc, sc)
    assert np.abs(out_rgb - g["out_rgb"]).max() <= IMG_TOL
    np.testing.assert_array_equal(counters.sum(0), g["counters"].sum(0))
    assert rel_err(d_sigma_w.sum(0), g["d_sigma_w"].sum(0)) <= GRAD_RTOL
    assert rel_err(d_sh_w.sum(0), g["d_sh_w"].sum(0)) <= GRAD_RTOL
    assert rel_err(d_pos_w.sum(0), g["d_pos_w"].sum(0)) <= GRAD_RTOL
    np.testing.assert_allclose(loss_w.sum(0), g["loss_w"].sum(0), rtol=1e-6)
    # render_rays drop-in on a frame
    f = load_golden("frame_2k_deg3")
    sa, origins, dirs, start, t_max = frame_rays(f)
    mm = len(dirs)
    rgb = np.empty((mm, 3))
    res = np.empty(mm)
    st = np.empty(mm, dtype=np.int8)
    ws = np.empty(mm)
    cnt = np.zeros((8, 2), dtype=np.int64)
    K.render_rays(sa.positions, sa.offsets, sa.neighbors, sa.sigma, sa.sh, sa.background, origins,
                  dirs, np.zeros(mm), np.full(mm, t_max), np.full(mm, start), 1e-3, 4096,
                  sa.width_floor, 8, rgb, res, st, ws, cnt)
    assert np.abs(rgb.reshape(f["img"].shape) - f["img"]).max() <= IMG_TOL
    assert cnt.sum(0)[0] == f["stats"][1] and cnt.sum(0)[1] == f["stats"][2]


def test_checkpoint_to_device_render(cuda_ok):
    """a reference-written RFOAM1 checkpoint rendered on the
    device matches the oracle on the same loaded scene."""
    import os

    from conftest import GOLDEN
    from paper_2502_01157_b200 import device as dv
    from paper_2502_01157_b200.camera import PINHOLE, CameraModel, look_at
    from paper_2502_01157_b200.checkpoint import load_device_scene
    from paper_2502_01157_b200.scene import softplus

    scene, ds = load_device_scene(os.path.join(GOLDEN, "scene300.rfoam"))
    assert ds.packed
    cam = CameraModel.from_angle_x(PINHOLE, 40, 30, 0.9, look_at((0.2, 0.1, 2.8), (0, 0, 0)))
    res = dv.render_image_device(ds, cam, f64=True, per_ray=True)
    torch.cuda.synchronize()
    adj = scene.adjacency
    sa = orc.SceneArrays(adj.positions, adj.offsets, adj.neighbors, softplus(scene.raw_density),
                         scene.sh_coeffs.reshape(-1, 48), scene.background)
    o = cam.position
    start = int(orc.nearest_sites(sa.positions, o[None, :])[0])
    t_max = float(np.linalg.norm(o - sa.center) + 2.0 * sa.diagonal + 1.0)
    ref = orc.render_rays(sa, np.broadcast_to(o, (1200, 3)), cam.ray_directions(), 0.0, t_max,
                          start)
    np.testing.assert_array_equal(res.ray_counters.cpu().numpy(), ref["counters"])
    assert np.abs(res.rgb.cpu().numpy() - ref["rgb"]).max() <= IMG_TOL


@pytest.mark.parametrize("rgb_scale", [None, 0.0])
@pytest.mark.parametrize("n_pairs", [1, 2, 3])
def test_train_batch_quantile_pairs_vs_oracle(cuda_ok, n_pairs, rgb_scale):
    """Pair counts other than the default P=2: the first two pairs are fused
    into the reverse pass, any further pairs take the per-lane scatter path;
    both must agree with kernels.py:456-567 (oracle).  rgb_scale=0 isolates
    the quantile gradient."""
    from paper_2502_01157_b200 import device as dv

    g = load_golden("train_2k_deg3_q")
    sa = golden_scene_arrays(g)
    m = len(g["origins"])
    rs = float(g["rgb_scale"]) if rgb_scale is None else rgb_scale
    up = np.random.default_rng(40 + n_pairs).uniform(0, 1, (m, n_pairs, 2))
    qs = 0.05 / (m * n_pairs)
    ref = orc.train_batch(sa, g["origins"], g["dirs"], np.zeros(m), g["t_max"], g["start"],
                          g["targets"], rs, qs, up, 1e-4,
                          epsilon=float(g["epsilon"]), threads=8)
    ds = dv.DeviceScene(golden_scene(g))
    gb = dv.GradBuffers(ds.n_sites, ds.device)
    loss = torch.zeros(2, dtype=torch.float64, device="cuda")
    dv.train_batch_device(ds, _dev(g["origins"]), _dev(g["dirs"]), _dev(np.zeros(m)),
                          _dev(g["t_max"]), _dev(g["start"], torch.int32), _dev(g["targets"]),
                          gb, loss, rgb_scale=rs, quantile_scale=qs,
                          u_pairs=_dev(up), weight_floor=1e-4, epsilon=float(g["epsilon"]))
    torch.cuda.synchronize()
    np.testing.assert_allclose(loss.cpu().numpy(), ref["loss_w"].sum(axis=0), rtol=1e-6)
    g4 = gb.g4.double().cpu().numpy()
    assert rel_err(g4[:, 3], ref["d_sigma_w"].sum(axis=0)) <= GRAD_RTOL
    assert rel_err(g4[:, :3], ref["d_pos_w"].sum(axis=0)) <= GRAD_RTOL
    assert rel_err(gb.sh.double().cpu().numpy(), ref["d_sh_w"].sum(axis=0)) <= GRAD_RTOL


@pytest.mark.parametrize("kind", ["mirror", "refract"])
def test_effect_rays_device(cuda_ok, kind):
    """rfb_effect_rays (batched apply_effect, rays.py:166-176) vs the
    reference's per-ray outputs, one plane per launch."""
    from paper_2502_01157_b200 import device as dv

    g = load_golden("effects")
    for i in range(0, len(g["d"]), 7):
        sel = [i]
        oo, od = dv.effect_rays_device(_dev(g["o"][sel]), _dev(g["d"][sel]), _dev(g["t_at"][sel]),
                                       g["normal"][i], kind, float(g["eta"][i]))
        np.testing.assert_allclose(oo.cpu().numpy()[0], g[f"{kind}_o"][i], rtol=0, atol=1e-15)
        np.testing.assert_allclose(od.cpu().numpy()[0], g[f"{kind}_d"][i], rtol=0, atol=1e-14)
    # a batch sharing one plane
    n = g["normal"][3]
    oo, od = dv.effect_rays_device(_dev(g["o"]), _dev(g["d"]), _dev(g["t_at"]), n, kind, 1.5)
    from paper_2502_01157_b200 import render as rd
    for i in range(len(g["d"])):
        r = rd.apply_effect(rd.Ray(g["o"][i], g["d"][i], 0.0, 9.0), n, kind, 1.5, g["t_at"][i])
        np.testing.assert_allclose(od.cpu().numpy()[i], r.direction, rtol=0, atol=1e-14)


@pytest.mark.parametrize("packed,cull", [(True, False), (True, True), (False, False)])
def test_fp64_positions_vs_oracle(cuda_ok, packed, cull):
    """Sites that are not fp32-representable (as after an Adam step on the
    positions): the packed layout with the widened pre-filter bound
    (positions_f64), also over view-culled rows (rfb_cull_scene with the fp64-site
    margin), and the generic fp64 layout; per-ray cell sequences, counters and
    status must be the oracle's bit for bit, the image within 1e-4."""
    from paper_2502_01157_b200 import device as dv
    from paper_2502_01157_b200.synthetic import delaunay_csr

    rng = np.random.default_rng(21)
    n = 3000
    pos = rng.uniform(-1, 1, (n, 3)) + rng.normal(0, 1e-9, (n, 3))  # fp64 positions
    assert not np.array_equal(pos.astype(np.float32).astype(np.float64), pos)
    off, nbr, _ = delaunay_csr(pos)
    raw = rng.normal(0, 1, n)
    sh = rng.normal(0, 0.3, (n, 48))
    from paper_2502_01157_b200.scene import softplus
    sa = orc.SceneArrays(pos, off, nbr, softplus(raw), sh, np.array([0.1, 0.2, 0.3]))
    ds = dv.DeviceScene.from_arrays(pos, off, nbr, softplus(raw), sh, np.array([0.1, 0.2, 0.3]),
                                    packed=packed)
    assert ds.packed == packed and ds.positions_f64
    m = 2048
    o = np.tile([0.0, 0.0, 3.0], (m, 1))
    d = rng.normal(size=(m, 3)) * [0.3, 0.3, 0.0] + [0.0, 0.0, -1.0]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    start = int(orc.nearest_sites(pos, o[:1])[0])
    tmax = ds.default_t_max(o[:1])
    ref = orc.render_rays(sa, o, d, 0.0, tmax, start)
    cone = None
    if cull:  # every direction is a positive multiple of (u, v, -1), (u, v) in this box
        uv = d[:, :2] / -d[:, 2:3]
        lo, hi = uv.min(0), uv.max(0)
        cone = np.array([[lo[0], lo[1], -1.0], [hi[0], lo[1], -1.0], [lo[0], hi[1], -1.0],
                         [hi[0], hi[1], -1.0]])
    res = dv.render_rays_device(ds, _dev(o), _dev(d), _dev(np.zeros(m)), _dev(np.full(m, tmax)),
                                _dev(np.full(m, start), torch.int32), f64=True, seg_capacity=512,
                                view_dirs=cone)
    torch.cuda.synchronize()
    if cull:
        dropped = int((ds._view_cells[:, 7] & 31).sum().item())
        assert dropped > 0.05 * ds.n_edges, dropped
    np.testing.assert_array_equal(res.status.cpu().numpy(), ref["status"])
    np.testing.assert_array_equal(res.ray_counters.cpu().numpy(), ref["counters"])
    assert np.abs(res.rgb.cpu().numpy() - ref["rgb"]).max() <= IMG_TOL
    cells = res.seg_cells.cpu().numpy()
    for q in range(0, m, 97):
        c, a, b, *_ = orc.walk_ray(sa, o[q], d[q], 0.0, tmax, start)
        np.testing.assert_array_equal(cells[q, :len(c)], c)


def test_train_batch_step_limit_failures_vs_oracle(cuda_ok):
    """Rays that hit the step limit render the background and contribute no
    gradient (kernels.py:230-236, 408-412); the rest are trained normally."""
    from paper_2502_01157_b200 import device as dv

    g = load_golden("train_2k_deg3_q")
    sa = golden_scene_arrays(g)
    m = len(g["origins"])
    ref = orc.train_batch(sa, g["origins"], g["dirs"], np.zeros(m), g["t_max"], g["start"],
                          g["targets"], float(g["rgb_scale"]), float(g["quantile_scale"]),
                          g["u_pairs"], 1e-4, epsilon=float(g["epsilon"]), step_limit=22,
                          threads=8)
    assert (ref["status"] == 2).any() and (ref["status"] == 0).any()
    ds = dv.DeviceScene(golden_scene(g))
    gb = dv.GradBuffers(ds.n_sites, ds.device)
    loss = torch.zeros(2, dtype=torch.float64, device="cuda")
    res = dv.train_batch_device(ds, _dev(g["origins"]), _dev(g["dirs"]), _dev(np.zeros(m)),
                                _dev(g["t_max"]), _dev(g["start"], torch.int32),
                                _dev(g["targets"]), gb, loss, rgb_scale=float(g["rgb_scale"]),
                                quantile_scale=float(g["quantile_scale"]),
                                u_pairs=_dev(g["u_pairs"]), weight_floor=1e-4,
                                epsilon=float(g["epsilon"]), step_limit=22, f64=True)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(res.status.cpu().numpy(), ref["status"])
    assert np.abs(res.rgb.cpu().numpy() - ref["rgb"]).max() <= IMG_TOL
    np.testing.assert_allclose(loss.cpu().numpy(), ref["loss_w"].sum(axis=0), rtol=1e-6)
    g4 = gb.g4.double().cpu().numpy()
    assert rel_err(g4[:, 3], ref["d_sigma_w"].sum(axis=0)) <= GRAD_RTOL
    assert rel_err(g4[:, :3], ref["d_pos_w"].sum(axis=0)) <= GRAD_RTOL
    assert rel_err(gb.sh.double().cpu().numpy(), ref["d_sh_w"].sum(axis=0)) <= GRAD_RTOL


def test_render_image_frames_are_independent(cuda_ok):
    """render_image returns frames backed by a small pool of pinned buffers:
    frames the caller keeps must never be overwritten by later renders."""
    from paper_2502_01157_b200 import render as rd
    from paper_2502_01157_b200.camera import PINHOLE, CameraModel, look_at

    g = load_golden("frame_2k_deg3")
    scene = golden_scene(g)
    from paper_2502_01157_b200 import device as dv
    ds = dv.DeviceScene(scene)
    cams = [CameraModel.from_angle_x(PINHOLE, 64, 48, 0.9, look_at((0.3 * k, 0.0, 3.0), (0, 0, 0)))
            for k in range(5)]
    kept = [rd.render_image(scene, c, device_scene=ds) for c in cams]
    again = [rd.render_image(scene, c, device_scene=ds).copy() for c in cams]
    for a, b in zip(kept, again):
        np.testing.assert_array_equal(a, b)
    assert not np.array_equal(kept[0], kept[1])


def test_render_image_zero_copy_equals_copy_path(cuda_ok, monkeypatch):
    """The walk kernel storing the frame straight into the mapped pinned buffer
    (render.ZERO_COPY_FRAMES) gives the same bits as rendering to HBM + D2H,
    and the mapped path is the one taken on the B200."""
    from paper_2502_01157_b200 import device as dv
    from paper_2502_01157_b200 import render as rd
    from paper_2502_01157_b200.camera import PINHOLE, CameraModel, look_at

    g = load_golden("frame_2k_deg3")
    scene = golden_scene(g)
    cams = [CameraModel.from_angle_x(PINHOLE, 96, 64, 0.9, look_at((0.2 * k, 0.1, 3.0), (0, 0, 0)))
            for k in range(3)]
    frames = {}
    for zc in (True, False):
        monkeypatch.setattr(rd, "ZERO_COPY_FRAMES", zc)
        ds = dv.DeviceScene(scene)
        frames[zc] = [rd.render_image(scene, c, device_scene=ds).copy() for c in cams]
        pool = rd._PINNED_POOLS[(str(ds.device), 96, 64, zc)]
        assert all((e[2] is not None) == zc for e in pool)
    for a, b in zip(frames[True], frames[False]):
        np.testing.assert_array_equal(a, b)
    cam = CameraModel(str(g["kind"]), int(g["width"]), int(g["height"]), float(g["focal"]), g["pose"])
    monkeypatch.setattr(rd, "ZERO_COPY_FRAMES", True)
    img = rd.render_image(scene, cam, epsilon=float(g["epsilon"]))
    assert np.abs(img - g["img"]).max() <= IMG_TOL


@pytest.mark.parametrize("name", FRAMES)
def test_trace_matches_reference_traces(cuda_ok, name):
    """render.trace (rays.py:81-115) against the reference's own trace() outputs
    (golden tr_*): cells, depths, status and counters bit-exact; the residual
    is walk_ray's exp(log_T) (bit-exact against the oracle's walk)."""
    from paper_2502_01157_b200 import device as dv
    from paper_2502_01157_b200 import render as R

    g = load_golden(name)
    sa, origins, dirs, start, t_max = frame_rays(g)
    scene = golden_scene(g)
    ds = dv.DeviceScene(scene)
    eps = float(g["epsilon"])
    off = 0
    for k, q in enumerate(g["tr_idx"]):
        L = int(g["tr_len"][k])
        cnt = np.zeros((1, 2), dtype=np.int64)
        segs = R.trace(scene, R.Ray(origins[q], dirs[q]), epsilon=eps, counters=cnt,
                       device_scene=ds)
        assert g["tr_status"][k] == 0 and segs.status == 0
        np.testing.assert_array_equal(segs.cells, g["tr_cells"][off:off + L])
        np.testing.assert_array_equal(segs.t_entry, g["tr_t0"][off:off + L])
        np.testing.assert_array_equal(segs.t_exit, g["tr_t1"][off:off + L])
        np.testing.assert_array_equal(cnt[0], g["tr_counters"][k])
        _, _, _, _, resid, _ = orc.walk_ray(sa, origins[q], dirs[q], 0.0, t_max, start,
                                            epsilon=eps)
        assert segs.residual_transmittance == resid
        off += L


def test_trace_failure_codes(cuda_ok):
    """trace() raises StepLimit / CycleDetected like rays.py:109-112."""
    from paper_2502_01157_b200 import device as dv
    from paper_2502_01157_b200 import render as R
    from paper_2502_01157_b200.errors import StepLimit

    g = load_golden("frame_2k_deg3")
    sa, origins, dirs, start, t_max = frame_rays(g)
    scene = golden_scene(g)
    ds = dv.DeviceScene(scene)
    q = int(g["tr_idx"][0])
    with pytest.raises(StepLimit):
        R.trace(scene, R.Ray(origins[q], dirs[q]), step_limit=3, device_scene=ds)
    # an explicit start cell and a finite t_max are honoured
    segs = R.trace(scene, R.Ray(origins[q], dirs[q], 0.0, 2.5), start_site=start,
                   device_scene=ds)
    c, a, b, st, resid, _ = orc.walk_ray(sa, origins[q], dirs[q], 0.0, 2.5, start)
    np.testing.assert_array_equal(segs.cells, c)
    np.testing.assert_array_equal(segs.t_exit, b)
    assert segs.residual_transmittance == resid


def test_flat_walk_ray_drop_in(cuda_ok):
    """kernels.walk_ray (kernels.py:76-162) with the reference's positional
    signature: fills the caller's segment buffers, returns (nseg, status,
    residual), counters[worker] +=, against the golden traces."""
    from paper_2502_01157_b200 import kernels as K

    g = load_golden("frame_3k_surface")
    sa, origins, dirs, start, t_max = frame_rays(g)
    eps = float(g["epsilon"])
    cells = np.empty(4096, dtype=np.int64)
    t0 = np.empty(4096)
    t1 = np.empty(4096)
    off = 0
    for k, q in enumerate(g["tr_idx"][:24]):
        L = int(g["tr_len"][k])
        cnt = np.zeros((3, 2), dtype=np.int64)
        nseg, status, resid = K.walk_ray(sa.positions, sa.offsets, sa.neighbors, sa.sigma,
                                         *origins[q], *dirs[q], 0.0, t_max, start, eps, 4096,
                                         sa.width_floor, cells, t0, t1, cnt, 2)
        assert (nseg, status) == (L, int(g["tr_status"][k]))
        np.testing.assert_array_equal(cells[:L], g["tr_cells"][off:off + L])
        np.testing.assert_array_equal(t0[:L], g["tr_t0"][off:off + L])
        np.testing.assert_array_equal(t1[:L], g["tr_t1"][off:off + L])
        np.testing.assert_array_equal(cnt[2], g["tr_counters"][k])
        assert not cnt[:2].any()
        *_, ref_resid, _ = orc.walk_ray(sa, origins[q], dirs[q], 0.0, t_max, start, epsilon=eps)
        assert resid == ref_resid
        off += L


def test_flat_render_rays_tracks_in_place_updates(cuda_ok):
    """kernels.render_rays keeps the CSR on the device between calls (cached on the
    adjacency arrays) but re-reads the parameters every call, like the
    reference: moving sites / new sigma / new SH in place are honoured."""
    from paper_2502_01157_b200 import kernels as K

    f = load_golden("frame_2k_deg3")
    sa, origins, dirs, start, t_max = frame_rays(f)
    m = len(dirs)
    pos = sa.positions.copy()
    sigma = sa.sigma.copy()
    sh = sa.sh.copy()
    off, nbr = sa.offsets, sa.neighbors
    rng = np.random.default_rng(4)
    for it in range(3):
        if it:  # the training loop's in-place updates between rebuilds
            pos += rng.normal(0.0, 1e-4, pos.shape)
            sigma *= rng.uniform(0.5, 1.5, sigma.shape)
            sh += rng.normal(0.0, 0.05, sh.shape)
        rgb = np.empty((m, 3))
        res = np.empty(m)
        st = np.empty(m, dtype=np.int8)
        ws = np.empty(m)
        cnt = np.zeros((1, 2), dtype=np.int64)
        K.render_rays(pos, off, nbr, sigma, sh, sa.background, origins, dirs, np.zeros(m),
                      np.full(m, t_max), np.full(m, start), 1e-3, 4096, sa.width_floor, 1, rgb,
                      res, st, ws, cnt)
        ref = orc.render_rays(orc.SceneArrays(pos, off, nbr, sigma, sh, sa.background), origins,
                              dirs, 0.0, t_max, start)
        np.testing.assert_array_equal(st, ref["status"])
        np.testing.assert_array_equal(cnt[0], ref["counters"].sum(0))
        assert np.abs(rgb - ref["rgb"]).max() <= IMG_TOL
