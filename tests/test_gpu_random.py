"""Randomised parity sweep: small random foams (uniform, clustered, surface,
non-fp32-exact positions -> generic layout), random cameras inside and
outside the hull, random epsilon / step limits.  Every ray's visited-cell
sequence, depths, counters and status must equal the oracle's bit for bit;
images 1e-4; gradients 1e-3 relative (per tensor)."""

import numpy as np
import pytest
import torch

from oracle import oracle as orc
from paper_2502_01157_b200.synthetic import delaunay_csr  # noqa: E402

pytestmark = pytest.mark.gpu


def _scene(seed):
    from paper_2502_01157_b200.scene import AdjacencyGraph, FoamScene
    from paper_2502_01157_b200.synthetic import delaunay_csr

    rng = np.random.default_rng(seed)
    n = int(rng.integers(20, 600))
    kind = seed % 4
    if kind == 0:
        pos = rng.uniform(-1, 1, (n, 3))
    elif kind == 1:
        c = rng.uniform(-1, 1, (4, 3))
        pos = c[rng.integers(0, 4, n)] + rng.normal(0, 0.15, (n, 3))
    elif kind == 2:
        u = rng.normal(0, 1, (n, 3))
        pos = 0.6 * u / np.linalg.norm(u, axis=1, keepdims=True) + rng.normal(0, 0.02, (n, 3))
    else:
        pos = rng.uniform(-1, 1, (n, 3)) * np.array([1.0, 0.3, 2.0])
    fp32 = seed % 3 != 0
    if fp32:
        pos = pos.astype(np.float32).astype(np.float64)
    off, nbr, hull = delaunay_csr(pos)
    raw = rng.normal(0, 1.5, n)
    sh = np.zeros((n, 16, 3))
    sh[:, 0] = rng.normal(0, 0.6, (n, 3))
    if seed % 2:
        sh[:, 1:] = rng.normal(0, 0.3, (n, 15, 3))
    bg = rng.uniform(0, 1, 3)
    return FoamScene(pos, raw, sh, bg, AdjacencyGraph(pos, off, nbr, hull)), rng, fp32


@pytest.mark.parametrize("seed", list(range(24)))
def test_random_scene_parity(cuda_ok, seed):
    from paper_2502_01157_b200 import device as dv
    from paper_2502_01157_b200.scene import softplus

    scene, rng, fp32 = _scene(seed)
    ds = dv.DeviceScene(scene)
    assert ds.packed and ds.positions_f64 == (not fp32)  # fp64 sites: widened bound
    adj = scene.adjacency
    sa = orc.SceneArrays(adj.positions, adj.offsets, adj.neighbors, softplus(scene.raw_density),
                         scene.sh_coeffs.reshape(-1, 48), scene.background)
    m = 700
    if seed % 5 == 0:  # origins inside the foam, per-ray
        o = rng.uniform(-0.8, 0.8, (m, 3))
    else:
        eye = rng.normal(0, 1, 3)
        eye = 2.5 * eye / np.linalg.norm(eye)
        o = np.broadcast_to(eye, (m, 3)).copy()
    tgt = rng.uniform(-0.7, 0.7, (m, 3))
    d = tgt - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    start = orc.nearest_sites(sa.positions, o)
    t_max = np.linalg.norm(o - sa.center, axis=1) + 2 * sa.diagonal + 1
    eps = [0.0, 1e-3, 0.05][seed % 3]
    step_limit = [4096, 40][int(seed % 7 == 3)]
    T = lambda a, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)  # noqa
    cap = 256
    res = dv.render_rays_device(ds, T(o), T(d), T(np.zeros(m)), T(t_max), T(start, torch.int32),
                                epsilon=eps, step_limit=step_limit, f64=True, seg_capacity=cap)
    torch.cuda.synchronize()
    ref = orc.render_rays(sa, o, d, 0.0, t_max, start, epsilon=eps, step_limit=step_limit)
    np.testing.assert_array_equal(res.status.cpu().numpy(), ref["status"])
    np.testing.assert_array_equal(res.ray_counters.cpu().numpy(), ref["counters"])
    np.testing.assert_array_equal(res.nseg.cpu().numpy(), ref["nseg"])
    assert np.abs(res.rgb.cpu().numpy() - ref["rgb"]).max() <= 1e-4
    cells = res.seg_cells.cpu().numpy()
    t1s = res.seg_t1.cpu().numpy()
    for q in range(0, m, 5):
        c, a, b, st, _, _ = orc.walk_ray(sa, o[q], d[q], 0.0, t_max[q], start[q], epsilon=eps,
                                         step_limit=step_limit)
        L = min(len(c), cap)
        np.testing.assert_array_equal(cells[q, :L], c[:L])
        np.testing.assert_array_equal(t1s[q, :L], b[:L])
    # gradients (generic adjoint)
    adjv = rng.normal(0, 1, (m, 3))
    gb = dv.GradBuffers(ds.n_sites, ds.device)
    dv.backward_rays_device(ds, T(o), T(d), T(np.zeros(m)), T(t_max), T(start, torch.int32),
                            T(adjv), gb, epsilon=eps, step_limit=step_limit)
    torch.cuda.synchronize()
    rgb, status, ds_, dsh, dp, _ = orc.render_rays_with_gradients(
        sa, o, d, adjv, np.zeros(m), t_max, start, epsilon=eps, step_limit=step_limit)
    g4 = gb.g4.double().cpu().numpy()

    def rel(a, b):
        den = np.abs(b).max()
        return np.abs(a - b).max() / den if den > 0 else np.abs(a).max()

    assert rel(g4[:, 3], ds_) <= 1e-3
    assert rel(g4[:, :3], dp) <= 1e-3
    assert rel(gb.sh.double().cpu().numpy(), dsh) <= 1e-3


@pytest.mark.parametrize("scale,offset", [(1e-3, 0.0), (1e-3, 0.02), (50.0, 0.0), (3.0, 2000.0)])
def test_fp64_sites_scaled_vs_oracle(cuda_ok, scale, offset):
    """The packed fp64-site bound (n1max + 2 max(X, 1/4)) across coordinate
    magnitudes: tiny scenes (X < 1/4), large ones, and a small scene far from
    the origin (X >> cell size); cell counters and status bit-exact."""
    from paper_2502_01157_b200 import device as dv
    from paper_2502_01157_b200.scene import softplus

    rng = np.random.default_rng(int(scale * 7 + offset))
    n = 2500
    pos = rng.uniform(-1, 1, (n, 3)) * scale + offset + rng.normal(0, 1e-9 * scale, (n, 3))
    off, nbr, _ = delaunay_csr(pos)
    raw = rng.normal(0, 1, n) - np.log(scale)  # keep optical depth O(1)
    sh = rng.normal(0, 0.4, (n, 48))
    bg = np.array([0.2, 0.1, 0.3])
    sa = orc.SceneArrays(pos, off, nbr, softplus(raw), sh, bg)
    ds = dv.DeviceScene.from_arrays(pos, off, nbr, softplus(raw), sh, bg)
    assert ds.packed and ds.positions_f64
    m = 1024
    eye = np.array([offset, offset, offset + 3.0 * scale])
    o = np.tile(eye, (m, 1))
    d = rng.normal(size=(m, 3)) * [0.3, 0.3, 0.0] + [0.0, 0.0, -1.0]
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    start = int(orc.nearest_sites(pos, o[:1])[0])
    tmax = ds.default_t_max(o[:1])
    ref = orc.render_rays(sa, o, d, 0.0, tmax, start)
    dev = lambda a, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)  # noqa
    res = dv.render_rays_device(ds, dev(o), dev(d), dev(np.zeros(m)), dev(np.full(m, tmax)),
                                dev(np.full(m, start), torch.int32), f64=True)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(res.status.cpu().numpy(), ref["status"])
    np.testing.assert_array_equal(res.ray_counters.cpu().numpy(), ref["counters"])
    assert np.abs(res.rgb.cpu().numpy() - ref["rgb"]).max() <= 1e-4
