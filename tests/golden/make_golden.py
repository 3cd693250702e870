"""Generate golden vectors by running the UNMODIFIED reference.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports ``rfoam`` read-only from /root/reference/pkg/src, builds small
synthetic foams (fixtures per SURVEY.md §8d, CSR from Qhull, cross-checked
against the reference's own ``delaunay.build``), and records the reference's
outputs of the hot-path entry points:

* ``render_image`` / ``render_ray_batch`` (rgb, residual, status, wsum, stats),
* ``trace`` per-ray cell sequences and depths for a ray subset,
* ``render_rays_with_gradients`` (rgb and the three gradient tensors),
* ``kernels.train_batch`` with the L2 adjoint and quantile pairs (W=2),
* SPEC known-answer tests (intersect_face, 2-site trace, composite, softplus).

The .npz files it writes are committed; tests/test_oracle.py pins the C
oracle to them and the GPU tests compare the CUDA path against the oracle.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from rfoam import foam as rfoam_foam  # noqa: E402
from rfoam.diffrender import composite as rcomp  # noqa: E402
from rfoam.diffrender.render import (RenderStats, render_image, render_ray_batch,  # noqa: E402
                                     render_rays_with_gradients)
from rfoam.foam import FoamScene  # noqa: E402
from rfoam.geometry import AdjacencyGraph, build  # noqa: E402
from rfoam.tracer import kernels  # noqa: E402
from rfoam.tracer.camera import FISHEYE, PINHOLE, CameraModel, look_at, orbit_poses  # noqa: E402
from rfoam.tracer.rays import WIDTH_FLOOR_SCALE, Ray, intersect_face, trace  # noqa: E402

from paper_2502_01157_b200.synthetic import delaunay_csr, random_positions  # noqa: E402


def ref_scene(n, seed, sh_degree, kind="uniform", check_delaunay=True):
    pos = random_positions(n, seed, kind)
    rng = np.random.default_rng(seed + 1_000_003)
    if kind == "surface":
        raw = np.where(np.linalg.norm(pos, axis=1) < 0.5, 20.0, -3.0)
    else:
        raw = rng.normal(0.0, 1.0, n)
    sh = np.zeros((n, 16, 3))
    sh[:, 0, :] = rng.normal(0.0, 0.5, (n, 3))
    if sh_degree >= 3:
        sh[:, 1:, :] = rng.normal(0.0, 0.15, (n, 15, 3))
    offsets, neighbors, hull = delaunay_csr(pos)
    if check_delaunay:
        tri = build(pos)
        ref_adj = AdjacencyGraph.from_triangulation(tri)
        assert np.array_equal(ref_adj.offsets, offsets), "Qhull CSR != reference Delaunay CSR"
        assert np.array_equal(ref_adj.neighbors, neighbors), "Qhull CSR != reference Delaunay CSR"
    adj = AdjacencyGraph(pos, offsets, neighbors, hull)
    scene = FoamScene(pos, raw, sh, np.array([0.1, 0.2, 0.3]), adj)
    adj.positions = scene.positions
    return scene


def scene_dict(scene):
    adj = scene.adjacency
    return dict(positions=scene.positions, raw_density=scene.raw_density,
                sh=scene.sh_coeffs.reshape(-1, 48), background=scene.background,
                offsets=adj.offsets.astype(np.int32), neighbors=adj.neighbors.astype(np.int32))


def traces_for(scene, origins, dirs, idx, epsilon, step_limit=4096):
    cells, t0, t1, lens, cnts, status = [], [], [], [], [], []
    for q in idx:
        cnt = np.zeros((1, 2), dtype=np.int64)
        ray = Ray(origins[q], dirs[q])
        try:
            segs = trace(scene, ray, epsilon=epsilon, step_limit=step_limit, counters=cnt)
            st = 0
        except Exception as e:  # StepLimit / CycleDetected
            segs = None
            st = 2 if type(e).__name__ == "StepLimit" else 3
        status.append(st)
        cnts.append(cnt[0])
        if segs is None:
            lens.append(0)
            continue
        cells.append(segs.cells)
        t0.append(segs.t_entry)
        t1.append(segs.t_exit)
        lens.append(len(segs))
    cat = lambda a, dt: np.concatenate(a).astype(dt) if a else np.zeros(0, dt)  # noqa: E731
    return dict(tr_idx=np.asarray(idx, dtype=np.int64), tr_len=np.asarray(lens, dtype=np.int64),
                tr_cells=cat(cells, np.int64), tr_t0=cat(t0, np.float64),
                tr_t1=cat(t1, np.float64), tr_counters=np.asarray(cnts, dtype=np.int64),
                tr_status=np.asarray(status, dtype=np.int8))


def frame_case(name, scene, eye, W, H, epsilon, n_trace=96, seed=0, angle=0.9, kind=PINHOLE):
    cam = CameraModel.from_angle_x(kind, W, H, angle, look_at(eye, (0.0, 0.0, 0.0)))
    stats = RenderStats()
    img, wsum, resid = render_image(scene, cam, epsilon=epsilon, workers=1, stats=stats,
                                    weight_check=True)
    dirs = cam.ray_directions()
    origins = np.broadcast_to(cam.position, (len(dirs), 3)).copy()
    rgb, residual, status = render_ray_batch(scene, origins, dirs, epsilon=epsilon, workers=1)
    assert np.array_equal(rgb.reshape(img.shape), img)
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(len(dirs), size=min(n_trace, len(dirs)), replace=False))
    d = dict(scene_dict(scene))
    d.update(pose=cam.pose, width=W, height=H, focal=cam.focal, epsilon=epsilon, dirs=dirs,
             kind=np.array(kind),
             img=img, wsum=wsum, residual=resid, status=status,
             stats=np.array([stats.rays, stats.cells_stepped, stats.neighbor_visits,
                             stats.failed_rays], dtype=np.int64))
    d.update(traces_for(scene, origins, dirs, idx, epsilon))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
    print(name, "rays", stats.rays, "cells/ray", stats.cells_stepped / stats.rays,
          "visits/ray", stats.neighbor_visits / stats.rays, "failed", stats.failed_rays)


def grad_case(name, scene, m, seed, epsilon, inside=False):
    rng = np.random.default_rng(seed)
    if inside:
        origins = rng.uniform(-0.5, 0.5, (m, 3))
    else:
        origins = np.broadcast_to(np.array([0.2, -0.1, 3.0]), (m, 3)).copy()
    target = rng.uniform(-0.4, 0.4, (m, 3))
    dirs = target - origins
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    adjoints = rng.normal(0.0, 1.0, (m, 3))
    rgb, grad = render_rays_with_gradients(scene, origins, dirs, adjoints, epsilon=epsilon)
    adj = scene.adjacency
    # the per-ray start sites / t_max the reference used (render.py:170-178)
    t_max = np.array([np.linalg.norm(0.5 * (adj.bbox_lo + adj.bbox_hi) - origins[k])
                      + 2.0 * adj.diagonal + 1.0 for k in range(m)])
    start = np.array([adj.nearest_site(origins[k]) for k in range(m)], dtype=np.int64)
    d = dict(scene_dict(scene))
    d.update(origins=origins, dirs=dirs, adjoints=adjoints, epsilon=epsilon, rgb=rgb,
             t_max=t_max, start=start, d_position=grad.d_position,
             d_raw_density=grad.d_raw_density, d_sh=grad.d_sh.reshape(-1, 48))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
    print(name, "max|d_sh|", np.abs(grad.d_sh).max(), "max|d_pos|", np.abs(grad.d_position).max())


def train_case(name, scene, m, seed, epsilon, quantile_scale, W=2):
    rng = np.random.default_rng(seed)
    eye = np.array([0.0, 0.3, 3.0])
    cam = CameraModel.from_angle_x(PINHOLE, 48, 32, 0.9, look_at(eye, (0.0, 0.0, 0.0)))
    all_dirs = cam.ray_directions()
    pix = rng.integers(0, len(all_dirs), size=m)
    dirs = np.ascontiguousarray(all_dirs[pix])
    origins = np.broadcast_to(cam.position, (m, 3)).copy()
    targets = rng.uniform(0.0, 1.0, (m, 3))
    u_pairs = rng.random((m, 2, 2))
    adj = scene.adjacency
    sigma = rfoam_foam.softplus(scene.raw_density)
    sh_flat = np.ascontiguousarray(scene.sh_coeffs.reshape(scene.n_sites, 48))
    start = np.full(m, adj.nearest_site(cam.position), dtype=np.int64)
    center = 0.5 * (adj.bbox_lo + adj.bbox_hi)
    t_far = float(np.linalg.norm(cam.position - center) + 2.0 * adj.diagonal + 1.0)
    t_min = np.zeros(m)
    t_max = np.full(m, t_far)
    n = scene.n_sites
    out_rgb = np.empty((m, 3))
    out_status = np.empty(m, dtype=np.int8)
    d_sigma_w = np.zeros((W, n))
    d_sh_w = np.zeros((W, n, 48))
    d_pos_w = np.zeros((W, n, 3))
    loss_w = np.zeros((W, 2))
    counters = np.zeros((W, 2), dtype=np.int64)
    sc = np.empty((W, 4096), dtype=np.int64)
    s0 = np.empty((W, 4096))
    s1 = np.empty((W, 4096))
    rgb_scale = 1.0 / (3.0 * m)
    kernels.train_batch(adj.positions, adj.offsets, adj.neighbors, sigma, sh_flat,
                        scene.background, origins, dirs, t_min, t_max, start, targets, epsilon,
                        4096, WIDTH_FLOOR_SCALE * adj.diagonal, rgb_scale, quantile_scale,
                        u_pairs, 1e-4, W, out_rgb, out_status, d_sigma_w, d_sh_w, d_pos_w,
                        loss_w, counters, sc, s0, s1)
    d = dict(scene_dict(scene))
    d.update(origins=origins, dirs=dirs, targets=targets, u_pairs=u_pairs, start=start,
             t_max=t_max, epsilon=epsilon, rgb_scale=rgb_scale, quantile_scale=quantile_scale,
             workers=W, out_rgb=out_rgb, out_status=out_status, d_sigma_w=d_sigma_w,
             d_sh_w=d_sh_w, d_pos_w=d_pos_w, loss_w=loss_w, counters=counters)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
    print(name, "loss_w", loss_w.sum(axis=0), "counters", counters.sum(axis=0))


def kat_case():
    """SPEC worked examples, recorded from the reference."""
    out = {}
    ray = Ray(np.zeros(3), np.array([1.0, 0.0, 0.0]))
    out["if_px"] = np.array(intersect_face(ray, np.zeros(3), np.array([2.0, 0, 0])), dtype=float)
    ray = Ray(np.zeros(3), np.array([-1.0, 0.0, 0.0]))
    out["if_mx"] = np.array(intersect_face(ray, np.zeros(3), np.array([2.0, 0, 0])), dtype=float)
    ray = Ray(np.zeros(3), np.array([0.6, 0.8, 0.0]))
    out["if_diag"] = np.array(intersect_face(ray, np.zeros(3), np.array([2.0, 0, 0])), dtype=float)
    pos = np.array([[0.0, 0, 0], [2.0, 0, 0]])
    sc = FoamScene.from_points(pos, raw_density=0.0)
    sc.adjacency = AdjacencyGraph.from_lists(pos, [[1], [0]])
    sc.adjacency.positions = sc.positions
    segs = trace(sc, Ray(np.array([-1.0, 0, 0]), np.array([1.0, 0, 0]), 0.0, 4.0), epsilon=0.0)
    out["two_site_cells"] = segs.cells
    out["two_site_t0"] = segs.t_entry
    out["two_site_t1"] = segs.t_exit
    out["two_site_pos"] = pos
    out["softplus_in"] = np.array([0.0, 10.0, -10.0, 1e-3, -3.0, 20.0])
    out["softplus_out"] = rfoam_foam.softplus(out["softplus_in"])
    out["softplus_grad_out"] = rfoam_foam.softplus_grad(out["softplus_in"])
    d = np.array([0.48, -0.6, 0.64])
    out["basis_dir"] = d
    basis = np.empty(16)
    kernels.sh_basis_into(d[0], d[1], d[2], basis)
    out["basis"] = basis
    # composite KATs
    out["ln2"] = np.log(2.0)
    np.savez_compressed(os.path.join(HERE, "kat.npz"), **out)
    print("kat", {k: v for k, v in out.items() if np.size(v) < 4})


def adam_case():
    """train.py:195-209 post-processing + adam.py:15-31 for two iterations
    (second with the SH warm-up mask off and positions frozen), on
    fp32-representable gradients so the device's fp32 buffer holds them
    exactly."""
    from rfoam.optim.adam import AdamState, adam_step

    rng = np.random.default_rng(21)
    n = 300
    pos = rng.uniform(-1, 1, (n, 3))
    raw = rng.normal(0, 1, n)
    sh = rng.normal(0, 0.3, (n, 16, 3))
    out = dict(pos0=pos.copy(), raw0=raw.copy(), sh0=sh.copy())
    st = [AdamState(pos.shape), AdamState(raw.shape), AdamState(sh.shape)]
    clip = 1e3
    for it, (lrs, warm) in enumerate([((2e-4, 1e-1, 5e-3), True), ((0.0, 5e-2, 2e-3), False)]):
        g_pos = (rng.normal(0, 1, (n, 3)) * 10).astype(np.float32).astype(np.float64)
        g_sig = (rng.normal(0, 1, n) * 2).astype(np.float32).astype(np.float64)
        g_sh = rng.normal(0, 1, (n, 16, 3)).astype(np.float32).astype(np.float64)
        g_pos[0, 0] = 5e3  # exercises the clip
        g_sh[1, 2, 1] = -2e3
        out[f"g_pos{it}"], out[f"g_sig{it}"], out[f"g_sh{it}"] = g_pos, g_sig, g_sh
        out[f"lrs{it}"] = np.array(lrs)
        out[f"warm{it}"] = np.array(warm)
        d_raw = g_sig * rfoam_foam.softplus_grad(raw)
        d_sh = g_sh.copy()
        if warm:
            d_sh[:, 1:, :] = 0.0
        d_pos = g_pos.copy()
        np.clip(d_raw, -clip, clip, out=d_raw)
        np.clip(d_sh, -clip, clip, out=d_sh)
        np.clip(d_pos, -clip, clip, out=d_pos)
        if lrs[0] > 0.0:
            adam_step(pos, d_pos, st[0], lrs[0])
        adam_step(raw, d_raw, st[1], lrs[1])
        adam_step(sh, d_sh, st[2], lrs[2])
        out[f"pos{it + 1}"], out[f"raw{it + 1}"], out[f"sh{it + 1}"] = pos.copy(), raw.copy(), sh.copy()
    np.savez_compressed(os.path.join(HERE, "adam.npz"), **out)
    print("adam", {k: v.shape for k, v in out.items() if k.startswith("pos")})


def checkpoint_case():
    """A reference-written RFOAM1 file (io/checkpoint.py:18-27)."""
    from rfoam.io.checkpoint import save_checkpoint

    sc = ref_scene(300, 31, 3, check_delaunay=False)
    save_checkpoint(sc, os.path.join(HERE, "scene300.rfoam"))
    np.savez_compressed(os.path.join(HERE, "scene300_expect.npz"),
                        positions=sc.positions.astype(np.float32).astype(np.float64),
                        raw=sc.raw_density.astype(np.float32).astype(np.float64),
                        sh=sc.sh_coeffs.astype(np.float32).astype(np.float64),
                        background=sc.background.astype(np.float32).astype(np.float64))


def adjacency_case():
    """geometry/delaunay.py build + adjacency.py from_triangulation on three
    point sets (uniform, surface shell, anisotropic Gaussian cluster):
    offsets, neighbors and hull flags, for the device builder."""
    out = {}
    rng = np.random.default_rng(99)
    sets = {
        "uniform2k": random_positions(2000, 7),
        "surface3k": random_positions(3000, 2, "surface"),
        "gauss1500": (rng.normal(size=(1500, 3)) * [1.0, 0.3, 2.0]).astype(np.float32)
        .astype(np.float64),
    }
    for name, pos in sets.items():
        adj = AdjacencyGraph.from_triangulation(build(pos))
        out[f"{name}_positions"] = pos
        out[f"{name}_offsets"] = adj.offsets
        out[f"{name}_neighbors"] = adj.neighbors.astype(np.int32)
        out[f"{name}_hull"] = adj.hull
        print(name, len(adj.neighbors), int(adj.hull.sum()))
    np.savez_compressed(os.path.join(HERE, "adjacency.npz"), **out)


def effects_case():
    """rays.py:60-176: intersect_face, reflect, refract (incl. back side and
    total internal reflection) and apply_effect on random unit vectors."""
    from rfoam.tracer.rays import EffectPlane, apply_effect, reflect, refract

    rng = np.random.default_rng(77)
    m = 64
    d = rng.normal(size=(m, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    o = rng.uniform(-1, 1, (m, 3))
    nr = rng.normal(size=(m, 3))
    nrm = np.stack([EffectPlane(np.zeros(3), v).normal for v in nr])
    eta = np.where(np.arange(m) % 2 == 0, 1.5, 1.0 / 1.5)
    t_at = rng.uniform(0, 2, m)
    out = {"d": d, "o": o, "normal": nrm, "eta": eta, "t_at": t_at}
    out["reflect"] = np.stack([reflect(d[i], nrm[i]) for i in range(m)])
    out["refract"] = np.stack([refract(d[i], nrm[i], eta[i]) for i in range(m)])
    for kind in ("mirror", "refract"):
        rs = [apply_effect(Ray(o[i], d[i], 0.0, 9.0), nrm[i], kind, eta[i], t_at[i])
              for i in range(m)]
        out[f"{kind}_o"] = np.stack([r.origin for r in rs])
        out[f"{kind}_d"] = np.stack([r.direction for r in rs])
    xs, xps = rng.uniform(-1, 1, (m, 3)), rng.uniform(-1, 1, (m, 3))
    xps[0] = xs[0] + np.cross(d[0], [0.0, 0.0, 1.0])  # face parallel to the ray
    f = [intersect_face(Ray(o[i], d[i]), xs[i], xps[i]) for i in range(m)]
    out.update(x=xs, xp=xps, face_t=np.array([v[0] for v in f]),
               face_front=np.array([v[1] for v in f]))
    tir = sum(1 for i in range(m) if np.allclose(out["refract"][i], out["reflect"][i] /
                                                 np.linalg.norm(out["reflect"][i])))
    np.savez_compressed(os.path.join(HERE, "effects.npz"), **out)
    print("effects", m, "tir/mirror-equal", tir)


if __name__ == "__main__":
    if len(sys.argv) > 1:  # regenerate only the named cases, e.g. `effects`
        for name in sys.argv[1:]:
            globals()[f"{name}_case"]()
        sys.exit(0)
    adjacency_case()
    effects_case()
    checkpoint_case()
    adam_case()
    kat_case()
    s2k = ref_scene(2000, 7, 3)
    frame_case("frame_2k_deg3", s2k, (0.0, 0.0, 3.0), 64, 48, 1e-3, seed=1)
    frame_case("frame_2k_deg3_eps0_orbit", s2k, tuple(orbit_poses(np.zeros(3), 3.0, 0.3, 8)[3][:3, 3]),
               40, 32, 0.0, seed=2)
    frame_case("frame_2k_deg3_fisheye", s2k, (0.3, 0.2, 2.6), 48, 36, 1e-3, seed=5,
               angle=1.4, kind=FISHEYE)
    s10k = ref_scene(10000, 0, 0, check_delaunay=False)
    frame_case("frame_10k_deg0", s10k, (0.0, 0.0, 3.0), 32, 32, 1e-3, seed=3)
    s3k = ref_scene(3000, 2, 3, kind="surface")
    frame_case("frame_3k_surface", s3k, tuple(orbit_poses(np.zeros(3), 3.0, 0.3, 8)[0][:3, 3]),
               48, 27, 1e-3, seed=4)
    grad_case("grad_2k_deg3", s2k, 64, 11, 1e-3)
    grad_case("grad_10k_deg0", s10k, 64, 15, 1e-3)
    grad_case("grad_2k_deg3_inside_eps0", s2k, 48, 12, 0.0, inside=True)
    train_case("train_2k_deg3_q", s2k, 192, 13, 1e-3, 0.01 / (192 * 2))
    train_case("train_3k_surface_q", s3k, 160, 14, 1e-3, 0.01 / (160 * 2))
