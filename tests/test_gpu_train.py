"""fused gradient post-processing + Adam on the GPU against
the reference's own numbers (tests/golden/adam.npz from optim/train.py:195-209
+ optim/adam.py), and a full device-resident training iteration
(train_batch + post-processing + Adam + scene refresh) against the oracle."""

import numpy as np
import pytest
import torch

from conftest import golden_scene, load_golden
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def test_post_grad_adam_matches_reference(cuda_ok):
    from paper_2502_01157_b200.scene import AdjacencyGraph, FoamScene
    from paper_2502_01157_b200.train import AdamHyper, DeviceTrainer

    g = load_golden("adam")
    n = len(g["pos0"])
    # a throwaway adjacency (the update does not walk)
    adj = AdjacencyGraph(g["pos0"], np.arange(n + 1), np.roll(np.arange(n), 1))
    tr = DeviceTrainer(FoamScene(g["pos0"], g["raw0"], g["sh0"], np.zeros(3), adj))
    for it in range(2):
        tr.grads.g4[:, :3] = torch.from_numpy(g[f"g_pos{it}"]).float().cuda()
        tr.grads.g4[:, 3] = torch.from_numpy(g[f"g_sig{it}"]).float().cuda()
        tr.grads.sh[:] = torch.from_numpy(g[f"g_sh{it}"].reshape(n, 48)).float().cuda()
        lp, ld, ls = g[f"lrs{it}"]
        tr.post_grad_adam(lp, ld, ls, bool(g[f"warm{it}"]), AdamHyper())
        torch.cuda.synchronize()
        np.testing.assert_array_equal(tr.positions.cpu().numpy(), g[f"pos{it + 1}"])
        np.testing.assert_array_equal(tr.sh.cpu().numpy().reshape(n, 16, 3), g[f"sh{it + 1}"])
        # d_raw uses exp(): CUDA vs numpy may differ in the last ulp
        np.testing.assert_allclose(tr.raw.cpu().numpy(), g[f"raw{it + 1}"], rtol=1e-13, atol=0)
    # the walk arrays were refreshed from the new parameters
    s4 = tr.ds.site4.cpu().numpy()
    np.testing.assert_array_equal(s4[:, :3], g["pos2"])
    from paper_2502_01157_b200.scene import softplus
    np.testing.assert_allclose(s4[:, 3], softplus(g["raw2"]), rtol=1e-13)
    if tr.ds.sh32 is not None:  # fp32 channel-major copy written by the Adam pass
        sh32 = tr.ds.sh32.cpu().numpy().reshape(n, 3, 16)
        if tr.ds.pk_of is not None:  # rows in the packed (Morton) order
            sh32 = sh32[tr.ds.pk_of.cpu().numpy()]
        np.testing.assert_array_equal(sh32, g["sh2"].astype(np.float32).transpose(0, 2, 1))


def test_device_training_iteration(cuda_ok):
    from paper_2502_01157_b200.scene import softplus, softplus_grad
    from paper_2502_01157_b200.train import AdamHyper, DeviceTrainer, adam_step_numpy

    g = load_golden("train_2k_deg3_q")
    scene = golden_scene(g)
    n = scene.n_sites
    m = len(g["origins"])
    d = lambda a, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)  # noqa
    tr = DeviceTrainer(scene)
    tr.step(d(g["origins"]), d(g["dirs"]), d(np.zeros(m)), d(g["t_max"]),
            d(g["start"], torch.int32), d(g["targets"]), lr_position=2e-4, lr_density=0.1,
            lr_sh=5e-3, sh_warmup=True, quantile_scale=float(g["quantile_scale"]),
            u_pairs=d(g["u_pairs"]))
    torch.cuda.synchronize()
    # reference iteration from the golden per-worker buffers (train.py:189-209)
    d_sigma = g["d_sigma_w"].sum(0)
    d_sh = g["d_sh_w"].sum(0).reshape(n, 16, 3)
    d_pos = g["d_pos_w"].sum(0)
    d_raw = d_sigma * softplus_grad(g["raw_density"])
    d_sh[:, 1:, :] = 0.0
    m_sh = np.zeros_like(d_sh)
    v_sh = np.zeros_like(d_sh)
    sh_ref = adam_step_numpy(g["sh"].reshape(n, 16, 3).copy(), np.clip(d_sh, -1e3, 1e3), m_sh,
                             v_sh, 1, 5e-3)
    st = tr.adam_state.cpu().numpy()
    m_pos, v_pos = st[:3 * n].reshape(n, 3), st[3 * n:6 * n].reshape(n, 3)
    m_raw = st[6 * n:7 * n]
    # moments are linear / quadratic in the gradient: 1e-3 relative per tensor
    rel = lambda a, b: np.abs(a - b).max() / np.abs(b).max()  # noqa
    assert rel(m_pos, 0.1 * d_pos) <= 1e-3
    assert rel(v_pos, 0.001 * d_pos ** 2) <= 2e-3
    assert rel(m_raw, 0.1 * d_raw) <= 1e-3
    # SH after one step: where the gradient is not negligible, Adam moves by ~lr*sign(g)
    big = np.abs(d_sh) > 1e-2 * np.abs(d_sh).max()
    got = tr.sh.cpu().numpy().reshape(n, 16, 3)
    np.testing.assert_allclose(got[big], sh_ref[big], rtol=0, atol=1e-9)
    assert float(tr.loss[0]) == pytest.approx(g["loss_w"].sum(0)[0], rel=1e-6)
    s4 = tr.ds.site4.cpu().numpy()
    np.testing.assert_allclose(s4[:, 3], softplus(tr.raw.cpu().numpy()), rtol=1e-13)


def test_device_training_loop_with_rebuilds(cuda_ok):
    """Several device-resident iterations (train_batch + Adam + refresh) with
    the Delaunay adjacency rebuilt on the device every few steps, as the
    reference's loop does (optim/train.py:247-256): the loss falls, and after
    each rebuild the device CSR equals a host (Qhull) triangulation of the
    moved sites."""
    from paper_2502_01157_b200 import device as dv
    from paper_2502_01157_b200.synthetic import delaunay_csr
    from paper_2502_01157_b200.train import DeviceTrainer

    g = load_golden("train_2k_deg3_q")
    scene = golden_scene(g)
    d = lambda a, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)  # noqa
    # targets: the scene's own render with perturbed colours (a reachable fit)
    rng = np.random.default_rng(8)
    m = 4096
    o = np.tile([0.0, 0.0, 3.0], (m, 1))
    dirs = rng.normal(size=(m, 3)) * [0.25, 0.25, 0.0] + [0.0, 0.0, -1.0]
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    tr = DeviceTrainer(scene)
    start = int(tr.ds.locate(d(o[:1])).item())
    tmax = tr.ds.default_t_max(o[:1])
    ref = dv.render_rays_device(tr.ds, d(o), d(dirs), d(np.zeros(m)), d(np.full(m, tmax)),
                                d(np.full(m, start), torch.int32), f64=True)
    targets = (ref.rgb * 0.8 + 0.1).contiguous()
    losses = []
    for it in range(12):
        start = int(tr.ds.locate(d(o[:1])).item())
        tmax = tr.ds.default_t_max(o[:1])
        loss = tr.step(d(o), d(dirs), d(np.zeros(m)), d(np.full(m, tmax)),
                       d(np.full(m, start), torch.int32), targets, lr_position=1e-4,
                       lr_density=0.05, lr_sh=2e-2)
        losses.append(float(loss[0].item()) / (3 * m))
        if (it + 1) % 4 == 0:
            info = tr.rebuild_adjacency()
            pos = tr.positions.cpu().numpy()
            off, nbr, _ = delaunay_csr(pos)
            np.testing.assert_array_equal(tr.ds.offsets.cpu().numpy(), off)
            np.testing.assert_array_equal(tr.ds.neighbors.cpu().numpy(), nbr)
            assert info["reverse_edges_added"] == 0
    assert losses[-1] < 0.7 * losses[0], losses


def test_trainer_dc_only_scene_after_warmup(cuda_ok):
    """A scene initialised with the DC band only (train.py:77 scene_from_sfm) gains
    higher SH bands once the warm-up ends; the trainer's walk must then colour
    with all 16 bands (the scene is pinned to SH degree 3) and its fp32 colour
    bound must follow the grown coefficients (rfb_scene.sh_absmax_dev)."""
    from paper_2502_01157_b200 import device as dv
    from paper_2502_01157_b200.train import DeviceTrainer

    g = load_golden("train_2k_deg3_q")
    scene = golden_scene(g)
    scene.sh_coeffs = scene.sh_coeffs.copy()
    scene.sh_coeffs[:, 1:, :] = 0.0
    n = scene.n_sites
    m = len(g["origins"])
    d = lambda a, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)  # noqa
    tr = DeviceTrainer(scene)
    assert tr.ds.sh_degree == 3
    bound0 = float(tr.ds.sh_absmax_dev.item())
    for _ in range(3):  # past the warm-up: bands 1..15 receive gradients
        tr.step(d(g["origins"]), d(g["dirs"]), d(np.zeros(m)), d(g["t_max"]),
                d(g["start"], torch.int32), d(g["targets"]), lr_position=0.0, lr_density=0.05,
                lr_sh=0.5, sh_warmup=False)
    torch.cuda.synchronize()
    sh = tr.sh.cpu().numpy()
    assert np.abs(sh.reshape(n, 16, 3)[:, 1:, :]).max() > 0.1
    assert float(tr.ds.sh_absmax_dev.item()) >= np.abs(sh).max().astype(np.float32)
    assert float(tr.ds.sh_absmax_dev.item()) > bound0
    # the trainer's scene renders exactly what the oracle renders from the updated
    # parameters (sigma read back from the device's site4)
    res = dv.render_rays_device(tr.ds, d(g["origins"]), d(g["dirs"]), d(np.zeros(m)),
                                d(g["t_max"]), d(g["start"], torch.int32), f64=True)
    torch.cuda.synchronize()
    s4 = tr.ds.site4.cpu().numpy()
    sa = orc.SceneArrays(s4[:, :3], g["offsets"], g["neighbors"], s4[:, 3], sh,
                         g["background"])
    ref = orc.render_rays(sa, g["origins"], g["dirs"], 0.0, g["t_max"], g["start"])
    np.testing.assert_array_equal(res.status.cpu().numpy(), ref["status"])
    assert np.abs(res.rgb.cpu().numpy() - ref["rgb"]).max() <= 1e-4


def test_trainer_rejects_moving_fixed_sites(cuda_ok):
    from paper_2502_01157_b200.train import AdamHyper, DeviceTrainer

    g = load_golden("train_2k_deg3_q")
    tr = DeviceTrainer(golden_scene(g), update_positions=False)
    with pytest.raises(ValueError):
        tr.post_grad_adam(1e-4, 0.1, 5e-3, False, AdamHyper())
