"""The multi-GPU path with real kernels in more than one process:
two ranks on cuda:0 joined by gloo (device tensors; the collectives are host
mediated, so no kernel of one rank waits on the other).  Each rank renders
its interleaved tiles through distributed.ShardedRenderer and trains its own
view through train.DeviceTrainer.step (global rgb_scale, one all-reduce of the
flat [n,52] gradients, then the fused Adam).  Checked against a single
process doing both views: the assembled frame bitwise, the all-reduced
gradients within 1e-3 relative, the loss to 1e-9, and both ranks' updated
parameters identical (reference: optim/train.py:168-209)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _views(W, H):
    import sys
    sys.path.insert(0, REPO)
    from bench import make_views

    return make_views(2, W, H)


def _batch(cam, ds, d):
    import torch

    dirs = cam.ray_directions()
    m = len(dirs)
    o = np.broadcast_to(cam.position, (m, 3)).copy()
    start = int(ds.locate(d(o[:1])).item())
    t_max = np.full(m, ds.default_t_max(cam.position[None, :]))
    targets = np.random.default_rng(30).uniform(0.0, 1.0, (m, 3))
    return (d(o), d(dirs), d(np.zeros(m)), d(t_max), d(np.full(m, start), torch.int32),
            d(targets))


def _worker(rank, world, port, ret):
    import sys
    sys.path.insert(0, REPO)
    sys.path.insert(0, os.path.join(REPO, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    from conftest import golden_scene, load_golden
    from paper_2502_01157_b200 import device as dv
    from paper_2502_01157_b200.distributed import ShardedRenderer
    from paper_2502_01157_b200.train import DeviceTrainer

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = load_golden("train_2k_deg3_q")
        scene = golden_scene(g)
        W, H = 160, 96
        cams = _views(W, H)
        ds = dv.DeviceScene(scene)
        d = lambda a, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)  # noqa
        # forward: this rank's tiles, frame assembled everywhere
        sr = ShardedRenderer(ds, W, H)
        frame = sr.render(cams[1], dst=None).clone()
        host = sr.render_to_host(cams[0], dst=0)
        full = [dv.render_image_device(ds, c, f64=True).rgb for c in cams]
        torch.cuda.synchronize()
        ok_frame = bool(torch.equal(frame, full[1]))
        ok_host = True if rank != 0 else bool(
            np.array_equal(host, full[0].cpu().numpy().reshape(H, W, 3)))
        # training: rank r trains view r; the reduced gradient is the two-view sum
        b = _batch(cams[rank], ds, d)
        m = b[0].shape[0]
        tr = DeviceTrainer(scene)
        tr.step(*b, lr_position=1e-4, lr_density=0.05, lr_sh=5e-3, m_global=2 * m)
        torch.cuda.synchronize()
        g_dist = tr.grads.flat.double().cpu().numpy()
        loss_dist = tr.loss.cpu().numpy().copy()
        # single-process reference over both views, same global scale
        gb = dv.GradBuffers(ds.n_sites, ds.device)
        loss = torch.zeros(2, dtype=torch.float64, device="cuda")
        for c in cams:
            bb = _batch(c, ds, d)
            dv.train_batch_device(ds, *bb, gb, loss, rgb_scale=1.0 / (3.0 * 2 * m))
        torch.cuda.synchronize()
        g_ref = gb.flat.double().cpu().numpy()
        n = ds.n_sites

        def rel(a, r):
            return float(np.abs(a - r).max() / np.abs(r).max())

        errs = [rel(g_dist[:4 * n].reshape(n, 4)[:, 3], g_ref[:4 * n].reshape(n, 4)[:, 3]),
                rel(g_dist[:4 * n].reshape(n, 4)[:, :3], g_ref[:4 * n].reshape(n, 4)[:, :3]),
                rel(g_dist[4 * n:], g_ref[4 * n:])]
        ok_grad = max(errs) <= 1e-3
        ok_loss = abs(loss_dist[0] - float(loss[0])) <= 1e-9 * abs(float(loss[0]))
        # both ranks applied the same update
        chk = torch.tensor([float(tr.positions.sum()), float(tr.sh.sum()), float(tr.raw.sum())],
                           dtype=torch.float64)
        lo, hi = chk.clone(), chk.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        ok_same = bool(torch.equal(lo, hi))
        ret[rank] = dict(frame=ok_frame, host=ok_host, grad=ok_grad, errs=errs, loss=ok_loss,
                         same=ok_same)
    finally:
        dist.destroy_process_group()


def test_two_ranks_render_and_train_on_one_gpu(cuda_ok):
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    ret = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ret)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    res = dict(ret)
    assert len(res) == world, res
    for r, v in res.items():
        assert v["frame"] and v["host"] and v["grad"] and v["loss"] and v["same"], (r, v)
