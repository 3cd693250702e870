"""world_size-2 gloo runs of the multi-GPU host logic:
tile-sharded frame assembly is bitwise identical to the unsharded frame and
the gradient all-reduce equals the sum of per-rank buffers."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_01157_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, W, H, ret):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)
        full = torch.from_numpy(rng.uniform(0, 1, (H * W, 3)).astype(np.float32))
        tiles = D.tile_assignment(W, H, rank, world)
        mask = torch.from_numpy(D.tile_pixel_mask(W, H, tiles).reshape(-1))
        local = torch.zeros_like(full)
        local[mask] = full[mask]   # this rank "renders" its tiles only
        D.assemble_frame(local, dst=None)
        ok_frame = bool(torch.equal(local, full))
        # gradients: each rank contributes its own buffer; all-reduce = sum
        n = 37
        g = torch.from_numpy(np.random.default_rng(100 + rank).normal(size=n * 52)
                             .astype(np.float32))
        loss = torch.tensor([float(rank + 1), 0.5], dtype=torch.float64)
        mine = g.clone()
        D.allreduce_gradients(g, loss)
        parts = [torch.from_numpy(np.random.default_rng(100 + r).normal(size=n * 52)
                                  .astype(np.float32)) for r in range(world)]
        ok_grad = bool(torch.allclose(g, sum(parts), rtol=0, atol=1e-6))
        ok_loss = abs(float(loss[0]) - world * (world + 1) / 2) < 1e-12
        ret[rank] = (ok_frame, ok_grad, ok_loss, bool(torch.equal(mine, parts[rank])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("W,H", [(96, 64), (130, 70)])
def test_gloo_world2_frame_and_gradients(W, H):
    world = 2
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    ret = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, W, H, ret)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert all(all(v) for v in ret.values()) and len(ret) == world, dict(ret)
