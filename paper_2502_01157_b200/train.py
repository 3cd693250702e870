"""Device-resident training step.

One iteration of the reference loop's hot part (optim/train.py:131-209) with
every array resident on the GPU:

  rfb_train_batch   walk + composite + L2 adjoint + reverse pass (+ quantile)
  all-reduce        one NCCL all-reduce of the flat [n, 52] fp32 gradients and
                    the loss pair (multi-GPU; rgb_scale uses the global ray
                    count, train.py:168-173)
  rfb_post_grad_adam  d_raw = dsigma * sigmoid(10 raw), SH warm-up mask,
                    +-clip, Adam with bias correction on the fp64 parameters
                    (train.py:195-209, adam.py:15-31)
  rfb_refresh_scene softplus -> site4 / packed headers, fp32 SH copy

Densify/prune/rebuild (train.py:211-256) stay out of scope: the adjacency is
used as given (stale between rebuilds exactly like the reference,
foam.py:70-80).  When positions are updated the scene is walked with the
generic fp64 layout (moved positions are no longer fp32-exact).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import device as dv
from .distributed import allreduce_gradients, world

# the Adam pass also writes the packed scene's fp32 SH copy (rfb_post_grad_adam
# sh32), so rfb_refresh_scene skips its fp64 -> fp32 SH pass
FUSE_SH32 = True


@dataclass
class AdamHyper:
    lr_position: float = 2e-4     # optim/config.py:20
    lr_density: float = 1e-1
    lr_sh: float = 5e-3
    beta1: float = 0.9            # optim/adam.py:15
    beta2: float = 0.999
    eps: float = 1e-8
    grad_clip: float = 1e3        # optim/config.py:44


class DeviceTrainer:
    """fp64 parameters + Adam moments on the GPU; one ``step`` = one training
    iteration's hot part.  ``scene`` is a FoamScene with adjacency."""

    def __init__(self, scene, device=None, update_positions=True):
        self.update_positions = bool(update_positions)
        # moving sites: packed layout with the fp64-position bound from the start
        # (rfb_refresh_scene then re-derives the fp32 copies after every step)
        # SH degree pinned to 3: a scene initialised with the DC band only
        # (train.py:77 scene_from_sfm) gains higher bands once the SH warm-up
        # ends, so the walk must read all 16 bands from the start
        self.ds = dv.DeviceScene(scene, device=device, sh_degree=3,
                                 positions_f64=True if update_positions else None)
        self.device = self.ds.device
        n = self.ds.n_sites
        self.n = n
        self.positions = torch.from_numpy(
            np.ascontiguousarray(scene.adjacency.positions, dtype=np.float64)).to(self.device)
        self.raw = torch.from_numpy(np.ascontiguousarray(scene.raw_density,
                                                         dtype=np.float64)).to(self.device)
        self.sh = self.ds.sh  # the walk reads this table: updated in place
        self.adam_state = torch.zeros(104 * n, dtype=torch.float64, device=self.device)
        self.steps = [0, 0, 0]  # Adam step counters per group (AdamState.step)
        self.grads = dv.GradBuffers(n, self.device)
        self.loss = torch.zeros(2, dtype=torch.float64, device=self.device)
        self.ws = dv.Workspace(self.device)
        self.lib = _lib.load()

    def post_grad_adam(self, lr_position, lr_density, lr_sh, sh_warmup, hyper: AdamHyper,
                       stream=None):
        do_pos = lr_position > 0.0
        if do_pos and not self.update_positions:
            # the packed fp32-exact layout cannot take moved sites in place
            # (rfb_refresh_scene would leave the fp32 edge records stale)
            raise ValueError("lr_position > 0 on a DeviceTrainer built with "
                             "update_positions=False")
        lrs = (lr_position, lr_density, lr_sh)
        h = np.zeros(18)
        for k in range(3):
            if k == 0 and not do_pos:
                continue
            self.steps[k] += 1
            s = self.steps[k]
            h[6 * k: 6 * k + 6] = (lrs[k], hyper.beta1, hyper.beta2, hyper.eps,
                                   1.0 - hyper.beta1 ** s, 1.0 - hyper.beta2 ** s)
        hp = np.ascontiguousarray(h)
        fuse = FUSE_SH32 and self.ds.sh32 is not None
        sh32 = dv._ptr(self.ds.sh32) if fuse else None
        _lib.check(self.lib.rfb_post_grad_adam(
            self.n, dv._ptr(self.grads.flat), dv._ptr(self.positions), dv._ptr(self.raw),
            dv._ptr(self.sh), dv._ptr(self.adam_state), float(hyper.grad_clip),
            1 if sh_warmup else 0, 1 if do_pos else 0,
            hp.ctypes.data_as(ctypes.c_void_p), sh32, dv._ptr(self.ds.sh_absmax_dev),
            dv._ptr(self.ds.pk_of), dv._stream(stream)), "rfb_post_grad_adam")
        _lib.check(self.lib.rfb_refresh_scene(self.ds.c, dv._ptr(self.positions),
                                              dv._ptr(self.raw), 0 if fuse else 1,
                                              dv._stream(stream)),
                   "rfb_refresh_scene")

    def rebuild_adjacency(self, stream=None) -> dict:
        """Re-triangulate the moved sites on the device (train.py:247-256's
        rebuild cadence; delaunay.build -> rfb_build_adjacency)."""
        return self.ds.rebuild_adjacency(self.positions, stream=stream)

    def step(self, origins, directions, t_min, t_max, start, targets, *, lr_position,
             lr_density, lr_sh, sh_warmup=False, quantile_scale=0.0, u_pairs=None,
             weight_floor=1e-4, m_global=None, epsilon=1e-3, step_limit=4096,
             hyper: AdamHyper | None = None, stream=None):
        """Returns (loss_rgb, loss_quantile) summed over ranks (device tensor)."""
        hyper = hyper or AdamHyper()
        m = origins.shape[0]
        _, ws = world()
        m_global = m_global or m * ws
        self.grads.zero_()
        self.loss.zero_()
        dv.train_batch_device(self.ds, origins, directions, t_min, t_max, start, targets,
                              self.grads, self.loss, rgb_scale=1.0 / (3.0 * m_global),
                              quantile_scale=quantile_scale, u_pairs=u_pairs,
                              weight_floor=weight_floor, epsilon=epsilon,
                              step_limit=step_limit, workspace=self.ws, stream=stream)
        allreduce_gradients(self.grads.flat, self.loss)
        self.post_grad_adam(lr_position, lr_density, lr_sh, sh_warmup, hyper, stream)
        return self.loss


def adam_step_numpy(params, grads, m, v, step, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """Host mirror of optim/adam.py:15-31 (same operation order), for tests."""
    m *= beta1
    m += (1.0 - beta1) * grads
    v *= beta2
    v += (1.0 - beta2) * grads * grads
    m_hat = m / (1.0 - beta1 ** step)
    v_hat = v / (1.0 - beta2 ** step)
    params -= lr * m_hat / (np.sqrt(v_hat) + eps)
    return params
