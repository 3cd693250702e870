"""Multi-GPU sharding of the hot path: one process per GPU,
``torch.distributed`` for the plumbing.

* Forward (configs 2/4): image tiles (32x32) are interleaved round-robin over
  the ranks, the scene is replicated, every rank renders its tiles into a
  full-frame buffer that is zero elsewhere, and a SUM reduction assembles the
  frame on the destination rank.  Each pixel is written by exactly one rank
  and x + 0 == x, so the assembled frame is bitwise identical to a 1-GPU
  render.  No collective is on the data path except this final gather.
* Training (configs 3/5): each rank renders its own view (or its share of the
  ray batch), accumulates per-site gradients into the flat fp32 [n, 52]
  buffer with ``rgb_scale = 1 / (3 * m_global)`` (train.py:168-173), and ONE
  all-reduce of that buffer (NCCL over NVLink/NVSwitch on B200; gloo in the
  CPU tests) makes every rank hold the global gradient.  Loss scalars are
  all-reduced too.

The rendering calls are librfb.so kernels; this module only decides which
tiles / rays a rank owns and issues the collectives.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def tile_grid(width: int, height: int, tile_w: int = 32, tile_h: int = 32):
    return (width + tile_w - 1) // tile_w, (height + tile_h - 1) // tile_h


def tile_assignment(width: int, height: int, rank: int, world_size: int, tile_w: int = 32,
                    tile_h: int = 32) -> np.ndarray:
    """Tile ids (ty * tiles_x + tx) owned by ``rank``: interleaved round-robin,
    so the expensive centre of the frame is spread over every rank."""
    tx, ty = tile_grid(width, height, tile_w, tile_h)
    return np.arange(tx * ty, dtype=np.int32)[rank::world_size].copy()


def tile_pixel_mask(width: int, height: int, tiles: np.ndarray, tile_w: int = 32,
                    tile_h: int = 32) -> np.ndarray:
    """Boolean (H, W) mask of the pixels covered by ``tiles`` (host helper)."""
    tx, _ = tile_grid(width, height, tile_w, tile_h)
    mask = np.zeros((height, width), dtype=bool)
    for t in np.asarray(tiles):
        y0, x0 = (int(t) // tx) * tile_h, (int(t) % tx) * tile_w
        mask[y0:y0 + tile_h, x0:x0 + tile_w] = True
    return mask


def assemble_frame(local_frame: torch.Tensor, dst: int | None = 0, group=None) -> torch.Tensor:
    """Sum the per-rank frames (zero outside each rank's tiles).  dst=None:
    every rank receives the frame (all-reduce)."""
    _, ws = world()
    if ws == 1:
        return local_frame
    # gloo reduces device tensors only through all-reduce (its reduce is host-only)
    gloo_dev = local_frame.is_cuda and dist.get_backend(group) == "gloo"
    if dst is None or gloo_dev:
        dist.all_reduce(local_frame, op=dist.ReduceOp.SUM, group=group)
    else:
        dist.reduce(local_frame, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return local_frame


def allreduce_gradients(flat: torch.Tensor, loss: torch.Tensor | None = None, group=None):
    """One all-reduce of the flat [n*52] gradient buffer (and the loss pair)."""
    _, ws = world()
    if ws == 1:
        return flat
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    if loss is not None:
        dist.all_reduce(loss, op=dist.ReduceOp.SUM, group=group)
    return flat


def shard_rays(m_global: int, rank: int, world_size: int):
    """Contiguous [lo, hi) ray range of ``rank`` (the reference's worker
    chunking, kernels.py:396-404, lifted to ranks)."""
    chunk = (m_global + world_size - 1) // world_size
    lo = min(m_global, rank * chunk)
    return lo, min(m_global, lo + chunk)


class ShardedRenderer:
    """Tile-sharded frame renderer over the ranks of the default group."""

    def __init__(self, device_scene, width: int, height: int, tile_w: int = 32,
                 tile_h: int = 32, lanes_per_ray: int | None = None):
        from . import device as dv

        self.dv = dv
        self.ds = device_scene
        self.rank, self.world = world()
        self.width, self.height = width, height
        self.tile_w, self.tile_h = tile_w, tile_h
        tiles = tile_assignment(width, height, self.rank, self.world, tile_w, tile_h)
        self.tiles = torch.from_numpy(tiles).to(device_scene.device)
        self.lanes = lanes_per_ray or dv.DEFAULT_LANES
        self.ws = dv.Workspace(device_scene.device)
        # fp64 frame: the reference's render_image contract (render.py:128-149)
        self.out = dv.alloc_forward(width * height, device_scene.device, f64=True, per_ray=False)

    def render(self, camera, epsilon=1e-3, step_limit=4096, dst: int | None = 0):
        """Render this rank's tiles and assemble the (H*W, 3) float64 frame on
        ``dst`` (None: everywhere)."""
        if self.world > 1:
            self.out.rgb.zero_()
        self.dv.render_image_device(self.ds, camera, epsilon=epsilon, step_limit=step_limit,
                                    tile_ids=self.tiles, tile_w=self.tile_w, tile_h=self.tile_h,
                                    lanes_per_ray=self.lanes, workspace=self.ws, out=self.out)
        return assemble_frame(self.out.rgb, dst=dst)

    def render_to_host(self, camera, epsilon=1e-3, step_limit=4096, dst: int = 0):
        """render() plus the device->host copy of the assembled frame on ``dst`` into a
        pinned buffer (two alternate, so the previous frame stays valid for one more call).
        Returns the (H, W, 3) float64 numpy image on ``dst`` -- render_image's contract
        (render.py:128-149) -- and None elsewhere."""
        frame = self.render(camera, epsilon=epsilon, step_limit=step_limit, dst=dst)
        if self.rank != dst:
            return None
        if not hasattr(self, "_pinned"):
            self._pinned = [torch.empty(frame.shape, dtype=frame.dtype, pin_memory=True)
                            for _ in range(2)]
            self._next = 0
        host = self._pinned[self._next]
        self._next ^= 1
        host.copy_(frame, non_blocking=True)
        torch.cuda.current_stream(frame.device).synchronize()
        return host.numpy().reshape(self.height, self.width, 3)
