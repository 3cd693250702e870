"""Reverse-pass iteration count per 32-ray warp (needs a RFB_COUNT_ITERS build)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import make_views  # noqa: E402
from paper_2502_01157_b200 import device as dv  # noqa: E402
from paper_2502_01157_b200.synthetic import make_foam  # noqa: E402

scene = make_foam(1_000_000, 1, 3)
ds = dv.DeviceScene(scene)
cam = make_views(1, 1920, 1080)[0]
dirs = cam.ray_directions_device()
m = dirs.shape[0]
o = torch.from_numpy(np.broadcast_to(cam.position, (m, 3)).copy()).cuda()
start = ds.locate(o[:1]).expand(m).contiguous()
tmin = torch.zeros(m, dtype=torch.float64, device="cuda")
tmax = torch.full((m,), ds.default_t_max(cam.position[None, :]), dtype=torch.float64, device="cuda")
tg = torch.from_numpy(np.random.default_rng(11).uniform(0, 1, (m, 3))).cuda()
gb = dv.GradBuffers(ds.n_sites, ds.device)
loss = torch.zeros(2, dtype=torch.float64, device="cuda")
res = dv.train_batch_device(ds, o, dirs, tmin, tmax, start, tg, gb, loss, rgb_scale=1.0 / (3 * m))
torch.cuda.synchronize()
it = int(res.counters[1].item())
seg = int(res.nseg.to(torch.int64).sum().item())
print(f"warps {m // 32}  reverse iterations/warp {it / (m / 32):.1f}  segments/ray {seg / m:.1f}  "
      f"avg group size {seg / it:.1f}")
