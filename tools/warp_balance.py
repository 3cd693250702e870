"""Per-warp step balance of the config-2 frame: lanes of a warp (a 4x8 pixel
patch) walk their own rays; the warp runs until its longest ray is done.
Prints sum(mean steps)/sum(max steps) over patches = lane utilisation bound
from ray-length divergence alone."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_01157_b200 import device as dv  # noqa: E402
from paper_2502_01157_b200.camera import PINHOLE, CameraModel, look_at  # noqa: E402
from paper_2502_01157_b200.synthetic import make_foam  # noqa: E402

W, H = 1920, 1080
scene = make_foam(1_000_000, 1, 3)
ds = dv.DeviceScene(scene)
cam = CameraModel.from_angle_x(PINHOLE, W, H, 0.9, look_at((0.0, 0.0, 3.0), (0.0, 0.0, 0.0)))
res = dv.render_image_device(ds, cam, per_ray=True)
torch.cuda.synchronize()
c = res.ray_counters[:, 0].cpu().numpy().reshape(H, W).astype(np.float64)
v = res.ray_counters[:, 1].cpu().numpy().reshape(H, W).astype(np.float64)
for name, a in (("cells", c), ("neighbour visits", v)):
    p = a[: H // 8 * 8, : W // 4 * 4].reshape(H // 8, 8, W // 4, 4).transpose(0, 2, 1, 3)
    p = p.reshape(-1, 32)
    print(f"{name}: mean {a.mean():.1f}, utilisation by ray length {p.mean(1).sum() / p.max(1).sum():.3f}")
