"""Per-8x4-tile ray-length divergence of the config-2 frame (tile mean/max of
cells stepped and neighbour visits per ray)."""
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
W, H = 1920, 1080
cam = make_views(1, W, H)[0]
res = dv.render_image_device(ds, cam, per_ray=True)
torch.cuda.synchronize()
rc = res.ray_counters.cpu().numpy().reshape(H, W, 2).astype(np.float64)
for name, ch in (("cells", 0), ("visits", 1)):
    a = rc[:, :, ch]
    t = a[: H // 4 * 4, : W // 8 * 8].reshape(H // 4, 4, W // 8, 8).transpose(0, 2, 1, 3).reshape(-1, 32)
    eff = t.sum() / (t.max(axis=1).sum() * 32)
    print(f"{name}: mean/ray {a.mean():.1f}  8x4-tile lockstep efficiency (sum/(32*max)) {eff:.3f}")
    t2 = a[: H // 8 * 8, : W // 4 * 4].reshape(H // 8, 8, W // 4, 4).transpose(0, 2, 1, 3).reshape(-1, 32)
    print(f"   4x8 tiles: {t2.sum() / (t2.max(axis=1).sum() * 32):.3f}")
    t3 = a[:, : W // 32 * 32].reshape(H, W // 32, 32).reshape(-1, 32)
    print(f"   1x32 rows: {t3.sum() / (t3.max(axis=1).sum() * 32):.3f}")
