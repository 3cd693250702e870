"""One training iteration as the reference runs it (optim/train.py:131-209):
65,536 random pixels of 8 views -> train_batch -> gradient chain + Adam ->
scene refresh, on the 1M-site scene, through train.DeviceTrainer.step."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_01157_b200 import device as dv  # noqa: E402
from paper_2502_01157_b200.camera import PINHOLE, CameraModel, orbit_poses  # noqa: E402
from paper_2502_01157_b200.synthetic import make_foam  # noqa: E402
from paper_2502_01157_b200.train import DeviceTrainer  # noqa: E402

W, H, V, m = 1920, 1080, 8, 65536
scene = make_foam(1_000_000, 1, 3)
tr = DeviceTrainer(scene)
cams = [CameraModel.from_angle_x(PINHOLE, W, H, 0.9, p) for p in orbit_poses(np.zeros(3), 3.0, 0.3, V)]
dirs_all = torch.stack([c.ray_directions_device(device="cuda") for c in cams])
orig = torch.from_numpy(np.stack([c.position for c in cams])).cuda()
images = torch.rand((V, W * H, 3), dtype=torch.float64, device="cuda")
gen = torch.Generator(device="cuda").manual_seed(0)


def iteration():
    flat = torch.randint(0, V * W * H, (m,), device="cuda", generator=gen)
    vi, pi = flat // (W * H), flat % (W * H)
    starts = tr.ds.locate(orig)
    t_far = tr.ds.default_t_max(orig.cpu().numpy())
    return tr.step(orig[vi], dirs_all[vi, pi], torch.zeros(m, dtype=torch.float64, device="cuda"),
                   torch.full((m,), t_far, dtype=torch.float64, device="cuda"),
                   starts[vi].contiguous(), images[vi, pi], lr_position=1e-5, lr_density=0.05,
                   lr_sh=5e-3)


for _ in range(3):
    iteration()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 20
e0.record()
for _ in range(n):
    loss = iteration()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print(f"training iteration (65,536 random pixels, 1M sites, moving fp64 sites): {ms:.2f} ms "
      f"= {m / ms / 1e3:.1f} M rays/s; loss {float(loss[0]) / (3 * m):.4f}")
