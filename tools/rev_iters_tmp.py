import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2502_01157_b200 import device as dv
from paper_2502_01157_b200.camera import PINHOLE, CameraModel, orbit_poses
from paper_2502_01157_b200.synthetic import make_foam
W, H = 1920, 1080
scene = make_foam(1_000_000, 1, 3); ds = dv.DeviceScene(scene)
cams = [CameraModel.from_angle_x(PINHOLE, W, H, 0.9, p) for p in orbit_poses(np.zeros(3), 3.0, 0.3, 8)]
dirs_all = torch.stack([c.ray_directions_device(device="cuda") for c in cams])
orig = torch.from_numpy(np.stack([c.position for c in cams])).cuda()
starts = ds.locate(orig); t_far = ds.default_t_max(np.stack([c.position for c in cams]))
m = 65536
flat = torch.from_numpy(np.random.default_rng(0).integers(0, 8 * W * H, size=m)).cuda()
vi, pi = flat // (W * H), flat % (W * H)
o = orig[vi].contiguous(); d = dirs_all[vi, pi].contiguous()
tmin = torch.zeros(m, dtype=torch.float64, device="cuda"); tmax = torch.full((m,), t_far, dtype=torch.float64, device="cuda")
st = starts[vi].contiguous(); tg = torch.rand((m, 3), dtype=torch.float64, device="cuda")
gb = dv.GradBuffers(ds.n_sites, ds.device); loss = torch.zeros(2, dtype=torch.float64, device="cuda")
for order in (None, "auto"):
    out = dv.train_batch_device(ds, o, d, tmin, tmax, st, tg, gb, loss, rgb_scale=1.0/(3*m), order=order)
    torch.cuda.synchronize()
    c0 = int(out.counters[0].item()); segs = int(out.nseg.sum().item())
    extra = c0 - segs
    print(order, "per_lane warps", extra // 1000000, "iterations", extra % 1000000, "segments", segs)
