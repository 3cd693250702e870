"""Training-batch throughput on the reference's sampling (optim/train.py:133-140):
m random pixels from random training views (8 orbit views at 1080p of the 1M-site
config-2 scene), processed in the given order vs the device coherent_order sort.
  python tools/train_batch_probe.py [--m 65536 262144 1048576] [--reps 5]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_01157_b200 import device as dv  # noqa: E402
from paper_2502_01157_b200.camera import PINHOLE, CameraModel, orbit_poses  # noqa: E402
from paper_2502_01157_b200.synthetic import make_foam  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, nargs="+", default=[65536, 262144, 1048576])
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--views", type=int, default=8)
ap.add_argument("--forward", action="store_true", help="time render_rays_device instead")
ap.add_argument("--lanes", type=int, default=1, help="lanes per ray (forward only)")
args = ap.parse_args()

W, H = 1920, 1080
scene = make_foam(1_000_000, 1, 3)
ds = dv.DeviceScene(scene)
cams = [CameraModel.from_angle_x(PINHOLE, W, H, 0.9, p)
        for p in orbit_poses(np.zeros(3), 3.0, 0.3, args.views)]
dirs_all = torch.stack([c.ray_directions_device(device="cuda") for c in cams])  # [V, HW, 3]
orig = torch.from_numpy(np.stack([c.position for c in cams])).cuda()
starts = ds.locate(orig)
t_far = ds.default_t_max(np.stack([c.position for c in cams]))
rng = np.random.default_rng(0)
for m in args.m:
    flat = torch.from_numpy(rng.integers(0, args.views * W * H, size=m)).cuda()
    vi, pi = flat // (W * H), flat % (W * H)
    o = orig[vi].contiguous()
    d = dirs_all[vi, pi].contiguous()
    tmin = torch.zeros(m, dtype=torch.float64, device="cuda")
    tmax = torch.full((m,), t_far, dtype=torch.float64, device="cuda")
    st = starts[vi].contiguous()
    tg = torch.rand((m, 3), dtype=torch.float64, device="cuda")
    gb = dv.GradBuffers(ds.n_sites, ds.device)
    loss = torch.zeros(2, dtype=torch.float64, device="cuda")
    ws = dv.Workspace(ds.device)
    out = dv.alloc_forward(m, ds.device, per_ray=True)
    for label in ("given order", "coherent_order"):
        def run():
            order = dv.coherent_order(o, d) if label == "coherent_order" else None
            if args.forward:
                dv.render_rays_device(ds, o, d, tmin, tmax, st, workspace=ws, out=out,
                                      order=order, lanes_per_ray=args.lanes)
            else:
                dv.train_batch_device(ds, o, d, tmin, tmax, st, tg, gb, loss,
                                      rgb_scale=1.0 / (3 * m), workspace=ws, out=out,
                                      order=order)
        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        print(f"m={m:8d} {label:15s}: {ms:8.2f} ms/batch  {m / ms / 1e3:7.2f} Mrays/s", flush=True)
