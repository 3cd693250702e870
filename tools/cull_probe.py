"""View-culling probe: time of rfb_cull_view alone and of the render on the culled
view (cull="last"), per region grid; share of neighbour records dropped."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import make_views  # noqa: E402
from paper_2502_01157_b200 import device as dv  # noqa: E402
from paper_2502_01157_b200.synthetic import make_foam  # noqa: E402

W, H = 1920, 1080
scene = make_foam(int(os.environ.get("N_SITES", 1_000_000)), 1, 3)
ds = dv.DeviceScene(scene)
cam = make_views(1, W, H)[0]
ws = dv.Workspace(ds.device)
out = dv.alloc_forward(W * H, ds.device, per_ray=False)


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


base = timed(lambda: dv.render_image_device(ds, cam, workspace=ws, out=out, cull=False))
print(f"no culling: render {base:.3f} ms", flush=True)
for g in os.environ.get("REGIONS", "1x1 2x2 3x2 4x2 4x3 4x4 8x4").split():
    rg = tuple(int(v) for v in g.split("x"))
    tc = timed(lambda: ds.view_camera(cam, regions=rg))
    tr = timed(lambda: dv.render_image_device(ds, cam, workspace=ws, out=out, cull="last"))
    R = rg[0] * rg[1]
    n1 = ds._view_cells[: R * ds.n_sites, 7]
    dropped = int((n1 & 31).sum().item())
    kept = int((ds._view_cells[: R * ds.n_sites, 6] - ds._view_cells[: R * ds.n_sites, 3]).to(torch.int64).sum().item())
    print(f"{g}: cull {tc:.3f} ms  render {tr:.3f} ms  total {tc + tr:.3f} ms  "
          f"dropped {dropped / (dropped + kept):.3f} of the records", flush=True)
