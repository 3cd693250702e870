import os, sys, torch
sys.path.insert(0, os.getcwd())
from bench import make_views
from paper_2502_01157_b200 import device as dv
from paper_2502_01157_b200.synthetic import make_foam
ds = dv.DeviceScene(make_foam(1_000_000, 1, 3))
cam = make_views(1, 1920, 1080)[0]
ws = dv.Workspace(ds.device)
out = dv.alloc_forward(1920 * 1080, ds.device, per_ray=False)
for tw, th in ((32, 32), (64, 32), (32, 64), (64, 64), (128, 32)):
    f = lambda: dv.render_image_device(ds, cam, workspace=ws, out=out, tile_w=tw, tile_h=th)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    import hashlib
    print(tw, th, round(e0.elapsed_time(e1) / 10, 3), "ms", hashlib.sha1(out.rgb.cpu().numpy().tobytes()).hexdigest()[:12], flush=True)
