"""Forward-kernel sweep / profiling driver (not part of the product).

python tools/sweep_fwd.py [--lanes 1,2,4,8] [--reps 5] [--train] [--once]
--once renders a single frame per variant (for ncu -k regex:k_render).
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import make_views  # noqa: E402
from paper_2502_01157_b200 import device as dv  # noqa: E402
from paper_2502_01157_b200.synthetic import make_foam  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lanes", default="1,2,4,8,16")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--sizes", default="", help="WxH list (e.g. 128x128,480x270): frame sizes to sweep")
ap.add_argument("--n-sites", type=int, default=1_000_000)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--sh-degree", type=int, default=3)
ap.add_argument("--width", type=int, default=1920)
ap.add_argument("--height", type=int, default=1080)
ap.add_argument("--train", action="store_true")
ap.add_argument("--once", action="store_true")
ap.add_argument("--view", type=int, default=0)
ap.add_argument("--cull", default="1", help="view culling modes to time: '0', '1' or '0,1'")
ap.add_argument("--packed", type=int, default=-1)
ap.add_argument("--quantile", action="store_true")
ap.add_argument("--morton", action="store_true", help="renumber sites in Morton order")
ap.add_argument("--force-deg0", action="store_true",
                help="timing probe: colour from the DC band only (walk unchanged)")
ap.add_argument("--fp64", action="store_true",
                help="perturb the sites by 1e-12 (not fp32-exact; same Delaunay graph)")
args = ap.parse_args()
print("lib", os.environ.get("RFB_LIB", "default"), flush=True)

scene = make_foam(args.n_sites, args.seed, args.sh_degree)
if args.fp64:
    import numpy as np
    scene.adjacency.positions += np.random.default_rng(0).normal(0, 1e-12, scene.adjacency.positions.shape)
    scene.positions = scene.adjacency.positions
if args.morton:  # experiment: renumber the sites along a Morton curve (same geometry)
    from paper_2502_01157_b200.scene import AdjacencyGraph, FoamScene
    adj = scene.adjacency
    q = np.clip(((adj.positions - adj.positions.min(0)) / np.ptp(adj.positions, 0).max()
                 * 1023).astype(np.int64), 0, 1023)
    def spread(x):
        x = x & 0x3FF
        x = (x | (x << 16)) & 0x30000FF
        x = (x | (x << 8)) & 0x300F00F
        x = (x | (x << 4)) & 0x30C30C3
        x = (x | (x << 2)) & 0x9249249
        return x
    key = spread(q[:, 0]) | (spread(q[:, 1]) << 1) | (spread(q[:, 2]) << 2)
    perm = np.argsort(key, kind="stable")      # new id -> old id
    inv = np.empty_like(perm); inv[perm] = np.arange(len(perm))
    deg = np.diff(adj.offsets)[perm]
    off = np.concatenate([[0], np.cumsum(deg)])
    E = int(off[-1])
    rid = np.repeat(np.arange(len(perm)), deg)
    src = np.repeat(adj.offsets[perm] - off[:-1], deg) + np.arange(E)
    vals = inv[adj.neighbors[src]]
    nbr = vals[np.lexsort((vals, rid))]
    a2 = AdjacencyGraph(adj.positions[perm], off, nbr)
    scene = FoamScene(adj.positions[perm], scene.raw_density[perm], scene.sh_coeffs[perm],
                      scene.background, a2)
ds = dv.DeviceScene(scene, packed=None if args.packed < 0 else bool(args.packed),
                    sh_degree=0 if args.force_deg0 else None)
print("packed", ds.packed, "positions_f64", getattr(ds, "positions_f64", None), flush=True)
cam = make_views(args.view + 1, args.width, args.height)[args.view]
ws = dv.Workspace(ds.device)
out = dv.alloc_forward(args.width * args.height, ds.device, per_ray=False)
sizes = [tuple(int(v) for v in x.split("x")) for x in args.sizes.split(",")] if args.sizes else []
for (sw, sh_) in sizes:
    c2 = make_views(args.view + 1, sw, sh_)[args.view]
    o2 = dv.alloc_forward(sw * sh_, ds.device, per_ray=False)
    for lanes in [int(x) for x in args.lanes.split(",")]:
        dv.render_image_device(ds, c2, lanes_per_ray=lanes, workspace=ws, out=o2)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            dv.render_image_device(ds, c2, lanes_per_ray=lanes, workspace=ws, out=o2)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        print(f"{sw}x{sh_} lanes={lanes:2d}: {ms:8.3f} ms  {sw * sh_ / ms / 1e3:8.2f} Mrays/s", flush=True)
if sizes:
    sys.exit(0)
culls = [int(c) for c in args.cull.split(",")]
for lanes in [int(x) for x in args.lanes.split(",")]:
  for cull in culls:
    reps = 1 if args.once else args.reps
    if not args.once:
        dv.render_image_device(ds, cam, lanes_per_ray=lanes, workspace=ws, out=out, cull=bool(cull))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        dv.render_image_device(ds, cam, lanes_per_ray=lanes, workspace=ws, out=out, cull=bool(cull))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    m = args.width * args.height
    import hashlib
    h = hashlib.sha1(out.rgb.cpu().numpy().tobytes()).hexdigest()[:12]
    print(f"fwd lanes={lanes:2d} cull={cull}: {ms:8.2f} ms/frame  {m / ms / 1e3:8.2f} Mrays/s  "
          f"rgb sha1 {h}", flush=True)

if args.train:
    perm = torch.from_numpy(dv.tile_order(args.width, args.height)).cuda()
    dirs = cam.ray_directions_device()[perm].contiguous()
    m = dirs.shape[0]
    o = torch.from_numpy(np.broadcast_to(cam.position, (m, 3)).copy()).cuda()
    start = ds.locate(o[:1]).expand(m).contiguous()
    tmin = torch.zeros(m, dtype=torch.float64, device="cuda")
    tmax = torch.full((m,), ds.default_t_max(cam.position[None, :]), dtype=torch.float64,
                      device="cuda")
    tg = torch.from_numpy(np.random.default_rng(11).uniform(0, 1, (m, 3))).cuda()
    gb = dv.GradBuffers(ds.n_sites, ds.device)
    loss = torch.zeros(2, dtype=torch.float64, device="cuda")
    wsb = dv.Workspace(ds.device)
    fo = dv.alloc_forward(m, ds.device)
    reps = 1 if args.once else args.reps
    for cull in culls:
      vw = (cam, perm) if cull else None
      loss.zero_()
      for r in range(reps + (0 if args.once else 1)):
          if r == 1 or (args.once and r == 0):
              torch.cuda.synchronize()
              t0 = time.perf_counter()
          if args.quantile:
              up = torch.rand((m, 2, 2), dtype=torch.float64, device="cuda")
              dv.train_batch_device(ds, o, dirs, tmin, tmax, start, tg, gb, loss,
                                    rgb_scale=1.0 / (3 * m), quantile_scale=0.01 / (2 * m),
                                    u_pairs=up, workspace=wsb, out=fo, order=None, view=vw)
          else:
              dv.train_batch_device(ds, o, dirs, tmin, tmax, start, tg, gb, loss,
                                    rgb_scale=1.0 / (3 * m), workspace=wsb, out=fo, order=None, view=vw)
      torch.cuda.synchronize()
      ms = (time.perf_counter() - t0) * 1e3 / reps
      import hashlib
      h = hashlib.sha1(fo.rgb.cpu().numpy().tobytes()).hexdigest()[:12]
      print(f"train cull={cull}: {ms:8.2f} ms/step  {m / ms / 1e3:8.2f} Mrays/s  "
            f"loss {float(loss[0]):.12g}  rgb sha1 {h}", flush=True)
