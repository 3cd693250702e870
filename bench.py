#!/usr/bin/env python
"""Benchmark: rays/s of the Radiant Foam hot path on B200 (BASELINE.json).

Workload (N=1): config 2 -- synthetic 1M-site foam (seed 1,
SH degree 3, uniform in [-1,1]^3, fp32-exact sites, Qhull CSR), pinhole
camera at (0,0,3) looking at the origin, camera_angle_x 0.9, 1920x1080,
epsilon 1e-3, step_limit 4096.  One step = one full forward frame
(rfb_render_image: ray generation + start cell + walk + SH-3 colour +
compositing).  ``fwd_bwd`` reports config 3 on the same scene: one step =
rfb_train_batch over every pixel of the view (L2 adjoint, quantile off) plus,
for N>1, the NCCL all-reduce of the per-site gradient buffer.

Multi-GPU (torchrun, one rank per GPU): every step renders N views (view k =
orbit pose k-1, view 0 = the config-2 camera); each view's 32x32 tiles are
interleaved round-robin over the ranks (scene replicated) and the frames are
summed onto rank 0.  Training: rank r trains on view r and the flat fp32
gradient buffer is all-reduced.  Per-rank work is fixed as N grows:
"scaling": "weak".

Timing: W untimed warm-up steps, then K steps bracketed by barrier +
synchronize, timed with CUDA events on the launching stream, max over ranks.
The scene (~950 MB packed at config 2) is larger than L2 (126 MB).  nvidia-smi clocks are
sampled during the timed region.  ``e2e`` times the public API
(render.render_image with a resident scene: camera in, (H,W,3) float64 image
copied to host) including the device->host copy of the image; at N>1 the
tile-sharded distributed.ShardedRenderer with the frame assembled on rank 0
and copied to the host there.  RFB_BENCH_DIST=1 takes the collective path at
N=1 too (a 1-rank NCCL group), to exercise it on one GPU.

--impl reference: the reference algorithm's CPU implementation on the host
cores (the C oracle port of rfoam/tracer/kernels.py, every host thread), on
a bounded row sample of the same frame.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "rays/sec fwd and fwd+bwd (1M-site foam, 1080p) at 1/2/4/8 B200; % of gather roofline"
UNIT = "rays/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n-sites", type=int, default=1_000_000)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--lanes", type=int, default=0, help="lanes per ray (0 = library default)")
    ap.add_argument("--no-fwd-bwd", action="store_true")
    ap.add_argument("--quantile", action="store_true",
                    help="fwd+bwd with the quantile regulariser on (lambda 0.01, P=2 pairs, "
                         "u_pairs from rng(12); optim/config.py:34-36)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-train-iter", action="store_true",
                    help="skip timing a reference-style training iteration (65,536 random pixels)")
    ap.add_argument("--no-adjacency", action="store_true",
                    help="skip timing the device Delaunay rebuild (SURVEY §8f row 2)")
    ap.add_argument("--cpu-row-stride", type=int, default=8)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 4, 5],
                    help="1: the reference's CPU-runnable case (10k sites, SH deg 0, "
                         "128x128); 2: config 2 forward + config 3 fwd+bwd (1M, 1080p; default); "
                         "4: 3M-site surface foam, one 4K frame tile-sharded over the ranks; "
                         "5: 3M surface foam, 8 orbit views at 1080p fwd+bwd split over the "
                         "ranks + NCCL gradient all-reduce")
    args = ap.parse_args()
    args.kind = "uniform"
    args.sh_degree = 3
    if args.config == 1:  # configs[0]: 10k-site foam, SH deg 0, one 128x128 frame
        if args.n_sites == 1_000_000:
            args.n_sites = 10_000
        if args.seed == 1:
            args.seed = 0
        if (args.width, args.height) == (1920, 1080):
            args.width, args.height = 128, 128
        args.sh_degree = 0
        args.cpu_row_stride = 1
    if args.config in (4, 5):
        args.kind = "surface"
        if args.n_sites == 1_000_000:
            args.n_sites = 3_000_000
        if args.seed == 1:
            args.seed = 2
    if args.config == 4 and (args.width, args.height) == (1920, 1080):
        args.width, args.height = 3840, 2160
        args.cpu_row_stride = max(args.cpu_row_stride, 32)
    return args


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def gather_ceilings():
    """Random-gather ceilings measured on a B200 by tools/gather_peak.cu, read from
    the committed profile so the bench line shows which memory level the walk runs at."""
    path = os.path.join(REPO, "profiles", "r09_gather_peak.jsonl")
    try:
        rows = [json.loads(x) for x in open(path) if x.startswith("{")]
    except OSError:
        return None
    g = [r for r in rows if r["kind"] == "gather"]

    def best(access, lo, hi):
        sel = [r["useful_GBps"] for r in g if r["access"] == access and lo <= r["working_set_bytes"] <= hi]
        return max(sel) if sel else None

    l2 = (4 << 20, 64 << 20)
    hbm = (1 << 30, 4 << 30)
    return {"unit": "GB/s useful",
            "l2_lane16": best("lane16", *l2), "l2_lane32": best("lane32", *l2),
            "l2_warp512": best("warp512", *l2),
            "hbm_lane16": best("lane16", *hbm), "hbm_lane32": best("lane32", *hbm),
            "hbm_warp512": best("warp512", *hbm),
            "latency_ns": {str(r["working_set_bytes"]): r["ns_per_hop"] for r in rows
                           if r["kind"] == "chase"},
            "source": "profiles/r09_gather_peak.jsonl (tools/gather_peak.cu)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(smax)) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_views(n_views, W, H):
    from paper_2502_01157_b200.camera import PINHOLE, CameraModel, look_at, orbit_poses

    poses = [look_at((0.0, 0.0, 3.0), (0.0, 0.0, 0.0))]
    poses += orbit_poses(np.zeros(3), 3.0, 0.3, 8)
    return [CameraModel.from_angle_x(PINHOLE, W, H, 0.9, poses[k % len(poses)])
            for k in range(n_views)]


def orbit_views(W, H, count=8):
    """orbit_poses(centre 0, r=3, elev 0.3, 8)."""
    from paper_2502_01157_b200.camera import PINHOLE, CameraModel, orbit_poses

    return [CameraModel.from_angle_x(PINHOLE, W, H, 0.9, p)
            for p in orbit_poses(np.zeros(3), 3.0, 0.3, count)]


def algorithmic_bytes(C, V, N, m, sh_bytes):
    """B_f = 24C + 16V + S_b N + 12 per ray (totals here)."""
    return 24.0 * C + 16.0 * V + sh_bytes * N + 12.0 * m


# ---------------------------------------------------------------------------
def _train_roofline():
    """k_train's measured binding unit and DRAM traffic (profiles/traffic.json, from the
    committed ncu capture)."""
    try:
        with open(os.path.join(REPO, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        return {"kernel": "k_train (walk + record + reverse pass)",
                "binding_unit": "l1tex data-pipe wavefronts",
                "binding_frac": tj.get("k_train_l1_data_pipe_frac"),
                "traffic": tj.get("k_train_dram_bytes_per_launch"),
                "source": tj.get("k_train_source", tj.get("source"))}
    except Exception:  # noqa: BLE001
        return None


def run_reference(args):
    """CPU reference arm: the oracle port on all host threads (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    line = cpu_baseline_measure(args, steps=args.steps, warmup=min(args.warmup, 1))
    out = {"metric": METRIC, "value": line["value"], "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "impl": "reference",
           "ms_per_step": line["ms_per_step"], "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"config {args.config}: {args.n_sites}-site {args.kind} foam, "
                                  f"SH deg {args.sh_degree}, {args.width}x{args.height} forward",
                      "sample": line["sample"], "n_sites": args.n_sites},
           "cpu_baseline": {"value": line["value"], "unit": UNIT, "cores": line["cores"],
                            "kind": "port", "sample": line["sample"]},
           "e2e": {"value": line["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def cpu_baseline_measure(args, steps=1, warmup=0, scene=None, cam=None):
    from oracle import oracle as orc
    from paper_2502_01157_b200.scene import softplus
    from paper_2502_01157_b200.synthetic import make_foam

    if scene is None:
        scene = make_foam(args.n_sites, args.seed, getattr(args, "sh_degree", 3),
                          kind=getattr(args, "kind", "uniform"))
    adj = scene.adjacency
    sa = orc.SceneArrays(adj.positions, adj.offsets, adj.neighbors, softplus(scene.raw_density),
                         scene.sh_coeffs.reshape(-1, 48), scene.background)
    if cam is None:
        cam = (make_views(1, args.width, args.height)[0] if getattr(args, "config", 2) == 2
               else orbit_views(args.width, args.height, 8)[0])
    rows = np.arange(0, args.height, args.cpu_row_stride)
    rr, cc = np.meshgrid(rows, np.arange(args.width), indexing="ij")
    dirs = cam.ray_directions(rr.reshape(-1), cc.reshape(-1))
    m = len(dirs)
    origin = cam.position
    start = int(orc.nearest_sites(sa.positions, origin[None, :])[0])
    t_max = float(np.linalg.norm(origin - sa.center) + 2.0 * sa.diagonal + 1.0)
    threads = os.cpu_count() or 1
    origins = np.broadcast_to(origin, (m, 3)).copy()
    for _ in range(warmup):
        orc.render_rays(sa, origins[:4096], dirs[:4096], 0.0, t_max, start, threads=threads)
    times = []
    for _ in range(max(steps, 1)):
        t0 = time.perf_counter()
        orc.render_rays(sa, origins, dirs, 0.0, t_max, start, threads=threads)
        times.append(time.perf_counter() - t0)
    dt = float(np.mean(times))
    return {"value": m / dt, "ms_per_step": dt * 1e3, "cores": threads,
            "sample": f"every {args.cpu_row_stride}th row of the {args.width}x{args.height} frame "
                      f"({m} rays/step, {len(times)} steps, C oracle port, {threads} threads)"}


# ---------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    from paper_2502_01157_b200 import device as dv
    from paper_2502_01157_b200 import render as rd
    from paper_2502_01157_b200.synthetic import make_foam

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # RFB_BENCH_DIST=1 runs the collective code path even at world size 1 (a 1-rank NCCL
    # group), so the N>1 plumbing can be exercised on the single GPU this round has
    dist_on = world > 1 or os.environ.get("RFB_BENCH_DIST") == "1"
    torch.cuda.set_device(local)
    if dist_on:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    def barrier():
        if dist_on:
            dist.barrier()

    W, H = args.width, args.height
    lanes = args.lanes if args.lanes > 0 else dv.DEFAULT_LANES
    t_build = time.perf_counter()
    scene = make_foam(args.n_sites, args.seed, args.sh_degree, kind=args.kind, verbose=(rank == 0))
    ds = dv.DeviceScene(scene, device=dev)
    build_s = time.perf_counter() - t_build
    scaling = "weak"
    if args.config in (1, 2):
        views = make_views(world, W, H)  # one view per rank per step, tile-sharded
        train_views = [views[rank]]
    elif args.config == 4:
        views = orbit_views(W, H, 8)[:1]  # one 4K frame per step, tile-sharded
        train_views = []
        scaling = "strong"
    else:
        views = orbit_views(W, H, 8)[:1]  # (forward probe only)
        train_views = orbit_views(W, H, 8)[rank::world]
        scaling = "strong"
    tx, ty = dv.tile_grid(W, H, 32, 32)
    all_tiles = np.arange(tx * ty, dtype=np.int32)
    my_tiles = torch.from_numpy(all_tiles[rank::world].copy()).to(dev)
    ws = dv.Workspace(dev)
    frames = [dv.alloc_forward(W * H, dev, per_ray=False) for _ in views]
    stream = torch.cuda.current_stream()

    def fwd_step():
        for k, cam in enumerate(views):
            if dist_on:
                frames[k].rgb.zero_()
            dv.render_image_device(ds, cam, tile_ids=my_tiles, lanes_per_ray=lanes, workspace=ws,
                                   out=frames[k])
        if dist_on:
            for fr in frames:
                dist.reduce(fr.rgb, dst=0)

    # -- untimed: counters for the roofline (view 0, full frame) ------------------
    probe = dv.render_image_device(ds, views[0], per_ray=True, lanes_per_ray=lanes, workspace=ws)
    torch.cuda.synchronize()
    C_tot, V_tot = [int(x) for x in probe.counters.cpu().tolist()]
    N_tot = int(probe.nseg.to(torch.int64).sum().item())
    failed = int((probe.status != 0).sum().item())
    m0 = W * H
    sh_bytes = 192 if ds.sh_degree == 3 else 12
    bytes_per_frame = algorithmic_bytes(C_tot, V_tot, N_tot, m0, sh_bytes)

    # -- forward timing ------------------------------------------------------------
    if args.config == 5:
        args.steps_fwd = 0
    for _ in range(args.warmup if args.config != 5 else 0):
        fwd_step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    if rank == 0:
        clk.start()
        time.sleep(0.3)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    ev0.record(stream)
    for s in range(args.steps):
        kev[s][0].record(stream)
        if args.config != 5:
            fwd_step()
        kev[s][1].record(stream)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    fwd_ms = ev0.elapsed_time(ev1)
    kernel_ms = float(np.mean([a.elapsed_time(b) for a, b in kev]))
    clocks = clk.stop() if rank == 0 else None
    t = torch.tensor([fwd_ms], dtype=torch.float64, device=dev)
    if dist_on:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    fwd_ms = float(t.item())
    rays_total = args.steps * W * H * len(views)
    fwd_value = rays_total / max(fwd_ms / 1e3, 1e-12)

    # -- fwd+bwd timing (config 3) -------------------------------------------------
    fb = None
    if not args.no_fwd_bwd and train_views:
        # each training view's rays in tile order (4x8 warp patches): the same
        # ray set, scheduled coherently (dv.tile_order); targets follow it
        perm = torch.from_numpy(dv.tile_order(W, H)).to(dev)
        rng = np.random.default_rng(11)
        batches = []
        for cam in train_views:
            dirs = cam.ray_directions_device(device=dev)[perm].contiguous()
            m = dirs.shape[0]
            origins = torch.from_numpy(np.broadcast_to(cam.position, (m, 3)).copy()).to(dev)
            start = ds.locate(origins[:1]).expand(m).contiguous()
            t_min = torch.zeros(m, dtype=torch.float64, device=dev)
            t_max = torch.full((m,), ds.default_t_max(cam.position[None, :]), dtype=torch.float64,
                               device=dev)
            targets = torch.from_numpy(rng.uniform(0.0, 1.0, (m, 3))).to(dev)[perm].contiguous()
            u_pairs = (torch.from_numpy(np.random.default_rng(12).uniform(0.0, 1.0, (m, 2, 2)))
                       .to(dev)[perm].contiguous() if args.quantile else None)
            batches.append((origins, dirs, t_min, t_max, start, targets, u_pairs))
        m = W * H
        n_train_views = len(train_views) * world if args.config in (1, 2) else 8
        gb = dv.GradBuffers(ds.n_sites, dev)
        loss = torch.zeros(2, dtype=torch.float64, device=dev)
        out_fb = dv.alloc_forward(m, dev, per_ray=True)
        rgb_scale = 1.0 / (3.0 * m * n_train_views)  # global ray count (train.py:168)
        q_scale = 0.01 / (m * n_train_views * 2) if args.quantile else 0.0  # lambda / (m P)
        wsb = dv.Workspace(dev)

        def fb_step():
            gb.zero_()
            loss.zero_()
            for (origins, dirs, t_min, t_max, start, targets, u_pairs) in batches:
                dv.train_batch_device(ds, origins, dirs, t_min, t_max, start, targets, gb, loss,
                                      rgb_scale=rgb_scale, quantile_scale=q_scale,
                                      u_pairs=u_pairs, workspace=wsb, out=out_fb,
                                      order=None)  # rays already in tile order
            if dist_on:
                dist.all_reduce(gb.flat)
                dist.all_reduce(loss)

        for _ in range(args.warmup):
            fb_step()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        clk2 = ClockSampler(local)
        if rank == 0:
            clk2.start()
            time.sleep(0.3)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            fb_step()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        fb_ms = e0.elapsed_time(e1)
        clocks_fb = clk2.stop() if rank == 0 else None
        t = torch.tensor([fb_ms], dtype=torch.float64, device=dev)
        if dist_on:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        fb_ms = float(t.item())
        fb_C = int(out_fb.ray_counters[:, 0].sum().item())
        fb_V = int(out_fb.ray_counters[:, 1].sum().item())
        fb_N = int(out_fb.nseg.to(torch.int64).sum().item())
        fb_bytes = algorithmic_bytes(fb_C, fb_V, fb_N, m, 192 if ds.sh_degree == 3 else 12) \
            + 12.0 * m + 2.0 * fb_N * (4 + (192 if ds.sh_degree == 3 else 12)) \
            + 2.0 * max(fb_N - m, 0) * 24  # B_fb, last view's counters
        fb = {"value": args.steps * m * n_train_views / (fb_ms / 1e3), "unit": UNIT,
              "ms_per_step": fb_ms / args.steps,
              "workload": ("config 3: 1080p forward+backward, per-site fp32 gradients"
                           if args.config == 2 else
                           "config 1 scene: 128x128 forward+backward" if args.config == 1 else
                           "config 5: 3M-site surface foam, 8 orbit views at 1080p "
                           "forward+backward split over the ranks")
                          + (", L2 adjoint + quantile regulariser (lambda 0.01, P=2)"
                             if args.quantile else ", L2 adjoint, quantile off")
                          + (", NCCL all-reduce" if dist_on else ""),
              "views_per_step": n_train_views,
              "algorithmic_bytes_per_view": fb_bytes,
              "achieved_GBps": fb_bytes * n_train_views / world / (fb_ms / args.steps / 1e3) / 1e9,
              "roofline": _train_roofline(),
              "cells_per_ray": int(out_fb.ray_counters[:, 0].sum().item()) / m,
              "loss_rgb": float(loss[0].item()) / (3.0 * m * n_train_views),
              "clocks": clocks_fb}

    # -- one training iteration as the reference's loop runs it (optim/train.py:131-209)
    train_iter = None
    if not args.no_train_iter and rank == 0 and world == 1 and args.config in (1, 2):
        from paper_2502_01157_b200.train import DeviceTrainer
        tr = DeviceTrainer(scene, device=dev)
        mb = 65536
        tv = orbit_views(W, H, 8)
        tdirs = torch.stack([c.ray_directions_device(device=dev) for c in tv])
        torig = torch.from_numpy(np.stack([c.position for c in tv])).to(dev)
        timgs = torch.rand((len(tv), W * H, 3), dtype=torch.float64, device=dev,
                           generator=torch.Generator(device=dev).manual_seed(13))
        tgen = torch.Generator(device=dev).manual_seed(14)
        t_far = tr.ds.default_t_max(np.stack([c.position for c in tv]))

        def train_step():
            flat = torch.randint(0, len(tv) * W * H, (mb,), device=dev, generator=tgen)
            vi, pi = flat // (W * H), flat % (W * H)
            st = tr.ds.locate(torig)
            return tr.step(torig[vi], tdirs[vi, pi],
                           torch.zeros(mb, dtype=torch.float64, device=dev),
                           torch.full((mb,), t_far, dtype=torch.float64, device=dev),
                           st[vi].contiguous(), timgs[vi, pi], lr_position=1e-5,
                           lr_density=0.05, lr_sh=5e-3)

        for _ in range(3):
            train_step()
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        n_it = 10
        a0.record(stream)
        for _ in range(n_it):
            train_step()
        a1.record(stream)
        torch.cuda.synchronize()
        it_ms = a0.elapsed_time(a1) / n_it
        train_iter = {"ms": it_ms, "rays_per_iteration": mb, "value": mb / (it_ms / 1e3),
                      "unit": UNIT,
                      "workload": "65,536 random pixels of 8 orbit views (the reference's "
                                  "batch_rays) -> start cells, train_batch, gradient chain + clip "
                                  "+ Adam on every parameter, scene refresh (moving fp64 sites); "
                                  "train.DeviceTrainer.step"}
        del tr, tdirs, timgs

    # -- device Delaunay rebuild of the same sites --------------
    adjacency = None
    if not args.no_adjacency and rank == 0:
        from paper_2502_01157_b200 import adjacency as adj_mod
        pos_d = torch.from_numpy(np.ascontiguousarray(scene.adjacency.positions)).to(dev)
        off_d, nbr_d, _, ainfo = adj_mod.build_device(pos_d)  # warm-up
        same = bool(torch.equal(off_d.cpu(), torch.from_numpy(scene.adjacency.offsets)) and
                    torch.equal(nbr_d.cpu(), torch.from_numpy(scene.adjacency.neighbors)))
        tms = []
        for _ in range(3):
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            adj_mod.build_device(pos_d)
            a1.record(stream)
            torch.cuda.synchronize()
            tms.append(a0.elapsed_time(a1))
        adjacency = {"ms": float(np.median(tms)), "sites": int(pos_d.shape[0]),
                     "edges": ainfo["edges"], "csr_equals_fixture": same,
                     "pass2_sites": ainfo["pass2_sites"],
                     "api": "adjacency.build_device(positions) -> CSR + hull (rfb_build_adjacency)",
                     "cpu_reference": "fixture CSR from scipy Qhull: ~127 s at 1M sites, 268 s "
                                      "at 3M (SURVEY §8c; .foam_cache build logs)"}
        del off_d, nbr_d

    # -- e2e through the public API (rank 0 view, host image out) -----------------
    e2e = None
    if not args.no_e2e and not dist_on:
        cam = views[0]
        rd.render_image(scene, cam, device_scene=ds, lanes_per_ray=lanes)
        torch.cuda.synchronize()
        ts = []
        for _ in range(max(3, min(args.steps, 10))):
            t0 = time.perf_counter()
            img = rd.render_image(scene, cam, device_scene=ds, lanes_per_ray=lanes)
            ts.append(time.perf_counter() - t0)
        e2e = {"value": W * H / float(np.median(ts)), "unit": UNIT, "h2d_bytes_per_step": 0,
               "d2h_bytes_per_step": int(img.nbytes),
               "api": "render.render_image(scene, camera, device_scene=ds) -> (H,W,3) f64 host"}
    elif not args.no_e2e:
        # N > 1: the sharded public API -- every rank renders its tiles of each view, the
        # frame is assembled on rank 0 and copied to the host there; max over ranks
        from paper_2502_01157_b200.distributed import ShardedRenderer
        sr = ShardedRenderer(ds, W, H, lanes_per_ray=lanes)

        def e2e_step():
            imgs = [sr.render_to_host(cam, dst=0) for cam in views]
            return [x for x in imgs if x is not None]

        e2e_step()
        torch.cuda.synchronize()
        ts = []
        for _ in range(max(3, min(args.steps, 10))):
            barrier()
            t0 = time.perf_counter()
            imgs = e2e_step()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        t = torch.tensor([float(np.median(ts))], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = {"value": len(views) * W * H / float(t.item()), "unit": UNIT,
               "h2d_bytes_per_step": 0,
               "d2h_bytes_per_step": int(sum(x.nbytes for x in imgs)) if rank == 0 else 0,
               "api": "distributed.ShardedRenderer(ds, W, H).render_to_host(camera) per view "
                      "(tile-sharded over the ranks, NCCL reduce to rank 0) -> pinned host frame",
               "timing": "median over steps of the per-rank wall clock, max over ranks"}

    if rank != 0:
        if dist_on:
            dist.destroy_process_group()
        return

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            cb = cpu_baseline_measure(args, steps=1, warmup=1, scene=scene, cam=views[0])
            cpu = {"value": cb["value"], "unit": UNIT, "cores": cb["cores"], "kind": "port",
                   "sample": cb["sample"]}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "port",
                   "sample": f"failed: {e}"}

    peak, peak_kind = peaks()
    achieved = bytes_per_frame * len(views) / world / max(kernel_ms / 1e3, 1e-12) / 1e9
    traffic = None
    l1_frac = None
    render_src = None
    tpath = os.path.join(REPO, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                tj = json.load(f)
            traffic = tj.get("k_render_dram_bytes_per_launch")
            l1_frac = tj.get("k_render_l1_data_pipe_frac")
            render_src = tj.get("k_render_source")
        except Exception:
            traffic = None
    workload = {
        1: "config 1: 10k-site foam (seed 0), SH deg 0, 128x128 forward render per view, "
           "camera (0,0,3)->origin, angle_x 0.9, eps 1e-3",
        2: "config 2: 1M-site foam (seed 1), SH deg 3, 1920x1080 forward render per view, "
           "camera (0,0,3)->origin, angle_x 0.9, eps 1e-3",
        4: "config 4: 3M-site surface foam (seed 2), SH deg 3, one 3840x2160 frame per step "
           "from orbit pose 0, 32x32 tiles interleaved over the ranks",
        5: "config 5: 3M-site surface foam (seed 2), 8 orbit views at 1920x1080 forward+backward "
           "per step split over the ranks, NCCL all-reduce of the [n,52] gradients",
    }[args.config]
    value = fwd_value
    ms_step = fwd_ms / args.steps
    if args.config == 5 and fb is not None:
        value = fb["value"]
        ms_step = fb["ms_per_step"]
        achieved = fb["achieved_GBps"]
        bytes_per_frame = fb["algorithmic_bytes_per_view"]
        kernel_ms = fb["ms_per_step"] / max(len(train_views), 1)
    scene_mb = sum(t.numel() * t.element_size() for t in
                   (ds.site4, ds.offsets, ds.neighbors, ds.sh, ds.cells, ds.edges, ds.sh32)
                   if t is not None) / 1e6
    l2_note = (f"inputs larger than L2 (scene {scene_mb:.0f} MB vs 126 MB L2); no flush"
               if scene_mb > 126 else
               f"scene ({scene_mb:.0f} MB) fits in L2; no flush (small-config case)")
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SURVEY.md §8d foam generator; random-init scene, no dataset)",
        "config": {"workload": workload,
                   "n_sites": args.n_sites, "n_edges": ds.n_edges, "views_per_step": len(views),
                   "tiles": "32x32 interleaved over ranks", "lanes_per_ray": lanes or "auto",
                   "l2": l2_note,
                   "cells_per_ray": C_tot / m0, "neighbor_visits_per_ray": V_tot / m0,
                   "segments_per_ray": N_tot / m0, "failed_rays": failed,
                   "scene_build_s": round(build_s, 1)},
        "fwd_bwd": fb,
        "e2e": e2e,
        "adjacency_rebuild": adjacency,
        "train_iteration": train_iter,
        "gpu_launches": (3 * args.steps * len(views) if args.config != 5
                         else args.steps * len(train_views)),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": "k_render (walk + SH + composite)" if args.config != 5 else
                               "k_train (walk + composite + reverse pass)",
                     "algorithmic_bytes_per_launch": bytes_per_frame,
                     "launch_ms": kernel_ms,
                     "note": "achieved counts the algorithmic gather bytes of SURVEY §8d "
                             "(no reuse); coherent rays share cells, so DRAM traffic per launch "
                             "is `traffic` and frac can exceed 1. The binding unit is the L1 "
                             "data pipe (binding_frac, from the ncu capture in profiles/).",
                     "traffic_source": render_src,
                     "binding_unit": "l1tex data-pipe wavefronts",
                     "binding_frac": l1_frac,
                     "gather_ceilings": gather_ceilings()},
        "cpu_baseline": cpu,
        "clocks": clocks,
    }
    print(json.dumps(out), flush=True)
    if dist_on:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
