"""Time the device Delaunay builder (rfb_build_adjacency) and compare its CSR
with the cached Qhull CSR of the bench scenes (.foam_cache).
  python tools/adjacency_probe.py [--kind uniform --n 1000000 --seed 1] [--reps 3]"""
import argparse
import os
import sys
import time

import numpy as np
import torch

os.environ["RFB_FIXTURE_BUILDER"] = "qhull"  # the comparison reference must be Qhull

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_01157_b200 import adjacency as A  # noqa: E402
from paper_2502_01157_b200.synthetic import cached_adjacency, random_positions  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--kind", default="uniform")
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--no-compare", action="store_true")
args = ap.parse_args()

pos = random_positions(args.n, args.seed, args.kind)
pd = torch.from_numpy(pos).cuda()
off, nbr, hull, info = A.build_device(pd)  # warm-up (+ module load)
torch.cuda.synchronize()
ts = []
for _ in range(args.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    off, nbr, hull, info = A.build_device(pd)
    e1.record()
    torch.cuda.synchronize()
    ts.append((e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3))
print(f"{args.kind} n={args.n}: device build {min(t[0] for t in ts):.1f} ms "
      f"(wall {min(t[1] for t in ts):.1f} ms) {info}", flush=True)
if not args.no_compare:
    tag = f"{args.kind}_n{args.n}_s{args.seed}"
    t0 = time.perf_counter()
    ref = cached_adjacency(pos, tag, verbose=True)
    print(f"reference CSR ({tag}) ready in {time.perf_counter() - t0:.1f}s", flush=True)
    o, nb, h = off.cpu().numpy(), nbr.cpu().numpy(), hull.cpu().numpy()
    same_off = np.array_equal(o, ref.offsets)
    same_nbr = same_off and np.array_equal(nb, ref.neighbors)
    print(f"offsets equal: {same_off}, neighbors equal: {same_nbr}, "
          f"hull equal: {np.array_equal(h, ref.hull)} (hull sites {int(h.sum())} vs "
          f"{int(ref.hull.sum())})")
    if not same_nbr:
        deg = np.diff(o)
        rdeg = np.diff(ref.offsets)
        bad = np.nonzero(deg != rdeg)[0]
        print(f"degree mismatches: {len(bad)} sites; first: {bad[:10]}")
        for i in bad[:5]:
            a = set(nb[o[i]:o[i + 1]].tolist())
            b = set(ref.neighbors[ref.offsets[i]:ref.offsets[i + 1]].tolist())
            print(f"  site {i} hull {bool(ref.hull[i])}: extra {sorted(a - b)} missing {sorted(b - a)}")
