"""Breakdown of the cold end-to-end call (bench.py e2e_cold): host scene ->
DeviceScene (upload + pack) -> render_image -> host image, per stage."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import make_views  # noqa: E402
from paper_2502_01157_b200 import device as dv  # noqa: E402
from paper_2502_01157_b200 import render as rd  # noqa: E402
from paper_2502_01157_b200.synthetic import make_foam  # noqa: E402

scene = make_foam(1_000_000, 1, 3)
cam = make_views(1, 1920, 1080)[0]
import cProfile  # noqa: E402
import pstats  # noqa: E402
for it in range(6):
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    t0 = time.perf_counter()
    ds = dv.DeviceScene(scene)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    pr.disable()
    if t1 - t0 > 0.2:
        pstats.Stats(pr).sort_stats("tottime").print_stats(6)
    img = rd.render_image(scene, cam, device_scene=ds)
    t2 = time.perf_counter()
    print(f"iter {it}: DeviceScene {1e3 * (t1 - t0):7.1f} ms, render_image {1e3 * (t2 - t1):6.1f} ms",
          flush=True)
    del ds, img
