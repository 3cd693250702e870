import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from bench import make_views
from paper_2502_01157_b200 import device as dv, render as rd
from paper_2502_01157_b200.synthetic import make_foam
scene = make_foam(10_000, 0, 0)
cam = make_views(1, 128, 128)[0]
for it in range(8):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ds = dv.DeviceScene(scene)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    img = rd.render_image(scene, cam, device_scene=ds)
    t2 = time.perf_counter()
    print(f"{it}: scene {1e3*(t1-t0):.1f} ms render {1e3*(t2-t1):.1f} ms", flush=True)
    del ds, img
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
ds = dv.DeviceScene(scene); img = rd.render_image(scene, cam, device_scene=ds); torch.cuda.synchronize()
pr.disable(); pstats.Stats(pr).sort_stats("cumtime").print_stats(15)
