"""Cold scene build (DeviceScene from a host FoamScene) timing, median of 6."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_01157_b200 import device as dv  # noqa: E402
from paper_2502_01157_b200.synthetic import make_foam  # noqa: E402
scene = make_foam(1_000_000, 1, 3)
ts = []
for it in range(8):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ds = dv.DeviceScene(scene)
    torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    del ds
print(f"chunk {dv._Uploader.CHUNK >> 20} MB threads {dv._Uploader.THREADS}: "
      f"DeviceScene median {1e3 * np.median(ts[2:]):.1f} ms", flush=True)
