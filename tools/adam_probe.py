"""Adam + scene refresh on the 1M-site scene (train.DeviceTrainer.post_grad_adam),
with the fp32 SH copy written by the Adam pass (FUSE_SH32) or by the refresh."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_01157_b200 import train  # noqa: E402
from paper_2502_01157_b200.synthetic import make_foam  # noqa: E402

tr = train.DeviceTrainer(make_foam(1_000_000, 1, 3))
tr.grads.flat.normal_(0, 1e-3)
for fuse in (True, False, True, False):
    train.FUSE_SH32 = fuse
    for _ in range(3):
        tr.post_grad_adam(1e-4, 0.1, 5e-3, False, train.AdamHyper())
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(50):
        tr.post_grad_adam(1e-4, 0.1, 5e-3, False, train.AdamHyper())
    b.record()
    torch.cuda.synchronize()
    print(f"fuse_sh32={fuse}: {a.elapsed_time(b) / 50:.4f} ms per Adam + refresh")
