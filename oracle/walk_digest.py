"""Per-ray digest of a walk's segment list (TEST INFRASTRUCTURE, like the rest
of oracle/): the same function as ``walk_digest`` in rfoam_oracle.c, computed
with torch from the device's segment dump (rfb_fwd_out.seg_cells/t0/t1), so a
large frame's visited-cell sequences and segment depths can be compared with
the oracle ray by ray without moving every segment list to the host.

digest = sum_s mix(mix(mix(cell_s + s * K) ^ bits(t0_s)) ^ bits(t1_s))  (mod 2^64)

Order-sensitive (the index enters every term) and exact on bits: equal
digests for every ray is the bit-exact cell / t0 / t1 check of SURVEY §8c.
torch has no uint64 arithmetic, so the mix runs on int64 with wrapping
multiplies and masked (logical) right shifts.
"""

from __future__ import annotations

import numpy as np
import torch

_M1 = 0xFF51AFD7ED558CCD
_M2 = 0xC4CEB9FE1A85EC53
_K = 0x9E3779B97F4A7C15


def _s64(x: int) -> int:
    """uint64 constant as the int64 with the same bits."""
    return x - (1 << 64) if x >= (1 << 63) else x


def _lsr33(x: torch.Tensor) -> torch.Tensor:
    return (x >> 33) & 0x7FFFFFFF


def _mix(x: torch.Tensor) -> torch.Tensor:
    x = x ^ _lsr33(x)
    x = x * _s64(_M1)
    x = x ^ _lsr33(x)
    x = x * _s64(_M2)
    return x ^ _lsr33(x)


def digests(seg_cells: torch.Tensor, seg_t0: torch.Tensor, seg_t1: torch.Tensor,
            nseg: torch.Tensor, chunk: int = 16384) -> np.ndarray:
    """(m,) uint64 digests from [m, cap] segment dumps; rays whose nseg
    exceeds cap raise (the dump would be truncated)."""
    m, cap = seg_cells.shape
    nseg = nseg.to(seg_cells.device, torch.int64)
    if m and int(nseg.max()) > cap:
        raise ValueError(f"segment dump capacity {cap} < max nseg {int(nseg.max())}")
    out = torch.empty(m, dtype=torch.int64, device=seg_cells.device)
    idx = torch.arange(cap, dtype=torch.int64, device=seg_cells.device)
    for lo in range(0, m, chunk):
        hi = min(m, lo + chunk)
        c = seg_cells[lo:hi].to(torch.int64)
        b0 = seg_t0[lo:hi].contiguous().view(torch.int64)
        b1 = seg_t1[lo:hi].contiguous().view(torch.int64)
        e = _mix(c + idx[None, :] * _s64(_K))
        e = _mix(e ^ b0)
        e = _mix(e ^ b1)
        e = torch.where(idx[None, :] < nseg[lo:hi, None], e, torch.zeros_like(e))
        out[lo:hi] = e.sum(dim=1)
    return out.cpu().numpy().view(np.uint64)
