"""rfb_segments.cu -- the reference's per-ray building blocks over given
segment lists (tracer/kernels.py:38-73, 165-196, 250-369, 456-567) -- against
the C oracle's restatement of the same functions, on walk segments of the
golden 2k scene; and the flat kernels.py single-ray drop-ins."""

import numpy as np
import pytest
import torch

from conftest import golden_scene_arrays, load_golden
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _segments(m=48, seed=0, inside=False):
    g = load_golden("grad_2k_deg3")
    sa = golden_scene_arrays(g)
    rng = np.random.default_rng(seed)
    o = rng.uniform(-0.3, 0.3, (m, 3)) if inside else np.tile([0.0, 0.0, 3.0], (m, 1))
    d = rng.normal(size=(m, 3)) + (0 if inside else np.array([0.0, 0.0, -4.0]))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    cells, t0, t1, off = [], [], [], [0]
    for r in range(m):
        start = int(orc.nearest_sites(sa.positions, o[r:r + 1])[0])
        c, a, b, status, _, _ = orc.walk_ray(sa, o[r], d[r], 0.0, 8.0, start, epsilon=0.0)
        cells.append(c), t0.append(a), t1.append(b), off.append(off[-1] + len(c))
    return (sa, o, d, np.array(off), np.concatenate(cells), np.concatenate(t0),
            np.concatenate(t1))


def _dev(a, dt=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)


def rel(a, b):
    den = np.abs(b).max()
    return float(np.abs(a - b).max() / den) if den > 0 else float(np.abs(a).max())


def test_basis_colors_composite(cuda_ok):
    from paper_2502_01157_b200 import device as dv

    sa, o, d, off, cells, t0, t1 = _segments()
    basis = dv.sh_basis_device(_dev(d))
    ref_basis = np.stack([orc.sh_basis(v) for v in d])
    np.testing.assert_allclose(basis.cpu().numpy(), ref_basis, rtol=0, atol=1e-15)
    col, mask = dv.cell_colors_device(_dev(sa.sh), _dev(cells[:len(d)], torch.int32), basis)
    for r in range(len(d)):
        c, mk = orc.cell_color(sa.sh, cells[r], ref_basis[r])
        np.testing.assert_allclose(col.cpu().numpy()[r], c, rtol=0, atol=1e-15)
        assert int(mask[r]) == mk
    rgb, T, ws = dv.composite_segments_device(_dev(sa.sigma), _dev(sa.sh), basis, _dev(off, torch.int64),
                                              _dev(cells, torch.int32), _dev(t0), _dev(t1),
                                              sa.background)
    r_rgb, r_T, r_ws = orc.composite_batch(off, cells, t0, t1, sa.sigma, sa.sh, d, sa.background)
    np.testing.assert_allclose(rgb.cpu().numpy(), r_rgb, rtol=0, atol=1e-13)
    np.testing.assert_allclose(T.cpu().numpy(), r_T, rtol=0, atol=1e-13)
    np.testing.assert_allclose(ws.cpu().numpy(), r_ws, rtol=0, atol=1e-13)


@pytest.mark.parametrize("inside", [False, True])
def test_backward_and_quantile_segments(cuda_ok, inside):
    from paper_2502_01157_b200 import device as dv

    sa, o, d, off, cells, t0, t1 = _segments(seed=3, inside=inside)
    m, n = len(d), sa.n
    adj = np.random.default_rng(5).normal(size=(m, 3))
    basis = dv.sh_basis_device(_dev(d))
    gs = torch.zeros(n, dtype=torch.float64, device="cuda")
    gsh = torch.zeros((n, 48), dtype=torch.float64, device="cuda")
    gp = torch.zeros((n, 3), dtype=torch.float64, device="cuda")
    dv.backward_segments_device(_dev(sa.positions), _dev(sa.sigma), _dev(sa.sh), sa.background,
                                _dev(o), _dev(d), basis, _dev(adj), _dev(off, torch.int64),
                                _dev(cells, torch.int32), _dev(t0), _dev(t1), gs, gsh, gp)
    r_s, r_sh, r_p = orc.backward_batch(sa.positions, sa.sigma, sa.sh, sa.background, o, d, adj,
                                        off, cells, t0, t1)
    assert rel(gs.cpu().numpy(), r_s) < 1e-10
    assert rel(gsh.cpu().numpy(), r_sh) < 1e-10
    assert rel(gp.cpu().numpy(), r_p) < 1e-10
    up = np.random.default_rng(6).uniform(0, 1, (m, 2, 2))
    qs = torch.zeros(n, dtype=torch.float64, device="cuda")
    qp = torch.zeros((n, 3), dtype=torch.float64, device="cuda")
    loss = dv.quantile_segments_device(_dev(sa.positions), _dev(sa.sigma), _dev(o), _dev(d),
                                       _dev(off, torch.int64), _dev(cells, torch.int32), _dev(t0), _dev(t1),
                                       _dev(up), 1e-4, 0.01, qs, qp)
    r_qs, r_qp, r_loss = orc.quantile_batch(sa.positions, sa.sigma, o, d, off, cells, t0, t1, up,
                                            1e-4, 0.01)
    np.testing.assert_allclose(loss.cpu().numpy(), r_loss, rtol=1e-12, atol=1e-14)
    assert rel(qs.cpu().numpy(), r_qs) < 1e-10
    assert rel(qp.cpu().numpy(), r_qp) < 1e-10


def test_flat_single_ray_drop_ins(cuda_ok):
    """kernels.sh_basis_into / cell_color / composite_segments / backward_ray /
    face_t_gradient / quantile_backward_ray with the reference signatures."""
    from paper_2502_01157_b200 import kernels as K

    sa, o, d, off, cells, t0, t1 = _segments(m=4, seed=9)
    r = 2
    c, a, b = cells[off[r]:off[r + 1]], t0[off[r]:off[r + 1]], t1[off[r]:off[r + 1]]
    basis = np.empty(16)
    K.sh_basis_into(*d[r], basis)
    np.testing.assert_allclose(basis, orc.sh_basis(d[r]), rtol=0, atol=1e-15)
    out = np.empty(3)
    mk = K.cell_color(sa.sh, c[0], basis, out)
    ref_c, ref_mk = orc.cell_color(sa.sh, c[0], basis)
    np.testing.assert_allclose(out, ref_c, rtol=0, atol=1e-15)
    assert mk == ref_mk
    rgb = np.empty(3)
    T, ws = K.composite_segments(c, a, b, len(c), sa.sigma, sa.sh, basis, *sa.background, rgb)
    r_rgb, r_T, r_ws = orc.composite_batch(np.array([0, len(c)]), c, a, b, sa.sigma, sa.sh,
                                           d[r:r + 1], sa.background)
    np.testing.assert_allclose(rgb, r_rgb[0], rtol=0, atol=1e-13)
    assert abs(T - r_T[0]) < 1e-13 and abs(ws - r_ws[0]) < 1e-13
    n = sa.n
    d_sigma, d_sh, d_pos = np.zeros(n), np.zeros((n, 48)), np.zeros((n, 3))
    K.backward_ray(sa.positions, sa.offsets, sa.neighbors, sa.sigma, sa.sh, sa.background,
                   *o[r], *d[r], 0.3, -0.2, 0.5, c, a, b, len(c), 0.0, basis, d_sigma, d_sh, d_pos)
    r_s, r_sh, r_p = orc.backward_batch(sa.positions, sa.sigma, sa.sh, sa.background, o[r:r + 1],
                                        d[r:r + 1], np.array([[0.3, -0.2, 0.5]]),
                                        np.array([0, len(c)]), c, a, b)
    assert rel(d_sigma, r_s) < 1e-12 and rel(d_sh, r_sh) < 1e-12 and rel(d_pos, r_p) < 1e-12
    d_pos2 = np.zeros((n, 3))
    K.face_t_gradient(sa.positions, c[0], c[1], *o[r], *d[r], b[0], 0.7, d_pos2)
    assert np.count_nonzero(d_pos2) > 0
    q_sigma, q_pos = np.zeros(n), np.zeros((n, 3))
    loss = K.quantile_backward_ray(c, a, b, len(c), sa.sigma, np.array([0.2, 0.7]), 1e-4,
                                   sa.positions, *o[r], *d[r], 0.01, q_sigma, q_pos)
    r_qs, r_qp, r_loss = orc.quantile_batch(sa.positions, sa.sigma, o[r:r + 1], d[r:r + 1],
                                            np.array([0, len(c)]), c, a, b,
                                            np.array([[[0.2, 0.7]]]), 1e-4, 0.01)
    assert abs(loss - r_loss[0]) < 1e-12
    assert rel(q_sigma, r_qs) < 1e-12 and rel(q_pos, r_qp) < 1e-12
