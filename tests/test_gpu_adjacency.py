"""Device Delaunay adjacency (rfb_build_adjacency) against
the reference's own builder (geometry/delaunay.py build +
adjacency.py from_triangulation, tests/golden/adjacency.npz) and, at sizes
the reference builder cannot reach, against Qhull (whose CSR the survey
verified bit-identical to the reference's at 2k/10k/100k)."""

import numpy as np
import pytest
import torch

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["uniform2k", "surface3k", "gauss1500"])
def test_adjacency_matches_reference_builder(cuda_ok, name):
    from paper_2502_01157_b200 import adjacency as A

    g = load_golden("adjacency")
    pos = g[f"{name}_positions"]
    off, nbr, hull, info = A.build_device(torch.from_numpy(pos).cuda())
    np.testing.assert_array_equal(off.cpu().numpy(), g[f"{name}_offsets"])
    np.testing.assert_array_equal(nbr.cpu().numpy(), g[f"{name}_neighbors"])
    np.testing.assert_array_equal(hull.cpu().numpy(), g[f"{name}_hull"])
    assert info["reverse_edges_added"] == 0


@pytest.mark.parametrize("kind,n,seed", [("uniform", 100_000, 5), ("surface", 60_000, 6)])
def test_adjacency_matches_qhull(cuda_ok, kind, n, seed):
    from paper_2502_01157_b200 import adjacency as A
    from paper_2502_01157_b200.synthetic import delaunay_csr, random_positions

    pos = random_positions(n, seed, kind)
    ref_off, ref_nbr, ref_hull = delaunay_csr(pos)
    off, nbr, hull, info = A.build_device(torch.from_numpy(pos).cuda())
    np.testing.assert_array_equal(off.cpu().numpy(), ref_off)
    np.testing.assert_array_equal(nbr.cpu().numpy(), ref_nbr)
    np.testing.assert_array_equal(hull.cpu().numpy(), ref_hull)
    assert info["reverse_edges_added"] == 0


def test_adjacency_errors_and_host_api(cuda_ok):
    from paper_2502_01157_b200 import adjacency as A
    from paper_2502_01157_b200.errors import DegenerateInput, DuplicatePoints

    g = load_golden("adjacency")
    pos = g["gauss1500_positions"].copy()
    adj = A.build(pos)
    np.testing.assert_array_equal(adj.offsets, g["gauss1500_offsets"])
    np.testing.assert_array_equal(adj.hull, g["gauss1500_hull"])
    dup = pos.copy()
    dup[7] = dup[3]
    with pytest.raises(DuplicatePoints):
        A.build(dup)
    bad = pos.copy()
    bad[2, 1] = np.nan
    with pytest.raises(DegenerateInput):
        A.build(bad)
    with pytest.raises(DegenerateInput):
        A.build(pos[:3])
