"""Host-side logic (no GPU): scene containers, activations, camera math, the
synthetic fixture generator and the distributed tile/ray partitioning."""

import numpy as np
import pytest

from conftest import golden_scene_arrays, load_golden
from oracle import oracle as orc
from paper_2502_01157_b200 import distributed as D
from paper_2502_01157_b200.camera import (PINHOLE, CameraModel, camera_rays, look_at,
                                          orbit_poses)
from paper_2502_01157_b200.errors import OutOfBounds, ShapeMismatch
from paper_2502_01157_b200.scene import (AdjacencyGraph, FoamScene, GradientBuffer, softplus,
                                         softplus_grad)
from paper_2502_01157_b200.synthetic import delaunay_csr, random_positions


def test_softplus_matches_reference_bits():
    g = load_golden("kat")
    np.testing.assert_array_equal(softplus(g["softplus_in"]), g["softplus_out"])
    np.testing.assert_array_equal(softplus_grad(g["softplus_in"]), g["softplus_grad_out"])
    assert softplus(0.0) == pytest.approx(0.0693147, abs=1e-7)
    assert float(softplus(-10.0)) == pytest.approx(3.72e-45, rel=1e-2)  # code value


def test_scene_validation():
    with pytest.raises(ShapeMismatch):
        FoamScene(np.zeros((3, 3)), np.zeros(2), np.zeros((3, 16, 3)))
    with pytest.raises(ShapeMismatch):
        FoamScene(np.zeros((3, 3)), np.zeros(3), np.zeros((3, 9, 3)))
    gb = GradientBuffer(4)
    gb.d_sh += 1.0
    assert gb.all_finite()
    gb.zero()
    assert not gb.d_sh.any()


def test_adjacency_from_lists_and_nearest():
    pos = np.array([[0.0, 0, 0], [2.0, 0, 0], [0, 2.0, 0]])
    adj = AdjacencyGraph.from_lists(pos, [[1, 2], [], []])
    assert adj.neighbor_list(0).tolist() == [1, 2]
    assert adj.neighbor_list(1).tolist() == [0]
    assert adj.degree(2) == 1
    # tie at the midpoint of sites 0 and 1: lowest id wins (adjacency.py:198)
    assert adj.nearest_site([1.0, 0.0, 0.0]) == 0
    g = load_golden("frame_2k_deg3")
    sa = golden_scene_arrays(g)
    adj = AdjacencyGraph(g["positions"], g["offsets"], g["neighbors"])
    q = np.random.default_rng(0).uniform(-1.5, 1.5, (200, 3))
    ref = orc.nearest_sites(sa.positions, q)
    assert [adj.nearest_site(x) for x in q] == ref.tolist()


@pytest.mark.parametrize("name", ["frame_2k_deg3", "frame_3k_surface"])
def test_camera_matches_reference(name):
    g = load_golden(name)
    cam = CameraModel(PINHOLE, int(g["width"]), int(g["height"]), float(g["focal"]), g["pose"])
    np.testing.assert_array_equal(cam.ray_directions(), g["dirs"])
    o, d = camera_rays(cam, (0, 0))
    np.testing.assert_array_equal(d, g["dirs"][0])
    with pytest.raises(OutOfBounds):
        camera_rays(cam, (int(g["height"]), 0))


def test_look_at_and_orbit():
    pose = look_at((0, 0, 3), (0, 0, 0))
    np.testing.assert_allclose(pose[:3, 2], [0, 0, 1])
    poses = orbit_poses(np.zeros(3), 3.0, 0.3, 8)
    assert len(poses) == 8
    for p in poses:
        np.testing.assert_allclose(np.linalg.norm(p[:3, 3]), 3.0)
        np.testing.assert_allclose(p[:3, :3] @ p[:3, :3].T, np.eye(3), atol=1e-12)


def test_synthetic_positions_fp32_exact_and_csr_symmetric():
    pos = random_positions(500, 3)
    np.testing.assert_array_equal(pos.astype(np.float32).astype(np.float64), pos)
    off, nbr, hull = delaunay_csr(pos)
    assert off[-1] == len(nbr)
    pairs = set()
    for i in range(len(pos)):
        row = nbr[off[i]:off[i + 1]]
        assert np.all(np.diff(row) > 0), "ascending neighbour ids per site"
        pairs.update((i, int(j)) for j in row)
    assert all((j, i) in pairs for i, j in pairs), "symmetric"
    assert hull.any()


def test_golden_csr_is_reference_delaunay():
    # make_golden.py asserted Qhull == rfoam.geometry.delaunay.build at 2k/3k;
    # the committed CSR must still be the Qhull CSR of the committed sites.
    g = load_golden("frame_2k_deg3")
    off, nbr, _ = delaunay_csr(g["positions"])
    np.testing.assert_array_equal(off, g["offsets"])
    np.testing.assert_array_equal(nbr, g["neighbors"])


@pytest.mark.parametrize("W,H,world", [(1920, 1080, 1), (1920, 1080, 2), (1920, 1080, 8),
                                       (130, 70, 3), (3840, 2160, 4)])
def test_tile_assignment_partitions_frame(W, H, world):
    cover = np.zeros((H, W), dtype=np.int32)
    for r in range(world):
        tiles = D.tile_assignment(W, H, r, world)
        cover += D.tile_pixel_mask(W, H, tiles)
    assert (cover == 1).all()


def test_shard_rays_partition():
    for m, w in [(10, 3), (65536, 8), (7, 8)]:
        ranges = [D.shard_rays(m, r, w) for r in range(w)]
        covered = np.concatenate([np.arange(lo, hi) for lo, hi in ranges])
        np.testing.assert_array_equal(covered, np.arange(m))


def test_rfoam1_checkpoint_roundtrip(tmp_path):
    """Reads the reference-written file; writes byte-identical files; rejects
    corrupt ones (io/checkpoint.py:30-60)."""
    import os

    from conftest import GOLDEN
    from paper_2502_01157_b200.checkpoint import (CorruptCheckpoint, load_checkpoint,
                                                  save_checkpoint)

    path = os.path.join(GOLDEN, "scene300.rfoam")
    e = load_golden("scene300_expect")
    sc = load_checkpoint(path, rebuild=True)
    np.testing.assert_array_equal(sc.positions, e["positions"])
    np.testing.assert_array_equal(sc.raw_density, e["raw"])
    np.testing.assert_array_equal(sc.sh_coeffs, e["sh"])
    np.testing.assert_array_equal(sc.background, e["background"])
    assert sc.adjacency.offsets[-1] == len(sc.adjacency.neighbors)
    out = tmp_path / "copy.rfoam"
    save_checkpoint(sc, out)
    assert out.read_bytes() == open(path, "rb").read()
    bad = tmp_path / "bad.rfoam"
    bad.write_bytes(b"RFOAM2" + out.read_bytes()[6:])
    with pytest.raises(CorruptCheckpoint):
        load_checkpoint(bad)
    bad.write_bytes(out.read_bytes()[:-4])
    with pytest.raises(CorruptCheckpoint):
        load_checkpoint(bad)
    blob = bytearray(out.read_bytes())
    blob[10:14] = np.array([np.nan], dtype="<f4").tobytes()
    bad.write_bytes(bytes(blob))
    with pytest.raises(CorruptCheckpoint):
        load_checkpoint(bad)


def test_tile_order_is_permutation():
    from paper_2502_01157_b200.device import tile_order

    for W, H in [(130, 70), (1920, 1080), (32, 32)]:
        o = tile_order(W, H)
        np.testing.assert_array_equal(np.sort(o), np.arange(W * H))
    o = tile_order(64, 32)
    # first warp = a 4 x 8 pixel patch
    np.testing.assert_array_equal(o[:8], [0, 1, 2, 3, 64, 65, 66, 67])


def test_effect_rays_host_match_reference():
    """render.reflect / refract / apply_effect / intersect_face against the
    reference's own outputs (tests/golden/effects.npz, rays.py:60-176)."""
    from paper_2502_01157_b200 import render as rd

    g = load_golden("effects")
    m = len(g["d"])
    for i in range(m):
        np.testing.assert_array_equal(rd.reflect(g["d"][i], g["normal"][i]), g["reflect"][i])
        np.testing.assert_allclose(rd.refract(g["d"][i], g["normal"][i], g["eta"][i]),
                                   g["refract"][i], rtol=0, atol=1e-15)
        for kind in ("mirror", "refract"):
            r = rd.apply_effect(rd.Ray(g["o"][i], g["d"][i], 0.0, 9.0), g["normal"][i], kind,
                                g["eta"][i], g["t_at"][i])
            np.testing.assert_array_equal(r.origin, g[f"{kind}_o"][i])
            np.testing.assert_allclose(r.direction, g[f"{kind}_d"][i], rtol=0, atol=1e-15)
            assert r.t_min == 0.0 and r.t_max == 9.0
        t, front = rd.intersect_face(rd.Ray(g["o"][i], g["d"][i]), g["x"][i], g["xp"][i])
        assert t == g["face_t"][i] and front == g["face_front"][i]
    with pytest.raises(ValueError):
        rd.EffectPlane(np.zeros(3), np.ones(3), kind="lens")
    with pytest.raises(ValueError):
        rd.intersect_face(rd.Ray(np.zeros(3), np.array([0.0, 0.0, 1.0])), np.ones(3), np.ones(3))


def test_csr_sha1_of_qhull_fixture():
    """synthetic.csr_sha1 over a Qhull CSR is deterministic and sensitive to one edge."""
    from paper_2502_01157_b200.synthetic import csr_sha1, delaunay_csr, random_positions

    pos = random_positions(3000, 9, "uniform")
    off, nbr, _ = delaunay_csr(pos)
    h = csr_sha1(off, nbr)
    assert h == csr_sha1(off.astype(np.int32), nbr.astype(np.int32))
    nbr2 = nbr.copy()
    nbr2[5] += 1
    assert csr_sha1(off, nbr2) != h


@pytest.mark.parametrize("W,H,angle", [(1920, 1080, 0.9), (320, 256, 1.4), (64, 1, 0.3)])
def test_view_cone_holds_every_pixel_direction(W, H, angle):
    """device.view_cone: every pixel direction of a pinhole camera (the reference's
    camera.py:78-92 arithmetic) is a positive combination of the four corner
    generators, so a face back-facing (with margin) for all four is back-facing
    for every pixel -- the premise of rfb_cull_scene."""
    from paper_2502_01157_b200 import device as dv

    cam = CameraModel.from_angle_x(PINHOLE, W, H, angle,
                                   look_at((0.3, -2.0, 2.5), (0.1, 0.2, -0.1)))
    cone = dv.view_cone(cam)
    c = cone / np.linalg.norm(cone, axis=1, keepdims=True)
    rng = np.random.default_rng(1)
    rows = rng.integers(0, H, 4000)
    cols = rng.integers(0, W, 4000)
    d = cam.ray_directions(rows, cols)
    n = rng.normal(size=(20000, 3))
    back = np.all(n @ c.T < -1e-9 * np.abs(n).sum(1)[:, None], axis=1)
    assert back.mean() > 0.1
    assert np.all(n[back] @ d.T < 0.0)
    # the corners are pixel directions themselves: the cone is tight
    corner = cam.ray_directions(np.array([0, 0, H - 1, H - 1]), np.array([0, W - 1, 0, W - 1]))
    np.testing.assert_allclose(corner, c, atol=1e-15)
    assert dv.view_cone(CameraModel.from_angle_x("fisheye", W, H, angle, cam.pose)) is None
