"""CPU: pin the fp64 oracle against the reference's golden vectors and KATs.

The fixtures under tests/golden/ were produced by running the reference
itself (tests/golden/make_golden.py); here the oracle (oracle/splat_oracle.c)
must reproduce them to ~1e-12 and the tile lists / n_contrib exactly.
"""

import numpy as np
import pytest

import oracle as O
from parity import golden_names, load_golden

NAMES = golden_names()


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    if b.size == 0:
        return 0.0
    s = np.max(np.abs(b))
    return float(np.max(np.abs(a - b)) / s) if s > 0 else float(np.max(np.abs(a)))


@pytest.fixture(scope="module", params=NAMES)
def run(request):
    g = load_golden(request.param)
    cam = g["camera"]
    fw = O.render(*g["inputs"], cam, g["background"], g["et"], nthreads=2)
    sb = O.scene_backward(*g["inputs"], cam, g["background"], fw, g["d_image"], nthreads=2)
    return request.param, g, fw, sb


def test_projection(run):
    name, g, fw, _ = run
    vis = np.nonzero(fw["visible"])[0]
    assert np.array_equal(vis, g["proj_source"])
    assert np.array_equal(fw["radius"][vis], g["proj_radius"])
    assert _rel(fw["mean2d"][vis], g["proj_mean2d"]) < 1e-13
    assert _rel(fw["cov2d"][vis], g["proj_cov2d"].reshape(-1, 4)[:, [0, 1, 3]]) < 1e-13
    assert _rel(fw["t_cam"][vis], g["proj_t_cam"]) < 1e-13
    assert _rel(fw["depth"][vis], g["proj_depth"]) < 1e-14


def test_bins_exact(run):
    name, g, fw, _ = run
    assert np.array_equal(fw["bin_ptr"], g["bin_ptr"])
    assert np.array_equal(fw["bin_idx"], g["bin_idx"])


def test_forward(run):
    name, g, fw, _ = run
    assert _rel(fw["image"], g["image"]) < 1e-12
    assert _rel(fw["final_T"], g["final_T"]) < 1e-12
    assert np.array_equal(fw["n_contrib"], g["n_contrib"])


def test_screen_space_grads(run):
    name, g, fw, sb = run
    for k in ("d_mean2d", "d_cov2d"):
        assert _rel(sb[k], g["s_" + k]) < 1e-11, k
    assert _rel(sb["d_color"], g["s_d_color"]) < 1e-11
    assert _rel(sb["d_opacity"], g["s_d_opacity"]) < 1e-11


def test_scene_grads(run):
    name, g, fw, sb = run
    for k in ("d_mean", "d_scale", "d_quat", "d_opacity", "d_color", "d_view"):
        assert _rel(sb[k], g["g_" + k]) < 1e-11, (name, k, _rel(sb[k], g["g_" + k]))


def test_thread_count_determinism():
    g = load_golden("cfg0_mini")
    cam = g["camera"]
    outs = []
    for nt in (1, 3):
        fw = O.render(*g["inputs"], cam, g["background"], g["et"], nthreads=nt)
        sb = O.scene_backward(*g["inputs"], cam, g["background"], fw, g["d_image"], nthreads=nt)
        outs.append((fw, sb))
    assert np.array_equal(outs[0][0]["image"], outs[1][0]["image"])
    for k in ("d_mean", "d_quat", "d_color"):
        assert _rel(outs[0][1][k], outs[1][1][k]) < 1e-13


# ---- known-answer tests restated from the reference's own unit tests ----

def _cam(w, h, fx, view=None, cx=None, cy=None, near=0.1, far=100.0):
    return O.Camera(np.eye(4) if view is None else view, fx, fx, (w - 1) / 2.0 if cx is None else cx,
                    (h - 1) / 2.0 if cy is None else cy, w, h, near, far)


def test_kat_optical_axis_maps_to_half_pixel():
    # tests/test_projection.py:63-71: cx = cy = 0 -> optical axis at (0.5, 0.5)
    cam = _cam(64, 64, 50.0, cx=0.0, cy=0.0)
    for z in (0.5, 2.0, 50.0):
        pr = O.project([[0.0, 0.0, z]], [[0.1, 0.1, 0.1]], [[1, 0, 0, 0]], cam)
        np.testing.assert_allclose(pr["mean2d"][0], [0.5, 0.5], atol=1e-12)


def test_kat_single_splat_half_opacity():
    # tests/test_forward.py:126-137: alpha = opacity at sigma = 0, T = 0.5
    cam = _cam(1, 1, 8.0)
    fw = O.render([[0.0, 0.0, 4.0]], [[0.5, 0.5, 0.5]], [[1, 0, 0, 0]], [0.5], [[1.0, 0.0, 0.0]], cam, np.zeros(3))
    np.testing.assert_allclose(fw["image"][0, 0], [0.5, 0.0, 0.0], rtol=1e-15)
    assert fw["final_T"][0, 0] == 0.5 and fw["n_contrib"][0, 0] == 1


def test_kat_two_splats_front_to_back():
    # tests/test_forward.py:139-151
    cam = _cam(1, 1, 8.0)
    fw = O.render([[0.0, 0.0, 3.0], [0.0, 0.0, 5.0]], [[0.5] * 3] * 2, [[1, 0, 0, 0]] * 2, [0.5, 0.5],
                  [[1.0, 0.0, 0.0], [0.0, 1.0, 0.0]], cam, np.zeros(3))
    np.testing.assert_allclose(fw["image"][0, 0], [0.5, 0.25, 0.0], rtol=1e-15)
    assert fw["final_T"][0, 0] == 0.25 and fw["n_contrib"][0, 0] == 2


def test_kat_single_splat_grads():
    # tests/test_backward_raster.py:67-96: d color = 0.5, d opacity = 1 (bg 0) / -2 (bg 1), d mean2d = 0
    cam = _cam(1, 1, 8.0)
    args = ([[0.0, 0.0, 4.0]], [[0.5] * 3], [[1, 0, 0, 0]], [0.5], [[1.0, 0.0, 0.0]])
    for bg, d_op in ((np.zeros(3), 1.0), (np.ones(3), -2.0)):
        fw = O.render(*args, cam, bg)
        sb = O.scene_backward(*args, cam, bg, fw, np.ones((1, 1, 3)))
        np.testing.assert_allclose(sb["d_color"][0], [0.5, 0.5, 0.5], rtol=1e-14)
        np.testing.assert_allclose(sb["d_opacity"][0], d_op, rtol=1e-13)
        np.testing.assert_allclose(sb["d_mean2d"][0], [0.0, 0.0], atol=1e-15)


def test_kat_binning_corner_and_interior():
    # tests/test_binning.py:48-59: interior splat -> 1 tile; corner splat radius 2 -> 4 tiles
    vis = np.ones(2, np.int8)
    ptr, idx = O.bin_tiles(vis, [[8.0, 8.0], [16.0, 16.0]], [1, 2], [1.0, 2.0], 64, 64)
    counts = np.diff(ptr)
    tiles_of = lambda j: sorted(int(t) for t in np.nonzero([j in idx[ptr[t]:ptr[t + 1]] for t in range(16)])[0])
    assert tiles_of(0) == [0]
    assert tiles_of(1) == [0, 1, 4, 5]
    assert counts.sum() == 5


def test_kat_sort_depth_then_index():
    # tests/test_binning.py:92-107: depths [3,1,2] -> [1,2,0]; equal depths -> ascending index
    vis = np.ones(3, np.int8)
    ptr, idx = O.bin_tiles(vis, [[8.0, 8.0]] * 3, [1, 1, 1], [3.0, 1.0, 2.0], 16, 16)
    assert idx.tolist() == [1, 2, 0]
    ptr, idx = O.bin_tiles(np.ones(6, np.int8), [[8.0, 8.0]] * 6, [1] * 6, [5.0, 9.0, 1.0, 9.0, 9.0, 1.0], 16, 16)
    assert idx.tolist() == [2, 5, 0, 1, 3, 4]


def test_errors_mirror_reference():
    cam = _cam(16, 16, 16.0)
    with pytest.raises(ValueError, match="gaussian 1: scale"):
        O.project([[0, 0, 4.0], [0, 0, 4.0]], [[0.1] * 3, [0.1, -1.0, 0.1]], [[1, 0, 0, 0]] * 2, cam)
    with pytest.raises(ValueError, match="gaussian 0: quaternion"):
        O.project([[0, 0, 4.0]], [[0.1] * 3], [[0, 0, 0, 0]], cam)
    # depth-culled splats never raise (sg/projection.py:124-125 precedes the checks)
    pr = O.project([[0, 0, -4.0]], [[-1.0] * 3], [[0, 0, 0, 0]], cam)
    assert pr["visible"][0] == 0
