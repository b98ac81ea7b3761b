"""GPU: the reference's per-splat helpers (paper_2312_02121_b200.helpers,
csrc/ops64.cu, float64) against golden vectors the real reference produced
(tests/golden/make_golden_helpers.py), the reference's own KATs
(tests/test_core.py, tests/test_projection.py, tests/test_backward_proj.py
of the reference) restated, and its ValueError messages."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "helpers.npz")


@pytest.fixture(scope="module")
def gold(cuda):
    return dict(np.load(GOLDEN))


def _cam(sg, z, i):
    fx, fy, cx, cy, W, H, near, far = z["intr"][i]
    return sg.Camera(view=z["view"][i], fx=fx, fy=fy, cx=cx, cy=cy, width=int(W), height=int(H), near=near, far=far)


def test_helpers_match_reference_goldens(gold):
    import paper_2312_02121_b200 as sg
    z = gold
    close = lambda a, b: np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12)
    for i in range(len(z["quat"])):
        cam = _cam(sg, z, i)
        close(sg.quat_to_rotmat(z["quat"][i]), z["R"][i])
        b = sg.compose_covariance_3d(z["quat"][i], z["scale"][i])
        assert isinstance(b, sg.Cov3DBundle)
        for k, key in (("R", "R"), ("S", "S"), ("M", "M"), ("sigma", "sigma")):
            close(getattr(b, k), z[key][i])
        close(sg.world_to_camera(z["mean"][i], cam), z["t_cam"][i])
        close(sg.camera_to_pixel(z["t_cam"][i], cam), z["mean2d"][i])
        close(sg.projection_jacobian(z["t_cam"][i], cam), z["J"][i])
        close(sg.project_covariance(z["J"][i], z["Rcw"][i], z["sigma"][i]), z["cov2d"][i])
        r = sg.bounding_radius(z["cov2d"][i])
        assert isinstance(r, int) and r == int(z["radius"][i])
        close(sg.mean2d_backward(z["d_mean2d"][i], z["t_cam"][i], cam), z["dt_mean2d"][i])
        ds, dt = sg.cov2d_backward(z["d_cov2d"][i], z["T_proj"][i], z["sigma"][i], z["J"][i], z["Rcw"][i],
                                   z["t_cam"][i], cam)
        close(ds, z["d_sigma"][i])
        close(dt, z["dt_cov2d"][i])
        dm, dv = sg.world_backward(z["d_t_total"][i], cam, z["mean"][i])
        close(dm, z["d_mean"][i])
        close(dv, z["d_view"][i])
        dq, dsc = sg.covariance3d_backward(z["dS"][i], b, z["quat"][i], z["scale"][i])
        close(dq, z["d_quat"][i])
        close(dsc, z["d_scale"][i])
        assert abs(sg.frobenius_inner(z["frob_x"][i], z["frob_y"][i]) - z["frob"][i]) <= 1e-12 * (1 + abs(z["frob"][i]))


def test_helper_kats_and_errors(cuda):
    """Known answers of the reference's tests, restated (not copied): identity
    quaternion -> I; scaled quaternions give the same R; optical axis maps to
    (0.5, 0.5) + principal point; radius of diag(1,1)+0.3 -> ceil(3 sqrt 1.3);
    d_scale = (2,2,2) for identity R, S = I and d_sigma = I; dq orthogonal to q;
    and the reference's ValueError texts."""
    import paper_2312_02121_b200 as sg
    np.testing.assert_allclose(sg.quat_to_rotmat([1, 0, 0, 0]), np.eye(3), atol=1e-15)
    q = np.array([0.3, -0.5, 0.2, 0.8])
    np.testing.assert_allclose(sg.quat_to_rotmat(q), sg.quat_to_rotmat(7.5 * q), atol=1e-14)
    R = sg.quat_to_rotmat(q)
    np.testing.assert_allclose(R @ R.T, np.eye(3), atol=1e-14)
    cam = sg.Camera(view=np.eye(4), fx=50.0, fy=60.0, cx=3.0, cy=4.0, width=64, height=48, near=0.1, far=100.0)
    np.testing.assert_allclose(sg.camera_to_pixel(np.array([0.0, 0.0, 2.0, 1.0]), cam), [3.5, 4.5], atol=1e-12)
    assert sg.bounding_radius(np.eye(2) + 0.3 * np.eye(2)) == int(np.ceil(3 * np.sqrt(1.3)))
    b = sg.compose_covariance_3d([1, 0, 0, 0], [1, 1, 1])
    dq, ds = sg.covariance3d_backward(np.eye(3), b, [1, 0, 0, 0], [1, 1, 1])
    np.testing.assert_allclose(ds, [2, 2, 2], atol=1e-12)
    dq, _ = sg.covariance3d_backward(np.arange(9.0).reshape(3, 3), sg.compose_covariance_3d(q, [0.2, 0.5, 1.0]), q,
                                     [0.2, 0.5, 1.0])
    assert abs(np.dot(dq, q)) < 1e-12 * np.linalg.norm(dq) * np.linalg.norm(q) + 1e-15
    _, dv = sg.world_backward(np.array([1.0, 2.0, 3.0, 4.0]), cam, [0.5, 0.5, 0.5])
    np.testing.assert_allclose(dv[3], np.outer([1, 2, 3, 4], [0.5, 0.5, 0.5, 1])[3])
    with pytest.raises(ValueError, match="quaternion norm is too small"):
        sg.quat_to_rotmat([0, 0, 0, 0])
    with pytest.raises(ValueError, match="quat must have shape"):
        sg.quat_to_rotmat([1, 0, 0])
    with pytest.raises(ValueError, match="scale components must be positive"):
        sg.compose_covariance_3d([1, 0, 0, 0], [1, 0, 1])
    with pytest.raises(ValueError, match="point is behind the camera"):
        sg.projection_jacobian([0, 0, -1.0, 1], cam)
    with pytest.raises(ValueError, match="degenerate projection"):
        sg.camera_to_pixel([0, 0, 0.0, 1], cam)
    with pytest.raises(ValueError, match="2d covariance must be positive definite"):
        sg.bounding_radius(np.zeros((2, 2)))
    with pytest.raises(ValueError, match="shape mismatch"):
        sg.frobenius_inner(np.zeros(3), np.zeros(4))
