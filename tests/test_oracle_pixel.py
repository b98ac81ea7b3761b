"""CPU: pin the oracle's per-pixel restatement (eval_alpha, composite_pixel,
composite_pixel_backward, transmittance_replay) against golden vectors made
by the reference itself (tests/golden/make_golden_pixel.py)."""

import numpy as np

import oracle as O
from parity import load_pixel_golden


def _q(z, q):
    sl = slice(int(z["bin_ptr"][q]), int(z["bin_ptr"][q + 1]))
    return np.array([0, sl.stop - sl.start]), z["bin_idx"][sl]


def test_eval_alpha_matches_reference():
    z = load_pixel_golden()
    n = len(z["ea_opacity"])
    out = O.eval_alpha(np.arange(n), z["ea_pix"], z["ea_mean2d"], z["ea_cov3"], z["ea_opacity"])
    ref = z["ea_out"]
    assert np.array_equal(out[:, 0] == 0, ref[:, 0] == 0)
    np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-15)


def test_composite_pixel_matches_reference():
    z = load_pixel_golden()
    o = O.composite_pixels(z["bin_ptr"], z["bin_idx"], z["q_pix"], z["q_et"], z["mean2d"], z["cov3"],
                           z["p_opacity"], z["p_color"], z["background"])
    assert np.array_equal(o["n_contrib"], z["q_nc"])
    np.testing.assert_allclose(o["color"], z["q_color"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(o["final_T"], z["q_T"], rtol=1e-12, atol=1e-300)
    # the fixture exercises every branch: empty bins, early stop, no early stop
    assert (np.diff(z["bin_ptr"]) == 0).any() and (z["q_nc"] > 0).any()
    assert (z["q_T"] < 1e-3).any() and (z["q_et"] == 0).any()


def test_composite_pixel_backward_and_replay_match_reference():
    z = load_pixel_golden()
    src = z["source_index"]
    n_q = len(z["q_T"])
    for q in range(n_q):
        ptr, idx = _q(z, q)
        b = O.composite_pixels_bwd(ptr, idx, z["q_pix"][q:q + 1], z["mean2d"], z["cov3"], z["p_opacity"],
                                   z["p_color"], z["background"], z["q_T"][q:q + 1], z["q_nc"][q:q + 1],
                                   z["d_pix"][q:q + 1], t_log=True)
        d9 = np.zeros_like(b["d9"])
        d9[src] = b["d9"]  # projected row j -> scene row src[j]
        cov = np.stack([d9[:, 6], d9[:, 7], d9[:, 7], d9[:, 8]], 1).reshape(-1, 2, 2)
        for got, ref in ((d9[:, :3], z["g_color"][q]), (d9[:, 3], z["g_opacity"][q]),
                         (d9[:, 4:6], z["g_mean2d"][q]), (cov, z["g_cov2d"][q])):
            np.testing.assert_allclose(got, ref, rtol=1e-10, atol=1e-12 * max(1.0, np.abs(ref).max()))
        t = b["t_log"]
        pairs = [(p, t[p]) for p in range(len(t) - 1, -1, -1) if np.isfinite(t[p])]
        r = slice(int(z["r_ptr"][q]), int(z["r_ptr"][q + 1]))
        assert [p for p, _ in pairs] == z["r_pos"][r].tolist()
        np.testing.assert_allclose([v for _, v in pairs], z["r_T"][r], rtol=1e-12)
