"""GPU: the float64 path (csrc/f64.cu) against the
fp64 oracle and the reference's golden vectors: projection, bins (exact),
image / final_T / n_contrib and every gradient class to ~1e-10 relative
(both sides compute the reference's fp64 expressions; differences are
rounding and summation order)."""

import numpy as np
import pytest
import torch

import oracle as O
from parity import golden_names, load_golden

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    s = np.max(np.abs(b)) if b.size else 0.0
    return float(np.max(np.abs(a - b)) / s) if s > 0 else float(np.max(np.abs(a)) if a.size else 0.0)


@pytest.mark.parametrize("name", golden_names())
def test_f64_frame_matches_reference(name, cuda):
    from paper_2312_02121_b200 import f64
    g = load_golden(name)
    t = [torch.as_tensor(np.asarray(a, np.float64), device=cuda) for a in g["inputs"]]
    fr = f64.render64(*t, g["camera"], g["background"], g["et"])
    torch.cuda.synchronize()
    vis = np.nonzero(fr.tiles.cpu().numpy() > 0)[0]
    assert np.array_equal(vis, g["proj_source"])
    assert np.array_equal(fr.radius.cpu().numpy()[vis], g["proj_radius"])
    if len(vis):
        assert _rel(fr.mean2d.cpu().numpy()[vis], g["proj_mean2d"]) < 1e-12
        assert _rel(fr.cov3.cpu().numpy()[vis], g["proj_cov2d"].reshape(-1, 4)[:, [0, 1, 3]]) < 1e-12
    # bins: identical lists (scene indices) to the reference's
    ptr, idx = g["bin_ptr"], g["bin_idx"]
    bins = fr.bins()
    assert [b for b in bins] == [idx[ptr[k]:ptr[k + 1]].tolist() for k in range(len(ptr) - 1)]
    assert np.array_equal(fr.n_contrib.cpu().numpy(), g["n_contrib"])
    assert _rel(fr.image.cpu().numpy(), g["image"]) < 1e-12
    assert _rel(fr.final_T.cpu().numpy(), g["final_T"]) < 1e-12
    d = torch.as_tensor(np.asarray(g["d_image"], np.float64), device=cuda)
    gr = f64.backward64(fr, *t, d)
    for key in ("d_color", "d_opacity", "d_mean2d", "d_cov2d"):
        assert _rel(gr[key].cpu().numpy(), g["s_" + key]) < 1e-10, key
    for key in ("d_mean", "d_scale", "d_quat", "d_opacity", "d_color", "d_view"):
        assert _rel(gr[key].cpu().numpy(), g["g_" + key]) < 1e-10, key


def test_f64_errors_like_reference(cuda):
    from paper_2312_02121_b200 import f64
    g = load_golden("config0")
    t = [torch.as_tensor(np.asarray(a, np.float64), device=cuda) for a in g["inputs"]]
    t[1] = -t[1]
    with pytest.raises(ValueError, match="scale"):
        f64.render64(*t, g["camera"], g["background"])
