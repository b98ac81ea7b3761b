"""Seeded synthetic scenes for BASELINE.json configs 0-4 (host side, numpy).

The reference publishes no dataset; BASELINE.json describes five synthetic
scenes by their distributions.  This module restates those descriptions with
the conventions SURVEY.md §8(d) fixes where BASELINE is silent:

* one ``np.random.default_rng(config_id)`` per config, draw order
  means -> scales -> quats -> opacity -> color -> camera(s) -> dL/dC;
* generated in fp64 and rounded to fp32 (the GPU sees fp32, the oracle sees
  ``fp64(fp32(x))`` so both sides start from identical values);
* quaternions are N(0, I4) / |.| stored (w, x, y, z) like the reference
  (``sg/core.py:146-171``); opacity is the raw [0, 1] value the reference
  consumes (no activation inside the path, ``sg/raster_forward.py:111``);
* look-at cameras: z = normalize(target - C), x = normalize(up x z) with
  up = (0, 1, 0), y = z x x, rows of R = [x; y; z], t = -R C.  Config 0's
  camera at (0, 0, -4) is then exactly the identity rotation.

These are interpretation, not reference content.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

NEAR = 0.01
FAR = 100.0


@dataclass
class CameraSpec:
    """Pinhole camera in the reference's convention (``sg/core.py:59-111``)."""

    view: np.ndarray  # (4, 4) float64 world -> camera (values are fp32-exact)
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    near: float = NEAR
    far: float = FAR


@dataclass
class SceneSpec:
    """Gaussian parameters as fp32 SoA arrays plus one or more cameras."""

    name: str
    means: np.ndarray      # (N, 3) float32
    scales: np.ndarray     # (N, 3) float32, > 0
    quats: np.ndarray      # (N, 4) float32, (w, x, y, z), unnormalised allowed
    opacities: np.ndarray  # (N,)  float32 in [0, 1]
    colors: np.ndarray     # (N, 3) float32 in [0, 1]
    cameras: list = field(default_factory=list)
    background: np.ndarray = field(default_factory=lambda: np.zeros(3, np.float32))
    d_images: list = field(default_factory=list)  # per camera (H, W, 3) float32

    @property
    def n(self) -> int:
        return int(self.means.shape[0])


def _f32(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64).astype(np.float32))


def look_at(center, target=(0.0, 0.0, 0.0), up=(0.0, 1.0, 0.0)) -> np.ndarray:
    """World-to-camera 4x4 for a camera at ``center`` looking at ``target``.

    The result is rounded through fp32 so the GPU (fp32) and the oracle (fp64)
    consume the same matrix.  Rotation rows are re-orthonormalised in fp64
    after rounding would break ``Camera.validate``'s 1e-9 check, so callers that
    validate use :func:`validated_view`.
    """
    c = np.asarray(center, dtype=np.float64)
    z = np.asarray(target, dtype=np.float64) - c
    z = z / np.linalg.norm(z)
    x = np.cross(np.asarray(up, dtype=np.float64), z)
    x = x / np.linalg.norm(x)
    y = np.cross(z, x)
    view = np.eye(4)
    view[0, :3], view[1, :3], view[2, :3] = x, y, z
    view[:3, 3] = -view[:3, :3] @ c
    return view.astype(np.float32).astype(np.float64)


def _random_direction(rng, up=(0.0, 1.0, 0.0)):
    upv = np.asarray(up)
    while True:
        d = rng.normal(size=3)
        d = d / np.linalg.norm(d)
        if abs(float(d @ upv)) <= 0.99:
            return d


def _sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def _unit_quats(rng, n):
    q = rng.normal(size=(n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def _clustered_means(rng, n, k=64, box=3.0, std_lo=0.05, std_hi=0.5):
    centers = rng.uniform(-box, box, size=(k, 3))
    stds = rng.uniform(std_lo, std_hi, size=(k, 3))
    assign = rng.integers(0, k, size=n)
    return centers[assign] + stds[assign] * rng.normal(size=(n, 3))


def make_config(config_id: int, *, n_override: int | None = None,
                n_views: int | None = None, with_grads: bool = True) -> SceneSpec:
    """Build BASELINE.json ``configs[config_id]`` (0..4).

    ``n_override`` shrinks the Gaussian count with the same distributions
    (used for quick tests); ``n_views`` trims config 3's 32-camera ring.
    """
    rng = np.random.default_rng(config_id)
    if config_id == 0:
        n = n_override or 10_000
        means = rng.uniform(-1.0, 1.0, size=(n, 3))
        scales = np.exp(rng.uniform(np.log(0.005), np.log(0.05), size=(n, 3)))
        quats = _unit_quats(rng, n)
        opac = _sigmoid(rng.normal(0.0, 1.0, size=n))
        colors = rng.uniform(0.0, 1.0, size=(n, 3))
        cams = [CameraSpec(look_at((0.0, 0.0, -4.0)), 256.0, 256.0, 128.0, 128.0, 256, 256)]
    elif config_id == 1:
        n = n_override or 100_000
        means = rng.uniform(-1.5, 1.5, size=(n, 3))
        scales = np.exp(rng.uniform(np.log(0.003), np.log(0.03), size=(n, 3)))
        quats = _unit_quats(rng, n)
        opac = _sigmoid(rng.normal(0.0, 1.0, size=n))
        colors = rng.uniform(0.0, 1.0, size=(n, 3))
        d = _random_direction(rng)
        cams = [CameraSpec(look_at(4.0 * d), 1100.0, 1100.0, 400.0, 400.0, 800, 800)]
    elif config_id in (2, 3):
        n = n_override or (1_000_000 if config_id == 2 else 3_000_000)
        means = _clustered_means(rng, n)
        scales = np.exp(rng.normal(np.log(0.01), 0.5, size=(n, 3)))
        quats = _unit_quats(rng, n)
        opac = _sigmoid(rng.normal(1.0, 1.0, size=n))
        colors = rng.uniform(0.0, 1.0, size=(n, 3))
        if config_id == 2:
            cams = [CameraSpec(look_at((0.0, 0.0, -8.0)), 1500.0, 1500.0, 960.0, 540.0, 1920, 1080)]
        else:
            nv = n_views or 32
            heights = rng.uniform(-1.0, 1.0, size=32)
            cams = []
            for k in range(nv):
                th = 2.0 * np.pi * k / 32.0
                c = (6.0 * np.cos(th), heights[k], 6.0 * np.sin(th))
                cams.append(CameraSpec(look_at(c), 1150.0, 1150.0, 648.5, 420.0, 1297, 840))
    elif config_id == 4:
        n = n_override or 6_000_000
        means = rng.uniform(-4.0, 4.0, size=(n, 3))
        scales = np.exp(rng.normal(np.log(0.008), 0.6, size=(n, 3)))
        quats = _unit_quats(rng, n)
        opac = _sigmoid(rng.normal(0.0, 1.5, size=n))
        colors = rng.uniform(0.0, 1.0, size=(n, 3))
        cams = [CameraSpec(look_at((0.0, 0.0, -10.0)), 3000.0, 3000.0, 1920.0, 1080.0, 3840, 2160)]
    else:
        raise ValueError(f"unknown config {config_id}")
    spec = SceneSpec(
        name=f"config{config_id}", means=_f32(means), scales=_f32(scales),
        quats=_f32(quats), opacities=_f32(opac), colors=_f32(colors), cameras=cams,
    )
    if with_grads:
        spec.d_images = [_f32(rng.normal(size=(c.height, c.width, 3))) for c in cams]
    return spec


def config_sizes(config_id: int) -> dict:
    """Static description used in bench/config JSON."""
    table = {
        0: dict(gaussians=10_000, width=256, height=256, views=1),
        1: dict(gaussians=100_000, width=800, height=800, views=1),
        2: dict(gaussians=1_000_000, width=1920, height=1080, views=1),
        3: dict(gaussians=3_000_000, width=1297, height=840, views=32),
        4: dict(gaussians=6_000_000, width=3840, height=2160, views=1),
    }
    return dict(table[config_id])
