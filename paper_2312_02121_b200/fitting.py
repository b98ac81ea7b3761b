"""Image fitting on the GPU path: sg/optimize.py (FitConfig, init_random, fit)
with every per-iteration array operation in CUDA kernels.

One iteration (sg/optimize.py:143-176): render (gs_frame_forward) -> L2
loss and d_image = 2 resid (gs_loss_l2) -> scene backward
(gs_frame_backward) -> chain to log-scale / logit space + Adam per class +
colour clip + activation for the next render (gs_adam_step).  Parameters,
Adam moments and the loss history stay on the device; the host reads one
16-byte meta word per iteration (status + intersection count, re-running the
iteration with a larger buffer if the capacity was too small) and the loss to
raise FloatingPointError like the reference (:159-160).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, api, ops
from ._lib import check


@dataclass
class FitConfig:
    """sg/optimize.py:16-33 (same fields and defaults)."""

    n_gaussians: int = 100
    iterations: int = 1000
    lr_mean: float = 2e-3
    lr_scale: float = 5e-3
    lr_quat: float = 2e-3
    lr_opacity: float = 2e-2
    lr_color: float = 1e-2
    seed: int = 0
    background: tuple = (0.0, 0.0, 0.0)
    loss: str = "l2"
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8


def init_random(config: FitConfig, camera, target):
    """sg/optimize.py:36-75: the same seeded draws in the same order (host
    set-up, not the hot path), returned as api.Gaussian3D."""
    rng = np.random.default_rng(config.seed)
    target = np.asarray(target, dtype=np.float64)
    depth_lo = camera.near + 2.0
    depth_hi = min(camera.far, depth_lo + 4.0)
    n = config.n_gaussians
    sigma_px = 0.5 * np.sqrt(camera.width * camera.height / n / np.pi) if n > 0 else 0.0
    view = np.asarray(camera.view, dtype=np.float64)
    R, t = view[:3, :3], view[:3, 3]
    scene = []
    for _ in range(n):
        px = rng.uniform(0.0, camera.width)
        py = rng.uniform(0.0, camera.height)
        depth = rng.uniform(depth_lo, depth_hi)
        t_cam = np.array([(px - 0.5 - camera.cx) * depth / camera.fx, (py - 0.5 - camera.cy) * depth / camera.fy,
                          depth])
        mean = R.T @ (t_cam - t)
        row = min(camera.height - 1, max(0, int(py)))
        col = min(camera.width - 1, max(0, int(px)))
        scene.append(api.Gaussian3D(mean=mean, scale=np.full(3, sigma_px * depth / camera.fx),
                                    quat=np.array([1.0, 0.0, 0.0, 0.0]), opacity=0.5, color=target[row, col].copy()))
    return scene


class GpuFit:
    """Device state of a fit: optimisation-space parameters, Adam moments,
    activated parameters and the per-iteration loss history."""

    def __init__(self, scene, camera, target, config: FitConfig, device=None):
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        self.cfg = config
        self.cam = ops.CameraParams.of(camera)
        n = len(scene)
        self.n = n
        f32 = lambda a: torch.as_tensor(np.ascontiguousarray(np.asarray(a, np.float64).astype(np.float32)),
                                        device=dev)
        self.means = f32(np.array([g.mean for g in scene]).reshape(n, 3))
        self.log_scales = f32(np.log(np.array([g.scale for g in scene]).reshape(n, 3)))
        self.quats = f32(np.array([g.quat for g in scene]).reshape(n, 4))
        op = np.clip(np.array([g.opacity for g in scene], np.float64), 1e-4, 1.0 - 1e-4)
        self.logits = f32(np.log(op) - np.log1p(-op))  # sg/optimize.py:92-93,132
        self.colors = f32(np.array([g.color for g in scene]).reshape(n, 3))
        self.scales = torch.empty_like(self.log_scales)
        self.opac = torch.empty_like(self.logits)
        self.m = torch.zeros((n, 14), device=dev, dtype=torch.float32)
        self.v = torch.zeros((n, 14), device=dev, dtype=torch.float32)
        self.target = f32(np.asarray(target, np.float64))
        self.d_image = torch.empty_like(self.target)
        self.losses = torch.zeros((max(config.iterations, 1),), device=dev, dtype=torch.float64)
        self.lrs = (C.c_float * 5)(config.lr_mean, config.lr_scale, config.lr_quat, config.lr_opacity,
                                   config.lr_color)
        self.bg = tuple(float(b) for b in config.background)
        self.capacity = None
        self.ws = None
        L = _lib.load()
        check(L.gs_activate(self.log_scales.data_ptr(), self.logits.data_ptr(), self.scales.data_ptr(),
                            self.opac.data_ptr(), n, ops._stream()), "gs_activate")

    def step(self, it: int) -> float:
        """One iteration; returns the loss measured before the update."""
        L = _lib.load()
        st = ops._stream()
        while True:
            fr = ops.frame_forward(self.means, self.scales, self.quats, self.opac, self.colors, self.cam, self.bg,
                                   True, capacity=self.capacity, check_meta=self.capacity is None, ws=self.ws)
            if self.capacity is None:  # first frame sized the buffers
                self.capacity = int(fr.needed_capacity * 1.5) + 4096
                self.ws = None
                continue
            meta = fr.meta().cpu()
            ops.raise_status(int(meta[0]))
            need = ops.needed_capacity(meta)
            if need <= self.capacity:
                self.ws = fr.ws
                break
            self.capacity = int(need * 1.5) + 4096
            self.ws = None
        loss_slot = self.losses[it:it + 1]
        check(L.gs_loss_l2(fr.image.data_ptr(), self.target.data_ptr(), self.target.numel(), self.d_image.data_ptr(),
                           loss_slot.data_ptr(), st), "gs_loss_l2")
        loss = float(loss_slot.item())
        if not np.isfinite(loss):
            raise FloatingPointError(f"loss diverged at iteration {it}")  # sg/optimize.py:159-160
        g = ops.frame_backward(fr, self.means, self.scales, self.quats, self.colors, self.d_image)
        check(L.gs_adam_step(self.means.data_ptr(), self.log_scales.data_ptr(), self.quats.data_ptr(),
                             self.logits.data_ptr(), self.colors.data_ptr(), self.scales.data_ptr(),
                             self.opac.data_ptr(), g["d_mean"].data_ptr(), g["d_scale"].data_ptr(),
                             g["d_quat"].data_ptr(), g["d_rgbo"].data_ptr(), self.m.data_ptr(), self.v.data_ptr(),
                             self.n, it + 1, self.lrs, self.cfg.beta1, self.cfg.beta2, self.cfg.eps, st),
              "gs_adam_step")
        return loss

    def scene(self):
        f = lambda t: t.detach().cpu().numpy().astype(np.float64)
        means, scales, quats, opac, colors = f(self.means), f(self.scales), f(self.quats), f(self.opac), f(self.colors)
        return [api.Gaussian3D(mean=means[i], scale=scales[i], quat=quats[i], opacity=opac[i], color=colors[i])
                for i in range(self.n)]


def fit(target, camera, config: FitConfig, init=None):
    """sg/optimize.py:96-190 on the GPU.  Returns (scene, loss_history)."""
    target = np.asarray(target, dtype=np.float64)
    if target.shape != (camera.height, camera.width, 3):
        raise ValueError(f"target shape {target.shape} does not match camera "
                         f"{(camera.height, camera.width, 3)}")
    if config.loss.lower() != "l2":
        raise ValueError(f"unsupported loss {config.loss!r}")
    scene = init_random(config, camera, target) if init is None else list(init)
    state = GpuFit(scene, camera, target, config)
    history = [state.step(it) for it in range(config.iterations)]
    return state.scene(), history
