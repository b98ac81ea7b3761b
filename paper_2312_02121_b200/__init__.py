"""B200-native (sm_100a) differentiable Gaussian-splatting hot path.

Drop-in for the reference `splatgrad` render path (project -> tile-bin/sort
-> rasterize forward -> rasterize backward -> projection backward).  Kernels
live in libsplat_b200.so (csrc/, C ABI in include/splat_b200.h); this package
is the host side: `ops` (device pipeline + torch.autograd.Function),
`engine` (captured multi-view steps), `dist` (multi-GPU), and the
reference's public API: every name of sg/__init__.py:64-119 resolves here
(`import paper_2312_02121_b200 as sg; sg.render(...)`), loaded lazily from

  api       render, scene_backward, ... and the value types
  helpers   the per-splat float64 helpers (quat_to_rotmat, cov2d_backward, ...)
  gradcheck finite-difference audit;  fitting  the training loop;  cli  formats + CLI
"""

__version__ = "0.1.0"

_SOURCES = {
    "api": ("ALPHA_MAX", "ALPHA_MIN", "DILATION", "SIGMA_CUT", "TILE_SIZE", "T_MIN", "Camera", "Gaussian3D",
            "ImageBuffer", "ProjectedGaussian", "RenderAux", "RenderResult", "SceneGradients", "Splat2DGrads",
            "TileGrid", "accumulate_image_backward", "assign_tiles", "composite_pixel", "composite_pixel_backward",
            "eval_alpha", "project_gaussian", "render", "render_brute_force", "scene_backward", "sort_bins",
            "transmittance_replay"),
    "helpers": ("Cov3DBundle", "bounding_radius", "camera_to_pixel", "compose_covariance_3d", "cov2d_backward",
                "covariance3d_backward", "frobenius_inner", "mean2d_backward", "project_covariance",
                "projection_jacobian", "quat_to_rotmat", "world_backward", "world_to_camera"),
    "gradcheck": ("AUDIT_CLASSES", "ClassCheck", "GradReport", "audit_scene", "finite_difference",
                  "make_audit_scene", "run_audit"),
    "fitting": ("FitConfig", "fit", "init_random"),
    "cli": ("main", "parse_scene", "read_image", "serialize_scene", "write_image"),
}
_WHERE = {name: mod for mod, names in _SOURCES.items() for name in names}

# the reference's sg/__init__.py:64-119 __all__, name for name
__all__ = sorted(_WHERE)


def __getattr__(name):
    mod = _WHERE.get(name)
    if mod is None:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
    import importlib
    value = getattr(importlib.import_module(f".{mod}", __name__), name)
    globals()[name] = value
    return value


def __dir__():
    return sorted(set(globals()) | set(_WHERE))
