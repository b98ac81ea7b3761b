"""CPU: the C-ABI library builds, loads and exports every declared symbol."""

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "splat_b200.h")


def header_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(gs_[a-z0-9_]+)\s*\(", src)))


def test_header_lists_exports():
    from paper_2312_02121_b200 import _lib
    assert header_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_symbol():
    from paper_2312_02121_b200 import _lib
    L = _lib.load()
    for name in header_symbols():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for name in header_symbols():
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_host_only_entry_points():
    from paper_2312_02121_b200 import _lib
    L = _lib.load()
    assert L.gs_version() == 1
    assert L.gs_scan_workspace_bytes(0) >= 16
    assert L.gs_scan_workspace_bytes(10_000_000) > L.gs_scan_workspace_bytes(10)
    assert L.gs_sort_workspace_bytes(1_000_000, 44) > 0
    assert L.gs_project_bwd_workspace_bytes(1000) >= 4 * 12 * 4


def test_set_option():
    from paper_2312_02121_b200 import _lib, ops
    for v in (1, 2, 3, 0):
        ops.set_option("binning", v)
        assert ops.get_option("binning") == v
    for v in (0, 1):
        ops.set_option("fuse_sort", v)
        assert ops.get_option("fuse_sort") == v
    for v in (0, 1):
        ops.set_option("tile_emit", v)
        assert ops.get_option("tile_emit") == v
    with pytest.raises(_lib.SplatLibError, match="binning"):
        ops.set_option("binning", 7)
    L = _lib.load()
    assert L.gs_frame_binning(100000, 800, 800) == 3  # auto: direct (2500 tiles)
    assert L.gs_frame_binning(100000, 1920, 1080) == 2  # 8160 tiles: scatter
    assert L.gs_frame_binning(1000000, 800, 800) == 1  # large scene: depth-first
    assert L.gs_frame_tile_emit(1000000, 800, 800) == 1  # ... with the tile-sorted emission (2500 tiles)
    assert L.gs_frame_tile_emit(1000000, 3840, 2160) == 0  # 32400 tiles: emission + onesweep by tile
    assert L.gs_frame_tile_emit(100000, 800, 800) == 0  # direct binning
    with pytest.raises(_lib.SplatLibError, match="fuse_sort"):
        ops.set_option("fuse_sort", 2)
    with pytest.raises(_lib.SplatLibError, match="unknown option"):
        ops.set_option("no_such_option", 1)
    with pytest.raises(_lib.SplatLibError, match="unknown option"):
        ops.get_option("no_such_option")
    L = _lib.load()
    assert L.gs_bin64_workspace_bytes(1000, 5000, 256) > 0
    assert L.gs_project64_bwd_workspace_bytes(1000) > 0


def test_kernels_are_sm100a():
    from paper_2312_02121_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out, out


def test_product_path_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2312_02121_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), f
                assert "splat_oracle" not in txt, f


def test_package_exports_the_reference_api():
    """Every name of the reference's sg/__init__.py:64-119 __all__ resolves
    on the package (lazily; device calls need a GPU, resolution does not)."""
    import paper_2312_02121_b200 as sg
    ref = ["ALPHA_MAX", "ALPHA_MIN", "AUDIT_CLASSES", "Camera", "ClassCheck", "Cov3DBundle", "DILATION", "FitConfig",
           "Gaussian3D", "GradReport", "ImageBuffer", "ProjectedGaussian", "RenderAux", "RenderResult", "SIGMA_CUT",
           "SceneGradients", "Splat2DGrads", "TILE_SIZE", "T_MIN", "TileGrid", "accumulate_image_backward",
           "assign_tiles", "audit_scene", "bounding_radius", "camera_to_pixel", "compose_covariance_3d",
           "composite_pixel", "composite_pixel_backward", "cov2d_backward", "covariance3d_backward", "eval_alpha",
           "finite_difference", "fit", "frobenius_inner", "init_random", "main", "make_audit_scene",
           "mean2d_backward", "parse_scene", "project_covariance", "project_gaussian", "projection_jacobian",
           "quat_to_rotmat", "read_image", "render", "render_brute_force", "run_audit", "scene_backward",
           "serialize_scene", "sort_bins", "transmittance_replay", "world_backward", "world_to_camera",
           "write_image"]
    assert sorted(sg.__all__) == sorted(ref)
    for name in ref:
        assert getattr(sg, name) is not None, name
    assert callable(sg.fit) and callable(sg.main) and sg.TILE_SIZE == 16 and sg.SIGMA_CUT == 4.5
