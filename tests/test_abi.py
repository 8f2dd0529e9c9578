"""The C-ABI library loads and exports every symbol include/fgs.h declares (CPU, no compute).

Also checks the pure-host entry points: workspace sizing and synchronous argument
validation (FGS_E_INVALID before any CUDA call), and that the ctypes struct
layouts match the header's field order/sizes.
"""
import ctypes
import os
import re

import pytest

from paper_2310_08528_b200 import build, fgs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fgs.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(fgs_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def L():
    build.build()
    return fgs.lib()


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("fgs_deform", "fgs_render", "fgs_deform_range", "fgs_render_batch", "fgs_render_status",
                 "fgs_render_workspace_bytes", "fgs_last_error"):
        assert must in names
    assert set(names) == set(fgs.EXPORTS)


def test_library_exports_every_declared_symbol(L):
    for name in declared_functions():
        assert hasattr(L, name), name


def test_version_and_error_strings(L):
    assert "sm_100a" in fgs.fgs_version()
    assert isinstance(fgs.fgs_last_error(), str)


def test_workspace_bytes_host_only(L):
    a = fgs.fgs_render_workspace_bytes(1000, 64, 64, 16000)
    b = fgs.fgs_render_workspace_bytes(1000, 64, 64, 32000)
    assert a > 0 and b > a and a % 256 == 0
    assert fgs.fgs_render_workspace_bytes(-1, 64, 64, 10) == 0
    assert fgs.fgs_render_workspace_bytes(10, 0, 64, 10) == 0


def test_validation_rejects_before_cuda(L):
    g = fgs.fgs_gaussians(10, 5, 0, 0, 0, 0, 0)          # sh_degree 5 is invalid
    rc = L.fgs_deform(ctypes.byref(g), None, None, ctypes.c_float(0.5), None, None)
    assert rc == fgs.FGS_E_INVALID and "sh_degree" in fgs.fgs_last_error()
    rc = L.fgs_deform(None, None, None, ctypes.c_float(0.5), None, None)
    assert rc == fgs.FGS_E_INVALID
    cam = fgs.fgs_camera()
    cam.width, cam.height, cam.fx, cam.fy = 0, 10, 1.0, 1.0
    d = fgs.fgs_deformed(0, 0, 0, 0, 0, 0, 0)
    img = ctypes.c_void_p(16)
    rc = L.fgs_render(ctypes.byref(cam), ctypes.byref(d), img, ctypes.c_void_p(256), 1 << 20, None)
    assert rc == fgs.FGS_E_INVALID and "image size" in fgs.fgs_last_error()
    rc = L.fgs_render_status(None, 0, 1, None)
    assert rc == fgs.FGS_E_INVALID


def test_struct_layouts():
    assert ctypes.sizeof(fgs.fgs_gaussians) == 8 + 8 + 5 * 8
    assert ctypes.sizeof(fgs.fgs_camera) == 4 * (9 + 3 + 4 + 2 + 3)
    assert fgs.fgs_hexplanes.planes.offset == 56
    assert ctypes.sizeof(fgs.fgs_render_aux) == 15 * 8
    assert ctypes.sizeof(fgs.fgs_mlp) == 8 + 12 * 8


def test_tuning_knob_host_only(L):
    cap0 = fgs.fgs_get_tuning(fgs.FGS_TUNE_TILE_SORT_CAP)
    assert cap0 == 1024
    fgs.fgs_set_tuning(fgs.FGS_TUNE_TILE_SORT_CAP, 64)
    assert fgs.fgs_get_tuning(fgs.FGS_TUNE_TILE_SORT_CAP) == 64
    fgs.fgs_set_tuning(fgs.FGS_TUNE_TILE_SORT_CAP, cap0)
    assert L.fgs_set_tuning(fgs.FGS_TUNE_TILE_SORT_CAP, 0) == fgs.FGS_E_INVALID
    assert L.fgs_set_tuning(fgs.FGS_TUNE_TILE_SORT_CAP, 4096) == fgs.FGS_E_INVALID
    assert L.fgs_set_tuning(99, 1) == fgs.FGS_E_INVALID
    assert fgs.fgs_get_tuning(99) == -1
    assert fgs.fgs_get_tuning(fgs.FGS_TUNE_BLEND_CULL) == 1
    with fgs.tuning(fgs.FGS_TUNE_BLEND_CULL, 0):
        assert fgs.fgs_get_tuning(fgs.FGS_TUNE_BLEND_CULL) == 0
    assert fgs.fgs_get_tuning(fgs.FGS_TUNE_BLEND_CULL) == 1
    assert L.fgs_set_tuning(fgs.FGS_TUNE_BLEND_CULL, 2) == fgs.FGS_E_INVALID
    assert fgs.fgs_get_tuning(fgs.FGS_TUNE_TILE_CULL) == 0
    with fgs.tuning(fgs.FGS_TUNE_TILE_CULL, 1):
        assert fgs.fgs_get_tuning(fgs.FGS_TUNE_TILE_CULL) == 1
    assert fgs.fgs_get_tuning(fgs.FGS_TUNE_TILE_CULL) == 0
    assert L.fgs_set_tuning(fgs.FGS_TUNE_TILE_CULL, 2) == fgs.FGS_E_INVALID
    assert fgs.fgs_get_tuning(fgs.FGS_TUNE_AGG_TILES) == 4096
    with fgs.tuning(fgs.FGS_TUNE_AGG_TILES, 1):
        assert fgs.fgs_get_tuning(fgs.FGS_TUNE_AGG_TILES) == 1
    assert fgs.fgs_get_tuning(fgs.FGS_TUNE_AGG_TILES) == 4096
    assert L.fgs_set_tuning(fgs.FGS_TUNE_AGG_TILES, 0) == fgs.FGS_E_INVALID
    assert L.fgs_set_tuning(fgs.FGS_TUNE_AGG_TILES, 4097) == fgs.FGS_E_INVALID
    assert L.fgs_set_tuning(1, 0) == fgs.FGS_E_INVALID          # retired key (single deform kernel)
    assert fgs.fgs_get_tuning(fgs.FGS_TUNE_RADIX) == 0 and fgs.fgs_get_tuning(fgs.FGS_TUNE_RADIX_MIN_LIST) == 768
    with fgs.tuning(fgs.FGS_TUNE_RADIX, 2):
        assert fgs.fgs_get_tuning(fgs.FGS_TUNE_RADIX) == 2
    assert L.fgs_set_tuning(fgs.FGS_TUNE_RADIX, 3) == fgs.FGS_E_INVALID
    assert L.fgs_set_tuning(fgs.FGS_TUNE_RADIX_MIN_LIST, 0) == fgs.FGS_E_INVALID
    assert fgs.fgs_get_tuning(fgs.FGS_TUNE_LONG_SORT) == 1
    with fgs.tuning(fgs.FGS_TUNE_LONG_SORT, 0):
        assert fgs.fgs_get_tuning(fgs.FGS_TUNE_LONG_SORT) == 0
    assert fgs.fgs_get_tuning(fgs.FGS_TUNE_LONG_SORT) == 1
    assert L.fgs_set_tuning(fgs.FGS_TUNE_LONG_SORT, 2) == fgs.FGS_E_INVALID


def test_stage_names_match_header():
    src = open(HEADER).read()
    stages = re.findall(r"FGS_STAGE_(\w+) ?=?", src)
    stages = [s for i, s in enumerate(stages) if s not in stages[:i]]
    assert [s.lower() for s in stages] == list(fgs.STAGES)
