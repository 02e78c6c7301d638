"""CPU-side checks of the C-ABI boundary (-m "not gpu"): the library builds for
sm_100a, loads without a GPU, exports every symbol include/csplat.h declares,
and rejects invalid arguments before touching the device."""
import ctypes as C
import math
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "csplat.h")


@pytest.fixture(scope="module")
def cs():
    from paper_2403_11247_b200 import _build, csplat
    _build.build()
    return csplat


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)          # drop comments
    return sorted(set(re.findall(r"^(?:int|size_t|const char\s*\*)\s*(csplat_[a-z_0-9]+)\s*\(",
                                 text, flags=re.M)))


def test_header_declares_the_six_entry_points():
    syms = declared_symbols()
    for s in ("csplat_project", "csplat_bin_tiles", "csplat_render_fwd", "csplat_render_bwd",
              "csplat_rvq_assign", "csplat_mask_prune"):
        assert s in syms


def test_library_exports_every_declared_symbol(cs):
    L = cs.lib()
    for s in declared_symbols():
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", cs.LIB_PATH], capture_output=True,
                         text=True).stdout
    for s in declared_symbols():
        assert re.search(r"\bT " + s + r"\b", out), s


def test_library_is_sm100a(cs):
    out = subprocess.run(["cuobjdump", "--list-elf", cs.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", cs.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "UBLKCP" in sass            # TMA bulk copies (R-VQ codebook staging)
    assert "UTMALDG.2D.GATHER4" in sass  # the renderers' tile::gather4 record loads
    assert "REDG.E.ADD.F32x4" in sass  # vector reductions in the backward


def test_version_and_strings(cs):
    L = cs.lib()
    assert L.csplat_version() >> 16 == 2
    assert L.csplat_status_string(0) == b"ok"
    assert L.csplat_status_string(3) == b"pair capacity exceeded"


def test_invalid_arguments_rejected_without_device(cs):
    L = cs.lib()
    cam = cs.camera(dict(fx=10, fy=10, cx=5, cy=5, width=16, height=16))
    bad = cs.camera(dict(fx=-1, fy=10, cx=5, cy=5, width=16, height=16))
    v, p = cs.view([1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0]), cs.params()
    g = cs.Gaussians(-1, None, None, None, None, None, None, None)
    assert L.csplat_project(C.byref(g), None, C.byref(cam), C.byref(v), C.byref(p), None, None,
                            None) == 1
    g0 = cs.Gaussians(0, None, None, None, None, None, None, None)
    assert L.csplat_project(C.byref(g0), None, C.byref(bad), C.byref(v), C.byref(p), None, None,
                            None) == 1
    assert L.csplat_rvq_assign(None, 10, None, 9, None, 1, 1, None, 1, None, None) == 1
    assert L.csplat_rvq_assign(None, 10, None, 3, None, 1, 300, None, 1, None, None) == 1
    assert L.csplat_rvq_assign(None, 10, None, 3, None, 17, 4, None, 1, None, None) == 1
    # misaligned record buffer
    g1 = cs.Gaussians(1, None, C.c_void_p(16), C.c_void_p(32), C.c_void_p(48), C.c_void_p(64),
                      C.c_void_p(80), C.c_void_p(96))
    assert L.csplat_project(C.byref(g1), None, C.byref(cam), C.byref(v), C.byref(p),
                            C.c_void_p(8), C.c_void_p(16), None) == 2
    # workspace too small
    assert L.csplat_bin_tiles(None, None, 0, C.byref(cam), 0, None, C.c_void_p(16),
                              C.c_void_p(16), 0, None, 0, None) == 4
    need = L.csplat_workspace_bytes(1, 100, 1000, C.byref(cam))
    assert need >= 8 * 1000
    assert L.csplat_workspace_bytes(2, 100, 0, None) >= 100 * 48 + 4 * 4
    assert L.csplat_workspace_bytes(2, 100, 0, None) % 256 == 0
    assert L.csplat_workspace_bytes(3, 100, 0, None) > 0
    buf = C.create_string_buffer(256)
    assert L.csplat_last_error(buf, 256) > 0


def test_composed_entry_points_reject_invalid_arguments_without_device(cs):
    """csplat_project_bin(_dv), csplat_project_bin_render(_dv), csplat_render_step and
    csplat_tracking_step validate their arguments before touching the device."""
    L = cs.lib()
    cam = cs.camera(dict(fx=10, fy=10, cx=5, cy=5, width=16, height=16))
    v, p = cs.view([1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0]), cs.params()
    gbad = cs.Gaussians(-1, None, None, None, None, None, None, None)
    g0 = cs.Gaussians(0, None, None, None, None, None, None, None)
    x = C.c_void_p(16)  # a non-NULL, 16-byte aligned placeholder (never dereferenced)
    gr = cs.Grads(*([None] * 7))
    # bad map / NULL view / NULL tile_range / small workspace
    assert L.csplat_project_bin(C.byref(gbad), None, C.byref(cam), C.byref(v), C.byref(p), x, x,
                                None, 0, None, x, x, 0, x, 1 << 20, None) == 1
    assert L.csplat_project_bin(C.byref(g0), None, C.byref(cam), None, C.byref(p), x, x,
                                None, 0, None, x, x, 0, x, 1 << 20, None) == 1
    assert L.csplat_project_bin_dv(C.byref(g0), None, C.byref(cam), None, C.byref(p), x, x,
                                   None, 0, None, x, x, 0, x, 1 << 20, None) == 1
    assert L.csplat_project_bin(C.byref(g0), None, C.byref(cam), C.byref(v), C.byref(p), x, x,
                                None, 0, None, None, x, 0, x, 1 << 20, None) == 1
    assert L.csplat_project_bin(C.byref(g0), None, C.byref(cam), C.byref(v), C.byref(p), x, x,
                                None, 0, None, x, x, 0, x, 0, None) == 4
    # misaligned record buffer
    assert L.csplat_project_bin(C.byref(g0), None, C.byref(cam), C.byref(v), C.byref(p),
                                C.c_void_p(8), x, None, 4, x, x, x, 0, x, 1 << 20, None) == 2
    # render: NULL image
    assert L.csplat_project_bin_render(C.byref(g0), None, C.byref(cam), C.byref(v), C.byref(p),
                                       x, x, 0, None, x, x, x, 1 << 20, None, x, x, x, x,
                                       None) == 1
    assert L.csplat_project_bin_render_dv(C.byref(g0), None, C.byref(cam), None, C.byref(p),
                                          x, x, 0, None, x, x, x, 1 << 20, x, x, x, x, x,
                                          None) == 1
    # step: NULL upstream, POSE_ONLY rejected, small backward workspace
    step = lambda dC, flags, wsb: L.csplat_render_step(  # noqa: E731
        C.byref(g0), None, C.byref(cam), C.byref(v), C.byref(p), x, x, 0, None, x, x, x,
        1 << 20, x, x, x, x, x, dC, x, x, flags, C.byref(gr), x, wsb, None)
    assert step(None, 0, 1 << 20) == 1
    assert step(x, cs.POSE_ONLY, 1 << 20) == 1
    assert step(x, 0, 0) == 4
    # tracking step: both / neither view, NULL observations
    track = lambda hv, dv, obs: L.csplat_tracking_step(  # noqa: E731
        C.byref(g0), None, C.byref(cam), hv, dv, C.byref(p), x, x, 0, None, x, x, x,
        1 << 20, x, x, x, x, x, obs, x, x, 1.0, 0.99, cs.POSE_ONLY, C.byref(gr), x, x, 1 << 20,
        None)
    assert track(C.byref(v), x, x) == 1
    assert track(None, None, x) == 1
    assert track(C.byref(v), None, None) == 1
