"""CPU-side checks of the C-ABI library (no GPU needed): it loads, exports every symbol
include/gs.h declares, its defaults equal the method constants, and argument validation
fails before any device work."""
import ctypes as ct
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2409_06765_b200 import build
    build.build()
    from paper_2409_06765_b200 import _lib
    return _lib


def _declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "gs.h")).read()
    return sorted(set(re.findall(r"GS_API\s+[\w\s\*]+?\b(gs_\w+)\s*\(", hdr)))


def test_header_declares_the_four_stages():
    syms = _declared_symbols()
    for s in ["gs_project", "gs_isect_tiles", "gs_rasterize_fwd", "gs_rasterize_bwd", "gs_project_bwd"]:
        assert s in syms


def test_library_exports_every_declared_symbol(L):
    lib = L.lib()
    for s in _declared_symbols():
        assert hasattr(lib, s), s
        assert s in L.SIGNATURES, f"binding lacks {s}"


def test_defaults_match_oracle_constants(L):
    """Appendix B constants are duplicated (not shared) between the CUDA path and the
    oracle; this cross-check keeps the two tables equal."""
    import oracle
    o = L.options()
    r = oracle.Options()
    assert o.tile_size == r.tile_size == 16
    for k in ["near_plane", "far_plane", "eps2d", "alpha_max", "alpha_min", "t_min"]:
        assert np.float32(getattr(o, k)) == np.float32(getattr(r, k)), k
    assert o.fov_clamp == r.fov_clamp and o.bbox_mode == r.bbox_mode


def test_status_strings_and_version(L):
    lib = L.lib()
    assert lib.gs_abi_version() == 11
    assert lib.gs_status_string(0) == b"ok"
    assert lib.gs_status_string(2) == b"unsupported"


def test_validation_before_device_work(L):
    lib = L.lib()
    o = L.options()
    null = None
    # NULL required pointers
    st = lib.gs_project(ct.byref(o), 10, 1, 64, 64, *([null] * 5), 1, null, null, null, null, null)
    assert st == 1
    # bad dimensions
    assert lib.gs_project(ct.byref(o), -1, 1, 64, 64, *([null] * 5), 1, null, null, null, null, null) == 1
    assert lib.gs_rasterize_fwd(ct.byref(o), 0, 1, 64, 64, *([null] * 8), null, 0, null, null) == 1
    # depth output with an unknown depth mode
    assert lib.gs_rasterize_fwd(ct.byref(o), 1, 1, 64, 64, *([null] * 8), 16, 3, null, null) == 1
    # pose gradients without a workspace
    assert lib.gs_project_bwd(ct.byref(o), 0, 1, 64, 64, *([null] * 5), 1, null, null, null, null, null, null,
                              null, null, null, 16, null, 0, null) == 1
    # packed entry points refuse dense options and vice versa
    assert lib.gs_project_packed(ct.byref(o), 0, 1, 64, 64, *([null] * 5), 1, null, null, 0, 8, 8, null, null,
                                 null, null, 256, 1 << 20, null) == 1
    op = L.options(packed=True)
    assert lib.gs_project(ct.byref(op), 0, 1, 64, 64, *([null] * 5), 1, null, null, null, null, null) == 1
    # unsupported tile size
    o2 = L.options(tile_size=8)
    assert lib.gs_project(ct.byref(o2), 10, 1, 64, 64, *([null] * 5), 1, null, null, null, null, null) == 2
    # sh degree out of range
    o3 = L.options(sh_degree=4)
    assert lib.gs_project(ct.byref(o3), 10, 1, 64, 64, *([null] * 5), 1, null, null, null, null, null) == 1
    # absgrad with N-D features needs one channel pass (D <= 4): refused before any launch
    P = 256   # any non-NULL, aligned address: the call must return before touching it
    assert lib.gs_rasterize_bwd_nd(ct.byref(o), 1, 10, 64, 64, P, P, 5, null, 10, null, P, P, P, P, P, null, 1,
                                   P, P, P, null) == 2
    # gs_project_bwd_range: the range must lie in [0, N] and be ordered
    bad_ranges = [(5, 3), (-1, 4), (0, 11)]
    for b0, b1 in bad_ranges:
        assert lib.gs_project_bwd_range(ct.byref(o), 10, b0, b1, 1, 64, 64, *([P] * 5), 16, P, P, P, P,
                                        *([P] * 5), null) == 1, (b0, b1)
    # packed options are refused by the dense range call
    assert lib.gs_project_bwd_range(ct.byref(op), 10, 0, 10, 1, 64, 64, *([P] * 5), 16, P, P, P, P,
                                    *([P] * 5), null) == 1
    # misaligned workspace
    assert lib.gs_isect_tiles(ct.byref(o), 1, 0, 64, 64, null, null, 0, 8, 8, null, null, 8, 1, 0, null) == 1
    # scheduling entry points: NULL buffers, bad dimensions, a bwd_zero_fill flag outside {0, 1}
    assert lib.gs_tile_order(ct.byref(o), 1, 64, 64, null, P, null) == 1
    assert lib.gs_tile_order(ct.byref(o), 0, 64, 64, P, P, null) == 1
    assert lib.gs_zero_splat_grads(ct.byref(o), 1, 10, null, null) == 1
    assert lib.gs_zero_splat_grads(ct.byref(o), 1, 10, P + 4, null) == 1   # misaligned
    oz = L.options()
    oz.bwd_zero_fill = 2
    assert lib.gs_zero_splat_grads(ct.byref(oz), 1, 0, null, null) == 1
    assert L.options().bwd_zero_fill == 1 and L.options(bwd_zero_fill=False).bwd_zero_fill == 0


def test_workspace_size_monotone(L):
    a = L.gs_isect_workspace_size(1, 1000, 64, 64, 1000)
    b = L.gs_isect_workspace_size(1, 1000, 64, 64, 100000)
    c = L.gs_isect_workspace_size(2, 1000, 64, 64, 100000)
    assert 0 < a < b < c


def test_product_package_never_imports_oracle():
    """The product path must not route through the oracle or any CPU fallback."""
    pkg = os.path.join(ROOT, "paper_2409_06765_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "gs_oracle" not in txt, f


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    from paper_2409_06765_b200 import _lib
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(_lib.GsError):
        _lib.lib()


def test_cpu_tensors_rejected(L):
    import torch
    with pytest.raises(L.GsError):
        L.ptr(torch.zeros(3), name="means")
