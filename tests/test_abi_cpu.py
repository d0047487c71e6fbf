"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every symbol that
include/nrt.h declares, and rejects bad arguments before touching the device."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def N():
    import __graft_entry__ as g
    g.build()
    import paper_2403_06648_b200 as N
    return N


def header_functions():
    src = open(os.path.join(ROOT, "include", "nrt.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nrt_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(N):
    L = N.lib()
    names = header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(L, name), name
    assert set(N.EXPORTED) == set(names)


def test_binding_fails_loudly_without_library(N, tmp_path, monkeypatch):
    monkeypatch.setattr(N, "_lib", None)
    monkeypatch.setattr(N, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        N.lib()


def test_record_layouts_match_header(N):
    assert N.COARSE_REC.itemsize == 184
    assert N.EVENT_REC.itemsize == 216
    assert N.REFINED_REC.itemsize == 4 + 4 + 32 + 32 + 192 + 16 + 16 + 32 + 8 + 16 + 8
    assert C.sizeof(N.nrt_edge) == 68


def test_host_side_validation(N):
    L = N.lib()
    h = C.c_void_p()
    # N = 0 -> EMPTY, before any CUDA call
    assert L.nrt_scene_build(None, None, 0, C.c_float(0.1), C.byref(h)) == 5
    assert b"no points" in L.nrt_last_error()
    d = N.nrt_scene_desc()
    d.n = 10
    d.voxel_size = -1.0
    pts = np.zeros((10, 3), np.float32)
    d.points = d.normals = pts.ctypes.data
    d.radius = 0.01
    assert L.nrt_scene_build_ex(C.byref(d), C.byref(h)) == 1
    # launch on a NULL scene
    tx = np.zeros(3, np.float32)
    assert L.nrt_launch(None, tx.ctypes.data, tx.ctypes.data, 1, 10, 2, 0, C.byref(h)) == 1
    # NULL-safe frees
    L.nrt_scene_free(None)
    L.nrt_paths_free(None)
    ld = N.nrt_launch_desc()
    L.nrt_launch_desc_default(C.byref(ld))
    assert (ld.kappa, ld.world, ld.stage) == (1, 1, 0)
    assert abs(ld.tau - 0.0015) < 1e-9 and abs(ld.dphi_deg - 2.5) < 1e-9
    rd = N.nrt_refine_desc()
    L.nrt_refine_desc_default(C.byref(rd))
    assert (rd.xi, rd.alpha, rd.beta, rd.max_iter) == (2.0, 0.4, 0.4, 100)
    assert L.nrt_paths_count(None, None) == 1
    assert N.nrt_version().startswith("nrt")
