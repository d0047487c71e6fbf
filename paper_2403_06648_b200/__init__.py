"""paper_2403_06648_b200 — Python binding of libnrt (include/nrt.h), the B200-native ray
launcher for arXiv 2403.06648.

Argument marshalling only (ctypes): every step of the path runs in the CUDA kernels of
libnrt.so.  There is no CPU fallback — importing works without a GPU (the library loads and
exports its symbols), but every compute call needs the CUDA device and raises NrtError on
failure.  Arrays may be numpy (host) or torch tensors (host or cuda); torch is only used for
device memory and streams.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NRT_LIB") or os.path.join(_HERE, "libnrt.so")  # NRT_LIB: tuning variants

NRT_MAX_INT = 8
STATUS = {0: "NRT_OK", 1: "NRT_E_INVALID", 2: "NRT_E_NOMEM", 3: "NRT_E_CUDA", 4: "NRT_E_OVERFLOW",
          5: "NRT_E_EMPTY", 6: "NRT_E_STATE"}
MEM_HOST, MEM_DEVICE = 0, 1
PATHS_COARSE, PATHS_REFINED, PATHS_EVENTS = 0, 1, 2
REF_STATUS = {0: "OK", 1: "NO_CONVERGE", 2: "OFF_EDGE", 3: "NO_SUPPORT", 4: "WRONG_SIDE",
              5: "OCCLUDED", 6: "DEGENERATE"}


class NrtError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


# ------------------------------------------------------------------------------------------
# ABI structs (include/nrt.h)
# ------------------------------------------------------------------------------------------
class nrt_edge(C.Structure):
    _fields_ = [("a", C.c_float * 3), ("b", C.c_float * 3), ("t0", C.c_float * 3),
                ("n0", C.c_float * 3), ("n1", C.c_float * 3), ("n_exp", C.c_float),
                ("label", C.c_int32)]


class nrt_scene_desc(C.Structure):
    _fields_ = [("points", C.c_void_p), ("normals", C.c_void_p), ("radii", C.c_void_p),
                ("radius", C.c_float), ("labels", C.c_void_p), ("n", C.c_int64),
                ("voxel_size", C.c_float), ("edges", C.c_void_p), ("n_edges", C.c_int32),
                ("mem", C.c_int), ("device", C.c_int32), ("stream", C.c_void_p),
                ("sdf_cell", C.c_float)]


class nrt_scene_info(C.Structure):
    _fields_ = [("n_surfels", C.c_int64), ("n_refs", C.c_int64), ("n_cells", C.c_int64),
                ("dims", C.c_int32 * 3), ("origin", C.c_float * 3), ("voxel", C.c_float),
                ("r_max", C.c_float), ("n_aabb", C.c_int64), ("n_aabb_refs", C.c_int64),
                ("sdf_cell", C.c_float)]


class nrt_launch_desc(C.Structure):
    _fields_ = [("kappa", C.c_int32), ("tau", C.c_float), ("c_R", C.c_float),
                ("dphi_deg", C.c_float), ("theta_ex_deg", C.c_float), ("edge_bin", C.c_float),
                ("rank", C.c_int32), ("world", C.c_int32), ("stage", C.c_int32),
                ("counters", C.c_int32), ("mem", C.c_int), ("stream", C.c_void_p),
                ("intersect", C.c_int32), ("sdf_r_s", C.c_float), ("sdf_t_sdf", C.c_float),
                ("sdf_xi", C.c_float), ("tracer", C.c_int32)]


class nrt_post_desc(C.Structure):
    _fields_ = [("lambda_m", C.c_double), ("angle_deg", C.c_double), ("r_s", C.c_double),
                ("stream", C.c_void_p)]


class nrt_refine_desc(C.Structure):
    _fields_ = [("xi", C.c_double), ("r_s", C.c_double), ("tol_m", C.c_double),
                ("max_iter", C.c_int32), ("alpha", C.c_double), ("beta", C.c_double),
                ("delta", C.c_double), ("tau", C.c_double), ("theta_ex_deg", C.c_double),
                ("rank", C.c_int32), ("world", C.c_int32), ("keep_invalid", C.c_int32),
                ("select", C.c_int32), ("blocks_per_sm", C.c_int32),
                ("stream", C.c_void_p), ("counters", C.c_int32), ("method", C.c_int32),
                ("gd_rho", C.c_int32), ("gd_t_sdf", C.c_double), ("gd_t_d", C.c_double),
                ("gd_t_a_deg", C.c_double)]


class nrt_paths_info(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n", C.c_int64), ("n_raw", C.c_int64),
                ("n_events", C.c_int64), ("n_fan_rays", C.c_int64), ("bounces", C.c_uint64),
                ("surfel_tests", C.c_uint64), ("cells_visited", C.c_uint64),
                ("cells_nonempty", C.c_uint64),
                ("ms_trace", C.c_float), ("ms_fans", C.c_float), ("ms_dedupe", C.c_float),
                ("ms_refine", C.c_float), ("ms_total", C.c_float),
                ("mls_value", C.c_uint64), ("mls_deriv", C.c_uint64)]


COARSE_REC = np.dtype([
    ("rx", "<u4"), ("n_int", "u1"), ("n_diff", "u1"), ("kinds", "<u2"),
    ("label", "<i4", (8,)), ("prim", "<u4", (8,)), ("v", "<f4", (8, 3)),
    ("s_edge", "<f4"), ("L", "<f4"), ("ray_id", "<u8")], align=True)
EVENT_REC = np.dtype([
    ("n_hist", "<i4"), ("n_diff", "<i4"), ("kinds", "<u2"), ("pad_", "<u2"),
    ("label", "<i4", (8,)), ("prim", "<u4", (8,)), ("v", "<f4", (8, 3)), ("s_edge", "<f4"),
    ("edge", "<u4"), ("sbin", "<i4"), ("s", "<f4"), ("d", "<f4", (3,)), ("L", "<f4"),
    ("dist2", "<f4"), ("ray_id", "<u8")], align=True)
REFINED_REC = np.dtype([
    ("rx", "<u4"), ("n_int", "u1"), ("n_diff", "u1"), ("kinds", "<u2"),
    ("label", "<i4", (8,)), ("prim", "<u4", (8,)), ("v", "<f8", (8, 3)),
    ("L", "<f8"), ("delay", "<f8"),
    ("aod_az", "<f4"), ("aod_el", "<f4"), ("aoa_az", "<f4"), ("aoa_el", "<f4"),
    ("inc", "<f4", (8,)), ("status", "<i4"), ("iters", "<i4"),
    ("resid", "<f8"), ("gradsq", "<f8"), ("ray_id", "<u8")], align=True)
assert COARSE_REC.itemsize == 184 and EVENT_REC.itemsize == 216
REC_DTYPE = {PATHS_COARSE: COARSE_REC, PATHS_REFINED: REFINED_REC, PATHS_EVENTS: EVENT_REC}

_VP = C.c_void_p
_P = C.POINTER
_SIGS = {
    "nrt_scene_build": ([_VP, _VP, C.c_int64, C.c_float, _P(_VP)], C.c_int),
    "nrt_scene_build_ex": ([_P(nrt_scene_desc), _P(_VP)], C.c_int),
    "nrt_scene_free": ([_VP], None),
    "nrt_scene_info_get": ([_VP, _P(nrt_scene_info)], C.c_int),
    "nrt_launch_desc_default": ([_P(nrt_launch_desc)], None),
    "nrt_launch": ([_VP, _VP, _VP, C.c_int32, C.c_int64, C.c_int32, C.c_int32, _P(_VP)], C.c_int),
    "nrt_launch_ex": ([_VP, _VP, _VP, C.c_int32, C.c_int64, C.c_int32, C.c_int32,
                       _P(nrt_launch_desc), _P(_VP)], C.c_int),
    "nrt_launch_fans": ([_VP, _VP, _VP, C.c_int64, C.c_int, _P(nrt_launch_desc)], C.c_int),
    "nrt_refine_desc_default": ([_P(nrt_refine_desc)], None),
    "nrt_refine": ([_VP, _VP, _P(_VP)], C.c_int),
    "nrt_refine_ex": ([_VP, _VP, _P(nrt_refine_desc), _P(_VP)], C.c_int),
    "nrt_post_desc_default": ([_P(nrt_post_desc)], None),
    "nrt_postprocess": ([_VP, _VP, _P(nrt_post_desc), _P(_VP)], C.c_int),
    "nrt_paths_count": ([_VP, _P(C.c_int64)], C.c_int),
    "nrt_paths_record_size": ([_VP, _P(C.c_int64)], C.c_int),
    "nrt_paths_info_get": ([_VP, _P(nrt_paths_info)], C.c_int),
    "nrt_paths_export": ([_VP, _VP, C.c_int64, C.c_int], C.c_int),
    "nrt_paths_export_events": ([_VP, _VP, C.c_int64, _P(C.c_int64), C.c_int], C.c_int),
    "nrt_paths_import": ([_VP, C.c_int64, C.c_int32, C.c_int, _VP, _VP, C.c_int32, _P(_VP)],
                         C.c_int),
    "nrt_paths_merge": ([_P(_VP), C.c_int32, C.c_int32, _P(_VP)], C.c_int),
    "nrt_paths_free": ([_VP], None),
    "nrt_debug_trace_rays": ([_VP, _VP, C.c_int64, C.c_int32, _P(nrt_launch_desc), _VP,
                              C.c_int64, _VP], C.c_int),
    "nrt_last_error": ([], C.c_char_p),
    "nrt_version": ([], C.c_char_p),
    "nrt_kernel_launches": ([], C.c_uint64),
    "nrt_probe_fp64_tflops": ([C.c_int], C.c_double),
    "nrt_workspace_bytes": ([], C.c_uint64),
    "nrt_workspace_trim": ([], None),
}
EXPORTED = tuple(_SIGS)

_lib = None


def lib():
    """Load libnrt.so (built by __graft_entry__.build()).  Raises if it is missing: the
    product path has no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libnrt.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(st):
    if st != 0:
        raise NrtError(st, lib().nrt_last_error().decode(errors="replace"))


# ------------------------------------------------------------------------------------------
# array marshalling
# ------------------------------------------------------------------------------------------
def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _ptr(x, dtype, keep):
    """-> (pointer, mem).  numpy arrays are made contiguous host arrays; torch tensors keep
    their device.  `keep` holds references for the duration of the call."""
    if x is None:
        return None, MEM_HOST
    if _is_torch(x):
        import torch
        tdt = {np.float32: torch.float32, np.int32: torch.int32, np.uint64: torch.int64,
               np.int64: torch.int64}[dtype]
        t = x.contiguous()
        if t.dtype != tdt:
            t = t.to(tdt)
        keep.append(t)
        return t.data_ptr(), (MEM_DEVICE if t.is_cuda else MEM_HOST)
    a = np.ascontiguousarray(x, dtype=dtype)
    keep.append(a)
    return a.ctypes.data, MEM_HOST


def _stream_ptr(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except Exception:
            pass
        return None
    return getattr(stream, "cuda_stream", stream)


def make_edges(edges):
    """nrt_gen.Edges (or None) -> ctypes array of nrt_edge."""
    n = 0 if edges is None else len(edges)
    arr = (nrt_edge * max(1, n))()
    for j in range(n):
        e = arr[j]
        e.a[:] = [float(x) for x in edges.a[j]]
        e.b[:] = [float(x) for x in edges.b[j]]
        e.t0[:] = [float(x) for x in edges.t0[j]]
        e.n0[:] = [float(x) for x in edges.n0[j]]
        e.n1[:] = [float(x) for x in edges.n1[j]]
        e.n_exp = float(edges.n_exp[j])
        e.label = int(edges.label[j])
    return arr, n


# ------------------------------------------------------------------------------------------
# handles
# ------------------------------------------------------------------------------------------
class Scene:
    """nrt_scene handle (A1)."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle)

    def info(self):
        i = nrt_scene_info()
        _check(lib().nrt_scene_info_get(self.h, C.byref(i)))
        return {"n_surfels": i.n_surfels, "n_refs": i.n_refs, "n_cells": i.n_cells,
                "dims": tuple(i.dims), "origin": tuple(i.origin), "voxel": i.voxel,
                "r_max": i.r_max, "n_aabb": i.n_aabb, "n_aabb_refs": i.n_aabb_refs,
                "sdf_cell": i.sdf_cell}

    def free(self):
        if self.h is not None and self.h.value:
            lib().nrt_scene_free(self.h)
        self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Paths:
    """nrt_paths handle (coarse or refined set)."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle)

    def count(self):
        n = C.c_int64()
        _check(lib().nrt_paths_count(self.h, C.byref(n)))
        return n.value

    def record_size(self):
        n = C.c_int64()
        _check(lib().nrt_paths_record_size(self.h, C.byref(n)))
        return n.value

    def info(self):
        i = nrt_paths_info()
        _check(lib().nrt_paths_info_get(self.h, C.byref(i)))
        return {k: getattr(i, k) for k, _ in nrt_paths_info._fields_}

    @property
    def kind(self):
        return self.info()["kind"]

    def export(self, out=None):
        """Records as a numpy structured array (host), or into a torch uint8 cuda tensor."""
        n, rs = self.count(), self.record_size()
        if out is not None:
            _check(lib().nrt_paths_export(self.h, C.c_void_p(out.data_ptr()), out.numel(),
                                          MEM_DEVICE if out.is_cuda else MEM_HOST))
            return out
        a = np.zeros(n, REC_DTYPE[self.kind])
        assert a.itemsize == rs
        _check(lib().nrt_paths_export(self.h, C.c_void_p(a.ctypes.data), a.nbytes, MEM_HOST))
        return a

    def export_events(self, device=None):
        """Stage-1 events (nrt_event_rec) of a launch handle: host numpy, or a torch uint8
        tensor on `device` (device-to-device copy)."""
        n = C.c_int64()
        st = lib().nrt_paths_export_events(self.h, None, 0, C.byref(n), MEM_HOST)
        if st not in (0, 4):
            _check(st)
        if device is not None:
            import torch
            t = torch.zeros(n.value * EVENT_REC.itemsize, dtype=torch.uint8, device=device)
            if n.value:
                _check(lib().nrt_paths_export_events(self.h, C.c_void_p(t.data_ptr()), t.numel(),
                                                     C.byref(n), MEM_DEVICE))
            return t
        a = np.zeros(n.value, EVENT_REC)
        if n.value:
            _check(lib().nrt_paths_export_events(self.h, C.c_void_p(a.ctypes.data), a.nbytes,
                                                 C.byref(n), MEM_HOST))
        return a

    def free(self):
        if self.h is not None and self.h.value:
            lib().nrt_paths_free(self.h)
        self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


# ------------------------------------------------------------------------------------------
# the ABI, one Python function per C entry point
# ------------------------------------------------------------------------------------------
def nrt_scene_build(points, normals, n, voxel_size) -> Scene:
    keep = []
    pp, _ = _ptr(points, np.float32, keep)
    pn, _ = _ptr(normals, np.float32, keep)
    h = C.c_void_p()
    _check(lib().nrt_scene_build(pp, pn, int(n), float(voxel_size), C.byref(h)))
    return Scene(h.value)


def nrt_scene_build_ex(points, normals, voxel_size, radii=None, radius=0.015, labels=None,
                       edges=None, device=0, stream=None, sdf_cell=0.0) -> Scene:
    keep = []
    pp, mem = _ptr(points, np.float32, keep)
    pn, mem2 = _ptr(normals, np.float32, keep)
    pr, mem3 = _ptr(radii, np.float32, keep)
    pl, mem4 = _ptr(labels, np.int32, keep)
    mems = {m for p, m in ((pp, mem), (pn, mem2), (pr, mem3), (pl, mem4)) if p is not None}
    if len(mems) != 1:
        raise ValueError("points/normals/radii/labels must all live in the same memory")
    ea, ne = make_edges(edges)
    d = nrt_scene_desc()
    d.points, d.normals, d.radii, d.labels = pp, pn, pr, pl
    d.radius = float(radius)
    d.n = int(len(points))
    d.voxel_size = float(voxel_size)
    d.edges = C.cast(ea, C.c_void_p)
    d.n_edges = ne
    d.mem = mems.pop()
    d.device = int(device)
    d.stream = _stream_ptr(stream)
    d.sdf_cell = float(sdf_cell)
    h = C.c_void_p()
    _check(lib().nrt_scene_build_ex(C.byref(d), C.byref(h)))
    return Scene(h.value)


def launch_desc(**kw) -> nrt_launch_desc:
    d = nrt_launch_desc()
    lib().nrt_launch_desc_default(C.byref(d))
    for k, v in kw.items():
        if k == "stream":
            v = _stream_ptr(v)
        setattr(d, k, v)
    return d


def nrt_launch(scene: Scene, tx, rx, n_rays, max_refl, max_diff) -> Paths:
    keep = []
    ptx, _ = _ptr(np.asarray(tx, np.float32), np.float32, keep)
    prx, _ = _ptr(np.asarray(rx, np.float32).reshape(-1, 3), np.float32, keep)
    h = C.c_void_p()
    _check(lib().nrt_launch(scene.h, ptx, prx, int(np.asarray(rx).reshape(-1, 3).shape[0]),
                            int(n_rays), int(max_refl), int(max_diff), C.byref(h)))
    return Paths(h.value)


def nrt_launch_ex(scene: Scene, tx, rx, n_rays, max_refl, max_diff, **desc) -> Paths:
    keep = []
    ptx, m1 = _ptr(tx if _is_torch(tx) else np.asarray(tx, np.float32), np.float32, keep)
    rxa = rx if _is_torch(rx) else np.asarray(rx, np.float32).reshape(-1, 3)
    prx, m2 = _ptr(rxa, np.float32, keep)
    if m1 != m2:
        raise ValueError("tx and rx must live in the same memory")
    d = launch_desc(mem=m1, stream=desc.pop("stream", None), **desc)
    h = C.c_void_p()
    _check(lib().nrt_launch_ex(scene.h, ptx, prx, int(rxa.shape[0]), int(n_rays), int(max_refl),
                               int(max_diff), C.byref(d), C.byref(h)))
    return Paths(h.value)


def nrt_launch_fans(scene: Scene, coarse: Paths, events, **desc):
    keep = []
    if _is_torch(events):
        pe, mem = events.data_ptr(), (MEM_DEVICE if events.is_cuda else MEM_HOST)
        n = events.numel() // EVENT_REC.itemsize
        keep.append(events)
    else:
        ev = np.ascontiguousarray(events, dtype=EVENT_REC)
        keep.append(ev)
        pe, mem, n = ev.ctypes.data, MEM_HOST, ev.shape[0]
    d = launch_desc(stream=desc.pop("stream", None), **desc)
    _check(lib().nrt_launch_fans(scene.h, coarse.h, pe, int(n), mem, C.byref(d)))
    return coarse


def refine_desc(**kw) -> nrt_refine_desc:
    d = nrt_refine_desc()
    lib().nrt_refine_desc_default(C.byref(d))
    for k, v in kw.items():
        if k == "stream":
            v = _stream_ptr(v)
        setattr(d, k, v)
    return d


def nrt_refine(scene: Scene, coarse: Paths) -> Paths:
    h = C.c_void_p()
    _check(lib().nrt_refine(scene.h, coarse.h, C.byref(h)))
    return Paths(h.value)


def nrt_refine_ex(scene: Scene, coarse: Paths, **desc) -> Paths:
    d = refine_desc(stream=desc.pop("stream", None), **desc)
    h = C.c_void_p()
    _check(lib().nrt_refine_ex(scene.h, coarse.h, C.byref(d), C.byref(h)))
    return Paths(h.value)


def gd_desc(case, **over) -> dict:
    """NEXT-4 refine-descriptor keywords of a case (paper GD, method = 1): Tables I-III defaults
    (noisy cloud, true normals) < case.gd < keyword overrides."""
    q = dict(r_s=0.01, t_sdf=0.001, xi=2.0, rho=2000, alpha=0.4, beta=0.4, delta=1e-4, t_d=0.02,
             t_a_deg=1.0)
    q.update(getattr(case, "gd", None) or {})
    q.update(over)
    return dict(method=1, xi=q["xi"], r_s=q["r_s"], gd_t_sdf=q["t_sdf"], gd_rho=int(q["rho"]),
                alpha=q["alpha"], beta=q["beta"], delta=q["delta"], gd_t_d=q["t_d"],
                gd_t_a_deg=q["t_a_deg"], tau=case.tau, theta_ex_deg=case.theta_ex_deg)


def nrt_postprocess(scene: Scene, refined: Paths, **desc) -> Paths:
    """NEXT-3 post-processing (exact labels, shortest per key, delay order, first-Fresnel-zone
    dedupe) of a refined set -> a new refined set in delay order."""
    d = nrt_post_desc()
    lib().nrt_post_desc_default(C.byref(d))
    for k, v in desc.items():
        setattr(d, k, _stream_ptr(v) if k == "stream" else v)
    if "stream" not in desc:
        d.stream = _stream_ptr(None)
    h = C.c_void_p()
    _check(lib().nrt_postprocess(scene.h, refined.h, C.byref(d), C.byref(h)))
    return Paths(h.value)


def nrt_paths_import(records, kind, tx, rx) -> Paths:
    keep = []
    if _is_torch(records):
        src, mem = records.data_ptr(), (MEM_DEVICE if records.is_cuda else MEM_HOST)
        n = records.numel() // REC_DTYPE[kind].itemsize
        keep.append(records)
    else:
        r = np.ascontiguousarray(records, dtype=REC_DTYPE[kind])
        keep.append(r)
        src, mem, n = r.ctypes.data, MEM_HOST, r.shape[0]
    ptx, _ = _ptr(np.asarray(tx, np.float32), np.float32, keep)
    rxa = np.asarray(rx, np.float32).reshape(-1, 3)
    prx, _ = _ptr(rxa, np.float32, keep)
    h = C.c_void_p()
    _check(lib().nrt_paths_import(src, int(n), int(kind), mem, ptx, prx, rxa.shape[0], C.byref(h)))
    return Paths(h.value)


def nrt_paths_merge(parts, kappa=1) -> Paths:
    arr = (C.c_void_p * len(parts))(*[p.h.value for p in parts])
    h = C.c_void_p()
    _check(lib().nrt_paths_merge(arr, len(parts), int(kappa), C.byref(h)))
    return Paths(h.value)


def nrt_debug_trace_rays(scene: Scene, tx, n_rays, max_refl, ray_ids, **desc) -> np.ndarray:
    keep = []
    ptx, _ = _ptr(np.asarray(tx, np.float32), np.float32, keep)
    ids = np.ascontiguousarray(ray_ids, dtype=np.uint64)
    out = np.zeros((ids.shape[0], max_refl + 1), np.int64)
    d = launch_desc(stream=desc.pop("stream", None), **desc)
    _check(lib().nrt_debug_trace_rays(scene.h, ptx, int(n_rays), int(max_refl), C.byref(d),
                                      ids.ctypes.data, ids.shape[0], out.ctypes.data))
    return out


def nrt_version() -> str:
    return lib().nrt_version().decode()


def nrt_kernel_launches() -> int:
    return int(lib().nrt_kernel_launches())


def nrt_probe_fp64_tflops(device=0) -> float:
    return float(lib().nrt_probe_fp64_tflops(int(device)))


def nrt_workspace_bytes() -> int:
    return int(lib().nrt_workspace_bytes())


def nrt_workspace_trim() -> None:
    lib().nrt_workspace_trim()


# ------------------------------------------------------------------------------------------
# convenience: a whole case (nrt_gen.LaunchCase) through the ABI
# ------------------------------------------------------------------------------------------
def build_case_scene(case, device_arrays=False, stream=None) -> Scene:
    """The case's scene; with case.sdf (NEXT-1) also its AABB primitives of edge sdf["cell"]."""
    s = case.scene
    a = float(getattr(case, "sdf", None)["cell"]) if getattr(case, "sdf", None) else 0.0
    if device_arrays:
        import torch
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        return nrt_scene_build_ex(t(s.points), t(s.normals), case.voxel, radii=t(s.radii),
                                  labels=t(s.labels), edges=s.edges, stream=stream, sdf_cell=a)
    return nrt_scene_build_ex(s.points, s.normals, case.voxel, radii=s.radii, labels=s.labels,
                              edges=s.edges, stream=stream, sdf_cell=a)


def case_desc(case) -> dict:
    """Launch-descriptor keywords of a case (with case.sdf: the NEXT-1 SDF intersection)."""
    desc = dict(kappa=case.kappa, tau=case.tau, c_R=case.c_R, dphi_deg=case.dphi_deg,
                theta_ex_deg=case.theta_ex_deg, edge_bin=case.edge_bin)
    q = getattr(case, "sdf", None)
    if q:
        desc.update(intersect=1, sdf_r_s=float(q["r_s"]), sdf_t_sdf=float(q["t_sdf"]),
                    sdf_xi=float(q["xi"]))
    return desc


def launch_case(scene: Scene, case, **kw) -> Paths:
    desc = case_desc(case)
    desc.update(kw)
    return nrt_launch_ex(scene, case.tx, case.rx, case.n_rays, case.max_refl, case.max_diff,
                         **desc)
