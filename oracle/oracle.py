"""ctypes wrapper of the CPU ORACLE (oracle/*.c).  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
may import this module.  It never imports the CUDA product path and vice versa.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SRCS = ["coarse.c", "grid.c", "sdf.c", "refine.c", "post.c", "gd.c", "env.c"]

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
          "-Wall", "-Wno-unused-function"]


def build(force: bool = False) -> str:
    srcs = [os.path.join(_HERE, s) for s in _SRCS if os.path.exists(os.path.join(_HERE, s))]
    if not force and os.path.exists(_LIB_PATH):
        mt = os.path.getmtime(_LIB_PATH)
        deps = srcs + [os.path.join(_HERE, "oracle.h")]
        if all(os.path.getmtime(s) <= mt for s in deps):
            return _LIB_PATH
    cmd = ["gcc", *CFLAGS, "-o", _LIB_PATH, *srcs, "-lm"]
    subprocess.run(cmd, check=True)
    return _LIB_PATH


COARSE_DTYPE = np.dtype([
    ("rx", "<u4"), ("n_int", "u1"), ("n_diff", "u1"), ("kinds", "<u2"),
    ("label", "<i4", (8,)), ("prim", "<u4", (8,)), ("v", "<f4", (8, 3)),
    ("s_edge", "<f4"), ("L", "<f4"), ("ray_id", "<u8")], align=True)
assert COARSE_DTYPE.itemsize == 184


HIST_FIELDS = [("n", "<i4"), ("n_diff", "<i4"), ("kinds", "<u2"), ("pad_", "<u2"),
               ("label", "<i4", (8,)), ("prim", "<u4", (8,)), ("v", "<f4", (8, 3)),
               ("s_edge", "<f4")]
EVENT_DTYPE = np.dtype([("h", np.dtype(HIST_FIELDS, align=True)), ("edge", "<u4"),
                        ("sbin", "<i4"), ("s", "<f4"), ("d", "<f4", (3,)), ("L", "<f4"),
                        ("dist2", "<f4"), ("ray_id", "<u8")], align=True)
assert EVENT_DTYPE.itemsize == 216


class _Edge(C.Structure):
    _fields_ = [("a", C.c_float * 3), ("b", C.c_float * 3), ("t0", C.c_float * 3),
                ("n0", C.c_float * 3), ("n1", C.c_float * 3), ("n_exp", C.c_float),
                ("label", C.c_int32)]


class _Scene(C.Structure):
    _fields_ = [("p", C.c_void_p), ("nrm", C.c_void_p), ("r", C.c_void_p), ("label", C.c_void_p),
                ("n", C.c_int64), ("edges", C.c_void_p), ("n_edges", C.c_int32),
                ("grid", C.c_void_p), ("sdf", C.c_void_p)]


class _SdfParams(C.Structure):
    _fields_ = [("cell", C.c_float), ("r_s", C.c_float), ("t_sdf", C.c_float), ("xi", C.c_float)]


class _Params(C.Structure):
    _fields_ = [("tx", C.c_float * 3), ("rx", C.c_void_p), ("n_rx", C.c_int32),
                ("n_rays", C.c_int64), ("max_refl", C.c_int32), ("max_diff", C.c_int32),
                ("kappa", C.c_int32), ("tau", C.c_float), ("c_R", C.c_float),
                ("dphi_deg", C.c_float), ("theta_ex_deg", C.c_float), ("edge_bin", C.c_float),
                ("rank", C.c_int32), ("world", C.c_int32), ("sdf", _SdfParams)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        L.or_sincos.argtypes = [C.c_double, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.or_fib_dir.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p]
        L.or_cos_ex.argtypes = [C.c_float]
        L.or_cos_ex.restype = C.c_float
        L.or_cRw.argtypes = [C.c_float, C.c_int64]
        L.or_cRw.restype = C.c_float
        L.or_hit.argtypes = [C.c_void_p] * 4 + [C.c_float, C.c_void_p, C.c_int, C.c_float,
                                                 C.c_float, C.POINTER(C.c_float)]
        L.or_reflect.argtypes = [C.c_void_p] * 3
        L.or_nearest.argtypes = [C.POINTER(_Scene), C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                 C.c_int64, C.c_float, C.c_float, C.POINTER(C.c_float)]
        L.or_nearest.restype = C.c_int64
        L.or_launch.argtypes = [C.POINTER(_Scene), C.POINTER(_Params), C.c_void_p, C.c_int64,
                                C.POINTER(C.c_int64), C.c_void_p, C.c_int64,
                                C.POINTER(C.c_int64), C.POINTER(C.c_uint64)]
        L.or_trace_rays.argtypes = [C.POINTER(_Scene), C.POINTER(_Params), C.c_void_p, C.c_int64,
                                    C.c_void_p, C.c_int64, C.POINTER(C.c_int64), C.c_void_p,
                                    C.POINTER(C.c_uint64)]
        L.or_trace_primary.argtypes = [C.POINTER(_Scene), C.POINTER(_Params), C.c_void_p,
                                       C.c_int64, C.POINTER(C.c_int64), C.c_void_p, C.c_int64,
                                       C.POINTER(C.c_int64), C.POINTER(C.c_uint64)]
        L.or_event_dedupe.argtypes = [C.c_void_p, C.c_int64]
        L.or_event_dedupe.restype = C.c_int64
        L.or_trace_fans.argtypes = [C.POINTER(_Scene), C.POINTER(_Params), C.c_void_p, C.c_int64,
                                    C.c_int32, C.c_int32, C.c_void_p, C.c_int64,
                                    C.POINTER(C.c_int64), C.POINTER(C.c_uint64)]
        L.or_dedupe.argtypes = [C.c_void_p, C.c_int64, C.c_int32]
        L.or_dedupe.restype = C.c_int64
        L.or_edge_closest.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(_Edge),
                                      C.POINTER(C.c_float), C.POINTER(C.c_float),
                                      C.POINTER(C.c_float)]
        L.or_fan_dirs.argtypes = [C.POINTER(_Edge), C.c_void_p, C.c_float, C.c_void_p, C.c_int]
        L.or_sdf_build.argtypes = [C.POINTER(_Scene), C.c_float]
        L.or_sdf_build.restype = C.c_void_p
        L.or_sdf_grid_build.argtypes = [C.c_void_p, C.c_double]
        L.or_sdf_free.argtypes = [C.c_void_p]
        L.or_sdf_count.argtypes = [C.c_void_p]
        L.or_sdf_count.restype = C.c_int64
        L.or_sdf_aabb.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                  C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.or_sdf_expf.argtypes = [C.c_float]
        L.or_sdf_expf.restype = C.c_float
        L.or_sdf_eval.argtypes = [C.POINTER(_Scene), C.c_void_p, C.c_int64, C.c_void_p, C.c_float,
                                  C.POINTER(C.c_float), C.c_void_p]
        L.or_sdf_nearest.argtypes = [C.POINTER(_Scene), C.c_void_p, C.POINTER(_SdfParams),
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int64,
                                     C.c_float, C.c_float, C.POINTER(C.c_float),
                                     C.POINTER(C.c_int64), C.c_void_p]
        L.or_sdf_nearest.restype = C.c_int64
        L.or_grid_build.argtypes = [C.POINTER(_Scene), C.c_double, C.c_void_p]
        L.or_grid_build.restype = C.c_void_p
        L.or_grid_free.argtypes = [C.c_void_p]
        L.or_grid_info.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_int64),
                                   C.POINTER(C.c_double)]
        _lib = L
    return _lib


def _f32(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float32)
    if shape is not None:
        a = a.reshape(shape)
    return a


class OracleScene:
    """Keeps the numpy arrays alive and the C view of them.  grid_voxel (m) attaches the
    tier-1 uniform grid (grid.c: the same argmin as the brute force, pinned to it bit for bit);
    shift (3,) moves the grid origin (invariance pins)."""

    def __init__(self, scene, grid_voxel=None, shift=None, sdf_cell=None, sdf_grid=None):
        self.p = _f32(scene.points, (-1, 3))
        self.nrm = _f32(scene.normals, (-1, 3))
        self.r = _f32(scene.radii, (-1,))
        self.label = np.ascontiguousarray(scene.labels, dtype=np.int32)
        E = scene.edges
        self.n_edges = len(E)
        self.edges = (_Edge * max(1, self.n_edges))()
        for j in range(self.n_edges):
            e = self.edges[j]
            e.a[:] = [float(x) for x in E.a[j]]
            e.b[:] = [float(x) for x in E.b[j]]
            e.t0[:] = [float(x) for x in E.t0[j]]
            e.n0[:] = [float(x) for x in E.n0[j]]
            e.n1[:] = [float(x) for x in E.n1[j]]
            e.n_exp = float(E.n_exp[j])
            e.label = int(E.label[j])
        self.c = _Scene(self.p.ctypes.data, self.nrm.ctypes.data, self.r.ctypes.data,
                        self.label.ctypes.data, self.p.shape[0],
                        C.cast(self.edges, C.c_void_p), self.n_edges, None)
        self.grid = None
        self.sdf = None
        if sdf_cell:
            self.sdf = lib().or_sdf_build(C.byref(self.c), float(sdf_cell))
            self.c.sdf = self.sdf
            if sdf_grid:  # tier 1 for the SDF intersection (same argmin, pinned)
                lib().or_sdf_grid_build(self.sdf, float(sdf_grid))
        if grid_voxel is not None:
            sh = np.ascontiguousarray(np.zeros(3) if shift is None else shift, np.float64)
            self.grid = lib().or_grid_build(C.byref(self.c), float(grid_voxel), sh.ctypes.data)
            self.c.grid = self.grid

    def grid_info(self):
        dims = np.zeros(3, np.int64)
        n, pad = C.c_int64(), C.c_double()
        lib().or_grid_info(self.grid, dims.ctypes.data, C.byref(n), C.byref(pad))
        return {"dims": dims.tolist(), "n_refs": n.value, "pad": pad.value}

    def __del__(self):
        try:
            if self.grid:
                lib().or_grid_free(self.grid)
            if self.sdf:
                lib().or_sdf_free(self.sdf)
        except Exception:
            pass


def coarse_scene(case, **kw):
    """The oracle scene of a coarse launch: with the NEXT-1 AABB primitives when the case asks
    for the SDF intersection (case.sdf = dict(cell, r_s, t_sdf, xi))."""
    sdf = getattr(case, "sdf", None)
    return OracleScene(case.scene, sdf_cell=sdf["cell"] if sdf else None, **kw)


def _params(case, rx=None, max_diff=None):
    rxa = _f32(case.rx if rx is None else rx, (-1, 3))
    p = _Params()
    p.tx[:] = [float(x) for x in np.asarray(case.tx, np.float32)]
    p.rx = rxa.ctypes.data
    p.n_rx = rxa.shape[0]
    p.n_rays = int(case.n_rays)
    p.max_refl = int(case.max_refl)
    p.max_diff = int(case.max_diff if max_diff is None else max_diff)
    p.kappa = int(case.kappa)
    p.tau = float(case.tau)
    p.c_R = float(case.c_R)
    p.dphi_deg = float(case.dphi_deg)
    p.theta_ex_deg = float(case.theta_ex_deg)
    p.edge_bin = float(case.edge_bin)
    p.rank = 0
    p.world = 1
    sdf = getattr(case, "sdf", None)  # NEXT-1: dict(cell=, r_s=, t_sdf=, xi=) or None
    if sdf:
        p.sdf.cell, p.sdf.r_s = float(sdf["cell"]), float(sdf["r_s"])
        p.sdf.t_sdf, p.sdf.xi = float(sdf["t_sdf"]), float(sdf["xi"])
    return p, rxa


def sincos(x: float):
    s, c = C.c_double(), C.c_double()
    lib().or_sincos(float(x), C.byref(s), C.byref(c))
    return s.value, c.value


def fib_dir(i: int, n: int) -> np.ndarray:
    d = np.zeros(3, np.float32)
    lib().or_fib_dir(int(i), int(n), d.ctypes.data)
    return d


def fib_dirs(n: int, ids=None) -> np.ndarray:
    ids = range(n) if ids is None else ids
    return np.stack([fib_dir(i, n) for i in ids]) if len(ids) else np.zeros((0, 3), np.float32)


def cos_ex(theta_deg: float) -> float:
    return lib().or_cos_ex(float(theta_deg))


def cRw(c_R: float, n_rays: int) -> float:
    return lib().or_cRw(float(c_R), int(n_rays))


def hit(o, d, p, n, r, lam=(), tau=0.0015, cosex=None):
    """R7-R8 predicate for one surfel -> t or None."""
    o, d, p, n = (_f32(x, (3,)) for x in (o, d, p, n))
    lam = np.ascontiguousarray(np.asarray(lam, np.float32).reshape(-1, 3))
    nl = lam.shape[0]
    if nl == 0:
        lam = np.zeros((1, 3), np.float32)
    t = C.c_float()
    ce = cos_ex(25.0) if cosex is None else cosex
    ok = lib().or_hit(o.ctypes.data, d.ctypes.data, p.ctypes.data, n.ctypes.data, float(r),
                      lam.ctypes.data, nl, float(tau), float(ce), C.byref(t))
    return t.value if ok else None


def reflect(d, n):
    d, n = _f32(d, (3,)), _f32(n, (3,))
    out = np.zeros(3, np.float32)
    lib().or_reflect(d.ctypes.data, n.ctypes.data, out.ctypes.data)
    return out


def nearest(scene: OracleScene, o, d, lam=(), prev=-1, tau=0.0015, cosex=None):
    o, d = _f32(o, (3,)), _f32(d, (3,))
    lama = np.ascontiguousarray(np.asarray(lam, np.float32).reshape(-1, 3))
    nl = lama.shape[0]
    if nl == 0:
        lama = np.zeros((1, 3), np.float32)
    t = C.c_float()
    ce = cos_ex(25.0) if cosex is None else cosex
    s = lib().or_nearest(C.byref(scene.c), o.ctypes.data, d.ctypes.data, lama.ctypes.data,
                         nl, int(prev), float(tau), float(ce),
                         C.byref(t))
    return int(s), float(t.value)


_FORK = {}


def _primary_worker(args):
    rank, world = args
    case, max_diff = _FORK["case"], _FORK["max_diff"]
    sc = _FORK.get("scene") or coarse_scene(case)
    p, rxa = _params(case, max_diff=max_diff)
    p.rank, p.world = rank, world
    rc, ec = 1 << 16, 1 << 16
    while True:
        raw = np.zeros(rc, COARSE_DTYPE)
        ev = np.zeros(ec, EVENT_DTYPE)
        nr, ne, nb = C.c_int64(), C.c_int64(), C.c_uint64()
        lib().or_trace_primary(C.byref(sc.c), C.byref(p), raw.ctypes.data, rc, C.byref(nr),
                               ev.ctypes.data, ec, C.byref(ne), C.byref(nb))
        if nr.value <= rc and ne.value <= ec:
            return raw[:nr.value].copy(), ev[:ne.value].copy(), int(nb.value)
        rc, ec = max(rc, nr.value), max(ec, ne.value)


def _fan_worker(args):
    part, parts = args
    case, max_diff, ev = _FORK["case"], _FORK["max_diff"], _FORK["events"]
    sc = _FORK.get("scene") or coarse_scene(case)
    p, rxa = _params(case, max_diff=max_diff)
    rc = 1 << 16
    while True:
        raw = np.zeros(rc, COARSE_DTYPE)
        nr, nb = C.c_int64(), C.c_uint64()
        lib().or_trace_fans(C.byref(sc.c), C.byref(p), ev.ctypes.data, ev.shape[0], part, parts,
                            raw.ctypes.data, rc, C.byref(nr), C.byref(nb))
        if nr.value <= rc:
            return raw[:nr.value].copy(), int(nb.value)
        rc = nr.value


def trace_primary(case, rank=0, world=1, scene: OracleScene | None = None):
    """or_trace_primary of lattice rays i == rank (mod world): raw records, raw events,
    bounces (no fans, no dedupe)."""
    sc = scene or coarse_scene(case)
    p, rxa = _params(case)
    p.rank, p.world = int(rank), int(world)
    rc, ec = 1 << 12, 1 << 12
    while True:
        raw = np.zeros(rc, COARSE_DTYPE)
        ev = np.zeros(ec, EVENT_DTYPE)
        nr, ne, nb = C.c_int64(), C.c_int64(), C.c_uint64()
        lib().or_trace_primary(C.byref(sc.c), C.byref(p), raw.ctypes.data, rc, C.byref(nr),
                               ev.ctypes.data, ec, C.byref(ne), C.byref(nb))
        if nr.value <= rc and ne.value <= ec:
            return raw[:nr.value].copy(), ev[:ne.value].copy(), int(nb.value)
        rc, ec = max(rc, nr.value), max(ec, ne.value)


def event_dedupe(ev):
    a = np.ascontiguousarray(ev.copy())
    m = lib().or_event_dedupe(a.ctypes.data, a.shape[0])
    return a[:m].copy()


def launch_phased(case, procs=1, max_diff=None, return_events=False, grid_voxel=None,
                  scene=None):
    """The same coarse operation run in phases over `procs` forked single-threaded
    processes (ray shards, then event shards); the merged set is identical (per-ray
    results are independent; the event set is global).  Returns (records, n_raw, bounces).
    grid_voxel: trace with the tier-1 grid (built once here, shared by the forked workers)."""
    import multiprocessing as mp
    lib()
    _FORK["case"], _FORK["max_diff"] = case, max_diff
    _FORK["scene"] = scene if scene is not None else (
        OracleScene(case.scene, grid_voxel=grid_voxel) if grid_voxel is not None else None)
    ctx = mp.get_context("fork")
    if procs > 1:
        with ctx.Pool(procs) as pool:
            parts = pool.map(_primary_worker, [(r, procs) for r in range(procs)])
    else:
        parts = [_primary_worker((0, 1))]
    raw = np.concatenate([x[0] for x in parts])
    ev = event_dedupe(np.concatenate([x[1] for x in parts]))
    nb = sum(x[2] for x in parts)
    _FORK["events"] = ev
    if ev.shape[0]:
        if procs > 1:
            with ctx.Pool(procs) as pool:
                fparts = pool.map(_fan_worker, [(r, procs) for r in range(procs)])
        else:
            fparts = [_fan_worker((0, 1))]
        raw = np.concatenate([raw] + [x[0] for x in fparts])
        nb += sum(x[1] for x in fparts)
    recs = dedupe(raw, case.kappa)
    _FORK.pop("scene", None)
    if return_events:
        return recs, raw.shape[0], nb, ev
    return recs, raw.shape[0], nb


def launch(case, scene: OracleScene | None = None, raw_cap=1 << 20, max_diff=None):
    """The coarse operation (C.1): returns (deduped records, n_raw, n_bounces)."""
    sc = scene or coarse_scene(case)
    p, rxa = _params(case, max_diff=max_diff)
    while True:
        raw = np.zeros(raw_cap, COARSE_DTYPE)
        out = np.zeros(raw_cap, COARSE_DTYPE)
        n_raw, n_out, nb = C.c_int64(), C.c_int64(), C.c_uint64()
        st = lib().or_launch(C.byref(sc.c), C.byref(p), raw.ctypes.data, raw_cap, C.byref(n_raw),
                             out.ctypes.data, raw_cap, C.byref(n_out), C.byref(nb))
        if st == 0:
            return out[:n_out.value].copy(), int(n_raw.value), int(nb.value)
        raw_cap = int(n_raw.value) + 1


def trace_rays(case, ray_ids, scene: OracleScene | None = None, raw_cap=1 << 16):
    """Primary rays only (no fans): raw records, per-segment hit ids, bounce count."""
    sc = scene or coarse_scene(case)
    p, rxa = _params(case)
    ids = np.ascontiguousarray(ray_ids, dtype=np.uint64)
    nseg = case.max_refl + 1
    while True:
        raw = np.zeros(raw_cap, COARSE_DTYPE)
        hits = np.zeros((ids.shape[0], nseg), np.int64)
        n_raw, nb = C.c_int64(), C.c_uint64()
        st = lib().or_trace_rays(C.byref(sc.c), C.byref(p), ids.ctypes.data, ids.shape[0],
                                 raw.ctypes.data, raw_cap, C.byref(n_raw), hits.ctypes.data,
                                 C.byref(nb))
        if st == 0:
            return raw[:n_raw.value].copy(), hits, int(nb.value)
        raw_cap = int(n_raw.value) + 1


def dedupe(recs: np.ndarray, kappa: int = 1) -> np.ndarray:
    a = np.ascontiguousarray(recs.copy())
    m = lib().or_dedupe(a.ctypes.data, a.shape[0], int(kappa))
    return a[:m].copy()


def make_edge(a, b, t0, n0, n1, n_exp=1.5, label=100):
    e = _Edge()
    e.a[:] = [float(x) for x in a]
    e.b[:] = [float(x) for x in b]
    e.t0[:] = [float(x) for x in t0]
    e.n0[:] = [float(x) for x in n0]
    e.n1[:] = [float(x) for x in n1]
    e.n_exp = float(n_exp)
    e.label = int(label)
    return e


def edge_closest(o, d, edge):
    o, d = _f32(o, (3,)), _f32(d, (3,))
    te, s, d2 = C.c_float(), C.c_float(), C.c_float()
    ok = lib().or_edge_closest(o.ctypes.data, d.ctypes.data, C.byref(edge), C.byref(te),
                               C.byref(s), C.byref(d2))
    return (te.value, s.value, d2.value) if ok else None


def fan_dirs(edge, d, dphi_deg=2.5):
    d = _f32(d, (3,))
    out = np.zeros((512, 3), np.float32)
    M = lib().or_fan_dirs(C.byref(edge), d.ctypes.data, float(dphi_deg), out.ctypes.data, 512)
    return out[:M].copy()


# ------------------------------------------------------------------------------------------
# refinement (refine.c)
# ------------------------------------------------------------------------------------------
REFINED_DTYPE = np.dtype([
    ("rx", "<u4"), ("n_int", "u1"), ("n_diff", "u1"), ("kinds", "<u2"),
    ("label", "<i4", (8,)), ("prim", "<u4", (8,)), ("v", "<f8", (8, 3)),
    ("L", "<f8"), ("delay", "<f8"),
    ("aod_az", "<f4"), ("aod_el", "<f4"), ("aoa_az", "<f4"), ("aoa_el", "<f4"),
    ("inc", "<f4", (8,)), ("status", "<i4"), ("iters", "<i4"),
    ("resid", "<f8"), ("gradsq", "<f8"), ("ray_id", "<u8")], align=True)
STATUS = {0: "OK", 1: "NO_CONVERGE", 2: "OFF_EDGE", 3: "NO_SUPPORT", 4: "WRONG_SIDE",
          5: "OCCLUDED", 6: "DEGENERATE"}


class _RefParams(C.Structure):
    _fields_ = [("xi", C.c_double), ("r_s", C.c_double), ("tol_m", C.c_double),
                ("max_iter", C.c_int32), ("alpha", C.c_double), ("beta", C.c_double),
                ("tau", C.c_double), ("theta_ex_deg", C.c_double), ("tx", C.c_float * 3),
                ("rx", C.c_void_p), ("jac_fd", C.c_int32)]


def _ref_params(case, rx=None, **over):
    rxa = _f32(case.rx if rx is None else rx, (-1, 3))
    p = _RefParams()
    p.xi = float(over.get("xi", case.xi))
    p.r_s = float(over.get("r_s", case.r_s))
    p.tol_m = float(over.get("tol_m", 1e-10))
    p.max_iter = int(over.get("max_iter", 100))
    p.alpha = float(over.get("alpha", 0.4))
    p.beta = float(over.get("beta", 0.4))
    p.tau = float(over.get("tau", case.tau))
    p.theta_ex_deg = float(over.get("theta_ex_deg", case.theta_ex_deg))
    p.tx[:] = [float(x) for x in np.asarray(case.tx, np.float32)]
    p.rx = rxa.ctypes.data
    p.jac_fd = int(over.get("jac_fd", 0))
    return p, rxa


def path_jacobian(case, rec, z=None, fd=False, h=1e-7, scene: OracleScene | None = None, **over):
    """Jacobian dr/dz of one coarse record's residual (pin helper): analytic (R37) or by central
    differences with step h -> (J m x m) or None."""
    refine(case, np.zeros(0, COARSE_DTYPE), scene)
    L = lib()
    if not hasattr(L, "_jac_setup"):
        L.or_path_jacobian.argtypes = [C.POINTER(_Scene), C.POINTER(_RefParams), C.c_void_p,
                                       C.c_void_p, C.c_int, C.c_double, C.c_void_p]
        L._jac_setup = True
    sc = scene or OracleScene(case.scene)
    p, rxa = _ref_params(case, **over)
    c = np.ascontiguousarray(np.asarray(rec, dtype=COARSE_DTYPE).reshape(1))
    J = np.zeros(24 * 24)
    zin = None if z is None else np.ascontiguousarray(z, np.float64)
    m = L.or_path_jacobian(C.byref(sc.c), C.byref(p), c.ctypes.data,
                           None if zin is None else zin.ctypes.data, int(bool(fd)), float(h),
                           J.ctypes.data)
    if m < 0:
        return None
    return J[: m * m].reshape(m, m).copy()


def refine(case, coarse, scene: OracleScene | None = None, **over):
    """Refine every coarse record (no dedupe): one or_refined per input, with status."""
    L = lib()
    if not hasattr(L, "_ref_setup"):
        L.or_refine.argtypes = [C.POINTER(_Scene), C.POINTER(_RefParams), C.c_void_p, C.c_int64,
                                C.c_void_p]
        L.or_mls.argtypes = [C.POINTER(_Scene), C.POINTER(_RefParams), C.c_int32, C.c_void_p,
                             C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_double)]
        L.or_refine_set_grid.argtypes = [C.c_int]
        L._ref_setup = True
    grid = over.pop("grid", True)
    sc = scene or OracleScene(case.scene)
    p, rxa = _ref_params(case, **over)
    cin = np.ascontiguousarray(coarse, dtype=COARSE_DTYPE)
    out = np.zeros(cin.shape[0], REFINED_DTYPE)
    L.or_refine_set_grid(1 if grid else 0)
    L.or_refine(C.byref(sc.c), C.byref(p), cin.ctypes.data, cin.shape[0], out.ctypes.data)
    L.or_refine_set_grid(1)
    return out


def _refine_worker(args):
    case, recs, over = args
    return refine(case, recs, _FORK.get("rscene"), **over)


def refine_par(case, coarse, procs=1, **over):
    """refine() over forked single-threaded processes (paths are independent; out[q] is
    bitwise the serial result for in[q])."""
    import multiprocessing as mp
    lib()
    cin = np.ascontiguousarray(coarse, dtype=COARSE_DTYPE)
    if procs <= 1 or len(cin) < 2:
        return refine(case, cin, **over)
    _FORK["rscene"] = OracleScene(case.scene)
    chunks = [cin[k::procs] for k in range(procs)]
    with mp.get_context("fork").Pool(procs) as pool:
        parts = pool.map(_refine_worker, [(case, c, over) for c in chunks if len(c)])
    _FORK.pop("rscene", None)
    out = np.zeros(len(cin), REFINED_DTYPE)
    for k, p in enumerate(parts):
        out[k::procs] = p
    return out


def mls(case, label, nseed, x, scene: OracleScene | None = None, **over):
    refine(case, np.zeros(0, COARSE_DTYPE), scene)  # argtypes
    sc = scene or OracleScene(case.scene)
    p, rxa = _ref_params(case, **over)
    ns = np.ascontiguousarray(nseed, np.float64)
    xx = np.ascontiguousarray(x, np.float64)
    pb, nb = np.zeros(3), np.zeros(3)
    f = C.c_double()
    ok = lib().or_mls(C.byref(sc.c), C.byref(p), int(label), ns.ctypes.data, xx.ctypes.data,
                      pb.ctypes.data, nb.ctypes.data, C.byref(f))
    return (pb, nb, f.value) if ok else None


def refine_dedupe(ref):
    """R28: among OK paths keep the shortest per key (then lowest ray id), key order."""
    ok = ref[ref["status"] == 0]
    best = {}
    for r in ok:
        k = (int(r["rx"]), int(r["n_int"]), int(r["kinds"]), tuple(int(x) for x in r["label"]))
        cur = best.get(k)
        if cur is None or (float(r["L"]), int(r["ray_id"])) < (float(cur["L"]), int(cur["ray_id"])):
            best[k] = r
    keys = sorted(best)
    return np.array([best[k] for k in keys], dtype=REFINED_DTYPE) if keys else np.zeros(0, REFINED_DTYPE)


def path_residual(case, rec, z=None, scene: OracleScene | None = None, **over):
    """Residual r(z) of one coarse record (at its seed when z is None) -> (r, z_seed)."""
    refine(case, np.zeros(0, COARSE_DTYPE), scene)
    L = lib()
    if not hasattr(L, "_res_setup"):
        L.or_path_residual.argtypes = [C.POINTER(_Scene), C.POINTER(_RefParams), C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p]
        L._res_setup = True
    sc = scene or OracleScene(case.scene)
    p, rxa = _ref_params(case, **over)
    c = np.ascontiguousarray(np.asarray(rec, dtype=COARSE_DTYPE).reshape(1))
    r = np.zeros(32)
    zs = np.zeros(32)
    zin = None if z is None else np.ascontiguousarray(z, np.float64)
    m = L.or_path_residual(C.byref(sc.c), C.byref(p), c.ctypes.data,
                           None if zin is None else zin.ctypes.data, r.ctypes.data, zs.ctypes.data)
    if m < 0:
        return None, None
    return r[:m].copy(), zs[:m].copy()


class _PostParams(C.Structure):
    _fields_ = [("lambda_m", C.c_double), ("angle_deg", C.c_double), ("r_s", C.c_double),
                ("tx", C.c_float * 3), ("rx", C.c_void_p)]


LAMBDA_60GHZ = 299792458.0 / 60e9   # Table I carrier frequency


def _post_params(case, lambda_m=LAMBDA_60GHZ, angle_deg=10.0, r_s=None):
    rxa = _f32(case.rx, (-1, 3))
    q = _PostParams()
    q.lambda_m = float(lambda_m)
    q.angle_deg = float(angle_deg)
    q.r_s = float(case.r_s if r_s is None else r_s)
    q.tx[:] = [float(x) for x in np.asarray(case.tx, np.float32)]
    q.rx = rxa.ctypes.data
    return q, rxa


def postprocess(case, refined, scene: OracleScene | None = None, **over):
    """NEXT-3 post-processing of refined records (status-OK ones): exact labels, shortest per
    key, delay order, greedy first-Fresnel-zone dedupe -> records in delay order."""
    L = lib()
    if not hasattr(L, "_post_setup"):
        L.or_postprocess.argtypes = [C.POINTER(_Scene), C.POINTER(_PostParams), C.c_void_p,
                                     C.c_int64, C.c_void_p]
        L.or_postprocess.restype = C.c_int64
        L.or_fresnel_dup.argtypes = [C.POINTER(_PostParams), C.c_double, C.c_void_p, C.c_void_p]
        L._post_setup = True
    sc = scene or OracleScene(case.scene)
    q, rxa = _post_params(case, **over)
    rin = np.ascontiguousarray(refined, dtype=REFINED_DTYPE)
    out = np.zeros(max(1, rin.shape[0]), REFINED_DTYPE)
    m = L.or_postprocess(C.byref(sc.c), C.byref(q), rin.ctypes.data, rin.shape[0], out.ctypes.data)
    return out[:m].copy()


def fresnel_dup(case, a, b, cos_max, **over):
    """The duplicate predicate of R36 for two refined records (pin helper)."""
    postprocess(case, np.zeros(0, REFINED_DTYPE), OracleScene(case.scene))
    q, rxa = _post_params(case, **over)
    ra = np.ascontiguousarray(np.asarray(a, REFINED_DTYPE).reshape(1))
    rb = np.ascontiguousarray(np.asarray(b, REFINED_DTYPE).reshape(1))
    return bool(lib().or_fresnel_dup(C.byref(q), float(cos_max), ra.ctypes.data, rb.ctypes.data))


# ---- NEXT-4: the paper's gradient-descent refinement (gd.c, readings R50-R56) ----------------
GD_DEFAULTS = dict(cell=0.0625, r_s=0.01, t_sdf=0.001, xi=2.0, rho=2000, alpha=0.4, beta=0.4,
                   delta=1e-4, t_d=0.02, t_a_deg=1.0)  # Tables I-III (noisy, true normals)


class _GdParams(C.Structure):
    _fields_ = [("sdf", _SdfParams), ("rho", C.c_int32), ("alpha", C.c_float), ("beta", C.c_float),
                ("delta", C.c_float), ("t_d", C.c_float), ("t_a_deg", C.c_float), ("tau", C.c_float),
                ("theta_ex_deg", C.c_float), ("tx", C.c_float * 3), ("rx", C.c_void_p)]


def gd_settings(case, **over):
    """The NEXT-4 parameters of a case: GD_DEFAULTS < case.gd < keyword overrides."""
    q = dict(GD_DEFAULTS)
    q.update(getattr(case, "gd", None) or {})
    q.update(over)
    return q


def _gd_params(case, **over):
    q = gd_settings(case, **over)
    rxa = _f32(case.rx, (-1, 3))
    p = _GdParams()
    p.sdf.cell, p.sdf.r_s, p.sdf.t_sdf, p.sdf.xi = q["cell"], q["r_s"], q["t_sdf"], q["xi"]
    p.rho, p.alpha, p.beta, p.delta = int(q["rho"]), q["alpha"], q["beta"], q["delta"]
    p.t_d, p.t_a_deg = q["t_d"], q["t_a_deg"]
    p.tau, p.theta_ex_deg = float(case.tau), float(case.theta_ex_deg)
    p.tx[:] = [float(x) for x in np.asarray(case.tx, np.float32)]
    p.rx = rxa.ctypes.data
    return p, rxa


def gd_scene(case, sdf_grid=None, **over):
    return OracleScene(case.scene, sdf_cell=gd_settings(case, **over)["cell"], sdf_grid=sdf_grid)


def gd_lib():
    """The oracle library with the NEXT-4 entry points' argument types set."""
    L = lib()
    if not hasattr(L, "_gd_setup"):
        L.or_refine_gd.argtypes = [C.POINTER(_Scene), C.POINTER(_GdParams), C.c_void_p, C.c_int64,
                                   C.c_void_p]
        L.or_gd_basis.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.or_gd_line_search.argtypes = [C.c_void_p] * 5 + [C.c_int, C.c_float, C.c_float, C.c_void_p]
        L.or_gd_line_search.restype = C.c_float
        L.or_sdf_normal27.argtypes = [C.POINTER(_Scene), C.c_void_p, C.c_int64, C.c_void_p, C.c_float,
                                      C.c_void_p]
        L.or_sdf_cell_of.argtypes = [C.POINTER(_Scene), C.c_void_p, C.c_int64]
        L.or_sdf_cell_of.restype = C.c_int64
        L._gd_setup = True
    return L


def refine_gd(case, coarse, scene: OracleScene | None = None, **over):
    """NEXT-4: refine every coarse record by the paper's GD (no dedupe), one or_refined each."""
    L = gd_lib()
    sc = scene or gd_scene(case, **over)
    p, rxa = _gd_params(case, **over)
    cin = np.ascontiguousarray(coarse, dtype=COARSE_DTYPE)
    out = np.zeros(cin.shape[0], REFINED_DTYPE)
    rc = L.or_refine_gd(C.byref(sc.c), C.byref(p), cin.ctypes.data, cin.shape[0], out.ctypes.data)
    assert rc == 0, rc
    return out


def _gd_worker(args):
    case, recs, over = args
    return refine_gd(case, recs, _FORK.get("gdscene"), **over)


def refine_gd_par(case, coarse, procs=1, sdf_grid=None, **over):
    """refine_gd() over forked single-threaded processes (out[q] is the serial result);
    sdf_grid: trace with the tier-1 SDF grid of that voxel (same results, pinned)."""
    import multiprocessing as mp
    lib()
    cin = np.ascontiguousarray(coarse, dtype=COARSE_DTYPE)
    if procs <= 1 or len(cin) < 2:
        return refine_gd(case, cin, scene=gd_scene(case, sdf_grid=sdf_grid, **over) if sdf_grid else None,
                         **over)
    _FORK["gdscene"] = gd_scene(case, sdf_grid=sdf_grid, **over)
    chunks = [cin[k::procs] for k in range(procs)]
    with mp.get_context("fork").Pool(procs) as pool:
        parts = pool.map(_gd_worker, [(case, c, over) for c in chunks if len(c)])
    _FORK.pop("gdscene", None)
    out = np.zeros(len(cin), REFINED_DTYPE)
    for k, part in enumerate(parts):
        out[k::procs] = part
    return out


# ---- NEXT-2: environment-driven launch + voxel cone tracing (env.c, readings R60-R67) -------
def env_lib():
    L = lib()
    if not hasattr(L, "_env_setup"):
        L.or_env_build.argtypes = [C.POINTER(_Scene), C.c_void_p, C.c_int32]
        L.or_env_build.restype = C.c_void_p
        L.or_env_free.argtypes = [C.c_void_p]
        L.or_env_count.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
        L.or_env_count.restype = C.c_int64
        L.or_env_ie.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(C.c_int32),
                                C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
        L.or_env_grid.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_float), C.POINTER(C.c_float),
                                  C.POINTER(C.c_void_p)]
        L.or_env_march.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]
        L.or_env_cone_sphere.argtypes = [C.c_void_p, C.c_void_p, C.c_float, C.c_float, C.c_void_p,
                                         C.c_float]
        L.or_env_launch.argtypes = [C.POINTER(_Scene), C.POINTER(_Params), C.c_void_p, C.c_int32,
                                    C.c_int32, C.c_void_p, C.c_int64, C.POINTER(C.c_int64),
                                    C.POINTER(C.c_uint64)]
        L._env_setup = True
    return L


class EnvScene:
    """The oracle scene with its SDF AABBs and the NEXT-2 IE tables for a case's RX set."""

    def __init__(self, case, sdf_grid=None):
        self.sc = coarse_scene(case, sdf_grid=sdf_grid)
        self.rx = _f32(case.rx, (-1, 3))
        self.E = env_lib().or_env_build(C.byref(self.sc.c), self.rx.ctypes.data, self.rx.shape[0])
        assert self.E

    def count(self):
        n_pc = C.c_int64()
        n = env_lib().or_env_count(self.E, C.byref(n_pc))
        return int(n), int(n_pc.value)

    def ie(self, i):
        p = np.zeros(3, np.float32)
        kind, label, vox = C.c_int32(), C.c_int32(), C.c_int64()
        env_lib().or_env_ie(self.E, int(i), p.ctypes.data, C.byref(kind), C.byref(label), C.byref(vox))
        return p, int(kind.value), int(label.value), int(vox.value)

    def grid(self):
        vd = np.zeros(3, np.int64)
        V, tc, mp = C.c_float(), C.c_float(), C.c_void_p()
        env_lib().or_env_grid(self.E, vd.ctypes.data, C.byref(V), C.byref(tc), C.byref(mp))
        nv = int(np.prod(vd))
        march = np.ctypeslib.as_array(C.cast(mp, C.POINTER(C.c_int32)), shape=(nv,)).copy()
        return vd, float(V.value), float(tc.value), march

    def __del__(self):
        try:
            env_lib().or_env_free(self.E)
        except Exception:
            pass


def _env_worker(args):
    case, part, parts = args
    es = _FORK["env"]
    p, rxa = _params(case)
    L = env_lib()
    cap = 1 << 16
    while True:
        raw = np.zeros(cap, COARSE_DTYPE)
        n, nr = C.c_int64(), C.c_uint64()
        st = L.or_env_launch(C.byref(es.sc.c), C.byref(p), es.E, part, parts, raw.ctypes.data, cap,
                             C.byref(n), C.byref(nr))
        if st == 0:
            return raw[: n.value].copy(), int(nr.value)
        cap = int(n.value) + 1


def env_launch(case, procs=1, sdf_grid=None):
    """NEXT-2 coarse set: transmission + cone tracing over forked processes (IE shards), then
    the R17 kappa dedupe -> (records, raw count, validation rays traced); sdf_grid: validate
    with the tier-1 SDF grid (same results, pinned)."""
    import multiprocessing as mp
    env_lib()
    _FORK["env"] = EnvScene(case, sdf_grid=sdf_grid)
    parts = max(1, procs)
    if parts == 1:
        res = [_env_worker((case, 0, 1))]
    else:
        with mp.get_context("fork").Pool(parts) as pool:
            res = pool.map(_env_worker, [(case, k, parts) for k in range(parts)])
    _FORK.pop("env", None)
    raw = np.concatenate([r for r, _ in res]) if res else np.zeros(0, COARSE_DTYPE)
    return dedupe(raw, case.kappa), len(raw), sum(n for _, n in res)
