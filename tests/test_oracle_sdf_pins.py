"""Pins of the oracle's NEXT-1 point-set SDF intersection (oracle/sdf.c; PAPER §II-B/§II-C
P:97-102; readings R40-R45 of DESIGN.md) against closed forms, libm and the image
method:
  * the FP32 exp of the Gaussian weights (written identically in the CUDA path) vs math.exp;
  * the AABB sizing rule on hand-placed points;
  * Eqs. 1-4 over a coplanar patch = the signed distance to its plane (closed form);
  * the march finds a plane within t_sdf of the exact intersection, with the plane's normal;
  * the departure rule keeps a ray that grazes away from its own wall free, and a corner wall hit;
  * a dense box room traced with the SDF intersection finds every image-method path of order <= 2.
"""
import ctypes as C
import math
import os

import numpy as np
import pytest

import nrt_gen as G

SDF = dict(cell=0.0625, r_s=0.015, t_sdf=0.0015, xi=2.0)


def plane_patch(z=0.0, h=0.012, ext=((-0.5, 0.5), (-0.5, 0.5)), nz=1.0, jitter=0.0, seed=0):
    rng = np.random.default_rng(seed)
    xs = np.arange(ext[0][0], ext[0][1], h)
    ys = np.arange(ext[1][0], ext[1][1], h)
    X, Y = np.meshgrid(xs, ys, indexing="ij")
    P = np.stack([X.ravel(), Y.ravel(), np.full(X.size, z)], 1)
    P[:, :2] += rng.uniform(-jitter, jitter, (len(P), 2))
    N = np.tile([0.0, 0.0, nz], (len(P), 1))
    return G.Scene(P.astype(np.float32), N.astype(np.float32), np.full(len(P), 0.01, np.float32),
                   np.zeros(len(P), np.int32), G.Edges.empty())


def sdf_case(scene, tx=(0, 0, 1), rx=(5, 5, 5), n_rays=100, max_refl=1, tau=0.0015):
    c = G.LaunchCase("sdf", scene, np.asarray(tx, np.float32), np.asarray(rx, np.float32).reshape(-1, 3),
                     n_rays, max_refl, 0, 0.5, tau=tau)
    c.sdf = dict(SDF)
    return c


def nearest(O, sc, o, d, lam=(), prev=-1, tau=0.0015, cos_ex=None):
    q = O._SdfParams(SDF["cell"], SDF["r_s"], SDF["t_sdf"], SDF["xi"])
    o, d = (np.ascontiguousarray(x, np.float32) for x in (o, d))
    lama = np.ascontiguousarray(np.asarray(lam, np.float32).reshape(-1, 3))
    nl = lama.shape[0]
    if nl == 0:
        lama = np.zeros((1, 3), np.float32)
    t, cell, n = C.c_float(), C.c_int64(), np.zeros(3, np.float32)
    ce = O.cos_ex(25.0) if cos_ex is None else cos_ex
    s = O.lib().or_sdf_nearest(C.byref(sc.c), sc.sdf, C.byref(q), o.ctypes.data, d.ctypes.data,
                               lama.ctypes.data, nl, int(prev), float(tau), float(ce), C.byref(t),
                               C.byref(cell), n.ctypes.data)
    return int(s), float(t.value), int(cell.value), n


def test_sdf_expf_vs_libm(O):
    L = O.lib()
    xs = np.concatenate([-np.linspace(0, 87, 20001), -np.random.default_rng(1).random(20000) * 20])
    worst = 0.0
    for x in xs.astype(np.float32):
        e = float(L.or_sdf_expf(float(x)))
        ref = math.exp(float(x))
        ulp = float(np.spacing(np.float32(ref)))
        worst = max(worst, abs(e - ref) / ulp)
    assert worst <= 2.0, worst
    assert L.or_sdf_expf(-88.0) == 0.0 and L.or_sdf_expf(0.0) == 1.0


def test_aabb_sizing_rule(O):
    """the points' extent per axis, or the cell's full extent where it exceeds a/2."""
    a = SDF["cell"]
    # one cell at the origin: spread 0.04 (> a/2) along x, 0.01 along y, 0 along z
    P = np.array([[0.001, 0.005, 0.0], [0.041, 0.015, 0.0], [0.02, 0.01, 0.0]], np.float32)
    s = G.Scene(P, np.tile(np.float32([0, 0, 1]), (3, 1)), np.full(3, 0.01, np.float32),
                np.zeros(3, np.int32), G.Edges.empty())
    sc = O.OracleScene(s, sdf_cell=a)
    lo, hi = np.zeros(3, np.float32), np.zeros(3, np.float32)
    cell, npt = C.c_int64(), C.c_int64()
    assert O.lib().or_sdf_count(sc.sdf) == 1
    O.lib().or_sdf_aabb(sc.sdf, 0, lo.ctypes.data, hi.ctypes.data, C.byref(cell), C.byref(npt))
    org = P.min(axis=0)
    assert npt.value == 3
    assert lo[0] == org[0] and hi[0] == np.float32(org[0] + np.float32(a))   # full extent
    assert lo[1] == np.float32(0.005) and hi[1] == np.float32(0.015)          # tight
    assert lo[2] == 0.0 and hi[2] == 0.0                                       # flat


def test_sdf_of_coplanar_patch_is_plane_distance(O):
    """Eqs. 1-4 over points of one plane with equal normals: pbar lies in the plane, nbar = n,
    so f(x) = (x - pbar) . n = the signed distance to the plane."""
    sc_ = plane_patch(z=0.25, jitter=0.003)
    sc = O.OracleScene(sc_, sdf_cell=SDF["cell"])
    rng = np.random.default_rng(3)
    L = O.lib()
    n_aabb = L.or_sdf_count(sc.sdf)
    for _ in range(200):
        j = int(rng.integers(n_aabb))
        lo, hi = np.zeros(3, np.float32), np.zeros(3, np.float32)
        cell, npt = C.c_int64(), C.c_int64()
        L.or_sdf_aabb(sc.sdf, j, lo.ctypes.data, hi.ctypes.data, C.byref(cell), C.byref(npt))
        x = np.float32((lo + hi) / 2 + rng.uniform(-0.05, 0.05, 3))
        f, nb = C.c_float(), np.zeros(3, np.float32)
        ok = L.or_sdf_eval(C.byref(sc.c), sc.sdf, j, x.ctypes.data, float(SDF["xi"] * SDF["r_s"]),
                           C.byref(f), nb.ctypes.data)
        assert ok
        assert abs(f.value - (float(x[2]) - 0.25)) < 2e-6
        assert np.allclose(nb, [0, 0, 1], atol=1e-6)


def test_march_hits_plane_within_t_sdf(O):
    sc_ = plane_patch(z=0.0, jitter=0.002)
    sc = O.OracleScene(sc_, sdf_cell=SDF["cell"])
    rng = np.random.default_rng(4)
    for _ in range(100):
        o = np.array([rng.uniform(-0.2, 0.2), rng.uniform(-0.2, 0.2), rng.uniform(0.05, 0.6)])
        d = np.array([rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3), -1.0])
        d /= np.linalg.norm(d)
        s, t, cell, n = nearest(O, sc, o, d)
        assert s >= 0
        t_exact = o[2] / -d[2]
        # the hit lies within t_sdf of the plane (|f| < t_sdf, or the linear zero of a sign change)
        assert abs((o[2] + t * d[2])) < SDF["t_sdf"] + 1e-6, (t, t_exact)
        assert np.allclose(n, [0, 0, 1], atol=1e-5)
    # a ray parallel above the plane, and one moving away, escape
    assert nearest(O, sc, (0, 0, 0.2), (1, 0, 0))[0] == -1
    assert nearest(O, sc, (0, 0, 0.2), (0, 0, 1))[0] == -1


def test_departure_rule(O):
    """A ray leaving the floor at a grazing angle is not stopped by the floor's neighbouring
    AABBs (their SDF at the origin is ~0 and their normal is the departure normal), while a ray
    toward a perpendicular wall 3 cm away is stopped before passing it (corners stay closed)."""
    floor = plane_patch(z=0.0, ext=((-0.5, 0.5), (-0.5, 0.5)))
    wall_pts = np.stack(np.meshgrid(np.float32([0.03]), np.arange(-0.5, 0.5, 0.012),
                                    np.arange(0.0, 0.5, 0.012), indexing="ij"), -1).reshape(-1, 3)
    P = np.concatenate([floor.points, wall_pts]).astype(np.float32)
    N = np.concatenate([floor.normals, np.tile(np.float32([-1, 0, 0]), (len(wall_pts), 1))])
    s = G.Scene(P, N.astype(np.float32), np.full(len(P), 0.01, np.float32),
                np.concatenate([np.zeros(len(floor.points), np.int32), np.ones(len(wall_pts), np.int32)]),
                G.Edges.empty())
    sc = O.OracleScene(s, sdf_cell=SDF["cell"])
    o = np.float32([-0.2, 0.0, 0.0])
    d = np.float32([-0.999, 0.0, 0.0447])
    d /= np.linalg.norm(d)
    assert nearest(O, sc, o, d, lam=[(0, 0, 1)])[0] == -1           # grazes away: free
    assert nearest(O, sc, o, d, lam=[])[0] >= 0                      # without the rule: stuck
    d2 = np.float32([0.999, 0.0, 0.0447])
    d2 /= np.linalg.norm(d2)
    o2 = np.float32([0.0, 0.0, 0.0])
    hit = nearest(O, sc, o2, d2, lam=[(0, 0, 1)])
    # stopped at the corner: by the wall, or by the corner AABB whose points mix both walls
    # (its SDF averages them, so the departure rule does not apply to it)
    assert hit[0] >= 0 and 0.0 < hit[1] < 0.035, hit


def test_dense_box_room_finds_every_image_path(O):
    """C1's room sampled 3x denser (1.8 cm spacing): with the SDF intersection every image-method
    path of order <= 2 is found (the coarse key set contains them; corner AABBs average two walls'
    normals, so a few extra coarse keys are the method's own)."""
    from tests.test_oracle_pins import _image_paths
    case = G.case("C1", n_rays=4000)
    case.scene = G.box_room(3)
    case.sdf = dict(SDF)
    recs, n_raw, nb = O.launch_phased(case, procs=os.cpu_count() or 1)
    keys = {tuple(int(x) for x in r["label"][: r["n_int"]]) for r in recs}
    img = _image_paths((4.0, 3.0, 2.5), case.tx.tolist(), case.rx[0].tolist(), 2)
    assert set(img) <= keys, set(img) - keys
    assert len(keys - set(img)) <= 4
    assert nb == case.n_rays * 3  # closed room: every ray traces max_refl + 1 segments


def test_sdf_eval_vs_fp64_eqs_1_4(O):
    """R41/R41b: the FP32 chunked-tree sums agree with Eqs. 1-4 evaluated in FP64 by numpy
    (exp from libm) within FP32 rounding, on AABBs of 1-600 noisy points (several chunks of 32
    and a ragged last chunk), so a dropped, duplicated or mis-weighted term fails."""
    rng = np.random.default_rng(7)
    P = rng.uniform(-0.3, 0.3, (60_000, 3))
    P[:, 2] = 0.02 * np.sin(7 * P[:, 0]) + rng.normal(0, 0.002, len(P))
    P = np.concatenate([P, [[0.29, 0.29, 0.3]]])  # a lone point: a 1-point AABB
    Nn = rng.normal(0, 0.15, (len(P), 3))
    Nn[:, 2] += 1.0
    Nn /= np.linalg.norm(Nn, axis=1, keepdims=True)
    s = G.Scene(P.astype(np.float32), Nn.astype(np.float32), np.full(len(P), 0.01, np.float32),
                np.zeros(len(P), np.int32), G.Edges.empty())
    sc = O.OracleScene(s, sdf_cell=SDF["cell"])
    L = O.lib()
    sigma = np.float32(SDF["xi"] * SDF["r_s"])
    pts64, nrm64 = s.points.astype(np.float64), s.normals.astype(np.float64)
    org = s.points.min(axis=0)
    a = np.float32(SDF["cell"])
    cells = np.floor((s.points - org) / a).astype(np.int64)
    n_aabb = L.or_sdf_count(sc.sdf)
    sizes = []
    for j in rng.permutation(n_aabb)[:60].tolist() + [n_aabb - 1]:
        lo, hi = np.zeros(3, np.float32), np.zeros(3, np.float32)
        cell, npt = C.c_int64(), C.c_int64()
        L.or_sdf_aabb(sc.sdf, j, lo.ctypes.data, hi.ctypes.data, C.byref(cell), C.byref(npt))
        dims = np.floor((s.points.max(axis=0) - org) / a).astype(np.int64) + 1
        lin = cells[:, 0] + dims[0] * (cells[:, 1] + dims[1] * cells[:, 2])
        ids = np.nonzero(lin == cell.value)[0]
        assert len(ids) == npt.value
        sizes.append(len(ids))
        x = np.float32((lo + hi) / 2 + rng.uniform(-0.03, 0.03, 3))
        f, nb = C.c_float(), np.zeros(3, np.float32)
        assert L.or_sdf_eval(C.byref(sc.c), sc.sdf, j, x.ctypes.data, float(sigma), C.byref(f), nb.ctypes.data)
        dd = pts64[ids] - x.astype(np.float64)
        w = np.exp(-(dd * dd).sum(1) / (2.0 * float(sigma) ** 2))
        pb = (w[:, None] * pts64[ids]).sum(0) / w.sum()
        nbar = (w[:, None] * nrm64[ids]).sum(0) / w.sum()
        f64 = float((x.astype(np.float64) - pb) @ nbar)
        assert np.allclose(nb, nbar, rtol=0, atol=2e-6), (j, nb, nbar)
        assert abs(f.value - f64) <= 2e-6 + 1e-5 * abs(f64), (j, f.value, f64)
    assert max(sizes) > 64 and min(sizes) == 1
