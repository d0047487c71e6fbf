"""Pins of the oracle's NEXT-4 refinement, the paper's own gradient descent (oracle/gd.c; PAPER
§II-E, Tables I-III; readings R50-R56 of DESIGN.md), against closed forms, FP64
re-evaluation and brute force — never against a retyped copy of its arithmetic:
  * a dense box room: every coarse path of order <= 2 refines to the image-method vertices;
  * a single diffraction converges to scipy's bounded minimiser of |a + t e - TX| + |. - RX|;
  * the line search: the accepted step satisfies Eq. 12's Armijo condition and gamma / beta
    violates it (FP64 re-evaluation); the gradient = FP64 central differences of f_k;
  * R53: the 27-cell normal of a plane is its normal, and equals numpy's FP64 Eq. 3 over the
    same points on a noisy cloud; R54: the basis is orthonormal, right-handed, axis rule.
"""
import ctypes as C
import os

import numpy as np
import pytest

import nrt_gen as G
from tests.test_oracle_refine_pins import coarse_rec, edge_case
from tests.test_oracle_sdf_pins import plane_patch

NPROC = max(1, min(32, os.cpu_count() or 1))
SDF = dict(cell=0.0625, r_s=0.015, t_sdf=0.0015, xi=2.0)
NOISELESS = dict(r_s=0.003, t_sdf=0.0005, t_d=0.002, t_a_deg=1.0)  # Tables II/III


def test_gd_box_room_equals_image_method(O):
    from tests.test_oracle_pins import _image_paths
    case = G.case("C1", n_rays=4000)
    case.scene = G.box_room(3)
    case.sdf = dict(SDF)
    recs, _, _ = O.launch_phased(case, procs=NPROC)
    case.gd = dict(NOISELESS)
    out = O.refine_gd_par(case, recs, procs=NPROC)
    paths = _image_paths((4.0, 3.0, 2.5), case.tx.astype(np.float64).tolist(),
                         case.rx[0].astype(np.float64).tolist(), 2)
    assert len(out) == 25
    for r in out:
        assert O.STATUS[int(r["status"])] == "OK", r
        assert int(r["iters"]) == 2000 and r["gradsq"] < 1e-4
        seq = tuple(int(x) for x in r["label"][: r["n_int"]])
        L_img, pts = paths[seq]
        walls = [(0, 0.0), (0, 4.0), (1, 0.0), (1, 3.0), (2, 0.0), (2, 2.5)]
        for k in range(r["n_int"]):
            # R42: the vertex is an SDF hit, within t_sdf of its wall (the room side), and it
            # sits at the mirror point along the wall
            ax, c = walls[seq[k]]
            off = abs(r["v"][k][ax] - c)
            assert off <= NOISELESS["t_sdf"] + 1e-6, (seq, r["v"][k])
            lat = np.delete(r["v"][k] - pts[k], ax)
            assert np.linalg.norm(lat) < 1e-3, (seq, r["v"][k], pts[k])
        # each vertex t_sdf inside the room shortens the path by at most 2 t_sdf
        assert L_img - 2 * NOISELESS["t_sdf"] * r["n_int"] - 1e-5 <= r["L"] <= L_img + 1e-5
        assert abs(r["delay"] - r["L"] / 299792458.0) < 1e-20


def test_gd_diffraction_vs_bounded_minimisation(O):
    from scipy.optimize import minimize_scalar
    rng = np.random.default_rng(5)
    done = 0
    for _ in range(30):
        a = rng.uniform(-1, 1, 3)
        b = a + rng.uniform(-2, 2, 3)
        tx = rng.uniform(-3, 3, 3)
        rx = rng.uniform(-3, 3, 3)
        a32, b32, tx32, rx32 = (np.float32(x) for x in (a, b, tx, rx))
        a, b, tx, rx = (x.astype(np.float64) for x in (a32, b32, tx32, rx32))
        e = (b - a) / np.linalg.norm(b - a)
        L = np.linalg.norm(b - a)
        f = lambda t: np.linalg.norm(a + t * e - tx) + np.linalg.norm(a + t * e - rx)
        res = minimize_scalar(f, bounds=(0, L), method="bounded", options={"xatol": 1e-12})
        if not (1e-2 < res.x < L - 1e-2):
            continue
        case = edge_case(O, tx32, rx32, a32, b32)
        c = coarse_rec(O, [a + 0.5 * L * e], [100], [0], kinds=1)
        r = O.refine_gd(case, c, rho=300)[0]
        assert O.STATUS[int(r["status"])] == "OK", r
        assert np.linalg.norm(r["v"][0] - (a + res.x * e)) < 2e-4
        assert abs(r["L"] - res.fun) < 1e-5
        done += 1
    assert done >= 8


def test_line_search_armijo_and_gradient(O):
    L = O.gd_lib()
    rng = np.random.default_rng(6)
    alpha = beta = 0.4
    f = lambda y, P, Q: np.linalg.norm(y - Q) + np.linalg.norm(y - P)
    for it in range(300):
        diff = it % 3 == 0
        x, P, Q = (rng.uniform(-2, 2, 3).astype(np.float32) for _ in range(3))
        n = rng.normal(size=3)
        n = (n / np.linalg.norm(n)).astype(np.float32)
        u, v = np.zeros(3, np.float32), np.zeros(3, np.float32)
        L.or_gd_basis(n.ctypes.data, u.ctypes.data, v.ctypes.data)
        y = np.zeros(3, np.float32)
        gam = L.or_gd_line_search(x.ctypes.data, P.ctypes.data, Q.ctypes.data, u.ctypes.data,
                                  v.ctypes.data, int(diff), alpha, beta, y.ctypes.data)
        X, P64, Q64, U, V = (a.astype(np.float64) for a in (x, P, Q, u, v))
        # gradient by FP64 central differences of f_k along u (and v)
        h = 1e-6
        gu = (f(X + h * U, P64, Q64) - f(X - h * U, P64, Q64)) / (2 * h)
        gv = 0.0 if diff else (f(X + h * V, P64, Q64) - f(X - h * V, P64, Q64)) / (2 * h)
        step = -gu * U - gv * V
        f0 = f(X, P64, Q64)
        slope = -(gu * gu + gv * gv)
        assert gam > 0
        assert np.allclose(y, X + gam * step, atol=1e-5)
        # Armijo (Eq. 12 shrink condition false) at gamma, true at gamma / beta (FP64, margins)
        assert f(X + gam * step, P64, Q64) <= f0 + alpha * gam * slope + 1e-5
        if gam < 1.0:
            g2 = gam / beta
            assert f(X + g2 * step, P64, Q64) > f0 + alpha * g2 * slope - 1e-5


def test_normal27_plane_and_fp64(O):
    L = O.gd_lib()
    sc_ = plane_patch(z=0.1, jitter=0.003)
    sc = O.OracleScene(sc_, sdf_cell=0.0625)
    sigma = np.float32(0.02)
    rng = np.random.default_rng(8)
    for _ in range(50):
        i = int(rng.integers(sc_.n))
        cell = L.or_sdf_cell_of(C.byref(sc.c), sc.sdf, i)
        x = (sc_.points[i] + rng.uniform(-0.01, 0.01, 3)).astype(np.float32)
        n = np.zeros(3, np.float32)
        assert L.or_sdf_normal27(C.byref(sc.c), sc.sdf, cell, x.ctypes.data, float(sigma), n.ctypes.data)
        assert np.allclose(n, [0, 0, 1], atol=1e-6)
    # noisy normals: FP64 Eq. 3 over the 3x3x3 cells' points
    P = rng.uniform(-0.3, 0.3, (40_000, 3))
    P[:, 2] = rng.normal(0, 0.004, len(P))
    Nn = rng.normal(0, 0.2, (len(P), 3))
    Nn[:, 2] += 1.0
    Nn /= np.linalg.norm(Nn, axis=1, keepdims=True)
    s = G.Scene(P.astype(np.float32), Nn.astype(np.float32), np.full(len(P), 0.01, np.float32),
                np.zeros(len(P), np.int32), G.Edges.empty())
    sc = O.OracleScene(s, sdf_cell=0.0625)
    org = s.points.min(axis=0)
    a = np.float32(0.0625)
    cells = np.floor((s.points - org) / a).astype(np.int64)
    for _ in range(30):
        i = int(rng.integers(s.n))
        cell = L.or_sdf_cell_of(C.byref(sc.c), sc.sdf, i)
        x = (s.points[i] + rng.uniform(-0.02, 0.02, 3)).astype(np.float32)
        n = np.zeros(3, np.float32)
        assert L.or_sdf_normal27(C.byref(sc.c), sc.sdf, cell, x.ctypes.data, float(sigma), n.ctypes.data)
        near = np.all(np.abs(cells - cells[i]) <= 1, axis=1)
        d = s.points[near].astype(np.float64) - x
        w = np.exp(-(d * d).sum(1) / (2.0 * float(sigma) ** 2))
        nb = (w[:, None] * s.normals[near].astype(np.float64)).sum(0) / w.sum()
        assert np.allclose(n, nb / np.linalg.norm(nb), atol=2e-5), (n, nb)


def test_basis_orthonormal_axis_rule(O):
    L = O.gd_lib()
    rng = np.random.default_rng(9)
    for _ in range(200):
        n = rng.normal(size=3)
        n = (n / np.linalg.norm(n)).astype(np.float32)
        u, v = np.zeros(3, np.float32), np.zeros(3, np.float32)
        L.or_gd_basis(n.ctypes.data, u.ctypes.data, v.ctypes.data)
        N, U, V = (a.astype(np.float64) for a in (n, u, v))
        assert abs(U @ N) < 1e-6 and abs(V @ N) < 1e-6 and abs(U @ V) < 1e-6
        assert abs(np.linalg.norm(U) - 1) < 1e-6 and abs(np.linalg.norm(V) - 1) < 1e-6
        assert np.allclose(np.cross(U, V), N, atol=1e-6)
        ax = int(np.argmin(np.abs(n)))
        assert abs(U[ax]) < 1e-7  # u = n x e_ax is perpendicular to the least axis
