"""Pins of the CPU oracle's REFINEMENT part (P6-P12) against closed
forms, convexity/brute force and invariants — never against a retyped copy of its formula."""
import json
import math
import os

import numpy as np
import pytest

import nrt_gen as G

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def plane_scene(planes, extent=((-1.0, 4.0), (-1.0, 1.0)), h=0.01, r=0.012):
    """Dense surfel grids on axis-aligned planes z = c (normal +-z), one label per plane."""
    P, N, L = [], [], []
    xs = np.arange(extent[0][0], extent[0][1] + 1e-9, h)
    ys = np.arange(extent[1][0], extent[1][1] + 1e-9, h)
    X, Y = np.meshgrid(xs, ys, indexing="ij")
    for lab, (zc, nz) in enumerate(planes):
        p = np.stack([X.ravel(), Y.ravel(), np.full(X.size, zc)], 1)
        P.append(p)
        N.append(np.tile([0.0, 0.0, nz], (p.shape[0], 1)))
        L.append(np.full(p.shape[0], lab, np.int32))
    P = np.concatenate(P).astype(np.float32)
    return G.Scene(P, np.concatenate(N).astype(np.float32), np.full(P.shape[0], r, np.float32),
                   np.concatenate(L), G.Edges.empty())


def make_case(scene, tx, rx, r_s=0.003):
    return G.LaunchCase("pin", scene, np.asarray(tx, np.float32),
                        np.asarray(rx, np.float32).reshape(-1, 3), 1000, 4, 1, 0.1, r_s=r_s,
                        tau=0.0015)


def coarse_rec(O, verts, labels, prims, kinds=0, rx=0):
    c = np.zeros(1, O.COARSE_DTYPE)
    c["rx"] = rx
    c["n_int"] = len(verts)
    c["kinds"] = kinds
    c["n_diff"] = bin(kinds).count("1")
    for k, (v, l, p) in enumerate(zip(verts, labels, prims)):
        c["v"][0, k] = v
        c["label"][0, k] = l
        c["prim"][0, k] = p
    return c


def nearest_id(scene, x, label):
    m = np.nonzero(scene.labels == label)[0]
    return int(m[np.argmin(np.sum((scene.points[m] - np.float32(x)) ** 2, 1))])


# ---------------------------------------------------------------- P6 / mirror point ------
def test_mirror_point(O):
    g = GOLD["mirror_point"]
    sc = plane_scene([(0.0, 1.0)])
    case = make_case(sc, g["tx"], g["rx"])
    c = coarse_rec(O, [(0.3, 0.05, 0.0)], [0], [nearest_id(sc, (0.3, 0.05, 0), 0)])
    r = O.refine(case, c)[0]
    assert O.STATUS[int(r["status"])] == "OK"
    assert np.allclose(r["v"][0], g["point"], atol=1e-9)
    assert abs(r["L"] - g["f"]) < 1e-7
    assert abs(r["L"] - 2 * math.sqrt(2)) < 1e-12
    assert r["gradsq"] < 1e-20


def test_two_planes_image_method(O):
    g = GOLD["two_planes"]
    sc = plane_scene([(0.0, 1.0), (1.0, -1.0)])
    case = make_case(sc, g["tx"], g["rx"])
    c = coarse_rec(O, [(0.6, 0.02, 0.0), (2.4, -0.03, 1.0)], [0, 1],
                   [nearest_id(sc, (0.6, 0, 0), 0), nearest_id(sc, (2.4, 0, 1), 1)])
    r = O.refine(case, c)[0]
    assert O.STATUS[int(r["status"])] == "OK"
    assert np.allclose(r["v"][0], g["I1"], atol=1e-9)
    assert np.allclose(r["v"][1], g["I2"], atol=1e-9)
    assert abs(r["L"] - math.sqrt(13)) < 1e-12 and abs(r["L"] - g["f"]) < 1e-6


# ---------------------------------------------------------------- P6 / box room ---------
def test_box_room_refined_equals_image_method(O):
    """C1: every refined vertex equals the closed-form image-method vertex to 1e-9 m."""
    from tests.test_oracle_pins import _image_paths
    case = G.case("C1")
    recs, _, _ = O.launch_phased(case, procs=os.cpu_count() or 1)
    ref = O.refine(case, recs)
    paths = _image_paths((4.0, 3.0, 2.5), case.tx.astype(np.float64).tolist(),
                         case.rx[0].astype(np.float64).tolist(), 2)
    assert (ref["status"] == 0).all()
    for r in ref:
        seq = tuple(int(x) for x in r["label"][: r["n_int"]])
        # image method evaluated at the f32 TX/RX the oracle uses
        L_img, pts = paths[seq]
        for k in range(r["n_int"]):
            assert np.linalg.norm(r["v"][k] - pts[k]) < 1e-9
        assert abs(r["L"] - L_img) < 1e-9
        assert abs(r["delay"] - r["L"] / 299792458.0) < 1e-20
        assert r["gradsq"] < GOLD.get("delta", 1e-4)


# ---------------------------------------------------------------- P7 diffraction --------
def edge_case(O, tx, rx, a=(0, 0, 0), b=(0, 0, 2)):
    far = G.Scene(np.array([[10.0, 10.0, 10.0]], np.float32), np.array([[0, 0, 1.0]], np.float32),
                  np.array([0.01], np.float32), np.array([0], np.int32),
                  G.Edges(np.array([a], np.float32), np.array([b], np.float32),
                          np.array([[0, 1, 0]], np.float32), np.array([[-1, 0, 0]], np.float32),
                          np.array([[0, -1, 0]], np.float32), np.array([1.5], np.float32),
                          np.array([100], np.int32)))
    return make_case(far, tx, rx)


def test_diffraction_example_t_equals_one(O):
    g = GOLD["edge_example"]
    case = edge_case(O, g["tx"], g["rx"], g["a"], g["b"])
    c = coarse_rec(O, [(0.0, 0.0, 0.7)], [100], [0], kinds=1)
    r = O.refine(case, c)[0]
    assert O.STATUS[int(r["status"])] == "OK"
    assert np.allclose(r["v"][0], [0, 0, g["t"]], atol=1e-9)
    # Keller condition: equal angles to the edge on both sides
    din = r["v"][0] - np.array(g["tx"])
    dout = np.array(g["rx"]) - r["v"][0]
    e = np.array([0, 0, 1.0])
    assert abs(din @ e / np.linalg.norm(din) - dout @ e / np.linalg.norm(dout)) < 1e-12


def test_diffraction_vs_bounded_scalar_minimisation(O):
    """f(t) = |a+te-TX| + |a+te-RX| is convex; scipy's bounded minimiser is the brute force."""
    from scipy.optimize import minimize_scalar
    rng = np.random.default_rng(4)
    done = 0
    for _ in range(40):
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
        if not (1e-3 < res.x < L - 1e-3):
            continue
        case = edge_case(O, tx32, rx32, a32, b32)
        c = coarse_rec(O, [a + 0.5 * L * e], [100], [0], kinds=1)
        r = O.refine(case, c)[0]
        assert int(r["status"]) == 0
        assert np.linalg.norm(r["v"][0] - (a + res.x * e)) < 1e-6
        assert r["L"] <= res.fun + 1e-12
        done += 1
    assert done >= 10


# ---------------------------------------------------------------- P9 residual identity --
def test_eq9_worked_example_and_finite_differences(O):
    g = GOLD["eq9_gradient_example"]
    sc = plane_scene([(0.0, 1.0)])
    case = make_case(sc, g["tx"], g["rx"])
    c = coarse_rec(O, [g["I"]], [0], [nearest_id(sc, g["I"], 0)])
    r, z = O.path_residual(case, c)
    # the oracle's basis for n = +z is u = +y, v = +z x +y = -x (R: least |n.a| axis, x first)
    assert abs(r[0]) < 1e-12
    assert abs(-r[1] - g["value"]) < 5e-8
    assert abs(r[2]) < 1e-12                      # on the plane: f_sdf = 0
    # Eqs. 9-10 are the derivatives of f_k = |I - I0| + |I - I2| along u and v
    tx, rx, I = (np.array(x, float) for x in (g["tx"], g["rx"], g["I"]))
    fk = lambda p: np.linalg.norm(p - tx) + np.linalg.norm(p - rx)
    h = 1e-6
    for vec, val in (((0, 1, 0), r[0]), ((-1, 0, 0), r[1])):
        vec = np.array(vec, float)
        fd = (fk(I + h * vec) - fk(I - h * vec)) / (2 * h)
        assert abs(fd - val) < 1e-5 * max(1.0, abs(fd))


# ---------------------------------------------------------------- P10 MLS -----------------
def test_mls_gaussian_weight_and_plane(O):
    sigma = 0.02
    case = make_case(G.Scene(np.array([[0.02, 0, 0], [0, 0, 0]], np.float32),
                             np.array([[0, 0, 1], [0, 0, 1]], np.float32),
                             np.full(2, 0.01, np.float32), np.zeros(2, np.int32), G.Edges.empty()),
                     (0, 0, 1), (1, 0, 1), r_s=sigma / 2.0)
    pb, nb, f = O.mls(case, 0, (0, 0, 1), (0.0, 0.0, 0.003))
    # p_bar_x = sigma w / (w + w0), w0 = exp(-(0.003^2)/(2 sigma^2)), w = exp(-(sigma^2+0.003^2)/(2 sigma^2))
    w0 = math.exp(-(0.003 ** 2) / (2 * sigma ** 2))
    w = pb[0] * w0 / (np.float32(0.02) - pb[0])
    assert abs(w / w0 - GOLD["gaussian_weight_at_sigma"]["value"]) < 2e-7
    assert abs(f - 0.003) < 1e-12 and np.allclose(nb, [0, 0, 1])
    # single point: f = (x - p).n
    pb, nb, f = O.mls(case, 0, (0, 0, 1), (0.0195, 0.0005, -0.002), r_s=0.0005)
    assert abs(f - (-0.002)) < 1e-12
    # coplanar noisy-free neighbourhood: f = signed plane distance, n = plane normal
    sc = plane_scene([(0.0, 1.0)])
    case = make_case(sc, (0, 0, 1), (1, 0, 1), r_s=0.01)
    pb, nb, f = O.mls(case, 0, (0, 0, 1), (0.123, -0.2, 0.0071))
    assert abs(f - np.float32(0.0071).astype(np.float64)) < 1e-9 or abs(f - 0.0071) < 1e-9
    assert np.allclose(nb, [0, 0, 1], atol=1e-15)


# ---------------------------------------------------------------- P11 delay ---------------
def test_delay_closed_form(O):
    g = GOLD["delay"]
    sc = plane_scene([(0.0, 1.0)])
    case = make_case(sc, (0, 0, 1), (3, 0, 1))
    c = coarse_rec(O, [], [], [])
    r = O.refine(case, c)[0]
    assert r["status"] == 0 and abs(r["L"] - g["length_m"]) < 1e-12
    assert abs(r["delay"] * 1e9 - g["delay_ns"]) < 1e-5


# ---------------------------------------------------------------- R25 validity ------------
def test_occlusion_and_wrong_side(O):
    sc = plane_scene([(0.0, 1.0)])
    # a blocker patch at z = 0.5 between TX and the mirror point
    blk = plane_scene([(0.5, 1.0)], extent=((0.3, 0.7), (-0.2, 0.2)))
    blk.labels[:] = 1
    both = G.Scene(np.concatenate([sc.points, blk.points]), np.concatenate([sc.normals, blk.normals]),
                   np.concatenate([sc.radii, blk.radii]), np.concatenate([sc.labels, blk.labels]),
                   G.Edges.empty())
    case = make_case(both, (0, 0, 1), (2, 0, 1))
    c = coarse_rec(O, [(0.9, 0, 0)], [0], [nearest_id(both, (0.9, 0, 0), 0)])
    r = O.refine(case, c)[0]
    assert O.STATUS[int(r["status"])] == "OCCLUDED"
    # TX above, RX below the plane: no specular point on the same side -> not OK
    case = make_case(sc, (0, 0, 1), (2, 0, -1))
    r = O.refine(case, coarse_rec(O, [(1.0, 0, 0)], [0], [nearest_id(sc, (1, 0, 0), 0)]))[0]
    assert O.STATUS[int(r["status"])] != "OK"


# ---------------------------------------------------------------- P12 reciprocity ---------
def test_reciprocity_box_room(O):
    """Refined set (TX->RX) == reversed refined set (RX->TX): vertices 1e-9 m, delays 1e-15 s."""
    a = G.case("C1")
    b = G.case("C1")
    b.tx, b.rx = a.rx[0].copy(), a.tx.reshape(1, 3).copy()
    ra = O.refine_dedupe(O.refine(a, O.launch_phased(a, procs=os.cpu_count() or 1)[0]))
    rb = O.refine_dedupe(O.refine(b, O.launch_phased(b, procs=os.cpu_count() or 1)[0]))
    A = {tuple(int(x) for x in r["label"][: r["n_int"]]): r for r in ra}
    B = {tuple(int(x) for x in r["label"][: r["n_int"]])[::-1]: r for r in rb}
    assert set(A) == set(B) and len(A) == 25
    for k, r in A.items():
        s = B[k]
        n = r["n_int"]
        if n:
            assert np.abs(r["v"][:n] - s["v"][:n][::-1]).max() < 1e-9
        assert abs(r["delay"] - s["delay"]) < 1e-15


# ---------------------------------------------------------------- R27 angles ------------
def _angles(r):
    return (float(r["aod_az"]), float(r["aod_el"]), float(r["aoa_az"]), float(r["aoa_el"]))


def _close_deg(a, b, tol=1e-4):
    """angle tuples equal within tol degrees; azimuths compared on the circle (+-180 alike)"""
    d = np.abs(np.asarray(a, float) - np.asarray(b, float))
    d = np.minimum(d, 360.0 - d)
    return bool(np.all(d <= tol))


def test_angles_closed_form_reflection(O):
    """R27: azimuth = atan2(y, x) about +z, elevation = asin(z); AoD along the
    first segment, AoA from the RX toward the last vertex; incidence = angle to the normal.
    Floor z = 0, TX (0,0,1), RX (2,0,1): vertex (1,0,0), AoD (0, -45), AoA (180, -45), 45 deg;
    the same turned by 90 deg about z: AoD (90, -45), AoA (-90, -45)."""
    sc = plane_scene([(0.0, 1.0)], extent=((-1.0, 3.0), (-1.0, 3.0)), h=0.02, r=0.02)
    for tx, rx, v, expect in (((0, 0, 1), (2, 0, 1), (1, 0, 0), (0.0, -45.0, 180.0, -45.0)),
                              ((0, 0, 1), (0, 2, 1), (0, 1, 0), (90.0, -45.0, -90.0, -45.0)),
                              ((0, 0, 1), (1, 1, 2), (1 / 3, 1 / 3, 0),
                               (45.0, -math.degrees(math.atan2(1, math.sqrt(2) / 3)), -135.0,
                                -math.degrees(math.atan2(2, 2 * math.sqrt(2) / 3))))):
        case = make_case(sc, tx, rx)
        seed = (v[0] + 0.02, v[1] - 0.01, 0.0)
        c = coarse_rec(O, [seed], [0], [nearest_id(sc, seed, 0)])
        r = O.refine(case, c)[0]
        assert O.STATUS[int(r["status"])] == "OK"
        assert np.allclose(r["v"][0], v, atol=1e-9)
        assert _close_deg(_angles(r), expect), (_angles(r), expect)
        inc = math.degrees(math.acos(tx[2] / math.dist(tx, v)))
        assert abs(float(r["inc"][0]) - inc) < 1e-4


def test_angles_los_and_diffraction(O):
    """LOS: AoD points TX -> RX, AoA RX -> TX.  Diffraction on the z-axis edge, TX (1,0,0), RX
    (0,1,2): vertex (0,0,1); the incidence angle is the Keller cone angle to the edge, 45 deg;
    AoD az 180, el 45; AoA from RX (0,1,2) toward (0,0,1): az -90, el -45."""
    g = GOLD["edge_example"]
    case = edge_case(O, g["tx"], g["rx"], g["a"], g["b"])
    los = np.zeros(1, O.COARSE_DTYPE)
    r = O.refine(case, los)[0]
    d = np.array(g["rx"], float) - g["tx"]
    az = math.degrees(math.atan2(d[1], d[0]))
    el = math.degrees(math.asin(d[2] / np.linalg.norm(d)))
    assert _close_deg(_angles(r), (az, el, math.degrees(math.atan2(-d[1], -d[0])), -el))
    c = coarse_rec(O, [(0.0, 0.0, 0.7)], [100], [0], kinds=1)
    r = O.refine(case, c)[0]
    assert O.STATUS[int(r["status"])] == "OK"
    assert _close_deg(_angles(r), (180.0, 45.0, -90.0, -45.0))
    assert abs(float(r["inc"][0]) - 45.0) < 1e-4


# ---------------------------------------------------------------- R37 analytic Jacobian --
def test_analytic_jacobian_equals_central_differences(O):
    """R37: the analytic Jacobian (chain rule through g, the MLS point/normal of Eqs. 2-4 and the
    (u, v) basis) equals central differences of the residual to their own accuracy (~1e-9
    relative at h = 1e-6..1e-7) on noisy synthetic-room paths with reflections and a
    diffraction; a wrong term (sign, index, transposed block) shows at 1e-3 or worse."""
    case = G.case("C2s", sigma=0.010, n=30_000, n_rays=15_000, max_diff=1, max_refl=2)
    co, _, _ = O.launch_phased(case, procs=os.cpu_count() or 1)
    sc = O.OracleScene(case.scene)
    checked = 0
    for i in range(0, len(co), max(1, len(co) // 30)):
        Ja = O.path_jacobian(case, co[i], scene=sc)
        if Ja is None:
            continue
        errs = []
        for h in (1e-5, 1e-6, 1e-7):
            Jf = O.path_jacobian(case, co[i], fd=True, h=h, scene=sc)
            errs.append(np.abs(Ja - Jf).max() / max(1e-12, np.abs(Ja).max()))
        assert min(errs) < 2e-8, (i, errs)
        checked += 1
    assert checked >= 20
    # and at a point away from the seed (z shifted by 3 mm on every unknown)
    r, z = O.path_residual(case, co[len(co) // 2], scene=sc)
    z2 = z + 0.003
    Ja = O.path_jacobian(case, co[len(co) // 2], z=z2, scene=sc)
    Jf = O.path_jacobian(case, co[len(co) // 2], z=z2, fd=True, h=1e-6, scene=sc)
    assert np.abs(Ja - Jf).max() / np.abs(Ja).max() < 1e-7


def test_analytic_jacobian_planar_closed_form(O):
    """On one plane z = 0 (noise-free, normals +z) the MLS point/normal derivatives are closed
    forms: dn/dx = 0, f = x_z, so the third residual row is (0, 0, 1) for the vertex and 0 for
    its neighbours; rows 1-2 are u, v projected (d g / d x)."""
    sc = plane_scene([(0.0, 1.0)])
    case = make_case(sc, (0.0, 0.0, 1.0), (2.0, 0.0, 1.0))
    c = coarse_rec(O, [(1.02, 0.01, 0.0)], [0], [nearest_id(sc, (1.02, 0.01, 0), 0)])
    J = O.path_jacobian(case, c)
    assert J.shape == (3, 3)
    assert np.allclose(J[2], [0, 0, 1], atol=1e-9)
    x = np.array([1.02, 0.01, 0.0])
    a, b = x - (0, 0, 1.0), x - (2.0, 0, 1.0)
    Ma = (np.eye(3) - np.outer(a, a) / (a @ a)) / np.linalg.norm(a)
    Mb = (np.eye(3) - np.outer(b, b) / (b @ b)) / np.linalg.norm(b)
    # basis of n = +z: axis x (smallest |n.a|, ties x<y<z), u = normalize(z x x) = +y, v = z x y = -x
    u, v = np.array([0, 1.0, 0]), np.array([-1.0, 0, 0])
    assert np.allclose(J[0], u @ (Ma + Mb), atol=1e-9)
    assert np.allclose(J[1], v @ (Ma + Mb), atol=1e-9)
