"""Pins of the CPU oracle's COARSE part against what the paper and mathematics fix
(P1, P3, P4, P5, P13, P14-style brute force, R13, R15, R17).

None of these re-types the oracle's formula: each compares it with a closed form, an
invariant, a library routine (numpy linear algebra, math.sin/cos) or brute force.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import nrt_gen as G

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


# ---------------------------------------------------------------- R2: sincos ------------
def test_sincos_matches_libm(O):
    rng = np.random.default_rng(1)
    xs = np.concatenate([rng.random(20000) * 2 * math.pi, np.linspace(0, 2 * math.pi, 4097),
                         [0.0, math.pi / 4, math.pi / 2, math.pi, 1.5 * math.pi]])
    for x in xs:
        s, c = O.sincos(float(x))
        assert abs(s - math.sin(x)) <= 4e-16, x
        assert abs(c - math.cos(x)) <= 4e-16, x


# ---------------------------------------------------------------- P1: Fibonacci ---------
@pytest.mark.parametrize("N", [10_000, 100_000])
def test_fibonacci_lattice_closed_form_and_covering(O, N):
    """R1: z_i exact, |d| = 1 to f32 rounding, covering radius <= 0.75 omega."""
    ids = np.arange(N)
    D = O.fib_dirs(N, ids) if N <= 10_000 else O.fib_dirs(N, ids)
    z_exact = (1.0 - (2.0 * ids + 1.0) / N).astype(np.float32)
    assert np.array_equal(D[:, 2], z_exact)
    nrm = np.linalg.norm(D.astype(np.float64), axis=1)
    assert np.max(np.abs(nrm - 1.0)) <= 2.0 ** -22
    # azimuth: phi = 2 pi frac(i g) -> compare with numpy's atan2 of the f32 direction
    g = (3.0 - math.sqrt(5.0)) / 2.0
    phi = 2 * math.pi * np.modf(ids * g)[0]
    phi_d = np.mod(np.arctan2(D[:, 1].astype(np.float64), D[:, 0].astype(np.float64)), 2 * math.pi)
    err = np.abs(np.angle(np.exp(1j * (phi - phi_d))))
    rr = np.sqrt(1 - z_exact.astype(np.float64) ** 2)
    ok = rr > 1e-3
    assert np.max(err[ok] * rr[ok]) < 1e-6
    from scipy.spatial import cKDTree
    rng = np.random.default_rng(7)
    q = rng.standard_normal((200_000, 3))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    dist, _ = cKDTree(D.astype(np.float64)).query(q)
    ang = 2 * np.arcsin(np.minimum(1.0, dist / 2))
    omega = math.sqrt(4 * math.pi / N)
    assert ang.max() <= 0.75 * omega
    assert abs(O.cRw(1.0, N) - omega) <= 1e-7 * omega


# ---------------------------------------------------------------- P3: HIT predicate -----
def test_hit_closed_forms(O):
    z = (0, 0, 1)
    # ray from (0,0,1) along -z onto a disk at the origin: t = 1 exactly
    assert O.hit((0, 0, 1), (0, 0, -1), (0, 0, 0), z, 0.1) == 1.0
    # two-sided: from below as well
    assert O.hit((0, 0, -2), (0, 0, 1), (0, 0, 0), z, 0.1) == 2.0
    # boundary q.q = r^2 is a hit (inclusive); just outside is not
    assert O.hit((0.5, 0, 1), (0, 0, -1), (0, 0, 0), z, 0.5) == 1.0
    assert O.hit((0.5, 0, 1), (0, 0, -1), (0, 0, 0), z, np.nextafter(np.float32(0.5), 0)) is None
    # parallel ray never hits; receding ray never hits
    assert O.hit((0, 0, 1), (1, 0, 0), (0, 0, 0), z, 10.0) is None
    assert O.hit((0, 0, 1), (0, 0, 1), (0, 0, 0), z, 10.0) is None
    # departure sheet: origin within tau of a parallel surfel -> transparent
    d = np.array([0.6, 0, -0.8], np.float32)
    assert O.hit((0, 0, 0.001), d, (0.0007, 0, 0), z, 0.05, lam=[z], tau=0.0015) is None
    assert O.hit((0, 0, 0.001), d, (0.0007, 0, 0), z, 0.05, lam=[], tau=0.0015) is not None
    # ...but beyond tau it is a surface again
    assert O.hit((0, 0, 0.01), d, (0.0075, 0, 0), z, 0.05, lam=[z], tau=0.0015) is not None
    # a perpendicular sheet is never excluded (corners stay closed)
    assert O.hit((0.001, 0, 0.5), (-0.8, 0, -0.6), (0, 0, 0.5), (1, 0, 0), 0.05,
                 lam=[z], tau=0.0015) is not None


def test_hit_vs_float64_brute_force(O):
    """Random disks: the predicate agrees with an FP64 ray-plane-disk solve (numpy linalg)
    away from the knife edges (|q| - r and f0 at least 1e-4 relative)."""
    rng = np.random.default_rng(3)
    agree = 0
    for _ in range(3000):
        o = rng.uniform(-1, 1, 3)
        d = rng.standard_normal(3)
        d /= np.linalg.norm(d)
        p = rng.uniform(-1, 1, 3)
        n = rng.standard_normal(3)
        n /= np.linalg.norm(n)
        r = rng.uniform(0.05, 1.0)
        o32, d32, p32, n32 = (x.astype(np.float32) for x in (o, d, p, n))
        r32 = np.float32(r)
        o, d, p, n, r = (x.astype(np.float64) for x in (o32, d32, p32, n32, r32))
        # plane solve: o + t d = p + a u + b v
        u = np.cross(n, [1, 0, 0] if abs(n[0]) < 0.9 else [0, 1, 0])
        u /= np.linalg.norm(u)
        v = np.cross(n, u)
        A = np.stack([d, -u, -v], 1)
        if abs(np.linalg.det(A)) < 1e-3:
            continue
        t, a, b = np.linalg.solve(A, p - o)
        rad = math.hypot(a, b)
        if abs(rad - r) < 1e-4 * max(r, 1) or abs(t) < 1e-4:
            continue
        expect = (t > 0) and rad <= r
        got = O.hit(o32, d32, p32, n32, r32, lam=[], tau=0.0)
        assert (got is not None) == expect
        if expect:
            assert abs(got - t) <= 1e-5 * max(1.0, t)
        agree += 1
    assert agree > 1500


def test_nearest_is_global_argmin_with_id_tiebreak(O):
    """Brute-force argmin semantics (R9): equal t -> lower id; prev is skipped."""
    z = np.array([0, 0, 1], np.float32)
    pts = np.array([[0, 0, 0], [0.01, 0, 0], [0, 0, 0.5], [0, 0, 0.5]], np.float32)
    sc = G.Scene(pts, np.repeat(z[None], 4, 0), np.full(4, 0.1, np.float32), np.zeros(4, np.int32),
                 G.Edges.empty())
    osc = O.OracleScene(sc)
    s, t = O.nearest(osc, (0, 0, 1), (0, 0, -1))
    assert (s, t) == (2, 0.5)               # two coincident surfels at z=0.5: lower id
    s, t = O.nearest(osc, (0, 0, 1), (0, 0, -1), prev=2)
    assert (s, t) == (3, 0.5)
    s, t = O.nearest(osc, (0, 0, 0.2), (0, 0, -1))
    assert (s, t) == (0, np.float32(0.2))   # (0,0,0) and (0.01,0,0) tie in t -> id 0
    s, t = O.nearest(osc, (0, 0, 1), (0, 0, 1))
    assert s == -1 and math.isinf(t)


# ---------------------------------------------------------------- P4: reflection -------
def test_reflection_identities(O):
    assert np.array_equal(O.reflect((0, 0, -1), (0, 0, 1)), np.float32([0, 0, 1]))
    s = np.float32(math.sqrt(0.5))
    r = O.reflect((s, 0, -s), (0, 0, 1))
    assert np.allclose(r, [s, 0, s], atol=1e-7)
    rng = np.random.default_rng(5)
    for _ in range(2000):
        d = rng.standard_normal(3)
        d /= np.linalg.norm(d)
        n = rng.standard_normal(3)
        n /= np.linalg.norm(n)
        d32, n32 = d.astype(np.float32), n.astype(np.float32)
        out = O.reflect(d32, n32).astype(np.float64)
        assert abs(np.linalg.norm(out) - 1) <= 2 ** -22
        assert abs(out @ n32 + d32.astype(np.float64) @ n32) <= 1e-6
        # reflection is an involution up to rounding
        back = O.reflect(out.astype(np.float32), n32).astype(np.float64)
        assert np.allclose(back, d32, atol=1e-6)


# ---------------------------------------------------------------- R13: edge closest ----
def test_edge_closest_point_vs_linear_solve(O):
    rng = np.random.default_rng(11)
    for _ in range(500):
        a = rng.uniform(-1, 1, 3).astype(np.float32)
        b = (a + rng.uniform(-1, 1, 3)).astype(np.float32)
        o = rng.uniform(-2, 2, 3).astype(np.float32)
        d = rng.standard_normal(3)
        d = (d / np.linalg.norm(d)).astype(np.float32)
        e = O.make_edge(a, b, (0, 0, 0), (0, 0, 0), (0, 0, 0))
        res = O.edge_closest(o, d, e)
        ev = b.astype(np.float64) - a
        L = np.linalg.norm(ev)
        ev /= L
        dd = d.astype(np.float64)
        # minimise |o + t d - a - s e|^2: normal equations (library solve)
        A = np.array([[dd @ dd, -dd @ ev], [-dd @ ev, ev @ ev]])
        if abs(np.linalg.det(A)) < 1e-4:
            continue
        w = a.astype(np.float64) - o
        t, s = np.linalg.solve(A, [dd @ w, -(ev @ w)])
        assert res is not None
        te, s32, d2 = res
        assert abs(te - t) < 2e-4 * max(1, abs(t)) and abs(s32 - s) < 2e-4 * max(1, abs(s))
        dist2 = np.sum((o + t * dd - a - s * ev) ** 2)
        assert abs(d2 - dist2) < 1e-4


# ---------------------------------------------------------------- R15: Keller fan ------
def test_keller_fan_counts_and_geometry(O):
    g = GOLD["keller_fan_counts"]
    e = O.make_edge((0, 0, 0), (0, 0, 2), (0, 1, 0), (-1, 0, 0), (0, -1, 0), n_exp=g["n_exp"])
    for theta, M in g["theta_deg_to_M"]:
        th = math.radians(theta)
        d = np.array([-math.sin(th), 0.0, math.cos(th)], np.float32)  # angle theta to e = +z
        F = O.fan_dirs(e, d, g["dphi_deg"])
        assert F.shape[0] == M
    # default 2.5 deg step: M0 = 108
    d = np.array([-1, 0, 0], np.float32)
    F = O.fan_dirs(e, d, 2.5).astype(np.float64)
    assert F.shape[0] == 108
    rng = np.random.default_rng(2)
    for _ in range(200):
        d = rng.standard_normal(3)
        d /= np.linalg.norm(d)
        d32 = d.astype(np.float32)
        F = O.fan_dirs(e, d32, 2.5).astype(np.float64)
        if F.shape[0] == 0:
            continue
        ct = float(d32.astype(np.float64)[2])
        # Keller cone: every fan ray keeps the incident angle to the edge (Eq. 14)
        assert np.allclose(F[:, 2], ct, atol=1e-6)
        assert np.allclose(np.linalg.norm(F, axis=1), 1.0, atol=1e-6)
        # M = max(1, ceil(108 |sin theta|))
        assert F.shape[0] == max(1, math.ceil(108 * math.sqrt(max(0.0, 1 - ct * ct)) - 1e-12))
        # no fan ray enters the solid (interior quadrant: x > 0 and y > 0 for this corner)
        interior = (F[:, 0] > 1e-6) & (F[:, 1] > 1e-6)
        assert not interior.any()


# ---------------------------------------------------------------- R17: dedupe law ------
def test_dedupe_kappa_bucket_law(O):
    rng = np.random.default_rng(9)
    n = 3000
    R = np.zeros(n, O.COARSE_DTYPE)
    R["rx"] = rng.integers(0, 3, n)
    R["n_int"] = rng.integers(0, 3, n)
    for k in range(2):
        R["label"][:, k] = np.where(R["n_int"] > k, rng.integers(0, 4, n), 0)
    R["L"] = rng.integers(0, 50, n).astype(np.float32) / 7
    R["ray_id"] = rng.permutation(n)
    for kappa in (1, 3, 100):
        out = O.dedupe(R, kappa)
        key = lambda r: (int(r["rx"]), int(r["n_int"]), int(r["kinds"]), tuple(int(x) for x in r["label"]))
        groups = {}
        for r in R:
            groups.setdefault(key(r), []).append((float(r["L"]), int(r["ray_id"])))
        expect = []
        for k in sorted(groups):
            expect += [(k, x) for x in sorted(groups[k])[:kappa]]
        got = [(key(r), (float(r["L"]), int(r["ray_id"]))) for r in out]
        assert got == expect


# ---------------------------------------------------------------- P5: image method -----
def _image_paths(room, tx, rx, kmax):
    """Independent FP64 image-method enumeration in a shoebox (textbook special case)."""
    walls = [(0, 0.0), (0, room[0]), (1, 0.0), (1, room[1]), (2, 0.0), (2, room[2])]
    out = {}
    for k in range(kmax + 1):
        for seq in itertools.product(range(6), repeat=k):
            if any(seq[i] == seq[i + 1] for i in range(k - 1)):
                continue
            imgs = [np.array(tx, float)]
            for w in seq:
                ax, c = walls[w]
                q = imgs[-1].copy()
                q[ax] = 2 * c - q[ax]
                imgs.append(q)
            pts = []
            tgt = np.array(rx, float)
            ok = True
            for j in range(k, 0, -1):
                ax, c = walls[seq[j - 1]]
                src = imgs[j]
                den = tgt[ax] - src[ax]
                if abs(den) < 1e-12:
                    ok = False
                    break
                t = (c - src[ax]) / den
                if not (0 < t < 1):
                    ok = False
                    break
                p = src + t * (tgt - src)
                if np.any(p < -1e-9) or np.any(p > np.array(room) + 1e-9):
                    ok = False
                    break
                pts.append(p)
                tgt = p
            if ok:
                out[seq] = (float(np.linalg.norm(imgs[-1] - np.array(rx, float))), pts[::-1])
    return out


def test_image_method_counts_match_paper_examples():
    g = GOLD["box_room_images"]
    paths = _image_paths(g["room"], g["tx"], g["rx"], 5)
    cnt = [sum(1 for s in paths if len(s) == k) for k in range(6)]
    assert cnt == g["count_by_order"]
    assert abs(paths[()][0] - g["los_length"]) < 1e-4
    assert abs(max(v[0] for s, v in paths.items() if len(s) == 2) - g["max_len_order2"]) < 1e-4


def test_box_room_coarse_set_is_the_image_method_set(O):
    """P5: C1's coarse key set == the 25 image paths of order <= 2; lengths and vertices close."""
    case = G.case("C1")
    recs, n_raw, nb = O.launch_phased(case, procs=os.cpu_count() or 1)
    paths = _image_paths((4.0, 3.0, 2.5), case.tx.tolist(), case.rx[0].tolist(), 2)
    keys = {tuple(int(x) for x in r["label"][: r["n_int"]]): r for r in recs}
    assert len(recs) == len(keys) == 25
    assert set(keys) == set(paths)
    omega = math.sqrt(4 * math.pi / case.n_rays)
    walls = [(0, 0.0), (0, 4.0), (1, 0.0), (1, 3.0), (2, 0.0), (2, 2.5)]
    for seq, r in keys.items():
        L_img, pts = paths[seq]
        assert abs(float(r["L"]) - L_img) < 0.05
        for k, w in enumerate(seq):
            ax, c = walls[w]
            assert abs(float(r["v"][k][ax]) - c) < 1e-5           # vertex on its wall plane
            assert np.linalg.norm(r["v"][k] - pts[k]) < 2 * omega * L_img
    # every primary ray traces at most max_refl+1 segments; the box is closed so exactly that
    assert nb == case.n_rays * (case.max_refl + 1)


# ---------------------------------------------------------------- P13: noise at 0 ------
def test_noise_generator_sigma_zero_is_bit_identical():
    a = G.synth_room(20_000, 0.0)
    b = G.synth_room(20_000, 0.0, seed=G.SEED)
    p = G.add_normal_noise(a.points, a.normals, 0.0, 123)
    assert p.tobytes() == a.points.tobytes() == b.points.tobytes()
    c = G.synth_room(20_000, 0.005)
    assert c.points.tobytes() != a.points.tobytes()
    disp = np.sum((c.points.astype(np.float64) - a.points) * a.normals, axis=1)
    assert abs(disp.std() - 0.005) < 0.0003
    tang = (c.points - a.points) - disp[:, None] * a.normals
    assert np.abs(tang).max() < 1e-6


def test_oracle_sharded_equals_single(O):
    """Per-ray independence: the phased multi-process oracle equals the single pass."""
    case = G.case("C2s", n=6000, n_rays=3000, max_refl=2)
    a = O.launch(case)
    b = O.launch_phased(case, procs=3)
    assert a[1:] == b[1:]
    assert a[0].tobytes() == b[0].tobytes()
