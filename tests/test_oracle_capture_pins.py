"""Pins of the oracle's capture and diffraction arithmetic (readings R12-R16 of DESIGN.md §2)
against closed-form geometry, a textbook group-by and an independent wedge scene.

  R12  RX reception sphere: capture iff 0 < t_j < t_hit and |perp| <= c_R omega (L + t_j)
       (the classical reception sphere; omega = sqrt(4 pi / N)).
  R13  edge capture: 0 <= s <= len, 0 < t_e < t_hit + b_e, dist <= c_R omega (L + t_e)
       (DEIE bias "reduce the maximum length by a small bias").
  R14  event dedupe: per (history, edge, floor(s / ds)) keep min (dist^2, ray id).
  R15/R16  Keller fan from an exterior wedge (Eq. 14) and the capture radius
       R_d = kR s' + ds/2, kR = c_R (n pi / M) |sin theta|.
None of these retypes an oracle formula: each builds a geometry whose answer is fixed by
construction (a receiver placed at a chosen perpendicular distance, an edge through a chosen
point, a wedge whose only path is the diffracted one) or compares with a numpy group-by.
"""
import math

import numpy as np

import nrt_gen as G

OMEGA_N = 100  # a coarse lattice: omega = 0.354 rad, so capture radii are large and exact


def far_scene(extra_pts=(), extra_n=(), r=0.01, edges=None):
    """A scene whose only surfels are far away (or the given ones)."""
    P = [[1000.0, 1000.0, 1000.0]] + [list(p) for p in extra_pts]
    Nn = [[0.0, 0.0, 1.0]] + [list(n) for n in extra_n]
    m = len(P)
    return G.Scene(np.array(P, np.float32), np.array(Nn, np.float32), np.full(m, r, np.float32),
                   np.arange(m, dtype=np.int32), edges or G.Edges.empty())


def case_of(scene, tx, rx, n_rays=OMEGA_N, max_refl=1, max_diff=0, **kw):
    c = G.LaunchCase("pin", scene, np.asarray(tx, np.float32),
                     np.asarray(rx, np.float32).reshape(-1, 3), n_rays, max_refl, max_diff, 0.5,
                     tau=0.0015)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def perp_unit(d):
    u = np.cross(d, [0.0, 0.0, 1.0])
    if np.linalg.norm(u) < 1e-3:
        u = np.cross(d, [1.0, 0.0, 0.0])
    return u / np.linalg.norm(u)


# ---------------------------------------------------------------- R12 -------------------
def test_rx_sphere_radius_closed_form(O):
    """An escaping primary ray i and a receiver at distance D along it, offset by delta
    perpendicular: captured iff delta <= c_R omega D (L = 0), with L_record = D."""
    tx = np.array([0.5, -0.3, 1.0])
    omega = math.sqrt(4 * math.pi / OMEGA_N)
    for i, D, c_R in ((7, 3.0, 1.0), (42, 1.7, 1.0), (63, 5.0, 0.5)):
        d = O.fib_dir(i, OMEGA_N).astype(np.float64)
        u = perp_unit(d)
        R = c_R * omega * D
        for f, expect in ((1 - 1e-5, True), (1 + 1e-5, False), (0.3, True), (2.0, False)):
            rx = tx + D * d + f * R * u
            case = case_of(far_scene(), tx, rx, c_R=c_R)
            raw, _, nb = O.trace_rays(case, [i])
            assert (len(raw) == 1) == expect, (i, D, f)
            assert nb == 1  # escape: one segment
            if expect:
                assert abs(raw[0]["L"] - D) < 1e-5 and raw[0]["n_int"] == 0
                assert raw[0]["ray_id"] == i
    # behind the origin (t_j < 0): never
    d = O.fib_dir(7, OMEGA_N).astype(np.float64)
    raw, _, _ = O.trace_rays(case_of(far_scene(), tx, tx - 2.0 * d), [7])
    assert len(raw) == 0


def test_rx_sphere_after_reflection_uses_unfolded_length(O):
    """One large disk on z = 0 below the TX: ray i reflects at h after L1, the receiver sits at
    D2 along the reflected ray, offset delta: captured iff delta <= omega (L1 + D2); a receiver
    beyond the disk plane (t_j >= t_hit) on the incident segment is never captured."""
    tx = np.array([0.2, 0.1, 1.0])
    omega = math.sqrt(4 * math.pi / OMEGA_N)
    sc = far_scene([(0.0, 0.0, 0.0)], [(0.0, 0.0, 1.0)], r=20.0)
    i = next(k for k in range(OMEGA_N) if O.fib_dir(k, OMEGA_N)[2] < -0.5)
    d = O.fib_dir(i, OMEGA_N).astype(np.float64)
    L1 = tx[2] / -d[2]
    h = tx + L1 * d
    dr = d * np.array([1, 1, -1])
    u = perp_unit(dr)
    D2 = 1.3
    R = omega * (L1 + D2)
    for f, expect in ((1 - 1e-5, True), (1 + 1e-5, False)):
        rx = h + D2 * dr + f * R * u
        raw, hits, nb = O.trace_rays(case_of(sc, tx, rx), [i])
        assert hits[0][0] == 1 and nb == 2
        got = [r for r in raw if r["n_int"] == 1]
        assert (len(got) == 1) == expect
        if expect:
            assert abs(got[0]["L"] - (L1 + D2)) < 1e-5
            assert np.allclose(got[0]["v"][0], h, atol=1e-5)
    # a receiver below the disk plane on the incident line: t_j > t_hit -> not captured
    rx = tx + (L1 + 0.5) * d
    raw, _, _ = O.trace_rays(case_of(sc, tx, rx), [i])
    assert not any(r["n_int"] == 0 for r in raw)


# ---------------------------------------------------------------- R13 -------------------
def edge_through(c, e, length, s0):
    """An edge along unit e whose parameter s0 sits at point c; faces irrelevant here."""
    a = c - s0 * e
    b = a + length * e
    z = np.zeros((1, 3), np.float32)
    return G.Edges(a[None].astype(np.float32), b[None].astype(np.float32), z + [[1, 0, 0]],
                   z + [[0, 1, 0]], z + [[0, 0, 1]], np.array([1.5], np.float32),
                   np.array([900], np.int32))


def events_of(O, case, i):
    raw, ev, nb = O.trace_primary(case, rank=i, world=case.n_rays)
    return ev


def test_edge_capture_windows_closed_form(O):
    """An edge crossing ray i perpendicularly at distance D, offset delta: the closest point is
    (t_e, s) = (D, s0), dist = delta; captured iff delta <= omega D, 0 <= s0 <= len and
    t_e < t_hit + b_e (b_e = r_max + tau)."""
    tx = np.array([0.0, 0.0, 1.0])
    omega = math.sqrt(4 * math.pi / OMEGA_N)
    i = 31
    d = O.fib_dir(i, OMEGA_N).astype(np.float64)
    e = perp_unit(d)
    n = np.cross(d, e)
    D, length = 2.0, 1.0
    R = omega * D

    def run(delta, s0, wall_at=None, rwall=0.02):
        extra = [] if wall_at is None else [tx + wall_at * d]
        extra_n = [] if wall_at is None else [d]
        sc = far_scene(extra, extra_n, r=rwall, edges=edge_through(tx + D * d + delta * n, e, length, s0))
        case = case_of(sc, tx, [[40.0, 40.0, 40.0]], max_diff=1, edge_bin=0.25)
        return events_of(O, case, i), case

    ev, _ = run(R * (1 - 1e-5), 0.4)
    assert len(ev) == 1
    assert abs(ev[0]["s"] - 0.4) < 1e-5 and abs(math.sqrt(ev[0]["dist2"]) - R * (1 - 1e-5)) < 1e-5
    assert abs(ev[0]["L"] - D) < 1e-5
    assert ev[0]["sbin"] * 0.25 <= ev[0]["s"] < (ev[0]["sbin"] + 1) * 0.25
    assert len(run(R * (1 + 1e-5), 0.4)[0]) == 0
    # s window [0, len]
    assert len(run(0.5 * R, -0.01)[0]) == 0
    assert len(run(0.5 * R, 0.01)[0]) == 1
    assert len(run(0.5 * R, length - 0.01)[0]) == 1
    assert len(run(0.5 * R, length + 0.01)[0]) == 0
    # t_e window: a wall across the ray at t_hit; b_e = r_max + tau = 0.02 + 0.0015
    b_e = 0.02 + 0.0015
    assert len(run(0.5 * R, 0.4, wall_at=D - b_e + 0.002)[0]) == 1
    assert len(run(0.5 * R, 0.4, wall_at=D - b_e - 0.002)[0]) == 0
    # behind the origin: t_e < 0
    sc = far_scene(edges=edge_through(tx - D * d, e, length, 0.4))
    assert len(events_of(O, case_of(sc, tx, [[40, 40, 40]], max_diff=1), i)) == 0


# ---------------------------------------------------------------- R14 -------------------
def test_event_dedupe_keeps_min_per_key(O):
    rng = np.random.default_rng(21)
    n = 4000
    E = np.zeros(n, O.EVENT_DTYPE)
    E["h"]["n"] = rng.integers(0, 3, n)
    for k in range(2):
        E["h"]["label"][:, k] = np.where(E["h"]["n"] > k, rng.integers(0, 3, n), 0)
    E["edge"] = rng.integers(0, 4, n)
    E["sbin"] = rng.integers(0, 3, n)
    E["dist2"] = rng.integers(0, 20, n).astype(np.float32) / 9
    E["ray_id"] = rng.permutation(n)
    out = O.event_dedupe(E)

    def key(r):
        h = r["h"]
        return (int(h["n"]), int(h["kinds"]), tuple(int(x) for x in h["label"]), int(r["edge"]),
                int(r["sbin"]))
    groups = {}
    for r in E:
        groups.setdefault(key(r), []).append((float(r["dist2"]), int(r["ray_id"])))
    expect = [(k, min(v)) for k, v in sorted(groups.items())]
    got = [(key(r), (float(r["dist2"]), int(r["ray_id"]))) for r in out]
    assert got == expect


# ---------------------------------------------------------------- R15/R16 wedge ---------
def wedge_scene(h=0.02, r=0.016, zmax=2.0, ext=1.5):
    """A solid occupying x < 0, y < 0 (0 <= z <= zmax): face 0 = plane y = 0 (x < 0, outward
    +y), face 1 = plane x = 0 (y < 0, outward +x); the exterior wedge (270 deg, n = 1.5) is the
    z axis.  Surfels on both faces, one label per face."""
    u = np.arange(h / 2, ext, h)
    z = np.arange(h / 2, zmax, h)
    U, Z = np.meshgrid(u, z, indexing="ij")
    f0 = np.stack([-U.ravel(), np.zeros(U.size), Z.ravel()], 1)
    f1 = np.stack([np.zeros(U.size), -U.ravel(), Z.ravel()], 1)
    P = np.concatenate([f0, f1]).astype(np.float32)
    Nn = np.concatenate([np.tile([0, 1.0, 0], (len(f0), 1)), np.tile([1.0, 0, 0], (len(f1), 1))])
    L = np.concatenate([np.zeros(len(f0), np.int32), np.ones(len(f1), np.int32)])
    E = G.Edges(np.array([[0, 0, 0]], np.float32), np.array([[0, 0, zmax]], np.float32),
                np.array([[-1, 0, 0]], np.float32), np.array([[0, 1, 0]], np.float32),
                np.array([[1, 0, 0]], np.float32), np.array([1.5], np.float32),
                np.array([77], np.int32))
    return G.Scene(P, Nn.astype(np.float32), np.full(len(P), r, np.float32), L, E)


def test_wedge_shadow_zone_only_the_diffraction_key(O):
    """TX above face 0, RX beside face 1: the direct line crosses the solid and no reflection
    connects them, so with max_refl = 0 the coarse key set is exactly {[edge]}; every fan record
    keeps Keller's cone (the angle to the edge of RX - v equals that of v - TX within the capture
    radius) and its receiver lies within R_d = kR t + ds/2 of its fan ray (Eq. 14 directions)."""
    sc = wedge_scene()
    tx, rx = np.array([-0.8, 0.3, 1.3]), np.array([0.3, -0.8, 0.9])
    case = case_of(sc, tx, rx, n_rays=20_000, max_refl=0, max_diff=1, kappa=1 << 30,
                   edge_bin=0.25, dphi_deg=2.5)
    recs, n_raw, nb, ev = O.launch_phased(case, procs=8, return_events=True)
    keys = {(int(r["n_int"]), int(r["kinds"]), tuple(int(x) for x in r["label"][: r["n_int"]]))
            for r in recs}
    assert keys == {(1, 1, (77,))}
    assert len(ev) > 0 and len(recs) > 0
    e = np.array([0.0, 0.0, 1.0])
    omega = math.sqrt(4 * math.pi / case.n_rays)
    edge = O.make_edge((0, 0, 0), (0, 0, 2), (-1, 0, 0), (0, 1, 0), (1, 0, 0), n_exp=1.5, label=77)
    for r in recs:
        v = r["v"][0].astype(np.float64)
        assert abs(v[0]) < 1e-6 and abs(v[1]) < 1e-6 and abs(v[2] - r["s_edge"]) < 1e-5
        rank, m = (int(r["ray_id"]) & ((1 << 63) - 1)) >> 8, int(r["ray_id"]) & 0xFF
        x = ev[rank]
        M = O.fan_dirs(edge, x["d"], 2.5).shape[0]
        f = O.fan_dirs(edge, x["d"], 2.5)[m].astype(np.float64)
        t = (rx - v) @ f
        perp = np.linalg.norm((rx - v) - t * f)
        st = math.sqrt(max(0.0, 1 - float(x["d"] @ e) ** 2))
        Rd = (1.5 * math.pi / M) * st * t + 0.125
        assert t > 0 and perp <= Rd * (1 + 1e-5) + 1e-6
        # Keller's cone: the incident ray's angle to the edge (the event's direction) equals the
        # fan ray's; RX - v deviates from the fan ray by at most perp
        assert abs(f @ e - float(x["d"] @ e)) < 1e-6
        ca = ((rx - v) @ e) / np.linalg.norm(rx - v)
        A = np.linalg.norm(rx - v)
        assert abs(ca - f @ e) <= perp / A + perp ** 2 / (2 * A * A) + 1e-6
        # the event's incident ray came from the TX within the capture radius of the edge point
        w = v - tx
        assert abs((w @ e) / np.linalg.norm(w) - float(x["d"] @ e)) < omega * 1.5
