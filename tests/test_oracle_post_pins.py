"""Pins of the CPU oracle's refined-path POST-PROCESSING (PAPER.md
§II-E, R33-R36): the first-Fresnel-zone radius of Eq. 13 in closed form
(P15 / S:556), the nearest-point label against a numpy brute force, and the greedy dedupe's
defining properties (min-delay representative, containment boundary, angle threshold,
duplicate-free output in delay order)."""
import math

import numpy as np
import pytest

import nrt_gen as G

C_LIGHT = 299792458.0


def two_label_plane(h=0.01):
    """Plane z = 0, x in [-0.5, 0.5], y in [-0.5, 0.5]; label 0 for x < 0, label 1 for x >= 0."""
    xs = np.arange(-0.5 + h / 2, 0.5, h)
    X, Y = np.meshgrid(xs, xs, indexing="ij")
    P = np.stack([X.ravel(), Y.ravel(), np.zeros(X.size)], 1).astype(np.float32)
    N = np.tile(np.float32([0, 0, 1]), (P.shape[0], 1))
    L = (P[:, 0] >= 0).astype(np.int32)
    return G.Scene(P, N, np.full(P.shape[0], 0.008, np.float32), L, G.Edges.empty())


def case_for(scene, tx, rx):
    return G.LaunchCase("post", scene, np.asarray(tx, np.float32),
                        np.asarray(rx, np.float32).reshape(-1, 3), 1000, 2, 0, 0.1, r_s=0.003,
                        tau=0.0015)


def rec(O, verts, labels, L=None, rx=0, tx=None, rxp=None):
    r = np.zeros(1, O.REFINED_DTYPE)
    r["rx"] = rx
    r["n_int"] = len(verts)
    for k, (v, l) in enumerate(zip(verts, labels)):
        r["v"][0, k] = v
        r["label"][0, k] = l
    if L is None:
        pts = [tx] + list(verts) + [rxp]
        L = sum(float(np.linalg.norm(np.subtract(pts[i + 1], pts[i]))) for i in range(len(pts) - 1))
    r["L"] = L
    r["delay"] = L / C_LIGHT
    return r


TX = (-0.6, 0.0, 0.8)
RXP = (0.6, 0.0, 0.8)


def test_fresnel_radius_closed_form_and_boundary(O):
    """s1 = s2 = 1 m, lambda = 5 mm: psi = sqrt(0.005 * 1 * 1 / 2) = 0.05 m."""
    assert abs(math.sqrt(0.005 * 1 * 1 / 2) - 0.05) < 1e-15
    case = case_for(two_label_plane(), TX, RXP)
    a = rec(O, [(0.0, 0.0, 0.0)], [0], tx=TX, rxp=RXP)
    cos10 = math.cos(math.radians(10.0))
    inside = rec(O, [(0.0499, 0.0, 0.0)], [1], tx=TX, rxp=RXP)
    outside = rec(O, [(0.0501, 0.0, 0.0)], [1], tx=TX, rxp=RXP)
    assert O.fresnel_dup(case, a, inside, cos10, lambda_m=0.005)
    assert not O.fresnel_dup(case, a, outside, cos10, lambda_m=0.005)
    # the same point offset turns the rays by ~2.8 deg: a 2 deg threshold rejects it
    assert not O.fresnel_dup(case, a, inside, math.cos(math.radians(2.0)), lambda_m=0.005)
    # containment is measured with the ACCEPTED path's radius: s1, s2 of `a`
    far = rec(O, [(0.0, 0.3, 0.0)], [0], tx=TX, rxp=RXP)
    assert not O.fresnel_dup(case, a, far, cos10, lambda_m=0.005)


def test_exact_label_is_nearest_point_label(O):
    sc = two_label_plane()
    case = case_for(sc, TX, RXP)
    rng = np.random.default_rng(3)
    for x in list(rng.uniform(-0.02, 0.02, (20, 1))) + [[-0.0001], [0.0001]]:
        v = (float(x[0]), float(rng.uniform(-0.2, 0.2)), 0.001)
        r = rec(O, [v], [7], tx=TX, rxp=RXP)  # coarse label 7 is wrong on purpose
        out = O.postprocess(case, r, r_s=0.003)
        d2 = np.sum((sc.points.astype(np.float64) - np.array(v)) ** 2, 1)
        want = int(sc.labels[np.argmin(d2)]) if d2.min() <= (2 * 0.003) ** 2 else 7
        assert int(out["label"][0, 0]) == want
    # nothing within 2 r_s: the coarse label stays
    r = rec(O, [(0.0, 0.0, 0.05)], [7], tx=TX, rxp=RXP)
    assert int(O.postprocess(case, r, r_s=0.003)["label"][0, 0]) == 7


def test_greedy_dedupe_properties(O):
    sc = two_label_plane()
    case = case_for(sc, TX, RXP)
    rng = np.random.default_rng(11)
    recs = []
    # cluster A near the origin (psi = sqrt(lambda s1 s2/(s1+s2)) ~ 5 cm at 60 GHz, s1 = s2 = 1 m):
    # jitter well inside psi
    for _ in range(6):
        recs.append(rec(O, [(rng.uniform(-0.001, 0.001), rng.uniform(-0.001, 0.001), 0.0)], [0],
                        tx=TX, rxp=RXP))
    # cluster B 3 psi away along y
    for _ in range(4):
        recs.append(rec(O, [(rng.uniform(-0.001, 0.001), 0.15 + rng.uniform(-0.001, 0.001), 0.0)],
                        [0], tx=TX, rxp=RXP))
    allr = np.concatenate(recs)
    # give every record its own (fake) label so that step 2 keeps all of them, then post-process
    # with a tiny r_s so that relabelling finds no point (labels stay distinct)
    allr["label"][:, 0] = np.arange(len(allr)) + 100
    out = O.postprocess(case, allr, r_s=1e-6)
    assert len(out) == 2
    d = allr["delay"]
    assert out["delay"][0] == d[:6].min() or out["delay"][0] == d[6:].min()
    assert set(out["delay"].tolist()) == {d[:6].min(), d[6:].min()}
    assert np.all(np.diff(out["delay"]) >= 0)
    cos10 = math.cos(math.radians(10.0))
    for i in range(len(out)):
        for j in range(i + 1, len(out)):
            assert not O.fresnel_dup(case, out[i], out[j], cos10)


def test_shortest_per_key_after_relabel(O):
    """Two records whose coarse labels differ but whose vertices lie on the same labelled
    region collapse to the shorter one (R28 with the exact labels)."""
    sc = two_label_plane()
    case = case_for(sc, TX, RXP)
    a = rec(O, [(0.2051, 0.0049, 0.0)], [3], L=2.0)
    b = rec(O, [(0.2551, 0.1049, 0.0)], [4], L=1.9)
    out = O.postprocess(case, np.concatenate([a, b]), r_s=0.003, lambda_m=1e-9)
    assert len(out) == 1 and out["L"][0] == pytest.approx(1.9) and out["label"][0, 0] == 1
    # invalid records never take part
    c = rec(O, [(0.2, 0.0, 0.0)], [3], L=1.0)
    c["status"] = 1
    out = O.postprocess(case, np.concatenate([a, c]), r_s=0.003)
    assert len(out) == 1 and out["L"][0] == pytest.approx(2.0)
