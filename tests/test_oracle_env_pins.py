"""Pins of the oracle's NEXT-2 coarse tracer, the paper's environment-driven launch with voxel
cone tracing (oracle/env.c; PAPER §II-B, §II-D, Alg. 1; readings
R60-R67 of DESIGN.md), against closed forms, numpy brute force and the image method:
  * R60 IEs: PCIE points = numpy means of each subvoxel's points, labels = the nearest point to
    the subvoxel centre, DEIE pieces tile the edge with one midpoint per crossed subvoxel;
  * R61 march distances = brute-force Chebyshev distances; the cone angle = atan(V / diagonal);
  * Alg. 1: the step equals the FP64 closed form of the first a-th boundary crossing (+ 1e-2);
  * R62 the cone-sphere test = the sphere's exact distance to the cone surface;
  * a dense box room: every image-method path of order <= 2 is found; a 270 deg wedge with TX
    and RX in the shadow zone: the key set is exactly {[edge]}.
"""
import math
import os

import numpy as np
import pytest

import nrt_gen as G
from tests.test_oracle_capture_pins import case_of, wedge_scene

NPROC = max(1, min(32, os.cpu_count() or 1))
SDF = dict(cell=0.0625, r_s=0.015, t_sdf=0.0015, xi=2.0)


def box_case():
    case = G.case("C1", n_rays=4000)
    case.scene = G.box_room(3)
    case.sdf = dict(SDF)
    case.kappa = 100
    return case


def test_ie_tables(O):
    case = G.case("C2", sigma=0.010, n_rays=1000)
    case.sdf = dict(SDF)
    es = O.EnvScene(case)
    n, n_pc = es.count()
    s = case.scene
    a = np.float32(SDF["cell"])
    org = s.points.min(axis=0)
    cell = np.floor((s.points - org) / a).astype(np.int64)
    dims = np.floor((s.points.max(axis=0) - org) / a).astype(np.int64) + 1
    cell = np.minimum(cell, dims - 1)
    sub = cell // 4
    sv = (dims + 3) // 4
    lin = sub[:, 0] + sv[0] * (sub[:, 1] + sv[1] * sub[:, 2])
    uniq, inv = np.unique(lin, return_inverse=True)
    assert n_pc == len(uniq)
    rng = np.random.default_rng(2)
    S4 = np.float32(4 * a)
    for q in rng.choice(n_pc, 60, replace=False):
        p, kind, label, vox = es.ie(q)
        m = np.nonzero(inv == q)[0]
        assert kind == 0
        assert np.array_equal(p, s.points[m].astype(np.float64).mean(axis=0).astype(np.float32))
        c = org + (sub[m[0]].astype(np.float32) + np.float32(0.5)) * S4
        d2 = ((s.points[m] - c) ** 2).sum(1)
        assert label == s.labels[m[np.argmin(d2)]]
    # DEIE pieces: consecutive along each edge, midpoints in distinct subvoxels
    edges = s.edges
    de = [es.ie(i) for i in range(n_pc, n - len(case.rx))]
    assert len(de) >= len(edges.a)
    for j in range(len(edges.a)):
        pts = [p for p, k, lab, v in de if lab == int(edges.label[j])]
        A, B = edges.a[j].astype(np.float64), edges.b[j].astype(np.float64)
        ev = B - A
        ts = sorted(float((p - A) @ ev / (ev @ ev)) for p in pts)
        assert 0 < ts[0] and ts[-1] < 1
        subs = {tuple(np.floor((p - org) / S4).astype(int)) for p in pts}
        assert len(subs) == len(pts)
        # one piece per subvoxel the segment crosses (FP64 count of boundary crossings + 1)
        cross = 0
        for k in range(3):
            lo, hi = sorted((A[k], B[k]))
            cross += len([m for m in range(-200, 400) if lo < org[k] + m * S4 < hi])
        assert len(pts) == cross + 1
    # RXIEs last, at the receivers
    p, kind, label, vox = es.ie(n - 1)
    assert kind == 2 and np.array_equal(p, case.rx[-1])


def test_march_distance_and_cone_angle(O):
    case = box_case()
    es = O.EnvScene(case)
    vd, V, tan_c, march = es.grid()
    n, _ = es.count()
    occ = np.zeros(int(np.prod(vd)), bool)
    for i in range(n):
        occ[es.ie(i)[3]] = True
    idx = np.stack(np.unravel_index(np.arange(len(occ)), tuple(vd[::-1])), 1)[:, ::-1]
    full = idx[occ]
    for v in range(len(occ)):
        dist = np.abs(full - idx[v]).max(axis=1).min()
        assert march[v] == max(1, dist)
    diag = np.linalg.norm(case.scene.points.max(axis=0).astype(np.float64) - case.scene.points.min(axis=0))
    assert V == np.float32(8 * SDF["cell"])
    assert abs(tan_c - V / diag) < 1e-6


def test_alg1_march_closed_form(O):
    L = O.env_lib()
    rng = np.random.default_rng(3)
    for _ in range(2000):
        v = rng.uniform(0, 20, 3).astype(np.float32)
        d = rng.normal(size=3)
        d = (d / np.linalg.norm(d)).astype(np.float32)
        a = int(rng.integers(1, 6))
        out = np.zeros(3, np.float32)
        L.or_env_march(v.ctypes.data, d.ctypes.data, a, out.ctypes.data)
        V64, D64 = v.astype(np.float64), d.astype(np.float64)
        # the parameter at which the ray has crossed a voxel boundaries along some axis first
        T = []
        for k in range(3):
            if D64[k] >= 0:
                T.append((np.floor(V64[k]) + a - V64[k]) / max(abs(D64[k]), 1e-16))
            else:
                T.append((V64[k] - np.floor(V64[k]) + a - 1) / max(abs(D64[k]), 1e-16))
        s = min(T) + 1e-2
        assert np.allclose(out, V64 + D64 * s, rtol=0, atol=2e-4 * max(1.0, s))
        # the new position lies past the crossing, at most a voxels further along that axis
        k = int(np.argmin(T))
        assert abs(np.floor(out[k]) - np.floor(v[k])) == a


def test_cone_sphere_exact_distance(O):
    L = O.env_lib()
    rng = np.random.default_rng(4)
    done = 0
    for _ in range(4000):
        o = rng.uniform(-1, 1, 3).astype(np.float32)
        d = rng.normal(size=3)
        d = (d / np.linalg.norm(d)).astype(np.float32)
        th = rng.uniform(0.01, 0.3)
        tan_c = np.float32(math.tan(th))
        sec_c = np.float32(math.sqrt(1 + float(tan_c) ** 2))
        c = (o + rng.uniform(-3, 3, 3)).astype(np.float32)
        r = np.float32(rng.uniform(0.01, 0.5))
        got = L.or_env_cone_sphere(o.ctypes.data, d.ctypes.data, float(tan_c), float(sec_c), c.ctypes.data,
                                   float(r))
        # exact distance from c to the (single-nappe) cone of half-angle th in FP64
        v = c.astype(np.float64) - o
        t = v @ d
        w = np.linalg.norm(v - t * d)
        thf = math.atan(float(tan_c))
        ang = math.atan2(w, t)  # angle between v and the axis
        if ang <= thf:
            dist = 0.0
        elif ang - thf >= math.pi / 2:
            dist = np.linalg.norm(v)  # nearest point is the apex
        else:
            dist = np.linalg.norm(v) * math.sin(ang - thf)
        if abs(dist - r) < 1e-4:
            continue  # knife edge
        done += 1
        # the paper's test is the lateral-surface distance without the apex cap: it may accept
        # spheres behind the apex within r of the axis line only when t >= -r
        if ang - thf >= math.pi / 2:
            continue
        assert bool(got) == (dist <= r), (dist, r, got)
    assert done > 3000


def test_box_room_finds_every_image_path(O):
    from tests.test_oracle_pins import _image_paths
    case = box_case()
    recs, n_raw, nrays = O.env_launch(case, procs=NPROC)
    keys = {tuple(int(x) for x in r["label"][: r["n_int"]]) for r in recs}
    img = _image_paths((4.0, 3.0, 2.5), case.tx.tolist(), case.rx[0].tolist(), 2)
    assert set(img) <= keys, set(img) - keys
    assert len(keys - set(img)) <= 12
    for r in recs:  # every record's unfolded length is at least its image path's (straight line)
        seq = tuple(int(x) for x in r["label"][: r["n_int"]])
        if seq in img:
            assert r["L"] >= img[seq][0] - 2e-3


def test_wedge_shadow_zone_only_the_diffraction_key(O):
    sc = wedge_scene()
    tx, rx = np.array([-0.8, 0.3, 1.3]), np.array([0.3, -0.8, 0.9])
    case = case_of(sc, tx, rx, n_rays=1000, max_refl=0, max_diff=1, kappa=100, dphi_deg=2.5)
    case.sdf = dict(SDF)
    recs, n_raw, nrays = O.env_launch(case, procs=NPROC)
    keys = {(int(r["n_int"]), int(r["kinds"]), tuple(int(x) for x in r["label"][: r["n_int"]])) for r in recs}
    assert keys == {(1, 1, (77,))}, keys
    for r in recs:
        v = r["v"][0]
        assert abs(v[0]) < 1e-6 and abs(v[1]) < 1e-6 and 0 < v[2] < 2
