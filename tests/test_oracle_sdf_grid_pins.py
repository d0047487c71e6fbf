"""Tier 1 of the oracle's SDF intersection (oracle/sdf.c or_sdf_grid_build): an independent
uniform grid over the AABB primitives walked in FP64 must give tier 0's argmin bit for bit —
random queries on the C2 cloud (origins inside, on surfaces, outside; axis-parallel rays; with
and without departure normals) and whole launches (dense box room with fans; the C2 scene), at
several voxel sizes."""
import ctypes as C
import os

import numpy as np
import pytest

import nrt_gen as G

NPROC = max(1, min(32, os.cpu_count() or 1))
SDF = dict(cell=0.0625, r_s=0.015, t_sdf=0.0015, xi=2.0)


def query(O, sc, o, d, lam, prev):
    q = O._SdfParams(SDF["cell"], SDF["r_s"], SDF["t_sdf"], SDF["xi"])
    o, d = (np.ascontiguousarray(x, np.float32) for x in (o, d))
    lama = np.ascontiguousarray(np.asarray(lam, np.float32).reshape(-1, 3))
    nl = lama.shape[0]
    if nl == 0:
        lama = np.zeros((1, 3), np.float32)
    t, cell, n = C.c_float(), C.c_int64(), np.zeros(3, np.float32)
    s = O.lib().or_sdf_nearest(C.byref(sc.c), sc.sdf, C.byref(q), o.ctypes.data, d.ctypes.data,
                               lama.ctypes.data, nl, int(prev), 0.0015, float(O.cos_ex(25.0)),
                               C.byref(t), C.byref(cell), n.ctypes.data)
    return int(s), t.value, int(cell.value), n.tobytes()


@pytest.mark.parametrize("voxel", [0.07, 0.125, 0.31])
def test_tier1_equals_tier0_random_queries(O, voxel):
    scene = G.synth_room(200_000, 0.010)
    t0 = O.OracleScene(scene, sdf_cell=SDF["cell"])
    t1 = O.OracleScene(scene, sdf_cell=SDF["cell"], sdf_grid=voxel)
    rng = np.random.default_rng(11)
    hits = 0
    for k in range(150):
        kind = k % 3
        if kind == 0:    # inside the room
            o = rng.uniform([0.5, 0.5, 0.3], [7.5, 5.5, 2.7])
        elif kind == 1:  # on a surface point
            o = scene.points[rng.integers(scene.n)].astype(np.float64)
        else:            # outside the room
            o = rng.uniform([-3, -3, -3], [11, 9, 6])
        d = rng.normal(size=3)
        if k % 10 == 0:
            d = np.zeros(3)
            d[k % 3] = 1.0 if k % 20 == 0 else -1.0
        d /= np.linalg.norm(d)
        lam = [scene.normals[rng.integers(scene.n)]] if kind == 1 else []
        r0 = query(O, t0, o, d, lam, -1)
        r1 = query(O, t1, o, d, lam, -1)
        assert r0 == r1, (k, r0, r1)
        hits += r0[0] >= 0
    assert hits > 60


def test_tier1_equals_tier0_whole_launches(O):
    case = G.case("C1", n_rays=3000, max_diff=1)
    case.scene = G.box_room(3)
    case.sdf = dict(SDF)
    a = O.launch_phased(case, procs=NPROC)
    b = O.launch_phased(case, procs=NPROC, scene=O.coarse_scene(case, sdf_grid=0.2))
    assert a[0].tobytes() == b[0].tobytes() and a[1:] == b[1:]
    case = G.case("C2", sigma=0.010, n_rays=2000, max_diff=0)
    case.sdf = dict(SDF)
    a = O.launch_phased(case, procs=NPROC)
    b = O.launch_phased(case, procs=NPROC, scene=O.coarse_scene(case, sdf_grid=0.125))
    assert a[0].tobytes() == b[0].tobytes() and a[1:] == b[1:]


def test_tier1_in_the_cone_tracer_and_gd(O):
    """The NEXT-2 and NEXT-4 oracles give the same results with the tier-1 SDF grid."""
    case = G.case("C1", n_rays=1000)
    case.scene = G.box_room(2)
    case.sdf = dict(SDF)
    case.kappa = 100
    a = O.env_launch(case, procs=NPROC)
    b = O.env_launch(case, procs=NPROC, sdf_grid=0.2)
    assert a[0].tobytes() == b[0].tobytes() and a[1:] == b[1:]
    case.gd = dict(r_s=0.003, t_sdf=0.0005, t_d=0.002, t_a_deg=1.0, rho=100)
    co = O.launch_phased(case, procs=NPROC)[0]
    g0 = O.refine_gd_par(case, co, procs=NPROC)
    g1 = O.refine_gd_par(case, co, procs=NPROC, sdf_grid=0.2)
    assert g0.tobytes() == g1.tobytes()
