"""Edge cases of the NEXT rows against the oracle (bit-exact): tiny and ragged lattices, a
one-point scene (a single flat AABB), no receivers, receivers outside the points' box, and the
degenerate GD settings (rho = 0, 1)."""
import os

import numpy as np
import pytest

import nrt_gen as G
from tests.test_gpu_coarse import assert_same_records

pytestmark = pytest.mark.gpu

NPROC = max(1, min(32, os.cpu_count() or 1))
SDF = dict(cell=0.0625, r_s=0.015, t_sdf=0.0015, xi=2.0)


@pytest.fixture(scope="module")
def N():
    import torch
    assert torch.cuda.is_available()
    import paper_2403_06648_b200 as N
    N.lib()
    return N


def box(n_rays=1000, density=3, **kw):
    case = G.case("C1", n_rays=n_rays, **kw)
    case.scene = G.box_room(density)
    case.sdf = dict(SDF)
    return case


@pytest.mark.parametrize("n_rays", [1, 2, 3, 33, 997])
def test_sdf_tiny_and_ragged_lattices(N, O, n_rays):
    case = box(n_rays)
    sc = N.build_case_scene(case)
    p = N.launch_case(sc, case)
    ref, n_raw, nb = O.launch(case)
    assert p.info()["bounces"] == nb
    assert_same_records(p.export(), ref, f"SDF n_rays={n_rays}")


def test_sdf_one_point_scene_and_no_receivers(N, O):
    s = G.Scene(np.array([[1.0, 1.0, 1.0]], np.float32), np.array([[0, 0, 1.0]], np.float32),
                np.array([0.01], np.float32), np.array([0], np.int32), G.Edges.empty())
    case = G.LaunchCase("one", s, np.array([1.0, 1.0, 2.0], np.float32), np.zeros((0, 3), np.float32),
                        5000, 2, 0, 0.1)
    case.sdf = dict(SDF)
    sc = N.build_case_scene(case)
    assert sc.info()["n_aabb"] == 1
    p = N.launch_case(sc, case)
    ref, n_raw, nb = O.launch(case)
    assert p.count() == 0 and len(ref) == 0
    assert p.info()["bounces"] == nb


def test_env_receivers_outside_and_none(N, O):
    case = box(1000, density=2)
    case.kappa = 100
    case.rx = np.array([[3.1, 2.2, 1.1], [9.0, -4.0, 7.0], [-1.0, 1.5, 1.0]], np.float32)
    sc = N.build_case_scene(case)
    p = N.launch_case(sc, case, tracer=1)
    ref, n_raw, nrays = O.env_launch(case, procs=NPROC)
    assert p.info()["bounces"] == nrays and p.info()["n_raw"] == n_raw
    assert_same_records(p.export(), ref, "NEXT-2 outside RX")
    case.rx = np.zeros((0, 3), np.float32)
    p = N.launch_case(N.build_case_scene(case), case, tracer=1)
    ref, n_raw, nrays = O.env_launch(case, procs=NPROC)
    assert p.count() == 0 == len(ref) and p.info()["bounces"] == nrays


@pytest.mark.parametrize("rho", [0, 1, 7])
def test_gd_rho_degenerate(N, O, rho):
    case = box(1000)
    case.gd = dict(r_s=0.003, t_sdf=0.0005, t_d=0.002, t_a_deg=1.0, rho=rho)
    sc = N.build_case_scene(case)
    co = N.launch_case(sc, case)
    got = N.nrt_refine_ex(sc, co, keep_invalid=1, **N.gd_desc(case)).export()
    ref = O.refine_gd(case, co.export())
    for f in ("v", "L", "status", "iters", "label", "prim"):
        assert np.array_equal(got[f], ref[f]), f
    g, r = got["gradsq"], ref["gradsq"]
    assert np.array_equal(np.isnan(g), np.isnan(r)) and np.array_equal(g[~np.isnan(g)], r[~np.isnan(r)])
    assert (got["iters"] == rho).sum() > 0
