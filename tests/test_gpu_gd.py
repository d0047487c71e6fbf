"""GPU parity of NEXT-4, the paper's own gradient-descent refinement (PAPER §II-E P:182-232,
Tables I-III; DESIGN R50-R56), against the oracle (oracle/gd.c), through the C ABI
(nrt_refine_desc.method = 1 on a scene built with sdf_cell > 0).

Bar: the refined records equal the oracle's bit for bit (vertices, length, delay, status,
iterations, ||grad f||^2, labels) — FP32 GD in the same operation order on both sides, the
reprojection traces and normals being the bit-exact SDF functions of NEXT-1; the FP64 angles
of R27 come from libm vs CUDA's atan2/asin/acos, compared within 1e-4 degrees.
"""
import os

import numpy as np
import pytest

import nrt_gen as G

pytestmark = pytest.mark.gpu

NPROC = max(1, min(32, os.cpu_count() or 1))
SDF = dict(cell=0.0625, r_s=0.015, t_sdf=0.0015, xi=2.0)
NOISELESS = dict(r_s=0.003, t_sdf=0.0005, t_d=0.002, t_a_deg=1.0)  # Tables II/III
EXACT = ("rx", "n_int", "n_diff", "kinds", "label", "prim", "v", "L", "delay", "inc", "status",
         "iters", "gradsq", "ray_id")


@pytest.fixture(scope="module")
def N():
    import torch
    assert torch.cuda.is_available()
    import paper_2403_06648_b200 as N
    N.lib()
    return N


def compare(got, ref, what):
    assert len(got) == len(ref), (what, len(got), len(ref))
    bad = {}
    for f in EXACT:
        if f == "inc":
            continue
        a, b = got[f].reshape(len(got), -1), ref[f].reshape(len(got), -1)
        ne = a != b
        if a.dtype.kind == "f":
            ne &= ~(np.isnan(a) & np.isnan(b))  # a degenerate path's 0/0 on both sides
        d = np.nonzero(np.any(ne, axis=1))[0]
        if len(d):
            bad[f] = (len(d), int(d[0]))
    assert not bad, (what, bad, got[list(bad.values())[0][1]] if bad else None,
                     ref[list(bad.values())[0][1]] if bad else None)
    for f in ("aod_az", "aod_el", "aoa_az", "aoa_el", "inc"):
        dd = np.abs(got[f].astype(np.float64) - ref[f].astype(np.float64))
        dd = np.minimum(dd, 360.0 - dd)
        assert dd.max() < 1e-4, (what, f, dd.max())


def run_gd(N, case, coarse_case=None, **over):
    """GPU: SDF coarse launch + GD refinement (keep_invalid) -> (coarse records, refined)."""
    cc = coarse_case or case
    sc = N.build_case_scene(cc)
    co = N.launch_case(sc, cc)
    ref = N.nrt_refine_ex(sc, co, keep_invalid=1, **N.gd_desc(case, **over))
    return co.export(), ref.export(), ref.info()


def test_gd_dense_box_room_bit_exact(N, O):
    case = G.case("C1", n_rays=4000)
    case.scene = G.box_room(3)
    case.sdf = dict(SDF)
    case.gd = dict(NOISELESS)
    coarse, got, info = run_gd(N, case)
    ref = O.refine_gd_par(case, coarse, procs=NPROC)
    compare(got, ref, "GD dense C1")
    assert (got["status"] == 0).all() and len(got) == 25
    assert info["n_raw"] == 25


@pytest.mark.parametrize("sigma", [0.0, 0.010])
def test_gd_c2_scene_bit_exact(N, O, sigma):
    """The C2 scene (1e6 surfels): SDF coarse set of a 2000-ray lattice, GD with Table II/III's
    parameters (noisy: r_s 0.01, t_sdf 0.001, t_d 0.02, t_a 1 deg), rho = 2000."""
    case = G.case("C2", sigma=sigma, n_rays=2000, max_diff=0)
    case.sdf = dict(SDF)
    if sigma == 0.0:
        case.gd = dict(NOISELESS)
    coarse, got, _ = run_gd(N, case)
    assert len(coarse) > 20
    ref = O.refine_gd_par(case, coarse, procs=NPROC)
    compare(got, ref, f"GD C2 sigma={sigma}")
    assert (got["status"] == 0).sum() > 5


def test_gd_c2_scene_diffraction_bit_exact(N, O):
    case = G.case("C2", sigma=0.005, n_rays=400, max_refl=2, max_diff=1)
    case.sdf = dict(SDF)
    coarse, got, _ = run_gd(N, case, rho=500)
    assert (coarse["n_diff"] > 0).sum() > 20
    ref = O.refine_gd_par(case, coarse, procs=NPROC, rho=500)
    compare(got, ref, "GD C2 diffraction")
    assert ((got["status"] == 0) & (got["n_diff"] > 0)).sum() > 3


def test_gd_c4_sampled_bit_exact(N, O):
    """Full C4 SDF coarse set (1e7 surfels, 1e7 rays, 85 RX): 16 sampled paths refined with the
    estimated-normal thresholds (t_a = 25 deg), rho = 300."""
    case = G.case("C4")
    case.sdf = dict(SDF)
    case.gd = dict(t_a_deg=25.0, rho=300)
    sc = N.build_case_scene(case)
    co = N.launch_case(sc, case).export()
    sample = co[np.random.default_rng(3).permutation(len(co))[:16]]
    sub = N.nrt_paths_import(sample, N.PATHS_COARSE, case.tx, case.rx)
    got = N.nrt_refine_ex(sc, sub, keep_invalid=1, **N.gd_desc(case)).export()
    ref = O.refine_gd_par(case, sample, procs=NPROC)
    compare(got, ref, "GD C4 sample")


def test_gd_errors(N):
    case = G.case("C1", n_rays=1000)
    sc = N.build_case_scene(case)  # no AABB primitives
    co = N.launch_case(sc, case)
    with pytest.raises(N.NrtError) as e:
        N.nrt_refine_ex(sc, co, **N.gd_desc(case))
    assert "sdf_cell" in str(e.value)
    case.sdf = dict(SDF)
    sc = N.build_case_scene(case)
    co = N.launch_case(sc, case)
    with pytest.raises(N.NrtError):
        N.nrt_refine_ex(sc, co, select=1, **N.gd_desc(case))


def test_gd_full_c2_sdf_set_bit_exact(N, O):
    """Every path of the whole C2 SDF coarse set (1864) refined by the paper's GD (rho = 2000):
    all records equal the oracle's (tier-1 SDF grid)."""
    case = G.case("C2", sigma=0.010)
    case.sdf = dict(SDF)
    coarse, got, _ = run_gd(N, case)
    assert len(coarse) > 1000
    ref = O.refine_gd_par(case, coarse, procs=NPROC, sdf_grid=0.125)
    compare(got, ref, "GD full C2")
    assert (got["status"] == 0).sum() > 500
