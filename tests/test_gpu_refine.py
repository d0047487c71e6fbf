"""GPU parity of the refinement rows (A9-A10) against the CPU oracle through the C ABI.

Bar (BASELINE.json north_star): refined vertices within 1e-5 m, delays within 1e-12 s; the
per-path status (OK / NO_CONVERGE / ...) must agree.  On noisy clouds a discrete validity
decision can flip at a knife edge between two FP64 implementations (SURVEY §7 "Refinement
robustness"); such flips are counted and must stay rare (<= 2 %), and are reported.
"""
import os

import numpy as np
import pytest

import nrt_gen as G

pytestmark = pytest.mark.gpu
NPROC = max(1, min(32, os.cpu_count() or 1))
TOL_V = 1e-5      # m
TOL_DELAY = 1e-12  # s
TOL_ANG = 1e-4     # degrees (R27 angles are float32)


@pytest.fixture(scope="module")
def N():
    import torch
    assert torch.cuda.is_available()
    import paper_2403_06648_b200 as N
    N.lib()
    return N


def refine_gpu(N, case, sc, coarse, keep_invalid=1, **kw):
    return N.nrt_refine_ex(sc, coarse, xi=case.xi, r_s=case.r_s, tau=case.tau,
                           theta_ex_deg=case.theta_ex_deg, keep_invalid=keep_invalid, **kw).export()


def compare(got, ref, max_flip_frac=0.0, what=""):
    assert len(got) == len(ref), what
    for f in ("rx", "n_int", "kinds", "label", "prim", "ray_id"):
        assert np.array_equal(got[f], ref[f]), (what, f)
    # A knife-edge flip is a path whose status differs, or which both sides refine to a valid
    # path but at different roots (|dv| > TOL_V): on noisy MLS surfaces the root is local to the
    # seed and a stalled Gauss-Newton trajectory is chaotic at the rounding level (SURVEY §8(c)
    # C.1 "a few knife-edge validity flips are possible. They are reported, not hidden").
    ok2 = (got["status"] == 0) & (ref["status"] == 0)
    dvp = np.abs(got["v"] - ref["v"]).reshape(len(got), -1).max(axis=1) if len(got) else np.zeros(0)
    root_flip = ok2 & (dvp > TOL_V)
    flips = np.nonzero((got["status"] != ref["status"]) | root_flip)[0]
    assert len(flips) <= max_flip_frac * len(got), (what, len(flips), got["status"][flips[:5]],
                                                    ref["status"][flips[:5]])
    both = ok2 & ~root_flip
    assert both.sum() > 0 or len(got) == 0
    # the paths both sides refine to the same root agree far inside the tolerance
    if both.sum() >= 10:
        assert np.median(dvp[both]) <= 1e-11, (what, np.median(dvp[both]))
    dv = np.abs(got["v"][both] - ref["v"][both]).max() if both.any() else 0.0
    dd = np.abs(got["delay"][both] - ref["delay"][both]).max() if both.any() else 0.0
    assert dv <= TOL_V, (what, dv)
    assert dd <= TOL_DELAY, (what, dd)
    # R27 angles (float32 degrees from the FP64 vertices; azimuths compared on the circle)
    da = 0.0
    if both.any():
        for f in ("aod_az", "aod_el", "aoa_az", "aoa_el", "inc"):
            d = np.abs(got[f][both].astype(np.float64) - ref[f][both])
            d = np.minimum(d, 360.0 - d)
            da = max(da, float(d.max()))
    assert da <= TOL_ANG, (what, da)
    print(f"[refine parity] {what}: {len(got)} paths, {len(flips)} knife-edge flips "
          f"({100.0 * len(flips) / max(1, len(got)):.2f} %; {int(root_flip.sum())} of them at "
          f"another root), {int(both.sum())} OK on both, "
          f"max |dv| {dv:.2e} m, |d delay| {dd:.2e} s, |d angle| {da:.2e} deg")
    return len(flips), dv, dd


def test_c1_refined_parity_and_image_method(N, O):
    case = G.case("C1")
    sc = N.build_case_scene(case)
    coarse = N.launch_case(sc, case)
    got = refine_gpu(N, case, sc, coarse)
    ref = O.refine(case, coarse.export())
    flips, dv, dd = compare(got, ref, 0.0, "C1")
    assert (got["status"] == 0).all() and len(got) == 25
    assert dv < 1e-9
    # the deduped (default) output equals the oracle's shortest-per-key set
    ded = N.nrt_refine_ex(sc, coarse, xi=case.xi, r_s=case.r_s, tau=case.tau).export()
    oref = O.refine_dedupe(ref)
    assert len(ded) == len(oref) == 25
    assert np.abs(ded["v"] - oref["v"]).max() < 1e-9


@pytest.mark.parametrize("sigma", [0.0, 0.010])
def test_sr_small_refined_parity(N, O, sigma):
    case = G.case("C2s", sigma=sigma, n=30_000, n_rays=15_000, max_diff=0)
    sc = N.build_case_scene(case)
    coarse = N.launch_case(sc, case)
    got = refine_gpu(N, case, sc, coarse)
    ref = O.refine(case, coarse.export())
    flips, dv, dd = compare(got, ref, 0.0 if sigma == 0 else 0.02, f"SR sigma={sigma}")
    assert (got["status"] == 0).sum() >= 10


def test_sr_small_diffraction_refined_parity(N, O):
    case = G.case("C2s", sigma=0.005, n=12_000, n_rays=8000, max_refl=2, max_diff=1)
    sc = N.build_case_scene(case)
    coarse = N.launch_case(sc, case)
    got = refine_gpu(N, case, sc, coarse)
    ref = O.refine(case, coarse.export())
    compare(got, ref, 0.02, "SR diffraction")
    assert ((got["status"] == 0) & (got["n_diff"] == 1)).sum() > 0


def test_sr_small_refined_parity_full_size_rs(N, O):
    """Small synthetic room refined at the full-size configurations' r_s = 0.01 m (sigma = 2 cm
    neighbourhoods, C2/C3's regime) rather than the sparse-cloud 0.03 m."""
    case = G.case("C2s", sigma=0.010, n=200_000, n_rays=20_000, max_diff=0)
    case.r_s = 0.01
    sc = N.build_case_scene(case)
    coarse = N.launch_case(sc, case)
    got = refine_gpu(N, case, sc, coarse)
    ref = O.refine_par(case, coarse.export(), procs=NPROC)
    compare(got, ref, 0.02, "SR 2e5 surfels r_s=0.01")
    assert (got["status"] == 0).sum() >= 10


def test_c2_full_set_refined_parity(N, O):
    """Full C2 (1e6 surfels, sigma = 1 cm, the bench's secondary workload): the GPU refines every
    coarse path, the oracle re-refines EVERY one of them; <= 0.5 % knife-edge status flips."""
    case = G.case("C2", sigma=0.010)
    sc = N.build_case_scene(case)
    coarse = N.launch_case(sc, case)
    got = refine_gpu(N, case, sc, coarse)
    cr = coarse.export()
    ref = O.refine_par(case, cr, procs=NPROC)
    compare(got, ref, 0.005, "C2 whole set")
    assert len(got) > 1000


def _sample(allg, n_ok, n_any, seed):
    rng = np.random.default_rng(seed)
    ok = np.nonzero(allg["status"] == 0)[0]
    rest = np.setdiff1d(np.arange(len(allg)), ok)
    return np.sort(np.concatenate([rng.choice(ok, min(n_ok, len(ok)), replace=False),
                                   rng.choice(rest, min(n_any, len(rest)), replace=False)]))


@pytest.mark.parametrize("name,seed", [("C4", 4), ("C5", 6)])
def test_full_size_sampled_refined_parity(N, O, name, seed):
    """Full C4 (1e7 surfels, fitted normals, 85 RX, diffraction) and C5 (879 RX, 1e8-ray
    lattice) — refinement in the throughput regime: the oracle re-refines 100 paths the GPU
    found valid and 100 others; <= 1 % status flips."""
    case = G.case(name)
    sc = N.build_case_scene(case, device_arrays=True)
    coarse = N.launch_case(sc, case)
    cr = coarse.export()
    allg = refine_gpu(N, case, sc, coarse)
    idx = _sample(allg, 100, 100, seed)
    ref = O.refine_par(case, cr[idx], procs=NPROC)
    compare(allg[idx], ref, 0.01, f"{name} sample")


def test_refine_sharding_union(N):
    case = G.case("C2s", sigma=0.0, n=20_000, n_rays=8000, max_diff=0)
    sc = N.build_case_scene(case)
    coarse = N.launch_case(sc, case)
    full = refine_gpu(N, case, sc, coarse)
    parts = [refine_gpu(N, case, sc, coarse, rank=r, world=3) for r in range(3)]
    merged = np.zeros_like(full)
    for r, p in enumerate(parts):
        merged[r::3] = p
    assert merged.tobytes() == full.tobytes()


def test_select_partitions(N):
    """select=1/2 split the coarse set by diffraction (disjoint R17/R28 keys): their refined
    records are exactly the full run's; blocks_per_sm only changes the schedule."""
    case = G.case("C2s", sigma=0.005, n=12_000, n_rays=8000, max_refl=2, max_diff=1)
    sc = N.build_case_scene(case)
    coarse = N.launch_case(sc, case)
    full = refine_gpu(N, case, sc, coarse)
    p1 = refine_gpu(N, case, sc, coarse, select=1)
    p2 = refine_gpu(N, case, sc, coarse, select=2, blocks_per_sm=1)
    assert len(p1) + len(p2) == len(full) and len(p2) > 0 and len(p1) > 0
    diff = coarse.export()["n_diff"] > 0
    assert p1.tobytes() == full[~diff].tobytes()
    assert p2.tobytes() == full[diff].tobytes()


def test_warp_and_block_kernels_agree(N, monkeypatch):
    """The two refinement kernels (warp per path, the throughput regime the C4/C5 bench runs;
    block of 12 warps per path, the latency regime) on the same C2 coarse set: every record
    equal, bit for bit (they share the device functions and take trials in the same order)."""
    case = G.case("C2", sigma=0.010)
    sc = N.build_case_scene(case)
    coarse = N.launch_case(sc, case)
    monkeypatch.setenv("NRT_REFINE_IMPL", "block")
    blk = refine_gpu(N, case, sc, coarse)
    monkeypatch.setenv("NRT_REFINE_IMPL", "warp")
    wrp = refine_gpu(N, case, sc, coarse)
    assert len(blk) == len(wrp) > 1000
    same = np.array([a.tobytes() == b.tobytes() for a, b in zip(blk, wrp)])
    assert same.all(), (int((~same).sum()), np.nonzero(~same)[0][:5])
