"""Pins of the oracle's tier-1 grid (oracle/grid.c) against tier 0 (the brute-force global
argmin of SURVEY §8(c) C.1, or_nearest) — the tier-1 grid only makes whole-configuration oracle
sets affordable; it must give the brute-force result bit for bit, for any voxel size and grid
origin (C.1 "Tier 1 ... must equal tier 0 bit-exactly on small scenes and must be invariant to
voxel size and origin").
"""
import numpy as np
import pytest

import nrt_gen as G


def _same(a, b):
    return a[0].tobytes() == b[0].tobytes() and a[1:] == b[1:]


@pytest.mark.parametrize("voxel,shift", [(0.05, (0, 0, 0)), (0.13, (0.011, 0.02, 0.0)),
                                         (0.4, (0.2, -0.1, 0.05)), (2.0, (0, 0, 0))])
def test_c1_tier1_equals_brute_force(O, voxel, shift):
    case = G.case("C1")
    ref = O.launch(case)
    sc = O.OracleScene(case.scene, grid_voxel=voxel, shift=shift)
    got = O.launch(case, scene=sc)
    assert _same(got, ref)
    assert len(got[0]) == 25


def test_sr_diffraction_tier1_equals_brute_force(O):
    """Synthetic room (sigma = 10 mm) with edges, diffraction on: records, raw count, bounces
    and the deduped event set."""
    case = G.case("C2s", sigma=0.010, n=12_000, n_rays=6000, max_refl=2, max_diff=1)
    ref = O.launch_phased(case, procs=8, return_events=True)
    got = O.launch_phased(case, procs=8, return_events=True, grid_voxel=0.07)
    assert ref[0].tobytes() == got[0].tobytes() and ref[1:3] == got[1:3]
    assert ref[3].tobytes() == got[3].tobytes()
    assert len(ref[3]) > 0 and (ref[0]["n_diff"] == 1).sum() > 0


def test_rr_many_rx_tier1_equals_brute_force(O):
    """Reconstructed-room recipe (clutter, holes, outliers, split labels, 879 RX)."""
    case = G.case("C5s", n_rays=3000)
    ref = O.launch_phased(case, procs=8)
    for v, sh in ((0.045, None), (0.11, (0.03, 0.01, 0.02))):
        got = O.launch_phased(case, procs=8,
                              scene=O.OracleScene(case.scene, grid_voxel=v, shift=sh))
        assert _same(got, ref), v


def test_pca_normals_tier1_equals_brute_force(O):
    case = G.case("C2s", sigma=0.010, n=20_000, n_rays=4000, max_diff=0, max_refl=4)
    case.scene = G.synth_room(20_000, 0.010, normals="pca")
    ref = O.launch_phased(case, procs=8)
    got = O.launch_phased(case, procs=8, grid_voxel=0.06)
    assert _same(got, ref)


def test_nearest_tier1_equals_brute_force_random_rays_full_c2(O):
    """Full C2 cloud (1e6 surfels): random origins (inside, on the bounds, outside the grid),
    random and axis-parallel directions, departure sheets and previous ids — the grid's
    nearest hit equals the brute-force argmin for every query."""
    case = G.case("C2")
    t0 = O.OracleScene(case.scene)
    t1 = O.OracleScene(case.scene, grid_voxel=0.05, shift=(0.013, 0.007, 0.021))
    rng = np.random.default_rng(11)
    P = case.scene.points
    n_q = 120
    hits = 0
    for q in range(n_q):
        kind = q % 4
        if kind == 0:      # inside the room
            o = rng.uniform([0.2, 0.2, 0.2], [7.8, 5.8, 2.8]).astype(np.float32)
        elif kind == 1:    # from a surfel (reflection origin), leaving its sheet
            i = rng.integers(len(P))
            o = P[i].copy()
        elif kind == 2:    # outside the grid
            o = rng.uniform([-3, -3, -3], [11, 9, 6]).astype(np.float32)
        else:              # on a grid-ish plane
            o = np.array([4.0, rng.uniform(0.1, 5.9), 1.5], np.float32)
        d = rng.standard_normal(3)
        if q % 5 == 0:     # axis-parallel / in-plane directions
            d[rng.integers(3)] = 0.0
        if q % 11 == 0:
            d[:] = 0.0
            d[rng.integers(3)] = rng.choice([-1.0, 1.0])
        d = (d / np.linalg.norm(d)).astype(np.float32)
        lam, prev = (), -1
        if kind == 1:
            lam, prev = (case.scene.normals[i],), int(i)
        a = O.nearest(t0, o, d, lam=lam, prev=prev, tau=case.tau)
        b = O.nearest(t1, o, d, lam=lam, prev=prev, tau=case.tau)
        assert a[0] == b[0] and np.float32(a[1]).tobytes() == np.float32(b[1]).tobytes(), (q, a, b)
        hits += a[0] >= 0
    assert hits > n_q // 2
