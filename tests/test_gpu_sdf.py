"""GPU parity of NEXT-1, the paper's point-set SDF intersection (DESIGN
R40-R45, §6.4), against the oracle's tier-0 SDF tracer (oracle/sdf.c: every AABB primitive
marched for every segment), through the C ABI (scene desc sdf_cell, launch desc intersect = 1).

Bar: coarse path sets bit-exact (the march, the FP32 Gaussian sums, the exp and the departure
rule are the same FP32 operations in the same order on both sides).
"""
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


def sdf_case(name, scene=None, **kw):
    c = G.case(name, **kw)
    if scene is not None:
        c.scene = scene
    c.sdf = dict(SDF)
    return c


def run(N, case, **kw):
    sc = N.build_case_scene(case)
    p = N.launch_case(sc, case, **kw)
    return p.export(), p.info(), sc


def test_dense_box_room_full_set_bit_exact(N, O):
    """C1's room at 1.8 cm surfel spacing (box_room(3)), 4000 rays, 2 reflections."""
    case = sdf_case("C1", G.box_room(3), n_rays=4000)
    got, info, sc = run(N, case)
    ref, n_raw, nb = O.launch_phased(case, procs=NPROC)
    assert info["bounces"] == nb == case.n_rays * 3
    assert info["n_raw"] == n_raw
    assert_same_records(got, ref, "SDF dense C1")
    si = sc.info()
    osc = O.coarse_scene(case)
    assert si["n_aabb"] == O.lib().or_sdf_count(osc.sdf)


def test_aabb_table_equals_oracle(N, O):
    """R40: the GPU build's AABB count equals the oracle's for the C2 scene (1e6 surfels)."""
    case = sdf_case("C2", sigma=0.010, n_rays=1000)
    sc = N.build_case_scene(case)
    osc = O.coarse_scene(case)
    si = sc.info()
    assert si["n_aabb"] == O.lib().or_sdf_count(osc.sdf) > 10_000
    assert si["n_aabb_refs"] >= si["n_aabb"]
    assert si["sdf_cell"] == np.float32(SDF["cell"])


@pytest.mark.parametrize("sigma", [0.0, 0.010, 0.020])
def test_c2_scene_full_set_bit_exact(N, O, sigma):
    """The C2 scene (1e6 surfels, noise sigma), 4000 rays, 3 reflections, no diffraction."""
    case = sdf_case("C2", sigma=sigma, n_rays=4000, max_diff=0)
    got, info, _ = run(N, case)
    ref, n_raw, nb = O.launch_phased(case, procs=NPROC)
    assert info["bounces"] == nb
    assert info["n_raw"] == n_raw
    assert_same_records(got, ref, f"SDF C2 sigma={sigma}")
    assert len(got) > 20


def test_c2_scene_with_diffraction_bit_exact(N, O):
    """Fans leave the edge with both face normals as departure normals (R43 with two)."""
    case = sdf_case("C2", sigma=0.005, n_rays=400, max_refl=2, max_diff=1)
    got, info, _ = run(N, case)
    ref, n_raw, nb, ev = O.launch_phased(case, procs=NPROC, return_events=True)
    assert info["n_events"] == len(ev)
    assert info["bounces"] == nb
    assert_same_records(got, ref, "SDF C2 diffraction")
    assert (got["n_diff"] == 1).sum() > 0


def test_forced_reorder_same_set(N, monkeypatch):
    """The per-bounce live-list reorder (forced on a small launch) does not change the set."""
    case = sdf_case("C2", sigma=0.010, n_rays=20_000, max_diff=0)
    base, bi, _ = run(N, case)
    monkeypatch.setenv("NRT_REORDER", "1")
    monkeypatch.setenv("NRT_SORT_MIN", "1")
    got, gi, _ = run(N, case)
    assert got.tobytes() == base.tobytes() and gi["bounces"] == bi["bounces"]


def test_full_c2_sampled_hit_sequences(N, O):
    """The full C2 lattice (1e6 rays): sampled rays' per-segment SDF hits (nearest AABB point
    ids) equal the oracle's tier-0 SDF tracer, through the production wavefront."""
    case = sdf_case("C2", sigma=0.010)
    sc = N.build_case_scene(case)
    ids = np.sort(np.random.default_rng(0).choice(case.n_rays, 48, replace=False)).astype(np.uint64)
    d = N.case_desc(case)
    d.pop("kappa"), d.pop("dphi_deg"), d.pop("edge_bin")
    gpu = N.nrt_debug_trace_rays(sc, case.tx, case.n_rays, case.max_refl, ids, **d)
    _, hits, _ = O.trace_rays(case, ids)
    assert np.array_equal(gpu, hits)
    assert (gpu[:, 1] >= 0).sum() > 10


def test_full_c2_records_retraced_by_oracle(N, O):
    """Full C2 SDF launch (1e6 rays, diffraction on): sampled primary records are reproduced
    exactly by the oracle re-tracing their rays; keys sorted and unique."""
    case = sdf_case("C2", sigma=0.010)
    sc = N.build_case_scene(case)
    p = N.launch_case(sc, case)
    got = p.export()
    prim = got[got["ray_id"] < (1 << 63)]
    assert len(prim) > 20
    sample = prim[np.random.default_rng(1).permutation(len(prim))[:40]]
    raw, _, _ = O.trace_rays(case, sample["ray_id"])
    rb = {r.tobytes() for r in raw}
    for r in sample:
        assert r.tobytes() in rb
    keys = [(int(r["rx"]), int(r["n_int"]), int(r["kinds"]), tuple(int(x) for x in r["label"]))
            for r in got]
    assert keys == sorted(keys) and len(set(keys)) == len(keys)


def test_sdf_errors(N):
    case = G.case("C1", n_rays=1000)
    sc = N.build_case_scene(case)  # no AABB primitives
    with pytest.raises(N.NrtError) as e:
        N.launch_case(sc, case, intersect=1)
    assert "sdf_cell" in str(e.value)
    s = case.scene
    with pytest.raises(N.NrtError):
        N.nrt_scene_build_ex(s.points, s.normals, 0.1, radii=s.radii, labels=s.labels, sdf_cell=-1.0)
    case.sdf = dict(SDF)
    sc = N.build_case_scene(case)
    with pytest.raises(N.NrtError):
        N.launch_case(sc, case, sdf_t_sdf=0.0)


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_fullsize_sdf_sampled_hit_sequences(N, O, name):
    """The reconstructed-room configs (1e7 surfels, 1e7 / 1e8-ray lattices) with the SDF
    intersection: sampled rays' per-segment hits equal the oracle's tier-0 SDF tracer."""
    case = sdf_case(name)
    sc = N.build_case_scene(case)
    ids = np.sort(np.random.default_rng(7).choice(case.n_rays, 12, replace=False)).astype(np.uint64)
    d = N.case_desc(case)
    d.pop("kappa"), d.pop("dphi_deg"), d.pop("edge_bin")
    gpu = N.nrt_debug_trace_rays(sc, case.tx, case.n_rays, case.max_refl, ids, **d)
    _, hits, _ = O.trace_rays(case, ids)
    assert np.array_equal(gpu, hits)
    assert (gpu[:, 1] >= 0).sum() > 3


def test_full_c2_sdf_set_bit_exact(N, O):
    """The whole C2 SDF launch (1e6 surfels, 1e6 rays, diffraction: 5.5e6 segments) equals the
    oracle's whole set (tier-1 SDF grid, pinned to tier 0), raw and bounce counts included."""
    case = sdf_case("C2", sigma=0.010)
    got, info, _ = run(N, case)
    ref, n_raw, nb = O.launch_phased(case, procs=NPROC, scene=O.coarse_scene(case, sdf_grid=0.125))
    assert info["bounces"] == nb and info["n_raw"] == n_raw
    assert_same_records(got, ref, "SDF full C2")
    assert len(got) > 1000


@pytest.mark.parametrize("name,rays", [("C4", 60_000), ("C5", 60_000)])
def test_fullsize_sdf_sharded_subset(N, O, name, rays):
    """A shard of the full-size C4 / C5 lattice (1e7 surfels; 1e7 / 1e8 rays) with the SDF
    intersection through the production path (stage 1): every raw record (kappa = 2^30), the
    events and the bounce count equal the oracle's (tier-1 SDF grid)."""
    import multiprocessing as mp
    case = sdf_case(name)
    case.kappa = 1 << 30
    world = case.n_rays // rays
    rank = world // 5
    sc = N.build_case_scene(case, device_arrays=True)
    p = N.launch_case(sc, case, rank=rank, world=world, stage=1)
    got, info, ev = p.export(), p.info(), p.export_events()
    O._FORK["case"], O._FORK["max_diff"] = case, None
    O._FORK["scene"] = O.coarse_scene(case, sdf_grid=0.125)
    with mp.get_context("fork").Pool(NPROC) as pool:
        parts = pool.map(O._primary_worker, [(rank + q * world, NPROC * world) for q in range(NPROC)])
    O._FORK.pop("scene")
    raw = np.concatenate([x[0] for x in parts])
    ref_ev = O.event_dedupe(np.concatenate([x[1] for x in parts]))
    ref = O.dedupe(raw, case.kappa)
    assert info["bounces"] == sum(x[2] for x in parts)
    assert len(got) == len(ref) and got.tobytes() == ref.tobytes()
    assert len(ev) == len(ref_ev) and ev.tobytes() == ref_ev.tobytes()
    assert len(got) > 0
