"""GPU parity of the coarse path (rows A1-A8) against the CPU oracle, through the C ABI.

Bar (BASELINE.json north_star): coarse path sets bit-exact.  Records are compared field by
field (key, representative ray id, vertices, L); the bounce counters must match too.
"""
import os

import numpy as np
import pytest

import nrt_gen as G

pytestmark = pytest.mark.gpu

NPROC = max(1, min(32, os.cpu_count() or 1))


@pytest.fixture(scope="module")
def N():
    import torch
    assert torch.cuda.is_available()
    import paper_2403_06648_b200 as N
    N.lib()
    return N


def assert_same_records(got, ref, what=""):
    assert got.dtype.names == ref.dtype.names
    if len(got) != len(ref) or got.tobytes() != ref.tobytes():
        gk = {(int(r["rx"]), int(r["n_int"]), int(r["kinds"]), tuple(r["label"])) for r in got}
        rk = {(int(r["rx"]), int(r["n_int"]), int(r["kinds"]), tuple(r["label"])) for r in ref}
        msg = [f"{what}: {len(got)} vs {len(ref)} records; keys only GPU {len(gk - rk)}, only "
               f"oracle {len(rk - gk)}"]
        if len(got) == len(ref):
            for f in got.dtype.names:
                bad = np.nonzero(np.any((got[f] != ref[f]).reshape(len(got), -1), axis=1))[0]
                if len(bad):
                    i = bad[0]
                    msg.append(f"field {f}: {len(bad)} differ, first at {i}: {got[i]} vs {ref[i]}")
        raise AssertionError("\n".join(msg))


def run_gpu(N, case, **kw):
    sc = N.build_case_scene(case)
    p = N.launch_case(sc, case, **kw)
    return p.export(), p.info(), sc


# ------------------------------------------------------------------ C1 (full set) -------
def test_c1_full_set_bit_exact(N, O):
    case = G.case("C1")
    got, info, sc = run_gpu(N, case)
    ref, n_raw, nb = O.launch_phased(case, procs=NPROC)
    assert info["bounces"] == nb
    assert info["n_raw"] == n_raw
    assert_same_records(got, ref, "C1")
    assert len(got) == 25


@pytest.mark.parametrize("voxel", [0.04, 0.0625, 0.3, 1.1])
def test_c1_invariant_to_voxel(N, O, voxel):
    case = G.case("C1")
    base, _, _ = run_gpu(N, case)
    case.voxel = voxel
    got, info, _ = run_gpu(N, case)
    assert_same_records(got, base, f"C1 voxel {voxel}")


def test_c1_device_arrays_and_host_arrays_agree(N):
    case = G.case("C1", n_rays=3000)
    a = N.launch_case(N.build_case_scene(case), case).export()
    b = N.launch_case(N.build_case_scene(case, device_arrays=True), case).export()
    assert a.tobytes() == b.tobytes()


def test_c1_kappa_100(N, O):
    case = G.case("C1", n_rays=4000, kappa=100)
    got, info, _ = run_gpu(N, case)
    ref, n_raw, nb = O.launch_phased(case, procs=NPROC)
    assert_same_records(got, ref, "C1 kappa=100")
    assert len(got) > 25


# ------------------------------------------------------------------ SR small ------------
@pytest.mark.parametrize("sigma", [0.0, 0.005, 0.010, 0.020])
def test_sr_small_no_diffraction_bit_exact(N, O, sigma):
    case = G.case("C2s", sigma=sigma, n=30_000, n_rays=15_000, max_diff=0)
    got, info, _ = run_gpu(N, case)
    ref, n_raw, nb = O.launch_phased(case, procs=NPROC)
    assert info["bounces"] == nb
    assert_same_records(got, ref, f"SR sigma={sigma}")
    assert len(got) > 10


def test_sr_small_with_diffraction_bit_exact(N, O):
    case = G.case("C2s", sigma=0.005, n=12_000, n_rays=8000, max_refl=2, max_diff=1)
    got, info, _ = run_gpu(N, case)
    ref, n_raw, nb, ev = O.launch_phased(case, procs=NPROC, return_events=True)
    assert info["n_events"] == len(ev)
    assert info["bounces"] == nb
    assert_same_records(got, ref, "SR diffraction")
    assert (got["n_diff"] == 1).sum() > 0


def test_pca_normals_small_bit_exact(N, O):
    case = G.case("C2s", sigma=0.010, n=30_000, n_rays=8000, max_diff=0, max_refl=4)
    case.scene = G.synth_room(30_000, 0.010, normals="pca")
    got, info, _ = run_gpu(N, case)
    ref, n_raw, nb = O.launch_phased(case, procs=NPROC)
    assert info["bounces"] == nb
    assert_same_records(got, ref, "SR pca normals")


# ------------------------------------------------------------------ full-size samples ---
@pytest.fixture(scope="module")
def c2():
    return G.case("C2", sigma=0.010)


def test_c2_full_size_sampled_hit_sequences(N, O, c2):
    """Per-ray hit sequences of sampled rays of the full C2 workload (1e6 surfels, 1e6 rays)
    equal the brute-force argmin, segment by segment."""
    sc = N.build_case_scene(c2)
    rng = np.random.default_rng(0)
    ids = np.sort(rng.choice(c2.n_rays, 48, replace=False)).astype(np.uint64)
    gpu = N.nrt_debug_trace_rays(sc, c2.tx, c2.n_rays, c2.max_refl, ids, tau=c2.tau,
                                 theta_ex_deg=c2.theta_ex_deg, c_R=c2.c_R)
    _, hits, _ = O.trace_rays(c2, ids)
    assert np.array_equal(gpu, hits)


def test_c2_full_size_records_retraced_by_oracle(N, O, c2):
    """Every primary-ray record of the full C2 launch is reproduced exactly by the oracle
    re-tracing its ray (property that holds at any size)."""
    sc = N.build_case_scene(c2)
    p = N.launch_case(sc, c2)
    got = p.export()
    info = p.info()
    assert info["n_events"] > 0 and info["n_fan_rays"] > 0
    prim = got[got["ray_id"] < (1 << 63)]
    assert len(prim) > 5
    sample = prim[np.random.default_rng(1).permutation(len(prim))[:40]]
    raw, _, _ = O.trace_rays(c2, sample["ray_id"])
    rb = {r.tobytes() for r in raw}
    for r in sample:
        assert r.tobytes() in rb
    # the set is sorted by key and unique per key (kappa = 1)
    keys = [(int(r["rx"]), int(r["n_int"]), int(r["kinds"]), tuple(int(x) for x in r["label"]))
            for r in got]
    assert keys == sorted(keys) and len(set(keys)) == len(keys)


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_full_size_sampled_hit_sequences_other_configs(N, O, name):
    """BASELINE configs[2..4] at full size (1e6 surfels with PCA normals / 1e7 surfels of the
    reconstructed-room recipe, 1e7 / 1e7 / 1e8-ray lattices): sampled rays' hit sequences
    equal the brute-force argmin segment by segment."""
    case = G.case(name)
    sc = N.build_case_scene(case)
    ids = np.sort(np.random.default_rng(5).choice(case.n_rays, 12, replace=False)).astype(np.uint64)
    gpu = N.nrt_debug_trace_rays(sc, case.tx, case.n_rays, case.max_refl, ids, tau=case.tau,
                                 theta_ex_deg=case.theta_ex_deg, c_R=case.c_R)
    _, hits, _ = O.trace_rays(case, ids)
    assert np.array_equal(gpu, hits)


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_full_size_records_retraced_other_configs(N, O, name):
    """Full C4 (85 RX, diffraction on) and C5 (879 RX, 1e8 rays) launches: sampled primary
    records are reproduced exactly by the oracle re-tracing their rays; keys unique+sorted."""
    case = G.case(name)
    sc = N.build_case_scene(case)
    p = N.launch_case(sc, case)
    got = p.export()
    prim = got[got["ray_id"] < (1 << 63)]
    assert len(prim) > 100
    sample = prim[np.random.default_rng(2).permutation(len(prim))[:12]]
    raw, _, _ = O.trace_rays(case, sample["ray_id"])
    rb = {r.tobytes() for r in raw}
    for r in sample:
        assert r.tobytes() in rb
    keys = [(int(r["rx"]), int(r["n_int"]), int(r["kinds"]), tuple(int(x) for x in r["label"]))
            for r in got]
    assert keys == sorted(keys) and len(set(keys)) == len(keys)


# ------------------------------------------------------------------ sharding ------------
def test_world_sharding_merge_equals_single(N, O):
    """R30: shards i == rank (mod world) merged by nrt_paths_merge == the world-1 set."""
    case = G.case("C2s", sigma=0.01, n=20_000, n_rays=12_000, max_diff=0)
    sc = N.build_case_scene(case)
    full = N.launch_case(sc, case).export()
    for world in (2, 3, 8):
        parts = [N.launch_case(sc, case, rank=r, world=world) for r in range(world)]
        merged = N.nrt_paths_merge(parts, 1).export()
        assert merged.tobytes() == full.tobytes(), world
        assert sum(p.info()["bounces"] for p in parts) == N.launch_case(sc, case).info()["bounces"]


def test_two_stage_diffraction_protocol_equals_single(N):
    """World > 1 with diffraction: stage 1 per rank -> gather events -> fans per rank -> merge."""
    case = G.case("C2s", sigma=0.005, n=12_000, n_rays=8000, max_refl=2, max_diff=1)
    sc = N.build_case_scene(case)
    full = N.launch_case(sc, case).export()
    for world in (2, 4):
        stage1 = [N.launch_case(sc, case, rank=r, world=world, stage=1) for r in range(world)]
        events = np.concatenate([p.export_events() for p in stage1])
        for r, p in enumerate(stage1):
            N.nrt_launch_fans(sc, p, events, rank=r, world=world, kappa=case.kappa, tau=case.tau,
                              c_R=case.c_R, dphi_deg=case.dphi_deg, theta_ex_deg=case.theta_ex_deg,
                              edge_bin=case.edge_bin)
        merged = N.nrt_paths_merge(stage1, case.kappa).export()
        assert merged.tobytes() == full.tobytes(), world


# ------------------------------------------------------------------ edge cases ----------
def test_edge_cases(N, O):
    case = G.case("C1", n_rays=1)
    got, info, sc = run_gpu(N, case)
    ref, _, nb = O.launch(case)
    assert got.tobytes() == ref.tobytes() and info["bounces"] == nb
    # no RX -> empty set, still traced
    p = N.nrt_launch_ex(sc, case.tx, np.zeros((0, 3), np.float32), 1000, 2, 0)
    assert p.count() == 0 and p.info()["bounces"] == 3000
    # max_refl = 0: LOS only
    p = N.nrt_launch_ex(sc, case.tx, case.rx, 10_000, 0, 0)
    r = p.export()
    assert len(r) == 1 and r[0]["n_int"] == 0
    # TX outside the grid: rays enter through the slab test; compare with the oracle
    c2 = G.case("C1", n_rays=3000)
    c2.tx = np.array([-3.0, 1.5, 1.2], np.float32)
    got, info, _ = run_gpu(N, c2)
    ref, _, nb = O.launch(c2)
    assert got.tobytes() == ref.tobytes() and info["bounces"] == nb


def test_errors(N):
    case = G.case("C1")
    s = case.scene
    bad = s.normals.copy()
    bad[7] *= 1.01
    with pytest.raises(N.NrtError) as e:
        N.nrt_scene_build_ex(s.points, bad, 0.1, radii=s.radii, labels=s.labels)
    assert e.value.status == 1 and "surfel 7" in str(e.value)
    lab = s.labels.copy()
    lab[3] = 5000
    with pytest.raises(N.NrtError):
        N.nrt_scene_build_ex(s.points, s.normals, 0.1, radii=s.radii, labels=lab)
    sc = N.build_case_scene(case)
    with pytest.raises(N.NrtError):
        N.nrt_launch_ex(sc, case.tx, case.rx, 0, 2, 0)
    with pytest.raises(N.NrtError):
        N.nrt_launch_ex(sc, case.tx, case.rx, 100, 6, 3)


def test_north_star_four_arg_build(N, O):
    """nrt_scene_build(points, normals, N, voxel): r = 0.015, pseudo-labels (R6)."""
    case = G.case("C1", n_rays=3000)
    s = case.scene
    sc = N.nrt_scene_build(s.points, s.normals, s.n, 0.1)
    p = N.nrt_launch(sc, case.tx, case.rx, case.n_rays, case.max_refl, 0)
    got = p.export()
    # the oracle on the same definition: r = 0.015, labels = 0.5 m cell index (R6)
    P = s.points.astype(np.float32)
    bmin = P.min(axis=0)
    bmax = P.max(axis=0)
    idx = np.floor((P - bmin) / np.float32(0.5)).astype(np.int64)
    lx = int(np.floor((bmax[0] - bmin[0]) / np.float32(0.5))) + 1
    ly = int(np.floor((bmax[1] - bmin[1]) / np.float32(0.5))) + 1
    lab = (idx[:, 0] + lx * (idx[:, 1] + ly * idx[:, 2])).astype(np.int32)
    s2 = G.Scene(s.points, s.normals, np.full(s.n, 0.015, np.float32), lab, G.Edges.empty())
    c = G.case("C1", n_rays=3000)
    c.scene = s2
    ref, _, nb = O.launch_phased(c, procs=NPROC)
    assert p.info()["bounces"] == nb
    assert_same_records(got, ref, "4-arg build")


# ------------------------------------------------------------------ RR room, many RX ----
@pytest.mark.parametrize("name", ["C4s", "C5s"])
def test_rr_small_many_rx_bit_exact(N, O, name):
    """Reconstructed-room-like clouds (clutter, holes, split labels, outliers, plane-fit
    normals) with 85 / 879 receivers: the receiver grid path must give the brute-force set."""
    case = G.case(name)
    assert len(case.rx) > 16
    got, info, _ = run_gpu(N, case)
    ref, n_raw, nb = O.launch_phased(case, procs=NPROC)
    assert info["bounces"] == nb
    assert info["n_raw"] == n_raw
    assert_same_records(got, ref, name)
    assert len(np.unique(got["rx"])) > 5


def test_rx_grid_equals_all_pairs(N, monkeypatch):
    case = G.case("C5s", n_rays=6000)
    a, _, _ = run_gpu(N, case)
    monkeypatch.setenv("NRT_RX_GRID_MIN", "1000000")  # force the all-receivers loop
    b, _, _ = run_gpu(N, case)
    monkeypatch.setenv("NRT_RX_GRID_MIN", "2")
    monkeypatch.setenv("NRT_RX_GRID_V", "0.17")       # another cell size
    c, _, _ = run_gpu(N, case)
    assert a.tobytes() == b.tobytes() == c.tobytes()
