"""Whole-configuration coarse parity through the production kernels (rows A1-A8 at the
BASELINE.json sizes), against the CPU oracle.

* Full sets: the GPU's complete coarse set of a full-size launch (`nrt_launch_ex`, the same
  call bench.py times: primary rays, events, Keller fans, dedupe) equals the oracle's set byte
  for byte, with the same raw-record, event and ray-bounce counts.  The oracle side is the
  tier-1 grid (oracle/grid.c, pinned to the brute force by tests/test_oracle_grid_pins.py):
  computed live for C2, and for the bigger configurations stored by scripts/make_golden.py
  (which calls only oracle/) as counts + SHA-256 in tests/golden/fullsize_sets.json.
* Sharded subsets vs the brute-force definition itself (tier 0): rank r of a large world
  traces ~300 primary rays of the full lattice through the production path (stage 1, kappa
  = 2^30 keeps every raw record); records, events and bounces equal tier 0's.
* Per-ray hit sequences dumped by the production TRACE/SHADE kernels (nrt_debug_trace_rays),
  with and without the forced live-list reorder.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import nrt_gen as G

pytestmark = pytest.mark.gpu
NPROC = max(1, min(64, os.cpu_count() or 1))
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fullsize_sets.json")))
KAPPA_ALL = 1 << 30


@pytest.fixture(scope="module")
def N():
    import torch
    assert torch.cuda.is_available()
    import paper_2403_06648_b200 as N
    N.lib()
    return N


def case_of(name):
    if name.startswith("C2s") and name[3:].isdigit():
        return G.case("C2", sigma=int(name[3:]) / 1000.0)
    return G.case(name)


def gpu_full(N, case):
    sc = N.build_case_scene(case, device_arrays=True)
    p = N.launch_case(sc, case)
    return p.export(), p.info()


# ------------------------------------------------------------------ full sets -----------
def test_c2_full_set_live_oracle(N, O):
    """C2 (the bench's secondary workload): the whole set, fans included, vs the tier-1 oracle
    computed now."""
    case = G.case("C2")
    got, info = gpu_full(N, case)
    ref, n_raw, nb, ev = O.launch_phased(case, procs=NPROC, return_events=True, grid_voxel=0.05)
    assert info["bounces"] == nb and info["n_raw"] == n_raw and info["n_events"] == len(ev)
    assert got.tobytes() == ref.tobytes()
    assert (got["n_diff"] == 1).sum() > 1000


@pytest.mark.parametrize("name", ["C2s0", "C2s5", "C2s20", "C3", "C4", "C5"])
def test_full_set_vs_stored_oracle(N, name):
    """Every other configuration at full size: counts and SHA-256 of the oracle's whole set."""
    if name not in GOLD:
        pytest.skip(f"{name} not in tests/golden/fullsize_sets.json (scripts/make_golden.py)")
    g = GOLD[name]
    case = case_of(name)
    assert case.n_rays == g["n_rays"] and case.scene.n == g["n_surfels"]
    got, info = gpu_full(N, case)
    assert info["bounces"] == g["bounces"], (info["bounces"], g["bounces"])
    assert info["n_raw"] == g["n_raw"]
    assert info["n_events"] == g["events"]
    assert len(got) == g["records"]
    assert hashlib.sha256(got.tobytes()).hexdigest() == g["sha256"]


# ------------------------------------------------------------------ sharded subsets -----
def _tier0_shard(O, case, rank, world):
    """Brute-force primary records/events/bounces of lattice rays i == rank (mod world),
    split over forked processes as i == rank + q world (mod P world)."""
    import multiprocessing as mp
    O._FORK["case"], O._FORK["max_diff"] = case, None
    O._FORK["scene"] = O.OracleScene(case.scene)
    with mp.get_context("fork").Pool(NPROC) as pool:
        parts = pool.map(O._primary_worker, [(rank + q * world, NPROC * world) for q in range(NPROC)])
    O._FORK.pop("scene")
    raw = np.concatenate([x[0] for x in parts])
    ev = O.event_dedupe(np.concatenate([x[1] for x in parts]))
    return O.dedupe(raw, KAPPA_ALL), ev, sum(x[2] for x in parts)


@pytest.mark.parametrize("name,rays", [("C2", 4000), ("C3", 300), ("C4", 300), ("C5", 1000)])
def test_sharded_subset_vs_brute_force(N, O, name, rays):
    """A shard of the full-size lattice through the production path (stage 1) equals tier 0:
    every raw record (kappa = 2^30), the locally deduped events and the bounce count."""
    case = case_of(name)
    world = case.n_rays // rays
    rank = world // 3
    sc = N.build_case_scene(case, device_arrays=True)
    p = N.launch_case(sc, case, rank=rank, world=world, stage=1, kappa=KAPPA_ALL)
    got, info = p.export(), p.info()
    ev = p.export_events()
    ref, ref_ev, nb = _tier0_shard(O, case, rank, world)
    assert info["bounces"] == nb
    assert len(got) == len(ref) and got.tobytes() == ref.tobytes()
    assert len(ev) == len(ref_ev) and ev.tobytes() == ref_ev.tobytes()
    # C3 (1 RX, 128 coarse paths from 1e7 rays) records nothing in 300 rays: bounces only
    assert len(got) + len(ev) > 0 or name == "C3"


# ------------------------------------------------------------------ hit dumps -----------
def _tier0_hits(O, case, ids):
    import multiprocessing as mp
    chunks = np.array_split(ids, NPROC)
    O._FORK["case"] = case
    with mp.get_context("fork").Pool(NPROC) as pool:
        parts = pool.map(_hits_worker, [c for c in chunks if len(c)])
    return np.concatenate(parts)


def _hits_worker(ids):
    from oracle import oracle as O
    case = O._FORK["case"]
    return O.trace_rays(case, ids)[1]


@pytest.mark.parametrize("name,n", [("C2", 256), ("C3", 96), ("C4", 64), ("C5", 64)])
def test_production_hit_sequences_vs_brute_force(N, O, name, n, monkeypatch):
    """Per-segment hit ids of sampled rays of the full lattices, dumped by the production
    k_trace/k_shade, equal the brute-force argmin segment by segment; also with the per-bounce
    live-list reorder forced on (NRT_REORDER=1, NRT_SORT_MIN=1)."""
    case = case_of(name)
    sc = N.build_case_scene(case, device_arrays=True)
    ids = np.sort(np.random.default_rng(17).choice(case.n_rays, n, replace=False)).astype(np.uint64)
    kw = dict(tau=case.tau, theta_ex_deg=case.theta_ex_deg, c_R=case.c_R)
    a = N.nrt_debug_trace_rays(sc, case.tx, case.n_rays, case.max_refl, ids, **kw)
    monkeypatch.setenv("NRT_REORDER", "1")
    monkeypatch.setenv("NRT_SORT_MIN", "1")
    b = N.nrt_debug_trace_rays(sc, case.tx, case.n_rays, case.max_refl, ids, **kw)
    ref = _tier0_hits(O, case, ids)
    assert np.array_equal(a, ref)
    assert np.array_equal(b, ref)
    assert (ref[:, 1] >= 0).sum() > n // 2


@pytest.mark.parametrize("name", ["C4s", "C5s", "C2s"])
def test_forced_reorder_full_set(N, O, name, monkeypatch):
    """The per-bounce reorder (normally only when the records exceed 4x L2) forced on small
    scenes: the whole coarse set still equals the brute-force oracle."""
    case = G.case(name) if name != "C2s" else G.case("C2s", sigma=0.005, n=12_000, n_rays=8000,
                                                        max_refl=2, max_diff=1)
    monkeypatch.setenv("NRT_REORDER", "1")
    monkeypatch.setenv("NRT_SORT_MIN", "1")
    sc = N.build_case_scene(case)
    p = N.launch_case(sc, case)
    got, info = p.export(), p.info()
    ref, n_raw, nb = O.launch_phased(case, procs=NPROC)
    assert info["bounces"] == nb and info["n_raw"] == n_raw
    assert got.tobytes() == ref.tobytes()
