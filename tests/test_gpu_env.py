"""GPU parity of NEXT-2, the paper's coarse tracer — environment-driven launch and voxel cone
tracing (PAPER §II-B/§II-D, Alg. 1; DESIGN R60-R67) — against the oracle (oracle/env.c),
through the C ABI (nrt_launch_desc.tracer = 1 with the SDF intersection).

Bar: the coarse path set (kappa = 100 shortest per key), the raw record count and the number of
validation rays equal the oracle's bit for bit.
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


def run(N, case, **kw):
    sc = N.build_case_scene(case)
    p = N.launch_case(sc, case, tracer=1, **kw)
    return p.export(), p.info()


def check(N, O, case, what, min_recs=1):
    got, info = run(N, case)
    ref, n_raw, nrays = O.env_launch(case, procs=NPROC)
    assert info["n_raw"] == n_raw, (what, info["n_raw"], n_raw)
    assert info["bounces"] == nrays, (what, info["bounces"], nrays)
    assert_same_records(got, ref, what)
    assert len(got) >= min_recs
    return got


def test_env_dense_box_room_bit_exact(N, O):
    case = G.case("C1", n_rays=1000)
    case.scene = G.box_room(3)
    case.sdf = dict(SDF)
    case.kappa = 100
    got = check(N, O, case, "NEXT-2 dense C1", 25)
    assert (got["n_int"] == 2).sum() > 10


def test_env_wedge_diffraction_bit_exact(N, O):
    from tests.test_oracle_capture_pins import case_of, wedge_scene
    sc = wedge_scene()
    case = case_of(sc, np.array([-0.8, 0.3, 1.3]), np.array([0.3, -0.8, 0.9]), n_rays=1000, max_refl=1,
                   max_diff=1, kappa=100, dphi_deg=2.5)
    case.sdf = dict(SDF)
    got = check(N, O, case, "NEXT-2 wedge")
    assert (got["n_diff"] == 1).sum() > 0


@pytest.mark.parametrize("max_diff", [0, 1])
def test_env_c2_scene_bit_exact(N, O, max_diff):
    """The C2 scene (1e6 surfels, sigma 10 mm, 20 exterior edges): one reflection, with and
    without a diffraction."""
    case = G.case("C2", sigma=0.010, n_rays=1000, max_refl=1, max_diff=max_diff)
    case.sdf = dict(SDF)
    case.kappa = 100
    got = check(N, O, case, f"NEXT-2 C2 max_diff={max_diff}", 10)
    if max_diff:
        assert (got["n_diff"] == 1).sum() > 100


def test_env_world_shards_merge(N):
    """Transmission rays sharded i == rank (mod world): the merged shards equal world 1."""
    case = G.case("C1", n_rays=1000)
    case.scene = G.box_room(2)
    case.sdf = dict(SDF)
    case.kappa = 100
    sc = N.build_case_scene(case)
    full = N.launch_case(sc, case, tracer=1)
    parts = [N.launch_case(sc, case, tracer=1, rank=r, world=3) for r in range(3)]
    merged = N.nrt_paths_merge(parts, case.kappa)
    assert merged.export().tobytes() == full.export().tobytes()
    assert sum(p.info()["bounces"] for p in parts) == full.info()["bounces"]


def test_env_errors(N):
    case = G.case("C1", n_rays=1000)
    case.sdf = dict(SDF)
    sc = N.build_case_scene(case)
    with pytest.raises(N.NrtError):
        N.launch_case(sc, case, tracer=1, intersect=0)


@pytest.mark.parametrize("name,parts", [("C4", 512), ("C5", 2048)])
def test_env_fullsize_sharded_subset_bit_exact(N, O, name, parts):
    """Full-size scenes (1e7 surfels; C4: 85 RX with diffraction, C5: 879 RX): the transmission
    shard i == 0 (mod parts) and its whole cone-traced subtree (rank 0 of world = parts) equals
    the oracle's part 0 — records (kappa = 2^30 keeps every one), raw and validation-ray counts."""
    case = G.case(name, max_refl=2)
    case.sdf = dict(SDF)
    case.kappa = 1 << 30
    sc = N.build_case_scene(case)
    p = N.launch_case(sc, case, tracer=1, rank=0, world=parts, stage=1)
    got, info = p.export(), p.info()
    O.env_lib()
    O._FORK["env"] = O.EnvScene(case)
    raw, rays = O._env_worker((case, 0, parts))
    O._FORK.pop("env", None)
    ref = O.dedupe(raw, case.kappa)
    assert info["n_raw"] == len(raw) and info["bounces"] == rays, (info["n_raw"], len(raw), info["bounces"], rays)
    assert_same_records(got, ref, f"NEXT-2 {name} shard 0/{parts}")
    assert len(got) > 0


def test_env_full_c2_bit_exact(N, O):
    """The paper's setting on the whole C2 scene: <= 3 reflections, <= 1 diffraction, kappa 100
    (1.3e7 validation rays): set, raw and validation-ray counts equal the oracle's (tier-1 SDF
    grid)."""
    case = G.case("C2", sigma=0.010, max_refl=3, max_diff=1)
    case.sdf = dict(SDF)
    case.kappa = 100
    got, info = run(N, case)
    ref, n_raw, nrays = O.env_launch(case, procs=NPROC, sdf_grid=0.125)
    assert info["n_raw"] == n_raw and info["bounces"] == nrays, (info["n_raw"], n_raw, info["bounces"], nrays)
    assert_same_records(got, ref, "NEXT-2 full C2")
    assert len(got) > 10_000
