"""GPU parity of the refined-path post-processing (PAPER §II-E
P:234-242, R33-R36) against the CPU oracle through the C ABI: the same refined
records post-processed on both sides give the same records, bit for bit (labels are integer
decisions taken on FP64 distances computed in the same order; the Fresnel and angle tests are
FP64 in the same order on both sides)."""
import math

import numpy as np
import pytest

import nrt_gen as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def N():
    import torch
    assert torch.cuda.is_available()
    import paper_2403_06648_b200 as N
    N.lib()
    return N


def refined_set(N, case):
    sc = N.build_case_scene(case)
    coarse = N.launch_case(sc, case)
    ref = N.nrt_refine_ex(sc, coarse, xi=case.xi, r_s=case.r_s, tau=case.tau,
                          theta_ex_deg=case.theta_ex_deg)
    return sc, ref


def check(N, O, case, angle_deg=10.0):
    sc, ref = refined_set(N, case)
    got = N.nrt_postprocess(sc, ref, r_s=case.r_s, angle_deg=angle_deg).export()
    want = O.postprocess(case, ref.export(), r_s=case.r_s, angle_deg=angle_deg)
    assert len(got) == len(want)
    assert got.tobytes() == want.tobytes()
    assert np.all(np.diff(got["delay"]) >= 0)
    return ref.count(), len(got)


def test_c1_post_equals_oracle(N, O):
    n_in, n_out = check(N, O, G.case("C1"))
    assert n_in == 25 and n_out == 25   # the box room's image paths are all distinct


@pytest.mark.parametrize("sigma", [0.0, 0.005])
def test_sr_small_post_equals_oracle(N, O, sigma):
    check(N, O, G.case("C2s", sigma=sigma, n=12_000, n_rays=8000, max_refl=2, max_diff=1))


def test_c2_full_post_equals_oracle_and_is_duplicate_free(N, O):
    case = G.case("C2", sigma=0.010)
    n_in, n_out = check(N, O, case)
    assert 0 < n_out <= n_in
    # a wide angle threshold and a long wavelength merge more: still equal to the oracle
    sc, ref = refined_set(N, case)
    got = N.nrt_postprocess(sc, ref, r_s=case.r_s, angle_deg=30.0, lambda_m=0.05).export()
    want = O.postprocess(case, ref.export(), r_s=case.r_s, angle_deg=30.0, lambda_m=0.05)
    assert got.tobytes() == want.tobytes() and len(got) <= n_out
    cmax = math.cos(math.radians(30.0))
    for i in range(len(got)):
        for j in range(i + 1, len(got)):
            if (got["rx"][i], got["n_int"][i], got["kinds"][i]) == (got["rx"][j], got["n_int"][j], got["kinds"][j]):
                assert not O.fresnel_dup(case, got[i], got[j], cmax, lambda_m=0.05)


def test_post_errors(N):
    case = G.case("C1", n_rays=3000)
    sc = N.build_case_scene(case)
    coarse = N.launch_case(sc, case)
    with pytest.raises(N.NrtError):
        N.nrt_postprocess(sc, coarse)          # not a refined set
    ref = N.nrt_refine_ex(sc, coarse, xi=case.xi, r_s=case.r_s, tau=case.tau)
    with pytest.raises(N.NrtError):
        N.nrt_postprocess(sc, ref, lambda_m=0.0)
