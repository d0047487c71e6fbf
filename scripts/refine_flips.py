"""Dump a refinement parity sample for offline study: coarse records, GPU refined records of the
warp and block kernels (keep_invalid).  Usage: python scripts/refine_flips.py C4 seed n_ok n_any"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import nrt_gen as G  # noqa: E402
import paper_2403_06648_b200 as N  # noqa: E402


def main():
    cfg, seed, n_ok, n_any = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    case = G.case(cfg)
    sc = N.build_case_scene(case, device_arrays=True)
    coarse = N.launch_case(sc, case)
    cr = coarse.export()
    out = {"coarse": cr}
    for impl in ("warp", "block"):
        os.environ["NRT_REFINE_IMPL"] = impl
        out[impl] = N.nrt_refine_ex(sc, coarse, xi=case.xi, r_s=case.r_s, tau=case.tau,
                                    theta_ex_deg=case.theta_ex_deg, keep_invalid=1).export()
    rng = np.random.default_rng(seed)
    allg = out["warp"]
    ok = np.nonzero(allg["status"] == 0)[0]
    rest = np.setdiff1d(np.arange(len(allg)), ok)
    idx = np.sort(np.concatenate([rng.choice(ok, min(n_ok, len(ok)), replace=False),
                                  rng.choice(rest, min(n_any, len(rest)), replace=False)]))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    np.savez(os.path.join(ROOT, "gpurun_out", f"flips_{cfg}.npz"), idx=idx, coarse=cr[idx],
             warp=out["warp"][idx], block=out["block"][idx])
    print("saved", len(idx))


if __name__ == "__main__":
    main()
