"""A/B of the refine kernels on one config (GPU): the block kernel (NRT_REFINE_IMPL=block) vs
the warp-per-path kernel (=warp) on the same coarse set, keep_invalid=1.  Prints times, status
counts and whether the records are bitwise equal (they must be: same arithmetic).
Usage: python scripts/refine_ab.py C4 [impl ...]"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import nrt_gen as G  # noqa: E402
import paper_2403_06648_b200 as N  # noqa: E402


def main():
    import torch
    cfg = sys.argv[1]
    args = sys.argv[2:]
    sub = 0
    if args and args[0].startswith("--sub="):
        sub = int(args.pop(0)[6:])
    impls = args or ["block", "warp"]
    case = G.case(cfg)
    sc = N.build_case_scene(case, device_arrays=True)
    coarse = N.launch_case(sc, case)
    if sub:  # every k-th coarse path (profiling runs)
        rec = coarse.export()
        coarse = N.nrt_paths_import(rec[:: max(1, len(rec) // sub)], N.PATHS_COARSE, case.tx, case.rx)
    out, recs = {"cfg": cfg, "coarse": coarse.count()}, {}
    for impl in impls:
        os.environ["NRT_REFINE_IMPL"] = impl
        ms = []
        for _ in range(2):
            r = N.nrt_refine_ex(sc, coarse, xi=case.xi, r_s=case.r_s, tau=case.tau,
                                theta_ex_deg=case.theta_ex_deg, keep_invalid=1)
            ms.append(round(r.info()["ms_refine"], 3))
        a = r.export()
        recs[impl] = a
        out[impl] = {"ms": ms, "status": np.bincount(a["status"], minlength=7).tolist(),
                     "iters": int(a["iters"].sum())}
        r.free()
    base = recs[impls[0]]
    for impl in impls[1:]:
        b = recs[impl]
        same = base.tobytes() == b.tobytes()
        ok = (base["status"] == 0) & (b["status"] == 0)
        out[f"{impl}_vs_{impls[0]}"] = {
            "bitwise": same,
            "status_diff": int((base["status"] != b["status"]).sum()),
            "max_dv_ok": float(np.abs(base["v"][ok] - b["v"][ok]).max()) if ok.any() else 0.0,
            "ok_far_1e-5": int((np.abs(base["v"][ok] - b["v"][ok]).reshape(ok.sum(), -1).max(1) > 1e-5).sum())
            if ok.any() else 0,
            "ok_both": int(ok.sum())}
    os.environ.pop("NRT_REFINE_IMPL", None)
    torch.cuda.synchronize()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
