"""Refinement workload statistics on one config (GPU): status x iteration histograms, time,
and the effect of the refine parameters (r_s, max_iter).  Saves the coarse set to
gpurun_out/<cfg>_coarse.npy for offline analysis.
Usage: python scripts/refine_stats.py C4 [r_s,max_iter ...]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import nrt_gen as G  # noqa: E402
import paper_2403_06648_b200 as N  # noqa: E402


def main():
    import torch
    cfg = sys.argv[1]
    variants = [tuple(float(x) for x in v.split(",")) for v in sys.argv[2:]]
    case = G.case(cfg)
    sc = N.build_case_scene(case, device_arrays=True)
    coarse = N.launch_case(sc, case)
    rec = coarse.export()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    if len(rec) * rec.itemsize < 48 << 20:
        np.save(os.path.join(ROOT, "gpurun_out", f"{cfg}_coarse.npy"), rec)
    out = {"cfg": cfg, "coarse": int(len(rec)),
           "n_int_hist": np.bincount(rec["n_int"], minlength=6).tolist(),
           "n_diff_hist": np.bincount(rec["n_diff"], minlength=2).tolist()}
    runs = [(case.r_s, 100)] + [(v[0], int(v[1])) for v in variants]
    for r_s, mi in runs:
        ms = []
        for rep in range(2):
            t0 = time.time()
            r = N.nrt_refine_ex(sc, coarse, xi=case.xi, r_s=r_s, tau=case.tau, keep_invalid=1,
                                max_iter=mi)
            ms.append(r.info()["ms_refine"])
        a = r.export()
        st = a["status"]
        it = a["iters"]
        key = f"r_s={r_s},max_iter={mi}"
        edges = [0, 1, 2, 3, 5, 8, 12, 20, 30, 50, 75, 99, 100, 101]
        h = {}
        for s in range(7):
            m = st == s
            h[N.REF_STATUS[s]] = np.histogram(it[m], bins=edges)[0].tolist()
        work = {"ms": ms, "status": np.bincount(st, minlength=7).tolist(),
                "iters_sum_by_status": [int(it[st == s].sum()) for s in range(7)],
                "iter_bins": edges, "hist": h,
                "valid_iters_p50_p90_p99_max": [float(np.percentile(it[st == 0], q)) if (st == 0).any() else 0
                                                for q in (50, 90, 99, 100)]}
        out[key] = work
        r.free()
        print(json.dumps({key: work}), flush=True)
    torch.cuda.synchronize()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
