"""Refinement latency probe: refine subsets of a saved C2 coarse set (variants/C2_coarse.npy):
all paths, the long-iteration ones (variants/long_ix.npy), the rest, and a single path."""
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
    case = G.case("C2")
    sc = N.build_case_scene(case)
    rec = np.load(os.path.join(ROOT, "variants", "C2_coarse.npy"))
    long_ix = np.load(os.path.join(ROOT, "variants", "long_ix.npy"))
    rest = np.setdiff1d(np.arange(len(rec)), long_ix)
    sets = {"all": np.arange(len(rec)), "long": long_ix, "rest": rest, "one": long_ix[:1]}
    out = {"lib": os.environ.get("NRT_LIB", "libnrt.so")}
    for name, ix in sets.items():
        ms = []
        for _ in range(3):
            p = N.nrt_paths_import(rec[ix], N.PATHS_COARSE, case.tx, case.rx)
            r = N.nrt_refine_ex(sc, p, xi=case.xi, r_s=case.r_s, tau=case.tau, keep_invalid=1)
            ms.append(r.info()["ms_refine"])
            st = np.bincount(r.export()["status"], minlength=7).tolist()
        torch.cuda.synchronize()
        out[name] = {"n": int(len(ix)), "ms": round(float(np.median(ms)), 3), "status": st}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
