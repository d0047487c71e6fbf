"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck / synccheck): C1 and a
small synthetic room with diffraction through scene build, launch (with the forced live-list
reorder), both refinement kernels (block and warp), post-processing and the debug hit dump."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import nrt_gen as G  # noqa: E402
import paper_2403_06648_b200 as N  # noqa: E402


def main():
    os.environ["NRT_REORDER"] = "1"
    os.environ["NRT_SORT_MIN"] = "1"
    for case in (G.case("C1", n_rays=2000),
                 G.case("C2s", sigma=0.005, n=8000, n_rays=3000, max_refl=2, max_diff=1)):
        sc = N.build_case_scene(case)
        p = N.launch_case(sc, case)
        for impl in ("block", "warp"):
            os.environ["NRT_REFINE_IMPL"] = impl
            r = N.nrt_refine_ex(sc, p, xi=case.xi, r_s=case.r_s, tau=case.tau,
                                theta_ex_deg=case.theta_ex_deg, counters=1)
            q = N.nrt_postprocess(sc, r, r_s=case.r_s)
            print(case.name, impl, p.count(), r.count(), q.count(), flush=True)
        ids = np.arange(0, case.n_rays, 97, dtype=np.uint64)
        h = N.nrt_debug_trace_rays(sc, case.tx, case.n_rays, case.max_refl, ids, tau=case.tau)
        print(case.name, "hits", int((h >= 0).sum()), flush=True)


if __name__ == "__main__":
    main()
