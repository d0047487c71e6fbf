"""Per-phase timing of one hot-path step on cuda:0 (scene build / launch / refine), printed
as JSON; used for profiling runs (also the target of ncu launch lists)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import nrt_gen as G
    import paper_2403_06648_b200 as N
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    voxel = float(sys.argv[3]) if len(sys.argv) > 3 and float(sys.argv[3]) > 0 else None
    case = G.case(cfg)
    if voxel:
        case.voxel = voxel
    if len(sys.argv) > 4:
        case.n_rays = int(float(sys.argv[4]))
    if os.environ.get("NRT_PROF_NO_REFINE"):
        globals()["_no_refine"] = True
    s = case.scene
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    pts, nrm, rad, lab = t(s.points), t(s.normals), t(s.radii), t(s.labels)
    st = torch.cuda.current_stream()
    out = []
    for r in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sc = N.nrt_scene_build_ex(pts, nrm, case.voxel, radii=rad, labels=lab, edges=s.edges,
                                  stream=st)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        p = N.launch_case(sc, case, stream=st, counters=1 if r == 0 else 0)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        info = p.info()
        if globals().get("_no_refine"):
            out.append({"build_ms": 1e3 * (t1 - t0), "launch_ms": 1e3 * (t2 - t1),
                        **{k: info[k] for k in ("ms_trace", "ms_fans", "bounces", "n",
                                                "surfel_tests", "cells_visited")}})
            continue
        rf = N.nrt_refine_ex(sc, p, xi=case.xi, r_s=case.r_s, tau=case.tau, keep_invalid=1,
                             stream=st)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        rr = rf.export()
        rinfo = rf.info()
        import collections
        out.append({"refine_ms": 1e3 * (t3 - t2), "ms_refine_kernel": rinfo["ms_refine"],
                    "status": dict(collections.Counter(int(x) for x in rr["status"])),
                    "iters_hist": np.histogram(rr["iters"], bins=[0, 2, 4, 8, 16, 32, 64, 101])[0].tolist(),
                    "iters_max": int(rr["iters"].max()) if len(rr) else 0})
        out.append({"build_ms": 1e3 * (t1 - t0), "launch_ms": 1e3 * (t2 - t1),
                    **{k: info[k] for k in ("ms_trace", "ms_fans", "ms_dedupe", "ms_total",
                                            "bounces", "n_raw", "n", "n_events", "n_fan_rays",
                                            "surfel_tests", "cells_visited", "cells_nonempty")},
                    "scene": sc.info()})
        del p, sc
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
