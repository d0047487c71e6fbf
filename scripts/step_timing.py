"""Host wall-clock per API call of the bench step (diagnosing step-time outliers)."""
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
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    case = G.case("C2")
    s = case.scene
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    pts, nrm, rad, lab = t(s.points), t(s.normals), t(s.radii), t(s.labels)
    tx, rx = t(case.tx), t(case.rx.reshape(-1, 3))
    st = torch.cuda.current_stream()
    desc = dict(kappa=case.kappa, tau=case.tau, c_R=case.c_R, dphi_deg=case.dphi_deg,
                theta_ex_deg=case.theta_ex_deg, edge_bin=case.edge_bin)
    rows = []
    flush = torch.empty((512 << 20) // 4, dtype=torch.float32, device=dev) if "flush" in sys.argv else None
    for r in range(reps):
        if flush is not None:
            flush.fill_(float(r))
        torch.cuda.synchronize()
        T = [time.perf_counter()]
        sc = N.nrt_scene_build_ex(pts, nrm, case.voxel, radii=rad, labels=lab, edges=s.edges, stream=st)
        T.append(time.perf_counter())
        co = N.nrt_launch_ex(sc, tx, rx, case.n_rays, case.max_refl, case.max_diff, stream=st, **desc)
        T.append(time.perf_counter())
        rf = N.nrt_refine_ex(sc, co, xi=case.xi, r_s=case.r_s, tau=case.tau, stream=st)
        T.append(time.perf_counter())
        i1, i2 = co.info(), rf.info()
        rf.free()
        co.free()
        sc.free()
        T.append(time.perf_counter())
        torch.cuda.synchronize()
        T.append(time.perf_counter())
        d = np.diff(T) * 1e3
        rows.append({"build": round(d[0], 2), "launch": round(d[1], 2), "refine": round(d[2], 2),
                     "free": round(d[3], 2), "sync": round(d[4], 2),
                     "launch_dev": round(i1["ms_total"], 2), "refine_kernel": round(i2["ms_refine"], 2)})
    print(json.dumps(rows, indent=0))


if __name__ == "__main__":
    main()
