"""NEXT-2 timing: the paper's environment-driven launch + cone tracing on a config, for several
interaction caps (device time of the cone-tracing kernels, whole launch, validation rays)."""
import json
import sys
import time

import torch

import nrt_gen as G
import paper_2403_06648_b200 as N

SDF = dict(cell=0.0625, r_s=0.015, t_sdf=0.0015, xi=2.0)
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
caps = [tuple(int(x) for x in c.split(",")) for c in (sys.argv[2:] or ["1,1", "2,1", "3,1"])]
kw = dict(sigma=0.010) if name.startswith("C2") else {}
for mr, md in caps:
    case = G.case(name, max_refl=mr, max_diff=md, **kw)
    case.sdf = dict(SDF)
    case.kappa = 100
    sc = N.build_case_scene(case)
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.time()
        p = N.launch_case(sc, case, tracer=1)
        torch.cuda.synchronize()
        wall = (time.time() - t) * 1e3
        i = p.info()
        print(json.dumps(dict(config=name, max_refl=mr, max_diff=md, rep=rep, wall_ms=round(wall, 1),
                              kernel_ms=round(i["ms_trace"], 2), rays=int(i["bounces"]), raw=int(i["n_raw"]),
                              paths=int(i["n"]), rays_per_s=round(i["bounces"] / wall * 1e3))), flush=True)
