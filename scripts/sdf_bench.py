"""NEXT-1 timing: the same launch with the disk hit (R7-R9) and with the paper's SDF
intersection (R40-R45); device-timed trace kernels (info ms_trace) and the whole launch."""
import argparse
import json
import time

import numpy as np
import torch

import nrt_gen as G
import paper_2403_06648_b200 as N

SDF = dict(cell=0.0625, r_s=0.015, t_sdf=0.0015, xi=2.0)

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--sigma", type=float, default=0.010)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--max_diff", type=int, default=None)
args = ap.parse_args()
kw = dict(sigma=args.sigma) if args.config.startswith("C2") else {}
if args.max_diff is not None:
    kw["max_diff"] = args.max_diff
case = G.case(args.config, **kw)
case.sdf = dict(SDF)
t = time.time()
sc = N.build_case_scene(case)
torch.cuda.synchronize()
print("build %.1f ms" % ((time.time() - t) * 1e3), sc.info())
for mode in (0, 1):
    for r in range(args.reps):
        torch.cuda.synchronize()
        t = time.time()
        p = N.launch_case(sc, case, intersect=mode)
        torch.cuda.synchronize()
        wall = (time.time() - t) * 1e3
        i = p.info()
        print(json.dumps(dict(mode="sdf" if mode else "disk", rep=r, wall_ms=round(wall, 2),
                              ms_trace=round(i["ms_trace"], 3), bounces=int(i["bounces"]),
                              n=int(i["n"]), n_raw=int(i["n_raw"]), fans=int(i["n_fan_rays"]),
                              gbounce_s=round(i["bounces"] / wall / 1e6, 3))))
# work counters (instrumented kernels): per segment cells, AABB marches, Gaussian terms
for mode in (0, 1):
    p = N.launch_case(sc, case, intersect=mode, counters=1)
    i = p.info()
    b = max(1, i["bounces"])
    print(json.dumps(dict(mode="sdf" if mode else "disk", counters=True, ms_trace=round(i["ms_trace"], 3),
                          cells_per_seg=round(i["cells_visited"] / b, 2),
                          nonempty_or_marches_per_seg=round(i["cells_nonempty"] / b, 2),
                          tests_or_terms_per_seg=round(i["surfel_tests"] / b, 1))))
