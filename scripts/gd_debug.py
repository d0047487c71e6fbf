"""Dump a GPU NEXT-4 run (coarse set + refined records with keep_invalid) for offline comparison
with the oracle: python scripts/gd_debug.py C2 0.0 2000 out.npz [rho]"""
import sys

import numpy as np

import nrt_gen as G
import paper_2403_06648_b200 as N

name, sigma, n_rays, out = sys.argv[1], float(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
rho = int(sys.argv[5]) if len(sys.argv) > 5 else 2000
case = G.case(name, sigma=sigma, n_rays=n_rays, max_diff=0) if name.startswith("C2") else G.case(name, n_rays=n_rays)
case.sdf = dict(cell=0.0625, r_s=0.015, t_sdf=0.0015, xi=2.0)
if sigma == 0.0:
    case.gd = dict(r_s=0.003, t_sdf=0.0005, t_d=0.002, t_a_deg=1.0)
sc = N.build_case_scene(case)
co = N.launch_case(sc, case)
ref = N.nrt_refine_ex(sc, co, keep_invalid=1, **N.gd_desc(case, rho=rho))
np.savez(out, coarse=co.export(), got=ref.export())
