"""Profiling target for the NEXT rows' kernels (ncu launch lists with DRAM bytes):
C4 SDF primary launch (k_trace_sdf, stage 1), C2 SDF primary launch, C2 cone tracer (k_env_*),
C2 SDF coarse set refined by the paper's GD (k_refine_gd)."""
import torch

import nrt_gen as G
import paper_2403_06648_b200 as N

SDF = dict(cell=0.0625, r_s=0.015, t_sdf=0.0015, xi=2.0)
for name in ("C4", "C2"):
    case = G.case(name, sigma=0.010) if name == "C2" else G.case(name)
    case.sdf = dict(SDF)
    sc = N.build_case_scene(case)
    N.launch_case(sc, case, stage=1)  # primary bounces only: the bench's roofline_trace launches
    torch.cuda.synchronize()
    if name == "C2":
        case.kappa = 100
        N.launch_case(sc, case, tracer=1)
        torch.cuda.synchronize()
        case.kappa = 1
        co = N.launch_case(sc, case)
        N.nrt_refine_ex(sc, co, **N.gd_desc(case))
        torch.cuda.synchronize()
print("done")
