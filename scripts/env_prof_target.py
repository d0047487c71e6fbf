import torch, nrt_gen as G, paper_2403_06648_b200 as N
case = G.case("C2", sigma=0.010, max_refl=3, max_diff=1); case.sdf = dict(cell=0.0625, r_s=0.015, t_sdf=0.0015, xi=2.0); case.kappa = 100
sc = N.build_case_scene(case); p = N.launch_case(sc, case, tracer=1); torch.cuda.synchronize(); print(p.info()["bounces"])
