import os, sys, json
sys.path.insert(0, "/root/repo")
import numpy as np
import nrt_gen as G
import paper_2403_06648_b200 as N
import torch
os.environ["NRT_PHASES"] = "1"
case = G.case("C5")
case.n_rays = 30_000_000
sc = N.build_case_scene(case, device_arrays=True)
for label, rx in (("879rx", case.rx), ("1rx", case.rx[:1]), ("0rx", case.rx[:0])):
    c2 = G.case("C5"); c2.scene = case.scene; c2.rx = rx; c2.n_rays = case.n_rays
    for rep in range(2):
        p = N.launch_case(sc, c2)
        torch.cuda.synchronize()
    print(label, p.info()["ms_trace"], flush=True)
