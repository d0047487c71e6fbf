"""SHA-256 of the refined records (keep_invalid=1) of one config's whole coarse set, for bitwise
A/B of refine builds (NRT_LIB=variant.so).  Usage: python scripts/refine_hash.py C5 [C2 ...]"""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import nrt_gen as G  # noqa: E402
import paper_2403_06648_b200 as N  # noqa: E402

for cfg in sys.argv[1:]:
    case = G.case(cfg)
    sc = N.build_case_scene(case, device_arrays=True)
    co = N.launch_case(sc, case)
    r = N.nrt_refine_ex(sc, co, xi=case.xi, r_s=case.r_s, tau=case.tau, theta_ex_deg=case.theta_ex_deg,
                        keep_invalid=1)
    a = r.export()
    print(cfg, len(a), hashlib.sha256(a.tobytes()).hexdigest()[:16], round(r.info()["ms_refine"], 1), flush=True)
