"""NEXT-1 path quality ("compare path quality vs disks at sigma = 5-20 mm").

On the C2 scene (1e6 surfels, 1e6 rays, diffraction) at noise sigma in {0, 5, 10, 20} mm, the
coarse launch runs with the disk hit (R7-R9) and with the paper's SDF intersection (R40-R45);
both coarse sets are refined by the same Gauss-Newton refinement (A9/A10).  Reference = the
valid refined paths of the noise-free cloud with the disk hit (the synthetic room's exact
specular/diffracted paths up to the refinement tolerance).  Reported per (sigma, mode): coarse
and valid refined counts, recall / precision of the reference keys (rx, kinds, labels), and the
median / 95th-percentile |delay - reference delay| over matched keys.
"""
import json
import sys

import numpy as np
import torch

import nrt_gen as G
import paper_2403_06648_b200 as N

SDF = dict(cell=0.0625, r_s=0.015, t_sdf=0.0015, xi=2.0)
OK = 0


def keyset(rec):
    out = {}
    for r in rec:
        if int(r["status"]) != OK:
            continue
        k = (int(r["rx"]), int(r["n_int"]), int(r["kinds"]), tuple(int(x) for x in r["label"]))
        out[k] = float(r["delay"])
    return out


def run(sigma, sdf):
    case = G.case("C2", sigma=sigma)
    if sdf:
        case.sdf = dict(SDF)
    sc = N.build_case_scene(case)
    torch.cuda.synchronize()
    c = N.launch_case(sc, case)
    ci = c.info()
    ref = N.nrt_refine_ex(sc, c, xi=case.xi, r_s=case.r_s, tau=case.tau,
                          theta_ex_deg=case.theta_ex_deg)
    rec = ref.export()
    return ci, rec


def main():
    sigmas = [float(x) for x in sys.argv[1:]] or [0.0, 0.005, 0.010, 0.020]
    _, rec0 = run(0.0, False)
    ref = keyset(rec0)
    rows = []
    for sg in sigmas:
        for sdf in (False, True):
            ci, rec = run(sg, sdf)
            ks = keyset(rec)
            both = sorted(set(ks) & set(ref))
            dd = np.array([abs(ks[k] - ref[k]) for k in both]) if both else np.zeros(1)
            row = dict(sigma_mm=sg * 1e3, mode="sdf" if sdf else "disk", coarse=ci["n"],
                       bounces=int(ci["bounces"]), valid=len(ks), ref_valid=len(ref),
                       recall=len(both) / max(1, len(ref)), precision=len(both) / max(1, len(ks)),
                       ddelay_med_ps=float(np.median(dd)) * 1e12,
                       ddelay_p95_ps=float(np.percentile(dd, 95)) * 1e12,
                       ms_trace=round(ci["ms_trace"] + ci["ms_fans"], 3))
            rows.append(row)
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
