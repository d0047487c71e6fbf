"""Host-time of each API call of the C5 step and the default mempool's state (diagnostics of
step-time variance)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import nrt_gen as G  # noqa: E402
import paper_2403_06648_b200 as N  # noqa: E402


def pool_stats():
    from cuda.bindings import runtime as rt
    _, pool = rt.cudaDeviceGetDefaultMemPool(0)
    out = []
    for a in (rt.cudaMemPoolAttr.cudaMemPoolAttrReservedMemCurrent, rt.cudaMemPoolAttr.cudaMemPoolAttrUsedMemCurrent,
              rt.cudaMemPoolAttr.cudaMemPoolAttrUsedMemHigh):
        err, v = rt.cudaMemPoolGetAttribute(pool, a)
        out.append(round(int(v) / 1e9, 2))
    return out


def main():
    import torch
    case = G.case(sys.argv[1] if len(sys.argv) > 1 else "C5")
    s = case.scene
    dev = torch.device("cuda", 0)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    pts, nrm, rad, lab = t(s.points), t(s.normals), t(s.radii), t(s.labels)
    tx, rx = t(case.tx), t(case.rx.reshape(-1, 3))
    st = torch.cuda.current_stream()
    flush = torch.empty((512 << 20) // 4, dtype=torch.float32, device="cuda")
    for k in range(10):
        flush.fill_(float(k))
        torch.cuda.synchronize()
        T = [time.perf_counter()]
        sc = N.nrt_scene_build_ex(pts, nrm, case.voxel, radii=rad, labels=lab, edges=s.edges, stream=st)
        T.append(time.perf_counter())
        p = N.nrt_launch_ex(sc, tx, rx, case.n_rays, case.max_refl, case.max_diff, kappa=case.kappa,
                            tau=case.tau, c_R=case.c_R, dphi_deg=case.dphi_deg,
                            theta_ex_deg=case.theta_ex_deg, edge_bin=case.edge_bin, stream=st)
        T.append(time.perf_counter())
        r = N.nrt_refine_ex(sc, p, xi=case.xi, r_s=case.r_s, tau=case.tau, stream=st)
        T.append(time.perf_counter())
        torch.cuda.synchronize()
        T.append(time.perf_counter())
        r.free(); p.free(); sc.free()
        torch.cuda.synchronize()
        T.append(time.perf_counter())
        print(k, [round(1e3 * (T[i + 1] - T[i]), 1) for i in range(len(T) - 1)], pool_stats(), flush=True)


if __name__ == "__main__":
    main()
