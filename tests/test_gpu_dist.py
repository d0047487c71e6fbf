"""The multi-GPU protocol (paper_2403_06648_b200/dist.py) executed by several
processes: scene replicated, rays i == rank (mod world), stage-1 events all-gathered before the
fans, coarse records all-gathered and merged, refinement sharded by path and merged.  The ranks
share cuda:0 and exchange through gloo (host-staged), so no kernel of one rank waits on another;
the global coarse and refined sets must equal the world-1 sets byte for byte (R30)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    import nrt_gen as G
    return G.case("C2s", sigma=0.005, n=12_000, n_rays=8000, max_refl=2, max_diff=1)


def _run(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    import paper_2403_06648_b200 as N
    from paper_2403_06648_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    case = _case()
    sc = N.build_case_scene(case)
    desc = dict(kappa=case.kappa, tau=case.tau, c_R=case.c_R, dphi_deg=case.dphi_deg,
                theta_ex_deg=case.theta_ex_deg, edge_bin=case.edge_bin)
    dev = torch.device("cuda", 0)
    coarse, info = D.launch_distributed(N, sc, case.tx, case.rx, case.n_rays, case.max_refl,
                                        case.max_diff, rank, world, has_edges=True, device=dev,
                                        **desc)
    ref, _ = D.refine_distributed(N, sc, coarse, case.tx, case.rx, rank, world, device=dev,
                                  xi=case.xi, r_s=case.r_s, tau=case.tau,
                                  theta_ex_deg=case.theta_ex_deg)
    np.save(os.path.join(outdir, f"coarse_{world}_{rank}.npy"), coarse.export())
    np.save(os.path.join(outdir, f"refined_{world}_{rank}.npy"), ref.export())
    np.save(os.path.join(outdir, f"bounces_{world}_{rank}.npy"), np.array([info["bounces"]]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_multiprocess_protocol_equals_single(world, tmp_path):
    import torch.multiprocessing as mp
    import paper_2403_06648_b200 as N
    case = _case()
    sc = N.build_case_scene(case)
    full = N.launch_case(sc, case)
    full_c = full.export()
    full_r = N.nrt_refine_ex(sc, full, xi=case.xi, r_s=case.r_s, tau=case.tau,
                             theta_ex_deg=case.theta_ex_deg).export()
    bounces = full.info()["bounces"]
    assert (full_c["n_diff"] == 1).sum() > 0 and len(full_r) > 10
    mp.start_processes(_run, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    tot = 0
    for r in range(world):
        c = np.load(tmp_path / f"coarse_{world}_{r}.npy")
        f = np.load(tmp_path / f"refined_{world}_{r}.npy")
        assert c.tobytes() == full_c.tobytes(), (world, r)
        assert f.tobytes() == full_r.tobytes(), (world, r)
        tot += int(np.load(tmp_path / f"bounces_{world}_{r}.npy")[0])
    assert tot == bounces


def _env_case():
    import nrt_gen as G
    case = G.case("C1", n_rays=1000)
    case.scene = G.box_room(2)
    case.sdf = dict(cell=0.0625, r_s=0.015, t_sdf=0.0015, xi=2.0)
    case.kappa = 100
    return case


def _run_env(rank, world, port, outdir):
    """NEXT-2 over processes: transmission rays sharded i == rank (mod world), records
    all-gathered and merged (kappa = 100) on every rank."""
    import torch
    import torch.distributed as dist
    import paper_2403_06648_b200 as N
    from paper_2403_06648_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    case = _env_case()
    sc = N.build_case_scene(case)
    desc = N.case_desc(case)
    desc["tracer"] = 1
    coarse, info = D.launch_distributed(N, sc, case.tx, case.rx, case.n_rays, case.max_refl,
                                        case.max_diff, rank, world, has_edges=False,
                                        device=torch.device("cuda", 0), **desc)
    np.save(os.path.join(outdir, f"env_{world}_{rank}.npy"), coarse.export())
    np.save(os.path.join(outdir, f"envb_{world}_{rank}.npy"), np.array([info["bounces"]]))
    dist.destroy_process_group()


def test_multiprocess_cone_tracer_equals_single(tmp_path):
    import torch.multiprocessing as mp
    import paper_2403_06648_b200 as N
    case = _env_case()
    sc = N.build_case_scene(case)
    full = N.launch_case(sc, case, tracer=1)
    world = 2
    mp.start_processes(_run_env, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    tot = 0
    for r in range(world):
        c = np.load(tmp_path / f"env_{world}_{r}.npy")
        assert c.tobytes() == full.export().tobytes(), r
        tot += int(np.load(tmp_path / f"envb_{world}_{r}.npy")[0])
    assert tot == full.info()["bounces"]
