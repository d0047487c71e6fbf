#!/usr/bin/env python
"""bench.py — one JSON line for the driver (see DESIGN.md §7 "Measurement").

Workload (default): BASELINE.json configs[4], "C5" — the reconstructed-room cloud (1e7 surfels,
fitted normals, 879 RX), a FIXED lattice of 1e8 Fibonacci rays from one TX, <= 4 reflections,
sharded i == rank (mod N) over the N GPUs (strong scaling: every N traces the same global set).
One step = one pass of the whole hot path over that workload:
  A1 scene build -> A2-A8 launch (primary rays, events/fans when the config has edges, dedupe,
  NCCL all-gather + global merge for N > 1) -> A9-A10 refinement (sharded by path, refined
  records all-gathered and merged).
`value` = ray-bounces per second of the whole job (device time, inputs resident in HBM, max over
ranks).  `--config C2` gives the secondary line (1e6 surfels, 1e6 rays, diffraction).
`--impl reference` times the CPU oracle (oracle/) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ray-bounces/sec and refined paths/sec at 1/2/4/8 B200; % of HBM roofline"
UNIT = "ray-bounces/s"
L2_FLUSH_BYTES = 512 << 20
# FP64 operations per neighbourhood term (k_refine rows): a value pass (Eqs. 2-4:
# difference 3, squared distance 5, weight 1 + exp 22, sums W/P/N 13) and a derivative pass of
# the analytic Jacobian (the same 31 + W, sum w d, sum w d d^T, sum w n, sum w n d^T = 43)
FLOPS_VALUE, FLOPS_DERIV = 44, 74
# NEXT-1 (--intersect sdf): FP32 operations per Gaussian term of the SDF evaluation (DESIGN.md
# §6.4: difference 3, |p-x|^2 5, weight 1, exp 21, products 7, tree sums 7)
FLOPS_SDF_TERM = 44
SDF = dict(cell=0.0625, r_s=0.015, t_sdf=0.0015, xi=2.0)  # Table I / P:131 (DESIGN R40-R45)
# FP32 peak (no measured figure in MEASURED_PEAKS.json): 148 SMs x 128 FP32 lanes x 2 flops
# (FFMA) x 1.965 GHz (B200_PROFILING.md: SM count and clocks.max.sm)
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12


def peaks():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(mp["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.p = None
        self.path = os.path.join("/tmp", f"nrt_clocks_{os.getpid()}.csv")

    def __enter__(self):
        if os.environ.get("NRT_BENCH_NO_CLOCKS"):
            return self
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", os.environ.get("NRT_CLOCKS_MS", "200")],
                stdout=self.f,
                stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        # keep nvidia-smi's start-up (NVML init) out of the timed region: start timing after its
        # first sample (interval: the profiling recipe's 200 ms; NRT_CLOCKS_MS overrides)
        t0 = time.time()
        while self.p is not None and time.time() - t0 < 10.0:
            self.f.flush()
            if os.path.getsize(self.path) > 0:
                time.sleep(0.3)
                break
            time.sleep(0.05)
        return self

    def __exit__(self, *a):
        if self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()
            self.f.close()

    def summary(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------------------
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def max_over_ranks(world, *vals):
    """Element-wise max of host floats over the ranks (NCCL all-reduce)."""
    if world == 1:
        return list(vals)
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(vals), dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def sum_over_ranks(world, *vals):
    if world == 1:
        return list(vals)
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(vals), dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(x) for x in t.tolist()]


class Runner:
    """One hot-path step on this rank, inputs resident in device memory.  Strong scaling: the
    lattice has case.n_rays directions for every N, rank r traces i == r (mod N); weak: the
    lattice grows to n_rays x N."""

    def __init__(self, N, case, world, rank, stream, scaling):
        import torch
        self.N, self.case, self.world, self.rank, self.stream = N, case, world, rank, stream
        s = case.scene
        dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        self.pts, self.nrm, self.rad, self.lab = t(s.points), t(s.normals), t(s.radii), t(s.labels)
        self.tx = t(case.tx)
        self.rx = t(case.rx.reshape(-1, 3))
        self.n_rays = case.n_rays * (world if scaling == "weak" else 1)
        self.desc = N.case_desc(case)  # with case.sdf: intersect = 1 and the SDF parameters
        if getattr(case, "tracer", 0):
            self.desc["tracer"] = 1
        self.sdf_cell = (float(case.sdf["cell"]) if getattr(case, "sdf", None)
                         else SDF["cell"] if getattr(case, "gd", None) is not None else 0.0)
        self.rdesc = dict(xi=case.xi, r_s=case.r_s, tau=case.tau, theta_ex_deg=case.theta_ex_deg)
        if getattr(case, "gd", None) is not None:  # NEXT-4: the paper's GD refinement
            self.rdesc = N.gd_desc(case)

    def step(self, counters=0):
        from paper_2403_06648_b200 import dist as D
        N, c = self.N, self.case
        import torch
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(self.stream)
        sc = N.nrt_scene_build_ex(self.pts, self.nrm, c.voxel, radii=self.rad, labels=self.lab,
                                  edges=c.scene.edges, stream=self.stream, sdf_cell=self.sdf_cell)
        ev[1].record(self.stream)
        if self.world == 1:
            coarse = N.nrt_launch_ex(sc, self.tx, self.rx, self.n_rays, c.max_refl, c.max_diff,
                                     counters=counters, stream=self.stream, **self.desc)
            info = coarse.info()
        else:
            coarse, info = D.launch_distributed(
                N, sc, c.tx, c.rx, self.n_rays, c.max_refl, c.max_diff, self.rank, self.world,
                has_edges=len(c.scene.edges) > 0, device=self.dev, stream=self.stream,
                counters=counters, **self.desc)
        ev[2].record(self.stream)
        refined, rinfo = D.refine_distributed(N, sc, coarse, c.tx, c.rx, self.rank, self.world,
                                              device=self.dev, stream=self.stream,
                                              counters=counters, **self.rdesc)
        ev[3].record(self.stream)
        ev[3].synchronize()
        out = {
            "phase_ms": [round(ev[i].elapsed_time(ev[i + 1]), 3) for i in range(3)],
            "bounces": info["bounces"],
            "coarse": coarse.count(),
            "refined": refined.count(),
            "ms_trace": info["ms_trace"],
            "ms_fans": info["ms_fans"],
            "ms_refine": rinfo["ms_refine"],
            "refine_paths": rinfo["n_raw"],
            "mls_value": rinfo["mls_value"],
            "mls_deriv": rinfo["mls_deriv"],
            "n_events": info["n_events"],
            "n_fan_rays": info["n_fan_rays"],
        }
        for h in (refined, coarse, sc):
            h.free()
        return out


def e2e_step(N, case, host, n_rays, world, rank, stream):
    """The public API with HOST buffers (pinned): H2D of the cloud inside the build, the
    distributed launch + refinement, D2H of the global refined set."""
    from paper_2403_06648_b200 import dist as D
    import torch
    sdf_cell = (float(case.sdf["cell"]) if getattr(case, "sdf", None)
                else SDF["cell"] if getattr(case, "gd", None) is not None else 0.0)
    sc = N.nrt_scene_build_ex(host["p"], host["n"], case.voxel, radii=host["r"],
                              labels=host["l"], edges=case.scene.edges, stream=stream,
                              sdf_cell=sdf_cell)
    desc = N.case_desc(case)
    if getattr(case, "tracer", 0):
        desc["tracer"] = 1
    if world == 1:
        coarse = N.nrt_launch_ex(sc, case.tx, case.rx, n_rays, case.max_refl, case.max_diff,
                                 stream=stream, **desc)
    else:
        coarse, _ = D.launch_distributed(N, sc, case.tx, case.rx, n_rays, case.max_refl,
                                         case.max_diff, rank, world,
                                         has_edges=len(case.scene.edges) > 0,
                                         device=torch.device("cuda", torch.cuda.current_device()),
                                         stream=stream, **desc)
    b = coarse.info()["bounces"]
    rdesc = (N.gd_desc(case) if getattr(case, "gd", None) is not None else
             dict(xi=case.xi, r_s=case.r_s, tau=case.tau, theta_ex_deg=case.theta_ex_deg))
    ref, _ = D.refine_distributed(N, sc, coarse, case.tx, case.rx, rank, world,
                                  device=torch.device("cuda", torch.cuda.current_device()),
                                  stream=stream, **rdesc)
    out = ref.export()  # D2H of the result
    for h in (ref, coarse, sc):
        h.free()
    return b, out.nbytes


# ------------------------------------------------------------------------------------------
def oracle_voxel(case):
    """The oracle's own tier-1 grid cell (independent of the GPU's voxel)."""
    return 0.03 if case.name in ("C4", "C5") else 0.05


def oracle_scene(case):
    """The oracle's scene: tier-1 grid (disk hit), or the tier-1 SDF tracer (case.sdf)."""
    from oracle import oracle as O
    if getattr(case, "sdf", None):
        return O.OracleScene(case.scene, sdf_cell=case.sdf["cell"], sdf_grid=0.125)
    return O.OracleScene(case.scene, grid_voxel=oracle_voxel(case))


def oracle_kind(case):
    return ("tier-1 SDF oracle (oracle/sdf.c, own 12.5 cm grid over the AABBs)" if getattr(case, "sdf", None)
            else "tier-1 grid oracle")


def _oracle_chunk(ids):
    """One forked worker's rays; the case and the oracle scene come from the fork (pickling the
    1e7-surfel case per task cost seconds per step)."""
    from oracle import oracle as O
    _, _, nb = O.trace_rays(O._FORK["case"], ids, scene=O._FORK.get("scene"))
    return nb


def cpu_baseline(case, seconds=15.0):
    """The oracle as it stands (tier-1 grid, oracle/grid.c) on this host's cores: forked
    processes over an evenly spaced sample of the lattice's primary rays."""
    import multiprocessing as mp
    from oracle import oracle as O
    O.lib()
    P = os.cpu_count() or 1
    O._FORK["scene"] = oracle_scene(case)
    O._FORK["case"] = case
    ids = np.arange(0, case.n_rays, max(1, case.n_rays // 997), dtype=np.uint64)
    t0 = time.perf_counter()
    nb0 = _oracle_chunk(ids[:64])
    per_bounce = max(1e-9, (time.perf_counter() - t0) / max(1, nb0))
    n_rays = max(P, int(seconds * P / (per_bounce * (case.max_refl + 1))))
    sample = np.linspace(0, case.n_rays - 1, n_rays).astype(np.uint64)
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(P) as pool:
        res = pool.map(_oracle_chunk, [sample[k::P] for k in range(P)])
    wall = time.perf_counter() - t0
    bounces = sum(res)
    one = sample[: max(1, len(sample) // (4 * P))]
    t1 = time.perf_counter()
    nb1 = _oracle_chunk(one)
    one_core = nb1 / max(1e-9, time.perf_counter() - t1)
    O._FORK.pop("scene", None)
    return {"value": bounces / wall, "unit": UNIT, "cores": P, "kind": "oracle",
            "value_1core": one_core,
            "sample": f"{len(sample)} primary rays of {case.name}'s lattice (evenly spaced ids; "
                      f"{oracle_kind(case)} over {case.scene.n} surfels, {len(case.rx)} RX; "
                      f"coarse tracing only), {wall:.1f} s wall on {P} processes"}


def _env_chunk(args):
    part, parts = args
    from oracle import oracle as O
    return O._env_worker((O._FORK["case"], part, parts))[1]


def cpu_baseline_env(case, parts=128):
    """NEXT-2: the oracle (env.c, tier-1 SDF validation) on this host's cores over the first P of
    `parts` transmission shards (IE i == k mod parts): validation rays per second."""
    import multiprocessing as mp
    from oracle import oracle as O
    O.env_lib()
    P = os.cpu_count() or 1
    O._FORK["env"] = O.EnvScene(case, sdf_grid=0.125)
    O._FORK["case"] = case
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(P) as pool:
        res = pool.map(_env_chunk, [(k, parts) for k in range(min(P, parts))])
    wall = time.perf_counter() - t0
    O._FORK.pop("env", None)
    return {"value": sum(res) / wall, "unit": UNIT, "cores": P, "kind": "oracle",
            "sample": f"transmission shards 0..{min(P, parts) - 1} of {parts} of {case.name} (NEXT-2 "
                      f"oracle, tier-1 SDF validation rays and their cone-traced subtrees), {wall:.1f} s "
                      f"wall on {P} processes"}


def run_config(case, world, scaling):
    n_total = case.n_rays * (world if scaling == "weak" else 1)
    hit = (" SDF intersection (NEXT-1: AABB edge %g m, r_s %g, t_sdf %g, xi %g);"
           % (case.sdf["cell"], case.sdf["r_s"], case.sdf["t_sdf"], case.sdf["xi"])
           if getattr(case, "sdf", None) else "")
    if getattr(case, "tracer", 0):
        hit += (" the paper's environment-driven launch + voxel cone tracing (NEXT-2; value = "
                "SDF validation rays/s, kappa %d);" % case.kappa)
    if getattr(case, "gd", None) is not None:
        hit += " the paper's GD refinement (NEXT-4: %s);" % ", ".join(
            "%s %s" % kv for kv in sorted(__import__("paper_2403_06648_b200").gd_desc(case).items())
            if kv[0] not in ("tau", "theta_ex_deg", "method"))
    return {"workload": f"{case.name}: {case.scene.name},{hit} 1 TX/{len(case.rx)} RX, "
                        f"{n_total} rays in total ({scaling} scaling over {world} GPU(s)), "
                        f"max_refl {case.max_refl}, max_diff {case.max_diff}; "
                        f"step = scene build + launch + refine",
            "voxel_m": case.voxel, "n_rays_total": n_total,
            "l2": "512 MiB write between steps (outside the timed events)",
            "parallelism": f"dp{world}: rays i == rank mod {world}, paths j == rank mod "
                           f"{world}, NCCL all-gather of events/coarse/refined records"}


def run_reference(args, case):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    O.lib()
    import multiprocessing as mp
    P = os.cpu_count() or 1
    O._FORK["scene"] = oracle_scene(case)
    O._FORK["case"] = case
    rays_per_step = (512 if getattr(case, "sdf", None) else 4096) * P
    times, bounces = [], []
    ctx = mp.get_context("fork")
    with ctx.Pool(P) as pool:
        for k in range(args.warmup + args.steps):
            sample = (np.arange(rays_per_step, dtype=np.uint64) * (case.n_rays // rays_per_step)
                      + k).astype(np.uint64)
            t0 = time.perf_counter()
            res = pool.map(_oracle_chunk, [sample[j::P] for j in range(P)])
            dt = time.perf_counter() - t0
            if k >= args.warmup:
                times.append(dt)
                bounces.append(sum(res))
    value = sum(bounces) / sum(times)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000 * statistics.mean(times),
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "impl": "reference",
            "config": dict(run_config(case, world, args.scaling),
                           sample=f"oracle: {rays_per_step} primary rays of the lattice per step"),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": P, "kind": "oracle",
                             "sample": f"{rays_per_step} primary rays per step of {case.name} "
                                       f"({oracle_kind(case)} over {case.scene.n} surfels, "
                                       f"coarse tracing only)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="nrt", choices=["nrt", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--sigma", type=float, default=0.010)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--intersect", default="disk", choices=["disk", "sdf"],
                    help="sdf: NEXT-1, the paper's point-set SDF intersection (secondary lines)")
    ap.add_argument("--tracer", default="fib", choices=["fib", "env"],
                    help="env: NEXT-2, the paper's environment-driven launch + voxel cone tracing "
                         "(implies --intersect sdf, kappa 100; secondary lines)")
    ap.add_argument("--refine", default="gn", choices=["gn", "gd"],
                    help="gd: NEXT-4, the paper's gradient-descent refinement (needs the AABB "
                         "primitives: implies sdf_cell; secondary lines)")
    args = ap.parse_args()

    import nrt_gen as G
    case = G.case(args.config, sigma=args.sigma) if args.config.startswith("C2") else G.case(args.config)
    if args.tracer == "env":
        args.intersect = "sdf"
        case.kappa = 100  # Table I
        case.tracer = 1
    if args.intersect == "sdf":
        case.sdf = dict(SDF)
    if args.refine == "gd":
        case.gd = {"t_a_deg": 25.0} if args.config in ("C3", "C4", "C5") else {}  # Table III
    if args.impl == "reference":
        run_reference(args, case)
        return

    import torch
    import paper_2403_06648_b200 as N
    N.lib()
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    R = Runner(N, case, world, rank, stream, args.scaling)

    # the L2-flush buffer exists before the warm-up, so that the memory pools are in their
    # steady state when the timed steps start
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    for k in range(args.warmup):
        flush.fill_(float(k))
        R.step()
    torch.cuda.synchronize()
    cnt = R.step(counters=1)  # instrumented (untimed): algorithmic byte and FLOP counts
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    outs = []
    launches0 = N.nrt_kernel_launches()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for k in range(args.steps):
            flush.fill_(float(k))          # L2 flush between steps (outside the event pair)
            ev[k][0].record(stream)
            outs.append(R.step())
            ev[k][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    launches = (N.nrt_kernel_launches() - launches0) / args.steps
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = max_over_ranks(world, sum(step_ms))[0]
    bounces = int(sum_over_ranks(world, float(outs[-1]["bounces"]))[0])
    value = bounces * args.steps / (total_ms / 1000.0)
    ms_trace = statistics.mean(o["ms_trace"] for o in outs)
    ms_fans = statistics.mean(o["ms_fans"] for o in outs)
    ms_refine = statistics.mean(o["ms_refine"] for o in outs)

    # ---- rooflines: the traversal (HBM, BJ's "% of HBM roofline") and the refinement (FP64)
    hbm, src = peaks()
    prim_only = prim_counts(N, R, case)
    if R.sdf_cell > 0:
        # NEXT-1: the SDF trace is FP32-ALU bound (Gaussian terms of Eqs. 1-4)
        fl = FLOPS_SDF_TERM * prim_only["tests"]
        achieved = fl / (ms_trace / 1000.0) / 1e12
        roof_trace = {"bound": "alu", "achieved": achieved, "peak": FP32_PEAK_TFLOPS,
                      "unit": "TFLOP/s", "frac": achieved / FP32_PEAK_TFLOPS,
                      "traffic": measured_traffic(case.name + ("_env" if getattr(case, "tracer", 0) else "_sdf")),
                      "kernel": ("k_env_tx + k_env_prop (cone tracing; SDF validation rays, one warp per "
                                 "ray)" if getattr(case, "tracer", 0) else
                                 "k_trace_sdf (primary bounces; one warp per segment)"),
                      "peak_source": "derived: 148 SM x 128 FP32 lanes x 2 x 1.965 GHz",
                      "flops_per_launch": fl, "gaussian_terms": prim_only["tests"],
                      "terms_per_bounce": prim_only["tests"] / max(1, prim_only["bounces"]),
                      "marches_per_bounce": prim_only["nonempty"] / max(1, prim_only["bounces"]),
                      "ms_per_launch": ms_trace}
    else:
        pb = 32 * prim_only["tests"] + 8 * prim_only["cells"]
        achieved = pb / (ms_trace / 1000.0) / 1e9
        roof_trace = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                      "frac": achieved / hbm, "traffic": measured_traffic(case.name),
                      "kernel": "k_trace (primary bounces)", "peak_source": src,
                      "bytes_per_launch": pb, "bytes_per_bounce": pb / max(1, prim_only["bounces"]),
                      "ms_per_launch": ms_trace}
    fp64 = N.nrt_probe_fp64_tflops(local)
    flops = FLOPS_VALUE * cnt["mls_value"] + FLOPS_DERIV * cnt["mls_deriv"]
    gd = getattr(case, "gd", None) is not None
    ach_f = flops / (ms_refine / 1000.0) / 1e12 if ms_refine else 0.0
    roof_refine = {"bound": "alu", "achieved": ach_f, "peak": fp64, "unit": "TFLOP/s",
                   "frac": ach_f / fp64 if fp64 > 0 else None,
                   "traffic": measured_traffic(case.name + "_refine"),
                   "kernel": "k_refine_w (FP64 Gauss-Newton, one warp per path)",
                   "peak_source": "measured FP64 FMA probe (nrt_probe_fp64_tflops); nominal "
                                  "148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz = 37.2 TFLOP/s",
                   "flops_per_launch": flops, "ms_per_launch": ms_refine,
                   "mls_terms": [cnt["mls_value"], cnt["mls_deriv"]]}
    if gd:
        # NEXT-4: FP32 ALU, Gaussian terms of its SDF evaluations (counted on device)
        fl = FLOPS_SDF_TERM * cnt["mls_value"]
        ach = fl / (ms_refine / 1000.0) / 1e12 if ms_refine else 0.0
        roof_refine = {"bound": "alu", "achieved": ach, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
                       "frac": ach / FP32_PEAK_TFLOPS, "traffic": measured_traffic(case.name + "_gd"),
                       "kernel": "k_refine_gd (the paper's GD, one warp per path)",
                       "peak_source": "derived: 148 SM x 128 FP32 lanes x 2 x 1.965 GHz",
                       "flops_per_launch": fl, "gaussian_terms": cnt["mls_value"],
                       "ms_per_launch": ms_refine}
    dominant_refine = ms_refine > ms_trace + ms_fans
    roof = roof_refine if dominant_refine else roof_trace
    post = post_timing(N, R, case) if world == 1 else None

    # ---- e2e through the public API with host (pinned) buffers, every rank
    e2e = None
    if not args.no_e2e:
        s = case.scene
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        host = {"p": pin(s.points), "n": pin(s.normals), "r": pin(s.radii), "l": pin(s.labels)}
        h2d = sum(v.nbytes for v in host.values()) + case.rx.nbytes + case.tx.nbytes
        e2e_step(N, case, host, R.n_rays, world, rank, stream)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        tot_b, d2h = 0, 0
        for _ in range(args.steps):
            b, ob = e2e_step(N, case, host, R.n_rays, world, rank, stream)
            tot_b += b
            d2h = ob
        torch.cuda.synchronize()
        dt = max_over_ranks(world, time.perf_counter() - t0)[0]
        tot_b = int(sum_over_ranks(world, float(tot_b))[0])
        e2e = {"value": tot_b / dt, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": 1000 * dt / args.steps}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": run_config(case, world, args.scaling),
        # refined paths/s: coarse paths refined (the refinement's input rate, as the paper's
        # Table IV refine times count) per second of the whole step, and of the refine kernel
        "refined_paths_per_s": outs[-1]["coarse"] * args.steps / (total_ms / 1000.0),
        "refine_kernel_paths_per_s": (outs[-1]["refine_paths"] / (ms_refine / 1000.0))
        if ms_refine else None,
        "coarse_paths": outs[-1]["coarse"], "refined_valid_paths": outs[-1]["refined"],
        "breakdown_ms": {"trace": ms_trace, "fans": ms_fans, "refine": ms_refine,
                         "step": total_ms / args.steps},
        "n_events": outs[-1]["n_events"], "n_fan_rays": outs[-1]["n_fan_rays"],
        "bounces_per_step": bounces,
        "step_ms": [round(x, 3) for x in step_ms],
        "phase_ms_build_launch_refine": [o["phase_ms"] for o in outs],
        "roofline": roof,
        "roofline_trace": roof_trace,
        "roofline_refine": roof_refine,
        # NEXT-3 post-processing (not a §8(a) row: timed separately, outside the step)
        "postprocess": post,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_env(case) if getattr(case, "tracer", 0) else cpu_baseline(case)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def post_timing(N, R, case, reps=3):
    """Device time of nrt_postprocess on this workload's refined set (median of reps)."""
    import torch
    sc = N.nrt_scene_build_ex(R.pts, R.nrm, case.voxel, radii=R.rad, labels=R.lab,
                              edges=case.scene.edges, stream=R.stream, sdf_cell=R.sdf_cell)
    coarse = N.nrt_launch_ex(sc, R.tx, R.rx, R.n_rays, case.max_refl, case.max_diff,
                             stream=R.stream, **R.desc)
    ref = N.nrt_refine_ex(sc, coarse, stream=R.stream, **R.rdesc)
    ms, n_out = [], 0
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(R.stream)
        p = N.nrt_postprocess(sc, ref, r_s=case.r_s, stream=R.stream)
        b.record(R.stream)
        b.synchronize()
        ms.append(a.elapsed_time(b))
        n_out = p.count()
        p.free()
    return {"ms": statistics.median(ms), "paths_in": ref.count(), "paths_out": n_out}


def measured_traffic(key):
    """DRAM bytes (read + write) per launch from the committed ncu launch list
    (profiles/r02_traffic.json, else r01): key = config name for the traversal kernel,
    config + "_refine" for the refinement kernel; None if not captured."""
    for name in ("r02_traffic.json", "r01_traffic.json"):
        try:
            t = json.load(open(os.path.join(ROOT, "profiles", name)))
            return float(t[key]["dram_bytes_per_launch"])
        except Exception:
            continue
    return None


def prim_counts(N, R, case):
    """Instrumented primary-only launch (stage 1: no fans) for the k_trace byte count."""
    sc = N.nrt_scene_build_ex(R.pts, R.nrm, case.voxel, radii=R.rad, labels=R.lab,
                              edges=case.scene.edges, stream=R.stream, sdf_cell=R.sdf_cell)
    p = N.nrt_launch_ex(sc, R.tx, R.rx, R.n_rays, case.max_refl, case.max_diff, counters=1,
                        stage=1, rank=R.rank, world=R.world, stream=R.stream, **R.desc)
    i = p.info()
    p.free()
    sc.free()
    return {"tests": i["surfel_tests"], "cells": i["cells_visited"], "bounces": i["bounces"],
            "nonempty": i["cells_nonempty"]}


if __name__ == "__main__":
    main()
