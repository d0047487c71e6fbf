"""Multi-GPU data parallelism over torch.distributed (NCCL on B200 / NVLink 5; gloo on CPU for
the plumbing tests).  SURVEY.md §8(e):

  * the scene is replicated: every rank builds it from the same input (deterministic);
  * primary rays are sharded by lattice index, i == rank (mod world);
  * diffraction events of every rank are all-gathered before the fans (R14 global event
    dedupe, so the result does not depend on world), fans are sharded by event rank;
  * coarse records are all-gathered and merged (R17) on every rank -> identical global set;
  * refinement is sharded by path, refined records all-gathered and merged (R28).

Only the raw fixed-size records cross the wire (nrt_paths_export / nrt_paths_import are the
ABI's byte interface); every merge runs in libnrt's kernels.
"""
from __future__ import annotations

import numpy as np


def shard_count(n: int, rank: int, world: int) -> int:
    """Number of items i in [0, n) with i == rank (mod world)."""
    return max(0, (n - rank + world - 1) // world) if n > rank else 0


def allgather_bytes(t, group=None):
    """All-gather variable-length 1-D uint8 tensors: exchange the lengths, then one padded
    all_gather_into_tensor (a single NCCL collective), concatenated in rank order.  With the
    gloo backend (CPU plumbing tests, several ranks on one GPU) device tensors are staged
    through the host and the result returned on the input's device."""
    import torch
    import torch.distributed as dist
    if t.device.type == "cuda" and dist.get_backend(group) == "gloo":
        return allgather_bytes(t.cpu(), group).to(t.device)
    world = dist.get_world_size(group)
    n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    ns = [int(x.item()) for x in ns]
    m = max(ns) if ns else 0
    if m == 0:
        return torch.zeros(0, dtype=torch.uint8, device=t.device)
    pad = torch.zeros(m, dtype=torch.uint8, device=t.device)
    pad[: t.numel()] = t
    if hasattr(dist, "all_gather_into_tensor") and t.device.type == "cuda":
        out = torch.zeros(world * m, dtype=torch.uint8, device=t.device)
        dist.all_gather_into_tensor(out, pad, group=group)
        parts = [out[r * m: r * m + ns[r]] for r in range(world)]
    else:
        outs = [torch.zeros(m, dtype=torch.uint8, device=t.device) for _ in range(world)]
        dist.all_gather(outs, pad, group=group)
        parts = [outs[r][: ns[r]] for r in range(world)]
    return torch.cat(parts)


def records_tensor(paths, device):
    """Export a path set's raw records into a uint8 tensor on `device`."""
    import torch
    nb = paths.count() * paths.record_size()
    buf = torch.zeros(nb, dtype=torch.uint8, device=device)
    if nb:
        paths.export(buf)
    return buf


def launch_distributed(N, scene, tx, rx, n_rays, max_refl, max_diff, rank, world, *, has_edges,
                       group=None, device="cuda", stream=None, counters=0, **desc):
    """Coarse launch over `world` ranks -> (global coarse set on every rank, local launch info)."""
    has_diff = max_diff > 0 and has_edges
    local = N.nrt_launch_ex(scene, tx, rx, n_rays, max_refl, max_diff, rank=rank, world=world,
                            stage=1 if has_diff else 0, counters=counters, stream=stream, **desc)
    if has_diff:
        ev = local.export_events(device=device)  # device-to-device copy of the stage-1 events
        evall = allgather_bytes(ev, group)
        N.nrt_launch_fans(scene, local, evall, rank=rank, world=world, stream=stream, **desc)
    info = local.info()
    allr = allgather_bytes(records_tensor(local, device), group)
    merged = N.nrt_paths_import(allr, N.PATHS_COARSE, np.asarray(tx, np.float32).reshape(3),
                                np.asarray(rx, np.float32).reshape(-1, 3))
    merged = N.nrt_paths_merge([merged], desc.get("kappa", 1))
    return merged, info


def refine_distributed(N, scene, coarse, tx, rx, rank, world, *, group=None, device="cuda",
                       stream=None, **desc):
    """Refinement sharded by path (j == rank mod world) -> global refined set on every rank."""
    local = N.nrt_refine_ex(scene, coarse, rank=rank, world=world, stream=stream, **desc)
    info = local.info()
    if world == 1:
        return local, info
    allr = allgather_bytes(records_tensor(local, device), group)
    imp = N.nrt_paths_import(allr, N.PATHS_REFINED, np.asarray(tx, np.float32).reshape(3),
                             np.asarray(rx, np.float32).reshape(-1, 3))
    return N.nrt_paths_merge([imp], 1), info
