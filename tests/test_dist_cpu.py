"""World-size-2 gloo tests of the multi-GPU plumbing (host side; no GPU needed).

The GPU path exchanges raw fixed-size records (events, coarse, refined) with allgather_bytes;
here the same function runs over gloo with variable per-rank lengths, and the ray / event /
path sharding arithmetic is checked against a brute-force enumeration."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_06648_b200.dist import allgather_bytes, shard_count


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rec = np.dtype([("key", "<u8"), ("L", "<f4"), ("id", "<u4")])
        rng = np.random.default_rng(rank)
        n = [5, 0, 17][rank % 3]
        a = np.zeros(n, rec)
        a["key"] = rng.integers(0, 1 << 60, n)
        a["L"] = rng.random(n).astype(np.float32)
        a["id"] = rank * 1000 + np.arange(n)
        out = allgather_bytes(torch.from_numpy(a.view(np.uint8).copy()))
        got = out.numpy().view(rec)
        empty = allgather_bytes(torch.zeros(0, dtype=torch.uint8))
        q.put((rank, got.tobytes(), int(empty.numel())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_allgather_bytes_variable_lengths_gloo(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rec = np.dtype([("key", "<u8"), ("L", "<f4"), ("id", "<u4")])
    expect = []
    for r in range(world):
        rng = np.random.default_rng(r)
        n = [5, 0, 17][r % 3]
        a = np.zeros(n, rec)
        a["key"] = rng.integers(0, 1 << 60, n)
        a["L"] = rng.random(n).astype(np.float32)
        a["id"] = r * 1000 + np.arange(n)
        expect.append(a)
    expect = np.concatenate(expect).tobytes()
    for rank, got, n_empty in res:
        assert got == expect, rank        # every rank holds the identical concatenation
        assert n_empty == 0


@pytest.mark.parametrize("n", [0, 1, 7, 1000, 1_000_003])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_counts_partition_the_lattice(n, world):
    counts = [shard_count(n, r, world) for r in range(world)]
    assert sum(counts) == n
    if n <= 1000:
        for r in range(world):
            assert counts[r] == len(range(r, n, world))
