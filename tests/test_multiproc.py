"""World-size-2 gloo tests (CPU) of the multi-GPU host logic in bench.py: SNP sharding, the single state
broadcast that replicates the setup, and max-over-ranks timing."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, w, _ = bench.dist_env()
        assert (r, w) == (rank, world)
        # rank 0 "sets up" a state; the others hold garbage until the broadcast
        state = torch.arange(1000, dtype=torch.uint8) if rank == 0 else torch.full((1000,), 7, dtype=torch.uint8)
        bench.replicate_state(state, world)
        ok_state = bool(torch.equal(state, torch.arange(1000, dtype=torch.uint8)))
        mx = bench.max_over_ranks(float(10 + rank), world)
        lo, hi = bench.shard_range(1000, rank, world, "weak")
        slo, shi = bench.shard_range(1001, rank, world, "strong")
        q.put((rank, ok_state, mx, (lo, hi), (slo, shi)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_broadcast_shards_and_max():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(world))
    assert all(r[1] for r in res)                       # every rank holds rank 0's state bytes
    assert all(r[2] == 11.0 for r in res)               # max over ranks
    assert [r[3] for r in res] == [(0, 1000), (1000, 2000)]   # weak: disjoint ranges of an N*m genome
    strong = [r[4] for r in res]
    assert strong[0][0] == 0 and strong[-1][1] == 1001 and strong[0][1] == strong[1][0]


@pytest.mark.parametrize("m,world", [(1_000_000, 8), (100_000, 3), (7, 4), (0, 2)])
def test_shard_ranges_partition(m, world):
    ranges = [bench.shard_range(m, r, world, "strong") for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == m
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    sizes = [h - l for l, h in ranges]
    assert max(sizes) - min(sizes) <= 1
    weak = [bench.shard_range(m, r, world, "weak") for r in range(world)]
    assert all(h - l == m for l, h in weak)


def test_work_model():
    f = bench.flops_per_block(10_000, 5, 1000, 8192)
    assert f["K1"] == 2 * 10_000 ** 2 * 8192
    assert f["K2"] == 2 * 10_000 * 8192 * 1000 * 7
    assert bench.k3_bytes(5, 1000, 8192) == 8192 * 1000 * (8 * 7 + 17)
