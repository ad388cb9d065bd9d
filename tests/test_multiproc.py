"""World-size-2 gloo tests (CPU) of the multi-GPU host logic in bench.py: SNP sharding, the single state
broadcast that replicates the setup, max-over-ranks timing, the per-rank parity cut + gather (rank 1's shard
included), and the launcher's refusal to label a run with the wrong GPU count."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import datagen


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _parity_worker(rank, world, port, q):
    """Every rank produces 'results' for its own shard (here by the oracle on CPU, standing in for the GPU run),
    cuts the parity subsample's SNPs of its shard, all_gather_object's them, and rank 0 merges and checks every
    rank's part -- bench.py's parity path with rank 1's shard included."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        cfg = datagen.custom_config(n=40, p=3, m=301, t=3, index=55, block_cols=64)
        ds = datagen.dataset(cfg)
        lo, hi = bench.shard_range(cfg.m, rank, world, "strong")
        snps, traits = bench.parity_subsample(cfg, cfg.m, world, "strong", 64, 60)
        glob, loc = bench.local_pairs(snps, lo, hi)
        G = datagen.xr_columns(cfg, np.arange(lo, hi))
        mine = oracle.gls_sequence(ds.Phi, ds.XL, G, ds.Y, ds.h2, ds.s2)
        b, v, s = mine["b"][..., -1], mine["Var"][..., -1, -1], mine["status"]
        cut = tuple(x[np.ix_(loc, traits)] for x in (b, v, s))
        parts = [None] * world
        dist.all_gather_object(parts, {"snps": glob, "res": {"fp64": cut}, "info": {"rank": rank}})
        if rank == 0:
            merged = bench.merge_gathered(parts, snps)["fp64"]
            ref = oracle.gls_sequence(ds.Phi, ds.XL, datagen.xr_columns(cfg, snps), ds.Y, ds.h2, ds.s2, traits=traits)
            ok = np.array_equal(merged[0], ref["b"][..., -1]) and np.array_equal(merged[2], ref["status"])
            shard1 = [int(x) for x in parts[1]["snps"]]
            q.put((ok, len(shard1), min(shard1) >= bench.shard_range(cfg.m, 1, world)[0], snps.size))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_parity_gather_checks_every_shard():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_parity_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    ok, n1, in_shard1, ns = q.get()
    assert ok            # rank 0's merged view of all shards equals the oracle on the whole subsample, bitwise
    assert n1 > 0 and in_shard1


def test_parity_edges_cover_shard_and_block_edges():
    m, world, k = 1_000_000, 8, 15104
    edges = bench.parity_edges(m, world, "strong", k)
    for r in range(world):
        lo, hi = bench.shard_range(m, r, world, "strong")
        assert lo in edges and hi - 1 in edges and lo + k - 1 in edges and lo + k in edges
        last = lo + (hi - lo - 1) // k * k
        assert last in edges
    cfg = datagen.CONFIGS[4]
    snps, traits = bench.parity_subsample(cfg, m, world, "strong", k, 10_000)
    assert set(edges) <= set(snps.tolist())
    assert snps.size * traits.size >= 10_000 * world
    # every rank gets at least 10^4 / T_s-ish SNPs of its own
    for r in range(world):
        lo, hi = bench.shard_range(m, r, world, "strong")
        g, l_ = bench.local_pairs(snps, lo, hi)
        assert np.array_equal(g - lo, l_) and g.size * traits.size >= 5_000


def test_bench_refuses_mislabelled_runs():
    """--gpus N without N GPUs fails loudly (exit 2), and a torchrun world that differs from --gpus is refused."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--config", "0"], cwd=root, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "needs 2 GPUs" in r.stderr
    env.update(WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "4", "--config", "0"], cwd=root, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr


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


def test_parity_edges_weak_scaling():
    """Weak scaling (opt-in): rank r owns [r m, (r+1) m) of an N m genome; its edges and block edges are forced."""
    m, world, k = 50_000, 4, 8192
    edges = bench.parity_edges(m, world, "weak", k)
    for r in range(world):
        lo, hi = bench.shard_range(m, r, world, "weak")
        assert (lo, hi) == (r * m, (r + 1) * m)
        assert lo in edges and hi - 1 in edges and lo + k in edges
    cfg = datagen.custom_config(n=32, p=2, m=m * world, t=3, index=77)
    snps, traits = bench.parity_subsample(cfg, m, world, "weak", k, 1_000)
    assert snps.max() < m * world and set(edges) <= set(snps.tolist())
