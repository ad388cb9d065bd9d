"""Shard and pipeline invariance on the GPU.

The paper makes "the number of markers accessed at once ... a user-configurable input parameter":
SNP blocks are independent given the replicated state, so a G-rank run (contiguous SNP shards, bench.py's strong
scaling) must give exactly the 1-rank result.  Shard emulation: shards 0..G-1 are run one after another on one GPU,
each by a context attached to a byte copy of the setup state (what a non-zero rank does after the broadcast), in the
launch configuration bench.py times (overlap on, auto block size), and the concatenation is compared BITWISE with the
1-shard run -- for G = 2, 4, 8, at full configuration sizes where it matters (n = 1e4 with K2 fused into K1's
epilogue, where a short tail block once took narrower tiles than a full block).

The pipeline stress test drives the three-stream pipeline (copy stream, auxiliary K2/K3 stream, D2H stream, joined
by events) with random block sizes, random placements (host / device inputs and outputs), back-to-back calls into
different buffers and random host-side delays between enqueues, and asserts bitwise-stable outputs.
"""
import random
import time

import numpy as np
import pytest

import datagen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _gw():
    import paper_1207_2169_b200 as gw
    return gw


def _ld(n):
    return (n + 15) // 16 * 16


def _shard(m, r, g):
    return (r * m) // g, ((r + 1) * m) // g


def _inputs(cfg, m=None):
    dev = torch.device("cuda", 0)
    c = cfg if m is None else datagen.Config(cfg.index, cfg.n, cfg.p, m, cfg.t, cfg.S, cfg.h2_range, cfg.s2_range)
    ds = datagen.dataset(c, device=dev)
    xr = torch.empty((c.m, _ld(c.n)), dtype=torch.uint8, pin_memory=True)
    datagen.xr_dosages(c, ld=_ld(c.n), out=xr.numpy())
    return c, ds, xr


def _emulate(c, ds, xr_dev, i8, block, groups):
    """1-shard run + G-shard emulations; asserts bitwise equality and returns the number of shard edges checked."""
    gw = _gw()
    eng = gw.Gwas(c.n, c.p, c.t, device=0, block_cols=block, int8_slices=i8, overlap=True)
    eng.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
    info = eng.run_info()
    ref = eng.run(xr_dev)
    torch.cuda.synchronize()
    edges = 0
    for g in groups:
        # a "rank" context: attached to a byte copy of rank 0's state, like the ranks after the NCCL broadcast
        rk = gw.Gwas(c.n, c.p, c.t, device=0, block_cols=block, int8_slices=i8, overlap=True)
        rk.state.copy_(eng.state)
        rk.attach()
        out = rk.alloc_outputs(c.m)
        for r in range(g):
            lo, hi = _shard(c.m, r, g)
            rk.run(xr_dev[lo:hi], out=(out[0][lo:hi], out[1][lo:hi], out[2][lo:hi]))
            edges += 1
        torch.cuda.synchronize()
        for a, b in zip(ref, out):
            assert torch.equal(a, b), f"G={g} shards differ from the 1-shard run (i8={i8}, k={info['block_cols']})"
        rk.close()
        del out
    eng.close()
    return info, ref


def test_shard_emulation_c3_full_fused():
    """C3 at full size (n = 1e4, m = 1e6, t = 1): K2 fused into K1 (t (p+2) = 7 <= 28); G = 2, 4, 8 shards and a
    different block size all reproduce the 1-shard run bit for bit."""
    c, ds, xr = _inputs(datagen.CONFIGS[3])
    xr_dev = xr.to("cuda")
    info, ref = _emulate(c, ds, xr_dev, 0, 0, (2, 4, 8))
    assert info["fused_k2"]
    # block size: auto vs the survey's 8192 (tail blocks of 576 vs 3136 columns) -- same bits
    gw = _gw()
    eng = gw.Gwas(c.n, c.p, c.t, device=0, block_cols=8192, overlap=False)
    eng.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
    other = eng.run(xr_dev)
    torch.cuda.synchronize()
    for a, b in zip(ref, other):
        assert torch.equal(a, b)
    eng.close()
    print(f"C3 full: auto k = {info['block_cols']}, shards 2/4/8 and k = 8192 bitwise equal")


@pytest.mark.parametrize("i8", [0, 7])
def test_shard_emulation_c4_columns(i8):
    """C4 shape (n = 1e4, p = 5, t = 1e3) on its first 60 000 SNPs: shard edges inside blocks, tail blocks of every
    size; FP64 (K2 unfused: t (p+2) = 7000) and the int8-sliced mode."""
    c, ds, xr = _inputs(datagen.CONFIGS[4], m=60_000)
    _emulate(c, ds, xr.to("cuda"), i8, 0 if i8 == 0 else 8192, (2, 4, 8))


@pytest.mark.parametrize("index", [1, 2])
def test_shard_emulation_c1_c2_full(index):
    """C1 (fused K2, 64-wide tiles) and C2 (many traits) at full size."""
    c, ds, xr = _inputs(datagen.CONFIGS[index])
    info, _ = _emulate(c, ds, xr.to("cuda"), 0, 0, (2, 4, 8))
    assert info["fused_k2"] == (index == 1)


@pytest.mark.parametrize("t", [64, 4])
def test_pipeline_stress_random_blocks_and_delays(t):
    """Random block sizes / placements / overlap, three back-to-back gwas_run calls per context into different
    buffers, random host sleeps between enqueues: every output bitwise equal to a serial device-resident run."""
    gw = _gw()
    cfg = datagen.custom_config(n=1000, p=4, m=20_000, t=t, index=700 + t)
    ds = datagen.dataset(cfg, device="cuda")
    xr_h = torch.empty((cfg.m, _ld(cfg.n)), dtype=torch.uint8, pin_memory=True)
    datagen.xr_dosages(cfg, ld=_ld(cfg.n), out=xr_h.numpy())
    xr_d = xr_h.to("cuda")
    base = gw.Gwas(cfg.n, cfg.p, cfg.t, device=0, block_cols=8192, overlap=False)
    base.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
    ref = [x.cpu() for x in base.run(xr_d)]
    torch.cuda.synchronize()
    rng = random.Random(12345 + t)
    for it in range(6):
        k = rng.choice([128, 640, 1000, 4096, 8192, 0])
        ovl = rng.random() < 0.7
        eng = gw.Gwas(cfg.n, cfg.p, cfg.t, device=0, block_cols=k, overlap=ovl)
        eng.state.copy_(base.state)
        eng.attach()
        outs = []
        for call in range(3):
            host_in, host_out = rng.random() < 0.6, rng.random() < 0.5
            out = eng.alloc_outputs(cfg.m, host=host_out)
            eng.run(xr_h if host_in else xr_d, out=out)
            outs.append((out, host_in, host_out))
            time.sleep(rng.uniform(0.0, 0.02))   # host-side delay while the GPU works on the enqueued call
        torch.cuda.synchronize()
        for out, hi, ho in outs:
            for a, b in zip(ref, out):
                assert torch.equal(a, b.cpu()), f"iteration {it}: k={k} overlap={ovl} host_in={hi} host_out={ho}"
        eng.close()
    base.close()
