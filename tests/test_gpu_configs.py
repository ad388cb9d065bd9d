"""GPU parity at BASELINE.json's full sizes (configs 1-4), in the launch configuration bench.py times
(uint8 X_R resident in HBM; FP64 mode: blocks pipelined over two streams (overlap) with the auto block size, the
headline; int8 mode: overlap, k = 8192), checked on the seeded stratified subsample of reading A18 (>= 10^4 pairs:
<= 16 traits incl. 0 and t-1, SNPs incl. 0, m-1 and the block edges of the k actually used) against the CPU
oracle."""
import numpy as np
import pytest

import datagen
import oracle
from gpu_helpers import TOL_B, TOL_VAR, compare

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("index,i8,lr", [(1, 0, 0), (2, 0, 0), (3, 0, 0), (4, 0, 0), (1, 8, 0), (2, 8, 0), (3, 8, 0),
                                         (4, 8, 0), (2, 0, -1), (4, 0, -1), (2, 8, -1), (4, 8, -1),
                                         (1, 7, 0), (4, 7, -1)])
def test_full_config_subsample(index, i8, lr):
    import paper_1207_2169_b200 as gw
    cfg = datagen.CONFIGS[index]
    dev = torch.device("cuda", 0)
    ds = datagen.dataset(cfg, device=dev)
    ld = (cfg.n + 15) // 16 * 16
    xr = torch.empty((cfg.m, ld), dtype=torch.uint8, pin_memory=True)
    datagen.xr_dosages(cfg, ld=ld, out=xr.numpy())
    xr_dev = xr.to(dev)
    eng = gw.Gwas(cfg.n, cfg.p, cfg.t, device=0, block_cols=0 if (i8 == 0 and lr == 0) else 8192, int8_slices=i8,
                  trait_rank=lr, overlap=True)
    eng.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
    rank = eng.trait_rank()[0]
    assert (rank > 0) == (lr != 0)  # C2 / C4 (t = 1000) compress
    k = eng.run_info()["block_cols"]
    b, v, s = eng.run(xr_dev)
    last = (cfg.m - 1) // k * k
    snps, traits = datagen.subsample(cfg, forced_snps=[k - 1, k, 2 * k - 1, last - 1, last])
    idx_s = torch.from_numpy(snps).to(dev)
    idx_t = torch.from_numpy(traits).to(dev)
    bs = b.index_select(0, idx_s).index_select(1, idx_t).cpu().numpy()
    vs = v.index_select(0, idx_s).index_select(1, idx_t).cpu().numpy()
    ss = s.index_select(0, idx_s).index_select(1, idx_t).cpu().numpy()
    assert int((s != 0).sum().item()) == int((s == 1).sum().item())  # no non-finite pairs anywhere
    eng.close()
    del xr_dev, b, v, s
    G = datagen.xr_columns(cfg, snps)
    ref = oracle.gls_sequence(ds.Phi, ds.XL, G, ds.Y, ds.h2, ds.s2, traits=traits)
    eb, ev = compare(bs, vs, ss, ref)
    print(f"C{index} int8_slices={i8} trait_rank={rank} k={k}: {snps.size} SNPs x {traits.size} traits = {snps.size * traits.size} pairs, "
          f"max|db|/SE={eb:.3e}, max Var rel={ev:.3e}")
    assert snps.size * traits.size >= 10_000
    assert eb <= TOL_B and ev <= TOL_VAR


@pytest.mark.parametrize("index,i8", [(1, 0), (3, 0), (1, 8), (3, 8)])
def test_full_config_subsample_chol(index, i8):
    """The single-trait configs through CLAK-Chol (Alg. 3) at full size, in both K1 modes."""
    import paper_1207_2169_b200 as gw
    cfg = datagen.CONFIGS[index]
    dev = torch.device("cuda", 0)
    ds = datagen.dataset(cfg, device=dev)
    ld = (cfg.n + 15) // 16 * 16
    xr = torch.empty((cfg.m, ld), dtype=torch.uint8, pin_memory=True)
    datagen.xr_dosages(cfg, ld=ld, out=xr.numpy())
    eng = gw.Gwas(cfg.n, cfg.p, cfg.t, device=0, block_cols=8192, int8_slices=i8, algorithm="chol", overlap=True)
    eng.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
    b, v, s = eng.run(xr.to(dev))
    snps, traits = datagen.subsample(cfg)
    idx_s = torch.from_numpy(snps).to(dev)
    bs = b.index_select(0, idx_s).cpu().numpy()
    vs = v.index_select(0, idx_s).cpu().numpy()
    ss = s.index_select(0, idx_s).cpu().numpy()
    eng.close()
    G = datagen.xr_columns(cfg, snps)
    ref = oracle.gls_sequence(ds.Phi, ds.XL, G, ds.Y, ds.h2, ds.s2, traits=traits)
    eb, ev = compare(bs, vs, ss, ref)
    print(f"C{index} chol int8_slices={i8}: {snps.size} pairs, max|db|/SE={eb:.3e}, max Var rel={ev:.3e}")
    assert eb <= TOL_B and ev <= TOL_VAR


def test_full_config_c1_fp64_dosages_staged_from_host():
    """C1 at full size with X_R as fp64 dosages in pinned HOST memory (staged block by block on the copy stream,
    results streamed back to pinned host memory) -- the bench's `modes.fp64_staged` path -- vs the oracle."""
    import paper_1207_2169_b200 as gw
    cfg = datagen.CONFIGS[1]
    ds = datagen.dataset(cfg, device=torch.device("cuda", 0))
    ld = (cfg.n + 1) // 2 * 2                       # 16-byte rows for fp64
    xr8 = torch.empty((cfg.m, ld), dtype=torch.uint8)
    datagen.xr_dosages(cfg, ld=ld, out=xr8.numpy())
    x64 = torch.empty((cfg.m, ld), dtype=torch.float64, pin_memory=True)
    x64.copy_(xr8)
    eng = gw.Gwas(cfg.n, cfg.p, cfg.t, device=0, block_cols=0, xr_dtype="f64", overlap=True)
    eng.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
    b, v, s = eng.alloc_outputs(cfg.m, host=True)
    eng.run(x64, out=(b, v, s))
    torch.cuda.synchronize()
    k = eng.run_info()["block_cols"]
    eng.close()
    snps, traits = datagen.subsample(cfg, forced_snps=[k - 1, k, (cfg.m - 1) // k * k])
    G = datagen.xr_columns(cfg, snps)
    ref = oracle.gls_sequence(ds.Phi, ds.XL, G, ds.Y, ds.h2, ds.s2, traits=traits)
    bs, vs, ss = (x.numpy()[np.ix_(snps, traits)] for x in (b, v, s))
    eb, ev = compare(bs, vs, ss, ref)
    print(f"C1 fp64 dosages from host: {snps.size * traits.size} pairs, max|db|/SE={eb:.3e}, max Var rel={ev:.3e}")
    assert eb <= TOL_B and ev <= TOL_VAR
