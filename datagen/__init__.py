"""Seeded synthetic inputs for the CLAK-Eig GLS-sequence hot path (shared by tests, oracle checks and bench).

This module holds NO arithmetic of the method (no M_j, no eigendecomposition, no GLS): it only draws
the inputs the paper's problem statement (Eq. probDef) consumes -- a kinship matrix
Phi, the fixed design X_L = [1 | L], SNP dosages X_R, phenotypes Y and per-trait (h2_j, sigma2_j) --
with the distributions BASELINE.json `configs` fix (readings A10-A14, A20, A22 of SURVEY.md §8(c),
restated in DESIGN.md §3).  The paper's own data are "artificial data sets which met pre-specified
values of t, m, p, and n"; no public dataset is involved.

Seeds: base = 12072169 + config index; each quantity draws from its own stream
numpy Philox(SeedSequence([base, s])):
    s=0 covariates, s=1 GRM SNPs, s=2 (h2, sigma2), s=3 beta, s=4 a (genetic), s=5 e (noise),
    s=6 parity subsample, [base, 7, b] = test-SNP generation block b (GEN_BLOCK SNPs each),
so any block of X_R can be regenerated on its own.
"""
from __future__ import annotations

import concurrent.futures as _cf
import dataclasses
import os

import numpy as np

BASE_SEED = 12072169
GEN_BLOCK = 8192  # SNPs per independently seeded generation block


@dataclasses.dataclass(frozen=True)
class Config:
    """One BASELINE.json config (index = position in BASELINE.json `configs`)."""
    index: int
    n: int            # individuals
    p: int            # columns of X_L (intercept + covariates)
    m: int            # SNPs
    t: int            # traits
    S: int            # SNPs used to build the GRM Phi
    h2_range: tuple   # (lo, hi) uniform, or (v, v) fixed
    s2_range: tuple
    block_cols: int = 8192

    @property
    def name(self) -> str:
        return f"C{self.index}"

    @property
    def seed(self) -> int:
        return BASE_SEED + self.index


CONFIGS = {
    0: Config(0, n=200, p=4, m=2000, t=4, S=5000, h2_range=(0.1, 0.9), s2_range=(0.5, 2.0), block_cols=2000),
    1: Config(1, n=1000, p=4, m=100_000, t=1, S=5000, h2_range=(0.4, 0.4), s2_range=(1.0, 1.0)),
    2: Config(2, n=1000, p=4, m=100_000, t=1000, S=5000, h2_range=(0.05, 0.95), s2_range=(0.5, 2.0)),
    3: Config(3, n=10_000, p=5, m=1_000_000, t=1, S=20_000, h2_range=(0.1, 0.9), s2_range=(0.5, 2.0)),
    4: Config(4, n=10_000, p=5, m=1_000_000, t=1000, S=20_000, h2_range=(0.05, 0.95), s2_range=(0.5, 2.0)),
}


def custom_config(n, p, m, t, S=None, h2_range=(0.1, 0.9), s2_range=(0.5, 2.0), index=100, block_cols=8192):
    """A config with config-0 generators at other sizes (used by tests)."""
    return Config(index, n=n, p=p, m=m, t=t, S=S if S is not None else max(4 * n, 64),
                  h2_range=h2_range, s2_range=s2_range, block_cols=block_cols)


def _rng(cfg_seed: int, *stream) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(np.random.SeedSequence([cfg_seed, *stream])))


def _dosages_from_uniform(u32: np.ndarray, maf: np.ndarray) -> np.ndarray:
    """Binomial(2, maf) from one uniform u32 per entry (reading A14): g = [u >= (1-f)^2] + [u >= 1-f^2].

    P(g=0) = (1-f)^2, P(g=1) = 2f(1-f), P(g=2) = f^2 exactly as Bern(f)+Bern(f), up to the 2^-32 grid.
    u32: (cols, n); maf: (cols,).  Returns uint8 (cols, n)."""
    scale = float(2 ** 32)
    top = float(2 ** 32 - 1)
    t0 = np.minimum(np.floor((1.0 - maf) ** 2 * scale), top).astype(np.uint32)[:, None]
    t1 = np.minimum(np.floor((1.0 - maf * maf) * scale), top).astype(np.uint32)[:, None]
    g = (u32 >= t0).view(np.uint8)
    g += (u32 >= t1).view(np.uint8)
    return g


def _draw_dosage_block(rng: np.random.Generator, cols: int, n: int):
    maf = rng.uniform(0.05, 0.5, size=cols)
    raw = rng.bit_generator.random_raw((cols * n + 1) // 2).view(np.uint32)[: cols * n]
    return _dosages_from_uniform(raw.reshape(cols, n), maf), maf


def snp_block(cfg: Config, b: int) -> np.ndarray:
    """Test-SNP generation block b: uint8 (cols, n) = columns b*GEN_BLOCK.. of X_R (SNP-major rows)."""
    c0 = b * GEN_BLOCK
    cols = min(GEN_BLOCK, cfg.m - c0)
    if cols <= 0:
        raise ValueError("block out of range")
    g, _ = _draw_dosage_block(_rng(cfg.seed, 7, b), GEN_BLOCK, cfg.n)
    return g[:cols]


def xr_dosages(cfg: Config, snp_lo: int = 0, snp_hi: int | None = None, ld: int | None = None,
               out: np.ndarray | None = None, threads: int | None = None) -> np.ndarray:
    """X_R columns [snp_lo, snp_hi) as uint8, shape (snp_hi-snp_lo, ld) -- i.e. column-major n x cols with
    leading dimension ld >= n (each SNP column contiguous, pad entries zero).  `out` may be a preallocated
    (e.g. pinned) array of that shape.  Generation blocks are drawn in parallel threads."""
    snp_hi = cfg.m if snp_hi is None else snp_hi
    ld = cfg.n if ld is None else ld
    cols = snp_hi - snp_lo
    if out is None:
        out = np.zeros((cols, ld), dtype=np.uint8)
    elif ld > cfg.n:
        out[:, cfg.n:] = 0
    b_lo, b_hi = snp_lo // GEN_BLOCK, (snp_hi - 1) // GEN_BLOCK + 1 if cols > 0 else snp_lo // GEN_BLOCK

    def work(b):
        g = snp_block(cfg, b)
        s0 = b * GEN_BLOCK
        lo, hi = max(s0, snp_lo), min(s0 + g.shape[0], snp_hi)
        out[lo - snp_lo: hi - snp_lo, : cfg.n] = g[lo - s0: hi - s0]

    nthr = threads or min(32, os.cpu_count() or 1)
    if b_hi - b_lo <= 1 or nthr == 1:
        for b in range(b_lo, b_hi):
            work(b)
    else:
        with _cf.ThreadPoolExecutor(nthr) as ex:
            list(ex.map(work, range(b_lo, b_hi)))
    return out


def covariates(cfg: Config) -> np.ndarray:
    """X_L = [1 | N(0,1) x (p-2) | Bernoulli(0.5) 'sex'], float64 (n, p) (readings A3, A12)."""
    rng = _rng(cfg.seed, 0)
    XL = np.empty((cfg.n, cfg.p), dtype=np.float64)
    XL[:, 0] = 1.0
    if cfg.p >= 2:
        XL[:, 1:cfg.p - 1] = rng.standard_normal((cfg.n, cfg.p - 2))
        XL[:, cfg.p - 1] = (rng.uniform(size=cfg.n) < 0.5).astype(np.float64)
    return XL


def grm_snps(cfg: Config) -> np.ndarray:
    """Standardised GRM genotypes G_s (n, S), float64: column s = (g_s - 2 f_s) / sqrt(2 f_s (1 - f_s)) with
    f_s the sample allele frequency (reading A10); monomorphic columns are redrawn."""
    rng = _rng(cfg.seed, 1)
    g, _ = _draw_dosage_block(rng, cfg.S, cfg.n)
    g = g.astype(np.float64)
    f = g.mean(axis=1) / 2.0
    while True:
        bad = np.nonzero((f <= 0.0) | (f >= 1.0))[0]
        if bad.size == 0:
            break
        g2, _ = _draw_dosage_block(rng, bad.size, cfg.n)
        g[bad] = g2
        f[bad] = g[bad].mean(axis=1) / 2.0
    Gs = (g - 2.0 * f[:, None]) / np.sqrt(2.0 * f * (1.0 - f))[:, None]
    return np.ascontiguousarray(Gs.T)


def _gram(Gs: np.ndarray, device) -> np.ndarray:
    if device is None or str(device) == "cpu":
        return Gs @ Gs.T
    import torch
    G = torch.from_numpy(Gs).to(device)
    return (G @ G.T).cpu().numpy()


def kinship(cfg: Config, Gs: np.ndarray | None = None, device=None) -> np.ndarray:
    """Phi = G_s G_s^T / S (BASELINE.json configs[0]: 'standardized GRM ... divided by 5000'), symmetrised
    exactly; float64 (n, n).  `device` (a torch device) only moves the Gram product off the host."""
    Gs = grm_snps(cfg) if Gs is None else Gs
    Phi = _gram(Gs, device) / float(cfg.S)
    Phi = 0.5 * (Phi + Phi.T)
    return np.ascontiguousarray(Phi)


def trait_params(cfg: Config):
    """(h2, sigma2) per trait, float64 (t,) each (config ranges; reading A22 for config 3)."""
    rng = _rng(cfg.seed, 2)
    h2 = rng.uniform(*cfg.h2_range, size=cfg.t) if cfg.h2_range[0] != cfg.h2_range[1] else np.full(cfg.t, cfg.h2_range[0])
    s2 = rng.uniform(*cfg.s2_range, size=cfg.t) if cfg.s2_range[0] != cfg.s2_range[1] else np.full(cfg.t, cfg.s2_range[0])
    return h2.astype(np.float64), s2.astype(np.float64)


def phenotypes(cfg: Config, XL: np.ndarray, Gs: np.ndarray, h2: np.ndarray, s2: np.ndarray, device=None) -> np.ndarray:
    """Y (n, t): y_j = X_L beta_j + sigma_j (sqrt(h2_j) G_s a_j / sqrt(S) + sqrt(1-h2_j) e_j) (reading A13):
    covariance exactly sigma2_j (h2_j Phi + (1-h2_j) I) because Phi = G_s G_s^T / S; null model (no SNP effect)."""
    beta = _rng(cfg.seed, 3).standard_normal((cfg.p, cfg.t))
    a = _rng(cfg.seed, 4).standard_normal((cfg.S, cfg.t))
    e = _rng(cfg.seed, 5).standard_normal((cfg.n, cfg.t))
    if device is None or str(device) == "cpu":
        Ga = Gs @ a
    else:
        import torch
        Ga = (torch.from_numpy(Gs).to(device) @ torch.from_numpy(a).to(device)).cpu().numpy()
    Y = XL @ beta + np.sqrt(s2)[None, :] * (np.sqrt(h2)[None, :] * Ga / np.sqrt(cfg.S) + np.sqrt(1.0 - h2)[None, :] * e)
    return np.asfortranarray(Y)


@dataclasses.dataclass
class Dataset:
    cfg: Config
    Phi: np.ndarray      # (n, n) float64 symmetric
    XL: np.ndarray       # (n, p) float64
    Y: np.ndarray        # (n, t) float64 (Fortran order: each trait contiguous)
    h2: np.ndarray       # (t,)
    s2: np.ndarray       # (t,)


def dataset(cfg: Config, device=None) -> Dataset:
    """Everything but X_R (which is streamed / generated per block with xr_dosages)."""
    XL = covariates(cfg)
    Gs = grm_snps(cfg)
    Phi = kinship(cfg, Gs, device)
    h2, s2 = trait_params(cfg)
    Y = phenotypes(cfg, XL, Gs, h2, s2, device)
    return Dataset(cfg, Phi, XL, Y, h2, s2)


def subsample(cfg: Config, n_pairs: int = 10_000, max_traits: int = 16, forced_snps=()):
    """Stratified seeded parity subsample (reading A18): T_s = min(t, max_traits) traits (always 0 and t-1)
    x ceil(n_pairs/T_s) SNPs, plus forced SNPs (0, m-1, block edges, shard edges).  Returns (snps, traits)
    sorted unique int64 arrays; the checked pairs are their Cartesian product."""
    rng = _rng(cfg.seed, 6)
    Ts = min(cfg.t, max_traits)
    traits = {0, cfg.t - 1}
    others = rng.permutation(cfg.t)
    for j in others:
        if len(traits) >= Ts:
            break
        traits.add(int(j))
    ns = min(cfg.m, -(-n_pairs // Ts))
    snps = set(int(s) for s in rng.choice(cfg.m, size=ns, replace=False))
    k = cfg.block_cols
    forced = {0, cfg.m - 1, min(k - 1, cfg.m - 1), min(k, cfg.m - 1), min(2 * k - 1, cfg.m - 1),
              ((cfg.m - 1) // k) * k}
    forced |= {int(s) for s in forced_snps if 0 <= s < cfg.m}
    snps |= forced
    return np.array(sorted(snps), dtype=np.int64), np.array(sorted(traits), dtype=np.int64)


def xr_columns(cfg: Config, snps) -> np.ndarray:
    """Selected X_R columns as float64 (n, len(snps)), regenerating only the blocks they live in."""
    snps = np.asarray(snps, dtype=np.int64)
    out = np.empty((cfg.n, snps.size), dtype=np.float64)
    by_block = {}
    for idx, s in enumerate(snps):
        by_block.setdefault(int(s) // GEN_BLOCK, []).append(idx)

    def work(b):
        g = snp_block(cfg, b)
        for idx in by_block[b]:
            out[:, idx] = g[int(snps[idx]) - b * GEN_BLOCK]

    nthr = min(16, os.cpu_count() or 1, max(1, len(by_block)))
    if nthr == 1:
        for b in by_block:
            work(b)
    else:
        with _cf.ThreadPoolExecutor(nthr) as ex:
            list(ex.map(work, list(by_block)))
    return out
