"""GPU parity of the variance-component estimation step (gwas_setup_estimate; DESIGN.md
readings E1-E4) against the CPU oracle (oracle/estimate.py, dense Cholesky likelihood, no eigendecomposition).

Tolerances (derived in DESIGN.md §6d): the estimate h2^ is a root of dl/dh located by bisection on both sides; the
derivative's rounding noise (~1e-13 relative to its terms) over its slope (~n) moves the root by < 1e-11, so
|h2_gpu - h2_ref| <= 1e-8 absolute, sigma2 relative <= 1e-8, log-likelihood relative <= 1e-10.  Where the two sides'
first grid maxima differ (a near-tie of two grid likelihoods), the tie itself is checked instead (<= 1e-9 relative)
and the trait is excluded from the h2 comparison -- at most 1 % of the traits (see _check).  End to end, (b, Var) after estimation match the oracle's GLS
evaluated at the oracle's own estimates within the north-star tolerances.
"""
import numpy as np
import pytest

import datagen
import oracle
import oracle.estimate as OE
from gpu_helpers import TOL_B, TOL_VAR, compare

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL_H2 = 1e-8
TOL_S2 = 1e-8
TOL_LL = 1e-10


def _gw():
    import paper_1207_2169_b200 as gw
    return gw


def _ld(n, es=1):
    q = 16 // es
    return (n + q - 1) // q * q


def _check(ds, method, gpu, ref, traits):
    """Compare GPU estimates (all traits) with oracle estimates on `traits`; returns max errors.

    A trait whose h2 differs by more than TOL_H2 is excluded from the h2 comparison only when it is a genuine near-tie
    of two grid likelihoods: the two sides' first grid argmaxes differ (GPU g_star from gwas_estimate_grid_argmax vs
    the oracle's), the oracle's likelihood at the GPU's h2 is within 1e-9 relative of the oracle's optimum, and the
    GPU's sigma2 and log-likelihood equal the oracle's evaluated AT the GPU's h2 (sigma2 rel <= 1e-8, ll rel <= 1e-10).
    At most 1 % of the compared traits (rounded down) may be excluded, so a broken estimator cannot pass by exclusion."""
    meth = OE.REML if method == "reml" else OE.ML
    eh = es = el = 0.0
    skipped = []
    for jj, j in enumerate(traits):
        if abs(gpu["h2"][j] - ref["h2"][jj]) > TOL_H2:
            assert int(gpu["g_star"][j]) != int(ref["g_star"][jj]), \
                (j, gpu["h2"][j], ref["h2"][jj], "same grid argmax: not a tie")
            alt = OE.profile_loglik(ds.Phi, ds.XL, ds.Y[:, j], gpu["h2"][j], meth)
            assert abs(alt["ll"] - ref["ll"][jj]) <= 1e-9 * abs(ref["ll"][jj]), (j, gpu["h2"][j], ref["h2"][jj])
            assert abs(gpu["sigma2"][j] - alt["sigma2"]) <= TOL_S2 * alt["sigma2"], j
            assert abs(gpu["loglik"][j] - alt["ll"]) <= TOL_LL * abs(alt["ll"]), j
            skipped.append(int(j))
            continue
        eh = max(eh, abs(gpu["h2"][j] - ref["h2"][jj]))
        es = max(es, abs(gpu["sigma2"][j] - ref["sigma2"][jj]) / ref["sigma2"][jj])
        el = max(el, abs(gpu["loglik"][j] - ref["ll"][jj]) / abs(ref["ll"][jj]))
    assert len(skipped) <= int(0.01 * len(traits)), f"near-tie exclusions {skipped} exceed 1% of {len(traits)} traits"
    return eh, es, el


def _estimate(cfg, ds, method, **kw):
    gw = _gw()
    eng = gw.Gwas(cfg.n, cfg.p, cfg.t, device=0, **kw)
    est = eng.setup_estimate(ds.Phi, ds.XL, ds.Y, method)
    est["ms"] = eng.estimate_ms()
    return eng, est


def _oracle_estimate(ds, method, traits):
    meth = OE.REML if method == "reml" else OE.ML
    rs = [OE.estimate_trait(ds.Phi, ds.XL, ds.Y[:, j], meth) for j in traits]
    return {"h2": np.array([r["h2"] for r in rs]), "sigma2": np.array([r["sigma2"] for r in rs]),
            "ll": np.array([r["ll"] for r in rs]), "g_star": np.array([r["g_star"] for r in rs]),
            "grid_ll": [r["grid_ll"] for r in rs]}


@pytest.mark.parametrize("method", ["ml", "reml"])
def test_estimate_c0_all_traits(method):
    cfg = datagen.custom_config(n=200, p=4, m=64, t=12, index=0)  # config 0's generators, 12 traits
    ds = datagen.dataset(cfg)
    eng, est = _estimate(cfg, ds, method)
    eng.close()
    traits = np.arange(cfg.t)
    ref = _oracle_estimate(ds, method, traits)
    eh, es, el = _check(ds, method, est, ref, traits)
    print(f"estimate {method} C0x12: max|dh2|={eh:.2e} sigma2 rel={es:.2e} ll rel={el:.2e}")
    assert eh <= TOL_H2 and es <= TOL_S2 and el <= TOL_LL


@pytest.mark.parametrize("p", [1, 2, 7])
def test_estimate_other_p(p):
    cfg = datagen.custom_config(n=150, p=p, m=16, t=5, index=7)
    ds = datagen.dataset(cfg)
    eng, est = _estimate(cfg, ds, "reml")
    eng.close()
    ref = _oracle_estimate(ds, "reml", np.arange(cfg.t))
    eh, es, el = _check(ds, "reml", est, ref, np.arange(cfg.t))
    assert eh <= TOL_H2 and es <= TOL_S2 and el <= TOL_LL, (eh, es, el)


def test_estimate_boundary_zero():
    """h2 = 0 truth, ML: many traits end at the h = 0 boundary, where both sides return exactly 0."""
    cfg = datagen.custom_config(n=120, p=3, m=16, t=16, h2_range=(0.0, 0.0), s2_range=(1.0, 1.0), index=8)
    ds = datagen.dataset(cfg)
    eng, est = _estimate(cfg, ds, "ml")
    eng.close()
    ref = _oracle_estimate(ds, "ml", np.arange(cfg.t))
    at0 = ref["h2"] == 0.0
    assert at0.sum() >= 3
    assert np.all(est["h2"][at0] == 0.0)
    eh, es, el = _check(ds, "ml", est, ref, np.arange(cfg.t))
    assert eh <= TOL_H2 and es <= TOL_S2 and el <= TOL_LL


def test_estimate_then_run_end_to_end():
    """Estimation + Alg. 4 in one call: (b, Var) vs the oracle's GLS at the oracle's estimates."""
    cfg = datagen.custom_config(n=200, p=4, m=300, t=6, index=0)
    ds = datagen.dataset(cfg)
    XR = datagen.xr_dosages(cfg, ld=_ld(cfg.n))
    eng, est = _estimate(cfg, ds, "reml", block_cols=128)
    b, v, s = eng.run(torch.from_numpy(XR).cuda())
    torch.cuda.synchronize()
    b, v, s = b.cpu().numpy(), v.cpu().numpy(), s.cpu().numpy()
    eng.close()
    ref_est = _oracle_estimate(ds, "reml", np.arange(cfg.t))
    ref = oracle.gls_sequence(ds.Phi, ds.XL, XR[:, :cfg.n].T.astype(np.float64), ds.Y, ref_est["h2"],
                              ref_est["sigma2"])
    eb, ev = compare(b, v, s, ref)
    print(f"estimate+run: max|db|/SE={eb:.2e} Var rel={ev:.2e}")
    assert eb <= TOL_B and ev <= TOL_VAR


def test_estimate_c2_sampled_traits_and_consistency():
    """C2 (n = 1000, t = 1000): all traits on the GPU; 3 seeded traits through the oracle; and the estimates
    track the simulated truth (h2_j ~ U(.05,.95), reading A13) -- mean error small, strong correlation."""
    cfg = datagen.CONFIGS[2]
    ds = datagen.dataset(cfg, device="cuda")
    eng, est = _estimate(cfg, ds, "reml")
    ms = est["ms"]
    eng.close()
    traits = np.array([0, 517, cfg.t - 1])
    ref = _oracle_estimate(ds, "reml", traits)
    eh, es, el = _check(ds, "reml", est, ref, traits)
    print(f"C2 estimate: {ms:.2f} ms for {cfg.t} traits; sampled max|dh2|={eh:.2e} s2 rel={es:.2e} ll rel={el:.2e}")
    assert eh <= TOL_H2 and es <= TOL_S2 and el <= TOL_LL
    assert abs(np.mean(est["h2"] - ds.h2)) < 0.03
    assert np.corrcoef(est["h2"], ds.h2)[0, 1] > 0.6
    assert abs(np.mean(est["sigma2"] / ds.s2) - 1.0) < 0.05


def test_estimate_errors():
    gw = _gw()
    cfg = datagen.custom_config(n=64, p=3, m=16, t=2, index=9)
    ds = datagen.dataset(cfg)
    eng = gw.Gwas(cfg.n, cfg.p, cfg.t, device=0)
    with pytest.raises(KeyError):
        eng.setup_estimate(ds.Phi, ds.XL, ds.Y, "mle")
    Y = ds.Y.copy()
    Y[:, 1] = ds.XL @ np.array([1.0, 2.0, -1.0])  # y in the span of X_L: R = 0
    with pytest.raises(gw.GwasError) as ei:
        eng.setup_estimate(ds.Phi, ds.XL, Y, "reml")
    assert "trait 1" in str(ei.value)
    eng.close()
    ch = gw.Gwas(cfg.n, cfg.p, 1, device=0, algorithm="chol")
    with pytest.raises(gw.GwasError):
        ch.setup_estimate(ds.Phi, ds.XL, ds.Y[:, :1], "ml")
    ch.close()


def test_estimate_with_lowrank_weights_and_int8():
    """Estimation feeds the low-rank weight factorisation and the int8-sliced run the same way as given (h2, s2)."""
    cfg = datagen.custom_config(n=240, p=4, m=500, t=48, index=0)
    ds = datagen.dataset(cfg)
    XR = datagen.xr_dosages(cfg, ld=_ld(cfg.n))
    eng, est = _estimate(cfg, ds, "reml", block_cols=256, trait_rank=-1, int8_slices=7)
    assert eng.trait_rank()[0] > 0
    b, v, s = eng.run(torch.from_numpy(XR).cuda())
    torch.cuda.synchronize()
    b, v, s = b.cpu().numpy(), v.cpu().numpy(), s.cpu().numpy()
    eng.close()
    ref_est = _oracle_estimate(ds, "reml", np.arange(cfg.t))
    eh, es, el = _check(ds, "reml", est, ref_est, np.arange(cfg.t))
    assert eh <= TOL_H2 and es <= TOL_S2 and el <= TOL_LL
    ref = oracle.gls_sequence(ds.Phi, ds.XL, XR[:, :cfg.n].T.astype(np.float64), ds.Y, ref_est["h2"],
                              ref_est["sigma2"])
    eb, ev = compare(b, v, s, ref)
    assert eb <= TOL_B and ev <= TOL_VAR, (eb, ev)
