"""Pins of the estimation oracle (oracle/estimate.py; readings E1-E4) against things other than itself.

Independent routes: hand-derived values (tests/golden/estimate_worked_examples.json), scipy's multivariate-normal
log-density (eigendecomposition-based), Harville's error-contrast likelihood through an SVD null-space basis, the
OLS closed form via numpy.linalg.lstsq at h = 0, central finite differences of the scipy log-density for the
derivative, scipy's bounded Brent search for the optimiser, invariances, and statistical consistency on traits
simulated with known (h2, sigma2).  None calls the CUDA path.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.optimize as sopt
from scipy.stats import multivariate_normal

import datagen
import oracle.estimate as E

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "estimate_worked_examples.json")))


def _problem(n=60, p=3, seed=5, h_true=0.6, s2=1.4):
    rng = np.random.default_rng(seed)
    G = rng.binomial(2, 0.3, size=(n, 3 * n)).astype(float)
    G = (G - 0.6) / math.sqrt(0.42)  # population-standardised: Phi is full rank (no null vector in span(X_L))
    Phi = G @ G.T / G.shape[1]
    XL = np.column_stack([np.ones(n), rng.standard_normal((n, p - 2)), rng.integers(0, 2, n)]).astype(float)
    V = h_true * Phi + (1 - h_true) * np.eye(n)
    y = XL @ rng.standard_normal(p) + np.linalg.cholesky(s2 * V + 1e-12 * np.eye(n)) @ rng.standard_normal(n)
    return Phi, XL, y


# ------------------------------------------------------------ hand values
@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: c["cite"][:30])
@pytest.mark.parametrize("key,method", [("ml", E.ML), ("reml", E.REML)])
def test_hand_values(case, key, method):
    r = E.profile_loglik(np.array(case["Phi"]), np.array(case["XL"]), np.array(case["y"]), case["h"], method,
                         with_derivative=True)
    want = case[key]
    assert r["ll"] == pytest.approx(eval(want["ll_expr"], {"math": math}), rel=1e-14, abs=1e-14)
    assert r["sigma2"] == pytest.approx(want["sigma2"], rel=1e-14)
    np.testing.assert_allclose(r["beta"], want["beta"], rtol=1e-14)
    if "dll" in want:
        assert r["dll"] == pytest.approx(want["dll"], abs=1e-14)


# ------------------------------------------------------------ library log-densities
@pytest.mark.parametrize("h", [0.0, 0.3, 0.75, 0.97])
def test_ml_equals_scipy_logpdf_and_profiles(h):
    Phi, XL, y = _problem()
    r = E.profile_loglik(Phi, XL, y, h, E.ML)
    V = h * Phi + (1 - h) * np.eye(len(y))
    ref = multivariate_normal(mean=XL @ r["beta"], cov=r["sigma2"] * V).logpdf(y)
    assert r["ll"] == pytest.approx(ref, rel=1e-11)
    # beta^ and sigma2^ maximise the full likelihood (profiling is correct): perturbations lower it
    for db in (np.eye(XL.shape[1])[0] * 1e-3, np.eye(XL.shape[1])[-1] * -1e-3):
        assert multivariate_normal(XL @ (r["beta"] + db), r["sigma2"] * V).logpdf(y) < ref
    for f in (0.99, 1.01):
        assert multivariate_normal(XL @ r["beta"], f * r["sigma2"] * V).logpdf(y) < ref


@pytest.mark.parametrize("h", [0.0, 0.4, 0.9])
def test_reml_equals_error_contrast_likelihood(h):
    Phi, XL, y = _problem()
    r = E.profile_loglik(Phi, XL, y, h, E.REML)
    K = sla.null_space(XL.T)  # n x (n-p) orthonormal, K^T X = 0 (SVD)
    V = h * Phi + (1 - h) * np.eye(len(y))
    ref = multivariate_normal(mean=np.zeros(K.shape[1]), cov=r["sigma2"] * (K.T @ V @ K)).logpdf(K.T @ y)
    assert r["ll"] == pytest.approx(ref, rel=1e-11)
    for f in (0.99, 1.01):  # sigma2^ = R/(n-p) maximises the contrast likelihood
        assert multivariate_normal(np.zeros(K.shape[1]), f * r["sigma2"] * (K.T @ V @ K)).logpdf(K.T @ y) < ref


def test_h0_is_ols():
    Phi, XL, y = _problem(seed=9)
    n, p = XL.shape
    beta, res, *_ = np.linalg.lstsq(XL, y, rcond=None)
    rss = float(res[0])
    r = E.profile_loglik(Phi, XL, y, 0.0, E.ML)
    np.testing.assert_allclose(r["beta"], beta, rtol=1e-12)
    assert r["sigma2"] == pytest.approx(rss / n, rel=1e-12)
    assert r["ll"] == pytest.approx(-n / 2 * (math.log(2 * math.pi * rss / n) + 1), rel=1e-13)
    rr = E.profile_loglik(Phi, XL, y, 0.0, E.REML)
    assert rr["sigma2"] == pytest.approx(rss / (n - p), rel=1e-12)


# ------------------------------------------------------------ derivative (reading E2) vs finite differences
@pytest.mark.parametrize("method", [E.ML, E.REML])
@pytest.mark.parametrize("h", [0.05, 0.5, 0.93])
def test_derivative_matches_finite_differences(method, h):
    Phi, XL, y = _problem(seed=3)
    d = E.profile_loglik(Phi, XL, y, h, method, with_derivative=True)["dll"]
    K = sla.null_space(XL.T)
    n = len(y)

    def ll_ref(hh):  # the profile likelihood through scipy only (independent of the oracle's formulas)
        V = hh * Phi + (1 - hh) * np.eye(n)
        if method == E.ML:
            Vi = np.linalg.inv(V)
            beta = np.linalg.solve(XL.T @ Vi @ XL, XL.T @ Vi @ y)
            rr = y - XL @ beta
            s2 = rr @ Vi @ rr / n
            return multivariate_normal(XL @ beta, s2 * V).logpdf(y)
        C = K.T @ V @ K
        z = K.T @ y
        s2 = z @ np.linalg.solve(C, z) / K.shape[1]
        return multivariate_normal(np.zeros(K.shape[1]), s2 * C).logpdf(z)

    step = 1e-5
    fd = (ll_ref(h + step) - ll_ref(h - step)) / (2 * step)
    assert d == pytest.approx(fd, rel=1e-6, abs=1e-6)


# ------------------------------------------------------------ optimiser (reading E3)
@pytest.mark.parametrize("method", [E.ML, E.REML])
def test_optimiser_matches_bounded_brent(method):
    Phi, XL, y = _problem(seed=11)
    est = E.estimate_trait(Phi, XL, y, method)
    gs = est["g_star"]
    assert est["ll"] >= np.max(est["grid_ll"]) - 1e-12
    lo, hi = max(0, gs - 1) / E.GRID, min(E.GRID, gs + 1) / E.GRID
    res = sopt.minimize_scalar(lambda h: -E.profile_loglik(Phi, XL, y, h, method)["ll"], bounds=(lo, hi),
                               method="bounded", options={"xatol": 1e-10})
    assert est["h2"] == pytest.approx(res.x, abs=1e-5)
    assert est["ll"] >= -res.fun - 1e-10
    if 0 < est["h2"] < 1:  # interior optimum: first-order condition
        assert abs(E.profile_loglik(Phi, XL, y, est["h2"], method, with_derivative=True)["dll"]) < 1e-6


def test_boundary_optimum_at_zero():
    # y with no kinship signal (iid noise), seed chosen so that the ML optimum sits at the h = 0 boundary:
    # l is decreasing at h = 0, so reading E3 returns exactly 0 without bisecting
    rng = np.random.default_rng(3)
    n = 50
    G = rng.standard_normal((n, 5))
    Phi = G @ G.T / 5 + 0.05 * np.eye(n)
    XL = np.column_stack([np.ones(n), rng.standard_normal(n)])
    y = XL @ np.array([1.0, -0.5]) + rng.standard_normal(n)
    est = E.estimate_trait(Phi, XL, y, E.ML)
    assert est["g_star"] == 0
    assert E.profile_loglik(Phi, XL, y, 0.0, E.ML, with_derivative=True)["dll"] < 0
    assert est["h2"] == 0.0
    res = sopt.minimize_scalar(lambda h: -E.profile_loglik(Phi, XL, y, h, E.ML)["ll"], bounds=(0.0, 0.01),
                               method="bounded", options={"xatol": 1e-12})
    assert res.x < 1e-6


def test_ml_degenerate_with_singular_kinship():
    """Reading E4: with a sample-centred GRM (Phi 1 = 0) and an intercept in X_L, the ML profile likelihood grows
    like -1/2 log(1 - h) as h -> 1 (log|V| -> -inf, R bounded); REML's log|A| cancels it exactly."""
    cfg = datagen.custom_config(n=80, p=3, m=10, t=1, index=43)
    ds = datagen.dataset(cfg)
    y = ds.Y[:, 0]
    h1, h2 = 0.999, 0.9999
    ml = [E.profile_loglik(ds.Phi, ds.XL, y, h, E.ML)["ll"] for h in (h1, h2)]
    rl = [E.profile_loglik(ds.Phi, ds.XL, y, h, E.REML)["ll"] for h in (h1, h2)]
    # the ML increment contains +1/2 log((1-h1)/(1-h2)) = 1/2 log 10 from the null direction; REML's does not
    assert (ml[1] - ml[0]) - (rl[1] - rl[0]) == pytest.approx(0.5 * math.log(10), abs=0.05)


def test_infeasible_grid_points_skipped():
    # sample-centred GRM: Phi 1 = 0, lambda_min ~ 0 -> h = 1 is infeasible (reading A7 margin)
    cfg = datagen.custom_config(n=80, p=3, m=10, t=2, index=41)
    ds = datagen.dataset(cfg)
    lam = float(np.linalg.eigvalsh(ds.Phi)[0])
    assert abs(lam) < 1e-10
    assert not E.feasible(lam, 1.0)
    est = E.estimate(ds.Phi, ds.XL, ds.Y, E.REML)
    assert np.all((est["h2"] >= 0) & (est["h2"] < 1))


# ------------------------------------------------------------ invariances
def test_invariances():
    Phi, XL, y = _problem(seed=21)
    a = E.estimate_trait(Phi, XL, y, E.REML)
    b = E.estimate_trait(Phi, XL, 4.0 * y, E.REML)  # y -> 4y: h unchanged, sigma2 x 16
    assert b["h2"] == pytest.approx(a["h2"], abs=1e-9)
    assert b["sigma2"] == pytest.approx(16 * a["sigma2"], rel=1e-9)
    perm = np.random.default_rng(0).permutation(len(y))
    c = E.estimate_trait(Phi[np.ix_(perm, perm)], XL[perm], y[perm], E.REML)
    assert c["h2"] == pytest.approx(a["h2"], abs=1e-7)
    assert c["ll"] == pytest.approx(a["ll"], rel=1e-10)


# ------------------------------------------------------------ statistical consistency (the model of P:12-14)
def test_consistency_on_simulated_traits():
    """Traits drawn from N(X beta, sigma2 (h2 Phi + (1-h2) I)) with known h2 = 0.6, sigma2 = 1.5 (datagen, reading
    A13): REML estimates average to the truth (per-trait SE ~ 0.1 at n = 300, so 24 traits give ~0.02)."""
    cfg = datagen.custom_config(n=300, p=3, m=10, t=24, h2_range=(0.6, 0.6), s2_range=(1.5, 1.5), index=42)
    ds = datagen.dataset(cfg)
    est = E.estimate(ds.Phi, ds.XL, ds.Y, E.REML, iters=30)
    assert abs(np.mean(est["h2"]) - 0.6) < 0.08
    assert abs(np.mean(est["sigma2"]) - 1.5) < 0.2


def test_exact_fit_is_an_error():
    """Reading E1: y in the span of X_L (R = 0 up to rounding) has no finite likelihood maximum -> ValueError."""
    Phi, XL, _ = _problem(seed=2)
    y = XL @ np.array([1.0, -2.0, 0.5])
    with pytest.raises(ValueError):
        E.profile_loglik(Phi, XL, y, 0.4, E.REML)
    with pytest.raises(ValueError):
        E.estimate_trait(Phi, XL, y, E.ML)
