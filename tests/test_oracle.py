"""Pins of the CPU oracle (oracle/) against things other than itself.

Every check here uses an independent route: hand-derived values, explicit inverses (LU, not Cholesky),
numpy.linalg.lstsq (QR/SVD) for OLS special cases, the n = w closed form, the Frisch-Waugh-Lovell
identity, or statistical calibration.  None calls the CUDA path.
"""
import json
import os

import numpy as np
import pytest

import datagen
import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


def _rand_problem(n, p, seed, h2=0.6, s2=1.7):
    rng = np.random.default_rng(seed)
    G = rng.binomial(2, 0.3, size=(n, 4 * n)).astype(float)
    G = (G - G.mean(0)) / np.maximum(G.std(0), 1e-3)
    Phi = G @ G.T / G.shape[1]
    XL = np.column_stack([np.ones(n), rng.standard_normal((n, p - 2)), rng.integers(0, 2, n)]).astype(float)
    g = rng.binomial(2, 0.25, size=n).astype(float)
    y = rng.standard_normal(n) * 1.3 + XL @ rng.standard_normal(p)
    return Phi, XL, g, y, h2, s2


def _brute(Phi, X, y, s2, h2):
    """P2: explicit inverses (LU), no Cholesky anywhere."""
    M = s2 * (h2 * Phi + (1 - h2) * np.eye(Phi.shape[0]))
    Minv = np.linalg.inv(M)
    A = X.T @ Minv @ X
    V = np.linalg.inv(A)
    return V @ (X.T @ Minv @ y), V


# ---------------------------------------------------------------- P1: worked values (tests/golden)
@pytest.mark.parametrize("case", GOLD["assemble_covariance"])
def test_p1_assemble_covariance(case):
    M = oracle.assemble_covariance(np.array(case["phi"]), case["sigma2"], case["h2"])
    np.testing.assert_allclose(M, case["M"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("case", GOLD["cholesky"])
def test_p1_cholesky(case):
    np.testing.assert_allclose(oracle.cholesky_lower(np.array(case["A"])), case["L"], atol=1e-15)
    R, piv = oracle.small_cholesky(np.array(case["A"]))
    np.testing.assert_allclose(R, case["L"], atol=1e-15)


@pytest.mark.parametrize("case", GOLD["forward_substitute"])
def test_p1_forward_substitute(case):
    np.testing.assert_allclose(oracle.forward_substitute(np.array(case["L"]), np.array(case["B"])), case["X"], atol=1e-15)


@pytest.mark.parametrize("case", GOLD["small_spd_solve"])
def test_p1_small_spd_solve(case):
    S = np.array(case["S"])
    R, _ = oracle.small_cholesky(S)
    np.testing.assert_allclose(oracle.small_spd_solve(R, np.array(case["rhs"])), case["x"], atol=1e-15)
    inv = oracle.small_spd_solve(R, np.eye(S.shape[0]))
    np.testing.assert_allclose(np.diag(inv), case["inv_diag"], atol=1e-15)


@pytest.mark.parametrize("case", GOLD["gls_single"])
def test_p1_gls_worked(case):
    b, V, st = oracle.gls_single(np.array(case["phi"], float), np.array(case["X"]), np.array(case["y"]),
                                 case["sigma2"], case["h2"])
    assert st == 0
    np.testing.assert_allclose(b, case["b"], rtol=1e-14, atol=1e-14)
    if case["var"] is not None:
        np.testing.assert_allclose(V, case["var"], rtol=1e-14, atol=1e-14)


def test_p1_not_spd_raises():
    with pytest.raises(ValueError):
        oracle.cholesky_lower(np.array([[1.0, 2.0], [2.0, 1.0]]))


# ---------------------------------------------------------------- P2: explicit-inverse brute force
@pytest.mark.parametrize("seed,n,p,h2,s2", [(1, 16, 3, 0.6, 1.7), (2, 40, 4, 0.95, 0.5), (3, 64, 5, 0.05, 2.0),
                                            (4, 33, 2, 0.5, 1.0)])
def test_p2_explicit_inverse(seed, n, p, h2, s2):
    Phi, XL, g, y, _, _ = _rand_problem(n, p, seed)
    X = np.column_stack([XL, g])
    b, V, st = oracle.gls_single(Phi, X, y, s2, h2)
    bb, VV = _brute(Phi, X, y, s2, h2)
    se = np.sqrt(np.diag(VV))
    assert st == 0
    assert np.max(np.abs(b - bb) / se) <= 1e-10
    assert np.max(np.abs(V - VV) / np.abs(VV).max()) <= 1e-10


# ---------------------------------------------------------------- P3: OLS special cases (lstsq)
@pytest.mark.parametrize("mode", ["h2=0", "phi=I"])
def test_p3_ols(mode):
    Phi, XL, g, y, _, _ = _rand_problem(50, 4, 7)
    X = np.column_stack([XL, g])
    s2 = 1.3
    if mode == "h2=0":
        b, V, _ = oracle.gls_single(Phi, X, y, s2, 0.0)
    else:
        b, V, _ = oracle.gls_single(np.eye(50), X, y, s2, 0.77)
    bols = np.linalg.lstsq(X, y, rcond=None)[0]
    # Var = sigma2 (X^T X)^-1 via an SVD pseudo-inverse (different algorithm)
    U, sv, Vt = np.linalg.svd(X, full_matrices=False)
    Vols = s2 * (Vt.T / sv ** 2) @ Vt
    se = np.sqrt(np.diag(Vols))
    assert np.max(np.abs(b - bols) / se) <= 1e-10
    assert np.max(np.abs(V - Vols) / np.abs(np.diag(Vols))) <= 1e-10


def test_p3_h2_zero_independent_of_phi():
    Phi, XL, g, y, _, _ = _rand_problem(30, 3, 8)
    Phi2, *_ = _rand_problem(30, 3, 9)
    X = np.column_stack([XL, g])
    b1, V1, _ = oracle.gls_single(Phi, X, y, 1.1, 0.0)
    b2, V2, _ = oracle.gls_single(Phi2, X, y, 1.1, 0.0)
    np.testing.assert_array_equal(b1, b2)
    np.testing.assert_array_equal(V1, V2)


# ---------------------------------------------------------------- P4 / P5: scaling laws
@pytest.mark.parametrize("alpha", [0.5, 4.0])
def test_p4_sigma2_scaling(alpha):
    Phi, XL, g, y, h2, s2 = _rand_problem(40, 4, 11)
    X = np.column_stack([XL, g])
    b1, V1, _ = oracle.gls_single(Phi, X, y, s2, h2)
    b2, V2, _ = oracle.gls_single(Phi, X, y, alpha * s2, h2)
    np.testing.assert_allclose(b2, b1, rtol=1e-12, atol=1e-12 * np.abs(b1).max())
    np.testing.assert_allclose(V2, alpha * V1, rtol=1e-12, atol=1e-14)            # textbook: linear
    _, L1, _ = oracle.gls_single(Phi, X, y, s2, h2, var_convention=1)
    _, L2, _ = oracle.gls_single(Phi, X, y, alpha * s2, h2, var_convention=1)
    np.testing.assert_allclose(L2, alpha ** 2 * L1, rtol=1e-12, atol=1e-14)       # paper-literal: quadratic


@pytest.mark.parametrize("alpha", [-3.0, 0.25])
def test_p5_y_scaling(alpha):
    Phi, XL, g, y, h2, s2 = _rand_problem(40, 4, 12)
    X = np.column_stack([XL, g])
    b1, V1, _ = oracle.gls_single(Phi, X, y, s2, h2)
    b2, V2, _ = oracle.gls_single(Phi, X, alpha * y, s2, h2)
    np.testing.assert_allclose(b2, alpha * b1, rtol=1e-12, atol=1e-13)
    np.testing.assert_array_equal(V2, V1)


# ---------------------------------------------------------------- P6: joint permutation of individuals
def test_p6_permutation():
    Phi, XL, g, y, h2, s2 = _rand_problem(48, 4, 13)
    X = np.column_stack([XL, g])
    P = np.random.default_rng(0).permutation(48)
    b1, V1, _ = oracle.gls_single(Phi, X, y, s2, h2)
    b2, V2, _ = oracle.gls_single(Phi[np.ix_(P, P)], X[P], y[P], s2, h2)
    se = np.sqrt(np.diag(V1))
    assert np.max(np.abs(b1 - b2) / se) <= 1e-10
    assert np.max(np.abs(V1 - V2) / np.abs(np.diag(V1))) <= 1e-10


# ---------------------------------------------------------------- P7: exact recovery
@pytest.mark.parametrize("h2", [0.0, 0.5, 0.99])
def test_p7_exact_recovery(h2):
    Phi, XL, g, _, _, s2 = _rand_problem(36, 4, 14)
    X = np.column_stack([XL, g])
    beta = np.array([0.3, -1.2, 2.5, 0.7, -0.05])
    b, _, st = oracle.gls_single(Phi, X, X @ beta, s2, h2)
    assert st == 0
    assert np.max(np.abs(b - beta)) <= 1e-10 * np.abs(beta).max()


# ---------------------------------------------------------------- P8: n = w closed form
def test_p8_square_closed_form():
    rng = np.random.default_rng(15)
    n = 5
    A = rng.standard_normal((n, n))
    Phi = A @ A.T / n + 0.1 * np.eye(n)
    X = np.column_stack([np.ones(n), rng.standard_normal((n, 3)), rng.integers(0, 3, n)])
    y = rng.standard_normal(n)
    s2, h2 = 1.4, 0.35
    b, V, _ = oracle.gls_single(Phi, X, y, s2, h2)
    M = s2 * (h2 * Phi + (1 - h2) * np.eye(n))
    Xi = np.linalg.inv(X)
    np.testing.assert_allclose(b, Xi @ y, rtol=1e-9, atol=1e-9 * np.abs(Xi @ y).max())
    np.testing.assert_allclose(V, Xi @ M @ Xi.T, rtol=1e-9, atol=1e-9 * np.abs(V).max())


# ---------------------------------------------------------------- P9: Frisch-Waugh-Lovell for the SNP entry
def test_p9_fwl():
    Phi, XL, g, y, h2, s2 = _rand_problem(60, 4, 16)
    M = s2 * (h2 * Phi + (1 - h2) * np.eye(60))
    Minv = np.linalg.inv(M)
    P = XL @ np.linalg.inv(XL.T @ Minv @ XL) @ XL.T @ Minv      # M^-1-orthogonal projector onto span(X_L)
    gt, yt = g - P @ g, y - P @ y
    bg = (gt @ Minv @ yt) / (gt @ Minv @ gt)
    vg = 1.0 / (gt @ Minv @ gt)
    b, V, _ = oracle.gls_single(Phi, np.column_stack([XL, g]), y, s2, h2)
    assert abs(b[-1] - bg) / np.sqrt(vg) <= 1e-10
    assert abs(V[-1, -1] - vg) / vg <= 1e-10


# ---------------------------------------------------------------- P10 + sequence == per-pair Alg. 1
def _small_cfg_data(n=48, p=4, m=37, t=5, seed_index=101):
    cfg = datagen.custom_config(n=n, p=p, m=m, t=t, index=seed_index)
    ds = datagen.dataset(cfg)
    XR = datagen.xr_dosages(cfg).T.astype(float)  # (n, m)
    return cfg, ds, XR


@pytest.mark.parametrize("p,chunk", [(4, 4096), (4, 7), (1, 5)])
def test_sequence_matches_single_per_pair(p, chunk):
    """the trait-cached sequence is BITWISE equal to the literal per-pair Alg. 1 (gls_single, which
    re-assembles and re-factors M_j for every pair), for every pair, including collinear (NaN-payload) pairs and
    chunk boundaries."""
    cfg, ds, XR = _small_cfg_data(p=p)
    XR = XR.copy()
    XR[:, 7] = 0.0                       # monomorphic SNP: collinear with the intercept (status 1)
    out = oracle.gls_sequence(ds.Phi, ds.XL, XR, ds.Y, ds.h2, ds.s2, snp_chunk=chunk)
    assert out["status"][7].tolist() == [oracle.STATUS_COLLINEAR] * cfg.t
    for i in range(cfg.m):
        for j in range(cfg.t):
            b, V, st = oracle.gls_single(ds.Phi, np.column_stack([ds.XL, XR[:, i]]), ds.Y[:, j], ds.s2[j], ds.h2[j])
            assert st == out["status"][i, j]
            np.testing.assert_array_equal(out["b"][i, j], b)
            np.testing.assert_array_equal(out["Var"][i, j], V)


def test_p10_identical_traits_and_slices():
    cfg, ds, XR = _small_cfg_data()
    Y2 = np.column_stack([ds.Y[:, 2], ds.Y[:, 2]])
    out = oracle.gls_sequence(ds.Phi, ds.XL, XR, Y2, ds.h2[[2, 2]], ds.s2[[2, 2]])
    np.testing.assert_array_equal(out["b"][:, 0], out["b"][:, 1])
    full = oracle.gls_sequence(ds.Phi, ds.XL, XR, ds.Y, ds.h2, ds.s2)
    np.testing.assert_array_equal(full["b"][:, 2], out["b"][:, 0])
    sub = oracle.gls_sequence(ds.Phi, ds.XL, XR, ds.Y, ds.h2, ds.s2, snps=[3, 9], traits=[4])
    np.testing.assert_array_equal(sub["b"][:, 0], full["b"][[3, 9], 4])


# ---------------------------------------------------------------- collinearity policy (reading A6)
def test_collinear_snps_flagged():
    cfg, ds, XR = _small_cfg_data()
    XR = XR.copy()
    XR[:, 0] = 1.0                    # monomorphic: multiple of the intercept
    XR[:, 1] = 2.0 * ds.XL[:, 1]      # copy of a covariate
    out = oracle.gls_sequence(ds.Phi, ds.XL, XR, ds.Y, ds.h2, ds.s2)
    assert (out["status"][:2] == oracle.STATUS_COLLINEAR).all()
    assert np.isnan(out["b"][:2]).all()
    assert (out["status"][2:] == 0).all()
    assert np.isfinite(out["b"][2:]).all()


def test_rank_deficient_xl_raises():
    cfg, ds, XR = _small_cfg_data()
    XL = ds.XL.copy()
    XL[:, 2] = XL[:, 1]
    with pytest.raises(ValueError):
        oracle.gls_sequence(ds.Phi, XL, XR, ds.Y, ds.h2, ds.s2)


# ---------------------------------------------------------------- P12: statistical calibration (pins reading A1)
def test_p12_calibration_pins_var_convention():
    cfg = datagen.custom_config(n=300, p=4, m=120, t=40, h2_range=(0.05, 0.95), s2_range=(0.5, 2.0), index=102)
    ds = datagen.dataset(cfg)
    XR = datagen.xr_dosages(cfg).T.astype(float)
    out0 = oracle.gls_sequence(ds.Phi, ds.XL, XR, ds.Y, ds.h2, ds.s2, var_convention=0)
    out1 = oracle.gls_sequence(ds.Phi, ds.XL, XR, ds.Y, ds.h2, ds.s2, var_convention=1)
    z0 = out0["b"][:, :, -1] ** 2 / out0["Var"][:, :, -1, -1]
    z1 = out1["b"][:, :, -1] ** 2 / out1["Var"][:, :, -1, -1]
    m0, m1 = z0.mean(0), z1.mean(0)
    inv = 1.0 / ds.s2
    slope0 = np.polyfit(inv, m0, 1)[0]
    slope1 = np.polyfit(inv, m1, 1)[0]
    assert 0.8 <= m0.mean() <= 1.2          # z ~ N(0,1) under the null with the textbook Var
    assert abs(slope0) < 0.3                # no dependence on 1/sigma2
    assert slope1 > 0.6                     # the paper-literal reading scales z^2 by 1/sigma2


# ---------------------------------------------------------------- generators (not the method)
def test_datagen_determinism_and_ranges():
    cfg = datagen.CONFIGS[0]
    a = datagen.xr_dosages(cfg, 100, 900)
    b = datagen.xr_dosages(cfg)[100:900]
    np.testing.assert_array_equal(a, b)
    assert set(np.unique(a)) <= {0, 1, 2}
    ds = datagen.dataset(cfg)
    np.testing.assert_array_equal(ds.Phi, ds.Phi.T)
    assert 0.8 < np.mean(np.diag(ds.Phi)) < 1.2
    assert ((ds.h2 >= 0.1) & (ds.h2 <= 0.9)).all() and ((ds.s2 >= 0.5) & (ds.s2 <= 2)).all()
    assert (ds.XL[:, 0] == 1).all() and set(np.unique(ds.XL[:, -1])) <= {0.0, 1.0}
    # dosage frequencies ~ Binomial(2, maf), maf ~ U(.05,.5): mean dosage 2*E[maf] = 0.55
    assert 0.5 < datagen.xr_dosages(cfg).mean() < 0.6
