"""CPU fp64 ORACLE for the variance-component estimation step (the "first step" of PAPER.md P:16).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this module.  It shares no code with the CUDA path and never imports it.

What the paper says: "In the first step, the reduced model (with X = [1 | L]) is fit to the data, thus
obtaining the estimates {sigma2^, h2^}";: "the model parameters are estimated using an iterative
procedure based on the Maximum Likelihood (GenABEL, FaST-LMM) or Restricted Maximum Likelihood (EMMAX)
methods".  The model: y = X_L beta + R, R ~ N(0, sigma2 (h2 Phi + (1 - h2) I)), h2 in [0, 1].
The paper prints no likelihood and no optimiser; readings E1-E4 fix them and this module follows
them literally, by the plain dense definitions (Cholesky of V, no eigendecomposition of Phi anywhere in the
likelihood):

  V(h)      = h Phi + (1 - h) I,   E = dV/dh = Phi - I                                (sigma2 factored out)
  A         = X^T V^-1 X,  beta^ = A^-1 X^T V^-1 y,  r = y - X beta^,  R = r^T V^-1 r     (GLS of the reduced model)
  ML   (E1): sigma2^ = R / n,        l(h) = -1/2 [ n log(2 pi R / n) + log|V| + n ]
  REML (E1): sigma2^ = R / (n - p),  l(h) = -1/2 [ (n-p) log(2 pi R / (n-p)) + log|V| + log|A| - log|X^T X| + (n-p) ]
            (beta and sigma2 profiled out in closed form; the REML form is Harville's likelihood of the error
             contrasts, including the log|X^T X| constant so that it equals that likelihood exactly)
  derivatives (E2, matrix calculus; envelope theorem for the profiled beta):
       R'   = - r^T V^-1 E V^-1 r,     A' = - X^T V^-1 E V^-1 X
  ML:  l'(h) = -1/2 [ n R'/R + tr(V^-1 E) ]
  REML:l'(h) = -1/2 [ (n-p) R'/R + tr(V^-1 E) + tr(A^-1 A') ]

Optimiser (reading E3): evaluate l on the grid h_g = g/G, g = 0..G (G = 100); a grid point is infeasible
(l = -inf) unless h lambda_min(Phi) + 1 - h > eps_spd (V SPD with the margin of reading A7).  g* = the first
argmax.  If l'(h_g*) > 0 and g*+1 is feasible, bisect [h_g*, h_g*+1]; if l'(h_g*) < 0 and g* > 0, bisect
[h_g*-1, h_g*]; otherwise h^ = h_g*.  Bisection: BISECT_ITERS times mid = (lo + hi)/2, lo = mid if l'(mid) > 0
else hi = mid; h^ = (lo + hi)/2.  sigma2^ and l are then evaluated at h^.

Pins: tests/test_oracle_estimate.py (scipy multivariate-normal log-density, the error-contrast likelihood,
the OLS closed form at h = 0, finite differences of the log-density, a bounded Brent search, invariances,
and statistical consistency on simulated traits).  No function here is "parity unpinned".
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

ML = 0
REML = 1
GRID = 100
BISECT_ITERS = 50
R_REL_MIN = 1e-24  # reading E1: R <= 1e-24 y^T V^-1 y (relative residual 1e-12) means y lies in span(X_L)


def _chol(V):
    return sla.cholesky(V, lower=True, check_finite=True)


def profile_loglik(Phi, XL, y, h, method=ML, with_derivative=False):
    """Profile log-likelihood of the reduced model at h (definitions in the module docstring).

    Returns dict(ll, sigma2, beta, R, dll (if with_derivative)).  Raises ValueError if V(h) is not SPD or
    R <= R_REL_MIN * y^T V^-1 y (y in the span of X_L)."""
    Phi = np.asarray(Phi, dtype=np.float64)
    X = np.asarray(XL, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    n, p = X.shape
    V = h * Phi + (1.0 - h) * np.eye(n)
    V = 0.5 * (V + V.T)
    try:
        L = _chol(V)
    except np.linalg.LinAlgError as exc:
        raise ValueError(f"V(h={h}) not SPD") from exc
    logdetV = 2.0 * np.sum(np.log(np.diag(L)))
    Xw = sla.solve_triangular(L, X, lower=True)
    yw = sla.solve_triangular(L, y, lower=True)
    A = Xw.T @ Xw
    cA = _chol(A)
    beta = sla.cho_solve((cA, True), Xw.T @ yw)
    r = y - X @ beta
    rw = sla.solve_triangular(L, r, lower=True)
    R = float(rw @ rw)
    if not (R > R_REL_MIN * float(yw @ yw)) or not np.isfinite(R):  # reading E1: exact fit is an error
        raise ValueError(f"residual R = {R} at h = {h}: y in the span of X_L")
    if method == ML:
        nn = n
        ll = -0.5 * (n * np.log(2.0 * np.pi * R / n) + logdetV + n)
    else:
        nn = n - p
        logdetA = 2.0 * np.sum(np.log(np.diag(cA)))
        logdetXX = 2.0 * np.sum(np.log(np.diag(_chol(X.T @ X))))
        ll = -0.5 * (nn * np.log(2.0 * np.pi * R / nn) + logdetV + logdetA - logdetXX + nn)
    out = {"ll": float(ll), "sigma2": R / nn, "beta": beta, "R": R}
    if with_derivative:
        E = Phi - np.eye(n)
        Vinv_r = sla.cho_solve((L, True), r)
        Vinv_E = sla.cho_solve((L, True), E)
        dR = -float(Vinv_r @ E @ Vinv_r)
        tr = float(np.trace(Vinv_E))
        dll = nn * dR / R + tr
        if method == REML:
            Vinv_X = sla.cho_solve((L, True), X)
            dA = -(Vinv_X.T @ E @ Vinv_X)
            dll += float(np.trace(sla.cho_solve((cA, True), dA)))
        out["dll"] = -0.5 * dll
    return out


def feasible(lam_min, h, eps_spd=1e-10):
    """Reading E3 / A7: V(h) = h Phi + (1-h) I is accepted iff its smallest eigenvalue exceeds eps_spd."""
    return h * lam_min + (1.0 - h) > eps_spd


def estimate_trait(Phi, XL, y, method=ML, grid=GRID, iters=BISECT_ITERS, eps_spd=1e-10, lam_min=None, grid_ll=None):
    """Reading E3 for one trait.  Returns dict(h2, sigma2, ll, g_star, grid_ll).

    lam_min: smallest eigenvalue of Phi (numpy eigvalsh if None) -- used only for the feasibility rule.
    grid_ll: precomputed grid log-likelihoods (for callers that share them); computed here if None."""
    if lam_min is None:
        lam_min = float(np.linalg.eigvalsh(np.asarray(Phi, dtype=np.float64))[0])
    hs = np.arange(grid + 1, dtype=np.float64) / grid
    ok = np.array([feasible(lam_min, h, eps_spd) for h in hs])
    if grid_ll is None:
        grid_ll = np.full(grid + 1, -np.inf)
        for g in range(grid + 1):
            if ok[g]:
                grid_ll[g] = profile_loglik(Phi, XL, y, hs[g], method)["ll"]
    gs = int(np.argmax(grid_ll))  # first maximum
    if not np.isfinite(grid_ll[gs]):
        raise ValueError("no feasible grid point")
    d0 = profile_loglik(Phi, XL, y, hs[gs], method, with_derivative=True)["dll"]
    lo = hi = None
    if d0 > 0 and gs + 1 <= grid and ok[gs + 1]:
        lo, hi = hs[gs], hs[gs + 1]
    elif d0 < 0 and gs > 0:
        lo, hi = hs[gs - 1], hs[gs]
    if lo is None:
        h = hs[gs]
    else:
        for _ in range(iters):
            mid = 0.5 * (lo + hi)
            if profile_loglik(Phi, XL, y, mid, method, with_derivative=True)["dll"] > 0:
                lo = mid
            else:
                hi = mid
        h = 0.5 * (lo + hi)
    fin = profile_loglik(Phi, XL, y, h, method)
    return {"h2": float(h), "sigma2": float(fin["sigma2"]), "ll": fin["ll"], "g_star": gs, "grid_ll": grid_ll}


def estimate(Phi, XL, Y, method=ML, traits=None, grid=GRID, iters=BISECT_ITERS, eps_spd=1e-10):
    """estimate_trait for each trait column of Y (n, t) (or the selected `traits`).
    Returns dict(h2 (nt,), sigma2 (nt,), ll (nt,), g_star (nt,), traits)."""
    Y = np.asarray(Y, dtype=np.float64).reshape(np.shape(Y)[0], -1)
    traits = np.arange(Y.shape[1]) if traits is None else np.asarray(traits)
    lam_min = float(np.linalg.eigvalsh(np.asarray(Phi, dtype=np.float64))[0])
    res = [estimate_trait(Phi, XL, Y[:, j], method, grid, iters, eps_spd, lam_min) for j in traits]
    return {k: np.array([r[k] for r in res]) for k in ("h2", "sigma2", "ll", "g_star")} | {"traits": traits}
