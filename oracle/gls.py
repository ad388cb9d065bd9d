"""CPU fp64 ORACLE for the 2-D sequence of GLS problems (PAPER.md Eq. probDef).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this module.  It shares no code with the CUDA path
(paper_1207_2169_b200/) and never imports it; the two meet only in the seeded generators of `datagen/`.

What it computes, for every SNP i and trait j, with X_i = [X_L | g_i] (n x w, w = p + 1):

    M_j      = sigma2_j (h2_j Phi + (1 - h2_j) I)
    b_ij     = (X_i^T M_j^-1 X_i)^-1 X_i^T M_j^-1 y_j                        (Eq. GLS)
    Var_ij   = (X_i^T M_j^-1 X_i)^-1                       var_convention=0 (reading A1)
             = sigma2_j (X_i^T M_j^-1 X_i)^-1              var_convention=1 (P:22/P:31 as printed)

CLAK-Eig (Alg. 4) reaches exactly this result ("by orthogonality of Z"), so the oracle
is the definition, evaluated by the paper's own per-problem procedure, CLAK-Chol for a single GLS
(Alg. 1; Table 1 "Naive" row P:193):

    1  M := sigma2 (h2 Phi + (1-h2) I)
    2  L L^T = M                                P:67   (textbook Cholesky; LAPACK dpotrf as the primitive)
    3  X := L^-1 X                              P:68   (forward substitution; LAPACK dtrtrs as the primitive)
    4  y := L^-1 y
    5  S := X^T X
    6  b := X^T y
    7  b := S^-1 b                              P:72   (w x w Cholesky S = R R^T, two substitutions)

Steps 1-4 depend on (i, j) only through j and through the column g_i of X: `gls_sequence` therefore runs
steps 1-2 once per trait and step 3 once per needed column -- the same numbers the per-pair loop would
produce, column by column.  Both entry points run the same primitives on the same shapes (the substitution
always has the X_L columns plus >= 1 SNP column as right-hand sides; lines 5-7 on a stack), so the trait-cached
sequence is bitwise equal to the literal per-pair Alg. 1 (test_oracle.py asserts it).  Nothing is blocked,
fused or reordered beyond that; no eigendecomposition appears anywhere in the oracle.

Collinearity (reading A6): in step 7 the last pivot R_ww^2 of S equals the Schur complement of the SNP
column; if R_ww^2 <= eps_collinear * S_ww the pair gets status 1 and NaN payload (the paper is silent).
The same relative test on an earlier pivot (R_kk^2 <= eps_collinear * S_kk, k < w-1) means X_L itself is
rank-deficient -> ValueError (the GPU path's GWAS_E_NOT_SPD).

Pins: tests/test_oracle.py (P1-P10, P12 of SURVEY.md §8(c)).  No function here is
"parity unpinned".
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

STATUS_OK = 0
STATUS_COLLINEAR = 1
STATUS_NONFINITE = 2


def assemble_covariance(Phi: np.ndarray, sigma2: float, h2: float) -> np.ndarray:
    """Alg. 1 line 1: M = sigma2 * (h2 * Phi + (1 - h2) * I); both triangles from one expression."""
    n = Phi.shape[0]
    M = sigma2 * (h2 * np.asarray(Phi, dtype=np.float64) + (1.0 - h2) * np.eye(n))
    return 0.5 * (M + M.T)


def cholesky_lower(A: np.ndarray) -> np.ndarray:
    """Alg. 1 line 2: L L^T = A, L lower triangular.  Raises ValueError if A is not SPD."""
    try:
        return sla.cholesky(A, lower=True, check_finite=True)
    except np.linalg.LinAlgError as exc:  # non-positive pivot
        raise ValueError(f"matrix not symmetric positive definite: {exc}") from exc


def forward_substitute(L: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Alg. 1 lines 3-4: X := L^-1 X column by column (lower-triangular solve)."""
    return sla.solve_triangular(L, B, lower=True, trans=0, check_finite=True)


def small_cholesky(S: np.ndarray):
    """Textbook (unblocked, left-looking) Cholesky S = R R^T for a stack of w x w SPD matrices, S: (..., w, w).

    Returns (R, pivots) where pivots[..., k] = S_kk - sum_{l<k} R_kl^2 (the squared diagonal R_kk^2 before the
    square root).  Non-positive pivots are left in `pivots`; R's entries from such a column on are NaN."""
    S = np.asarray(S, dtype=np.float64)
    w = S.shape[-1]
    R = np.zeros_like(S)
    piv = np.zeros(S.shape[:-1], dtype=np.float64)
    for k in range(w):
        d = S[..., k, k] - np.sum(R[..., k, :k] * R[..., k, :k], axis=-1)
        piv[..., k] = d
        with np.errstate(invalid="ignore", divide="ignore"):
            rkk = np.where(d > 0, np.sqrt(np.where(d > 0, d, 1.0)), np.nan)
            R[..., k, k] = rkk
            for i in range(k + 1, w):
                R[..., i, k] = (S[..., i, k] - np.sum(R[..., i, :k] * R[..., k, :k], axis=-1)) / rkk
    return R, piv


def small_spd_solve(R: np.ndarray, rhs: np.ndarray) -> np.ndarray:
    """Alg. 1 line 7: x = S^-1 rhs with S = R R^T: forward (R z = rhs) then backward (R^T x = z).
    R: (..., w, w) lower, rhs: (..., w) or (..., w, q)."""
    vec = rhs.ndim == R.ndim - 1
    B = rhs[..., None] if vec else rhs
    w = R.shape[-1]
    z = np.zeros(B.shape, dtype=np.float64)
    for k in range(w):
        z[..., k, :] = (B[..., k, :] - np.einsum("...l,...lq->...q", R[..., k, :k], z[..., :k, :])) / R[..., k, k, None]
    x = np.zeros_like(z)
    for k in range(w - 1, -1, -1):
        x[..., k, :] = (z[..., k, :] - np.einsum("...l,...lq->...q", R[..., k + 1:, k], x[..., k + 1:, :])) / R[..., k, k, None]
    return x[..., 0] if vec else x


def normal_equations(Xw: np.ndarray, yw: np.ndarray):
    """Alg. 1 lines 5-6 on a stack of whitened designs Xw (k, n, w) and one whitened y (n,):
    S = X^T X (k, w, w), r = X^T y (k, w).  Each entry is the same dot product whatever k is."""
    Xw = np.ascontiguousarray(Xw)   # one memory layout, so one summation order, whatever the caller passed
    yw = np.ascontiguousarray(yw)
    S = np.einsum("kna,knb->kab", Xw, Xw)
    r = np.einsum("kna,n->ka", Xw, yw)
    return S, r


def _finish(S, r, sigma2, eps_collinear, var_convention):
    """Steps 7 (+Var) on a stack of normal equations S (..., w, w), r (..., w).
    Returns b (..., w), Var (..., w, w), status (...)."""
    w = S.shape[-1]
    R, piv = small_cholesky(S)
    diag = np.diagonal(S, axis1=-2, axis2=-1)
    if np.any(~(piv[..., : w - 1] > eps_collinear * diag[..., : w - 1])):
        raise ValueError("S_TL not SPD: X_L is rank-deficient for some trait")
    last = piv[..., w - 1]
    collinear = ~(last > eps_collinear * S[..., w - 1, w - 1])
    Rs = np.where(collinear[..., None, None], np.eye(w), R)  # keep arithmetic finite on flagged pairs
    b = small_spd_solve(Rs, r)
    Var = small_spd_solve(Rs, np.broadcast_to(np.eye(w), S.shape).copy())
    if var_convention == 1:
        Var = Var * np.asarray(sigma2)[..., None, None]
    status = np.where(collinear, STATUS_COLLINEAR, STATUS_OK)
    finite = np.isfinite(b).all(axis=-1) & np.isfinite(Var).all(axis=(-2, -1))
    status = np.where((status == STATUS_OK) & ~finite, STATUS_NONFINITE, status)
    bad = status != STATUS_OK
    b = np.where(bad[..., None], np.nan, b)
    Var = np.where(bad[..., None, None], np.nan, Var)
    return b, Var, status.astype(np.int8)


def gls_single(Phi, X, y, sigma2, h2, var_convention=0, eps_collinear=1e-10):
    """One GLS problem by Alg. 1.  X: (n, w) with the SNP (if any) in the last column.
    Returns (b (w,), Var (w, w), status)."""
    X = np.asarray(X, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    M = assemble_covariance(Phi, sigma2, h2)          # line 1
    L = cholesky_lower(M)                              # line 2
    Xw = forward_substitute(L, X)                      # line 3
    yw = forward_substitute(L, y)                      # line 4
    S, r = normal_equations(Xw[None], yw)              # lines 5-6
    b, Var, st = _finish(S, r, np.array([sigma2], dtype=np.float64), eps_collinear, var_convention)  # line 7
    return b[0], Var[0], int(st[0])


def gls_sequence(Phi, XL, XR, Y, h2, sigma2, snps=None, traits=None, var_convention=0,
                 eps_collinear=1e-10, snp_chunk=4096):
    """The 2-D sequence (Eq. probDef) over SNP columns `snps` of XR (n, m) and traits `traits`.

    XR may also be given as the already-selected columns (n, len(snps)) with snps=None.
    Returns dict with b (ns, nt, w), Var (ns, nt, w, w), status (ns, nt) int8 -- indexed [i][j] in the
    order of `snps` / `traits`.  Per trait: Alg. 1 lines 1-2 once, line 3 per column (see module doc)."""
    Phi = np.asarray(Phi, dtype=np.float64)
    XL = np.asarray(XL, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    n, p = XL.shape
    w = p + 1
    G = np.asarray(XR) if snps is None else np.asarray(XR)[:, np.asarray(snps)]
    ns = G.shape[1]
    traits = np.arange(Y.shape[1]) if traits is None else np.asarray(traits)
    nt = traits.size
    b = np.empty((ns, nt, w))
    Var = np.empty((ns, nt, w, w))
    status = np.empty((ns, nt), dtype=np.int8)
    snp_chunk = max(1, min(snp_chunk, int(5e7 // (n * w))))
    for jj, j in enumerate(traits):
        M = assemble_covariance(Phi, float(sigma2[j]), float(h2[j]))     # line 1
        L = cholesky_lower(M)                                           # line 2
        yw = forward_substitute(L, Y[:, j])                             # line 4
        for c0 in range(0, ns, snp_chunk):
            c1 = min(ns, c0 + snp_chunk)
            # line 3 on [X_L | g_c0 .. g_c1-1]: the X_L part of every X_i and the SNP columns in one substitution
            # (>= 2 right-hand sides, like gls_single's [X_L | g_i]: every column takes the same arithmetic path)
            Xc = forward_substitute(L, np.column_stack([XL, G[:, c0:c1].astype(np.float64)]))
            k = c1 - c0
            Xw = np.empty((k, n, w))                                    # X_i := L^-1 X_i for each i
            Xw[:, :, :p] = Xc[None, :, :p]
            Xw[:, :, p] = Xc[:, p:].T
            S, r = normal_equations(Xw, yw)                             # lines 5-6
            bb, VV, st = _finish(S, r, np.full(k, float(sigma2[j])), eps_collinear, var_convention)  # line 7
            b[c0:c1, jj] = bb
            Var[c0:c1, jj] = VV
            status[c0:c1, jj] = st
    return {"b": b, "Var": Var, "status": status, "traits": traits}
