// Setup kernels for gwas_setup (Alg. 4 lines 6-11, batched over all traits).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gw {

// Alg. 4 lines 6, 8, 9 folded into one operand.  d_j[k] = 1/(s2_j (h2_j w_k + 1 - h2_j))
// (D of line 6; K K^T = D of line 7 is never formed: K^T x . K^T y = x^T D y).  Row `col` of B2 (K = Kpad
// contiguous doubles) is
//   col = f t + j, f < p :  d_j * X_L'[:, f]          col = p t + j :  d_j * y'_j
//   t(p+1) <= col < nsq  :  0 (alignment pad)         col = nsq + j :  d_j   (used with A∘A in K2)
// Entries k >= n are written as 0.  A non-positive / tiny denominator (reading A7) records the smallest
// offending (j, k) as j * n + k in *err (initialised to ~0ull).
__global__ void build_b2(const double* __restrict__ XLp, const double* __restrict__ Yp, const double* __restrict__ W,
                         const double* __restrict__ h2, const double* __restrict__ s2, int n, int p, int t, int kpad,
                         int nsq, int n2, double eps_spd, double* __restrict__ B2, unsigned long long* err) {
  for (int col = blockIdx.y; col < n2; col += gridDim.y) {  // grid-stride in y: n2 = t (p + 2) may exceed 65535
  int j = -1, f = -1;
  if (col < t * (p + 1)) {
    f = col / t;
    j = col - f * t;
  } else if (col >= nsq) {
    j = col - nsq;
  }
  double* out = B2 + (long long)col * kpad;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < kpad; k += gridDim.x * blockDim.x) {
    double val = 0.0;
    if (j >= 0 && k < n) {
      const double hj = h2[j], sj = s2[j];
      const double den = sj * (hj * W[k] + (1.0 - hj));
      if (!(den > eps_spd)) {
        atomicMin(err, (unsigned long long)j * (unsigned long long)n + (unsigned long long)k);
      }
      const double d = 1.0 / den;
      if (f < 0) val = d;
      else if (f < p) val = d * XLp[(long long)f * kpad + k];
      else val = d * Yp[(long long)j * kpad + k];
    }
    out[k] = val;
  }
  }
}

// Alg. 4 lines 10-11 finished per trait: S_TL_j[f][l] = STL[f][l t + j], b_T_j[f] = STL[f][p t + j]
// (both produced by K2 with A = X_L'^T).  Cholesky S_TL_j = L L^T (lower triangle of S_TL read), v = L^-1 b_T,
// and for the full output mode betaT = S_TL^-1 b_T = L^-T v and dinv = diag(S_TL^-1) = column sums of L^-1 squared.
// A pivot <= eps_rel * S_kk (X_L rank-deficient, reading A6) records the smallest such j in *err.
template <int PMAX>
__global__ void trait_factor(const double* __restrict__ STL, long long lds, int p, int t, double eps_rel,
                             double* __restrict__ Lpk, double* __restrict__ v, double* __restrict__ betaT,
                             double* __restrict__ dinv, unsigned long long* err) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= t) return;
  double L[PMAX][PMAX];
  double bt[PMAX];
  for (int f = 0; f < p; ++f) {
    bt[f] = STL[(long long)f * lds + (long long)p * t + j];
    for (int l = 0; l <= f; ++l) L[f][l] = STL[(long long)f * lds + (long long)l * t + j];
  }
  bool ok = true;
  for (int k = 0; k < p; ++k) {
    const double skk = L[k][k];
    double d = skk;
    for (int l = 0; l < k; ++l) d -= L[k][l] * L[k][l];
    // relative pivot test (reading A6 applied to X_L): a column of X_L' numerically in the span of the others
    if (!(d > eps_rel * skk) || !isfinite(d)) { ok = false; d = 1.0; }
    const double rkk = sqrt(d);
    L[k][k] = rkk;
    for (int i = k + 1; i < p; ++i) {
      double s = L[i][k];
      for (int l = 0; l < k; ++l) s -= L[i][l] * L[k][l];
      L[i][k] = s / rkk;
    }
  }
  if (!ok) atomicMin(err, (unsigned long long)j);
  double vv[PMAX];
  for (int f = 0; f < p; ++f) {
    double s = bt[f];
    for (int l = 0; l < f; ++l) s -= L[f][l] * vv[l];
    vv[f] = s / L[f][f];
    v[(long long)f * t + j] = vv[f];
    for (int l = 0; l <= f; ++l) Lpk[(long long)(f * (f + 1) / 2 + l) * t + j] = L[f][l];
  }
  // betaT = L^-T v
  double bb[PMAX];
  for (int f = p - 1; f >= 0; --f) {
    double s = vv[f];
    for (int l = f + 1; l < p; ++l) s -= L[l][f] * bb[l];
    bb[f] = s / L[f][f];
    betaT[(long long)f * t + j] = bb[f];
  }
  // dinv[f] = sum_k (L^-1)_{k f}^2 ; column f of L^-1 by forward substitution on e_f
  for (int f = 0; f < p; ++f) {
    double x[PMAX];
    double acc = 0.0;
    for (int k = 0; k < p; ++k) {
      double s = (k == f) ? 1.0 : 0.0;
      for (int l = 0; l < k; ++l) s -= L[k][l] * x[l];
      x[k] = (k < f) ? 0.0 : s / L[k][k];
      acc += x[k] * x[k];
    }
    dinv[(long long)f * t + j] = acc;
  }
}

// Column-major n x c (ld = ld_src) -> row-per-column layout with leading dimension kpad, zero padding.
__global__ void pad_columns(const double* __restrict__ src, long long ld_src, int n, int c, int kpad,
                            double* __restrict__ dst) {
  for (int col = blockIdx.y; col < c; col += gridDim.y)
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < kpad; k += gridDim.x * blockDim.x)
      dst[(long long)col * kpad + k] = (k < n) ? src[(long long)col * ld_src + k] : 0.0;
}

}  // namespace gw

namespace gw {

// Low-rank trait weights (reading L1): with D = U S V^T (cusolver gesvd, U n x t, ld ldu) truncated to r
// columns, the K2 operand becomes (rows of kpad doubles, K-contiguous; entries k >= n are 0)
//   row f r + rr (f < p) :  U[:, rr] * X_L'[:, f]          row p r + j :  B2_old row p t + j  (= d_j * y'_j)
//   rows p r + t .. nsq_lr - 1 : 0                          row nsq_lr + rr :  U[:, rr]        (used with A∘A)
// written to `out` (not in place: the y rows move up).
// U(k, rr) = U[k su_k + rr su_r] (column-major U of D, or the transposed VT of D^T when t > n).
__global__ void build_lowrank_b2(const double* __restrict__ U, long long su_k, long long su_r,
                                 const double* __restrict__ XLp, const double* __restrict__ B2, int n, int p, int t,
                                 int kpad, int r, int nsq_lr, double* __restrict__ out) {
  for (int row = blockIdx.y; row < nsq_lr + r; row += gridDim.y) {
  double* o = out + (long long)row * kpad;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < kpad; k += gridDim.x * blockDim.x) {
    double v = 0.0;
    if (k < n) {
      if (row < p * r) {
        const int f = row / r, rr = row - f * r;
        v = U[(long long)k * su_k + (long long)rr * su_r] * XLp[(long long)f * kpad + k];
      } else if (row < p * r + t) {
        v = B2[(long long)(p * t + (row - p * r)) * kpad + k];
      } else if (row >= nsq_lr) {
        v = U[(long long)k * su_k + (long long)(row - nsq_lr) * su_r];
      }
    }
    o[k] = v;
  }
  }
}

// W^T (t x r, row j = the trait's r mixing weights): Wt[j][rr] = S[rr] V(j, rr), V(j, rr) = V[j sv_j + rr sv_r].
__global__ void build_lowrank_wt(const double* __restrict__ S, const double* __restrict__ V, long long sv_j,
                                 long long sv_r, int t, int r, double* __restrict__ Wt) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= t * r) return;
  const int j = idx / r, rr = idx - j * r;
  Wt[idx] = S[rr] * V[(long long)j * sv_j + (long long)rr * sv_r];
}

// dst (rows x cols, column-major, ld ldd) = the rows x cols matrix stored row-major in src (row stride lds).
__global__ void rows_to_colmajor(const double* __restrict__ src, long long lds, int rows, int cols,
                                 double* __restrict__ dst, long long ldd) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)rows * cols) return;
  const int r = (int)(idx % rows), c = (int)(idx / rows);
  dst[(long long)c * ldd + r] = src[(long long)r * lds + c];
}

}  // namespace gw
