// Variance-component estimation in the eigenbasis (the paper's "first step"; SURVEY.md
// §8(f) NEXT-3; readings E1-E4).  For every trait j the reduced model y_j = X_L beta + R,
// R ~ N(0, sigma2 V(h)), V(h) = h Phi + (1 - h) I, is fitted by ML or REML with beta and sigma2 profiled out.
// After Alg. 4 lines 1, 2, 4 (Phi = Z W Z^T, X_L' = Z^T X_L, y'_j = Z^T y_j) every quantity is a weighted sum
// over the eigen-index k with v_k = h w_k + 1 - h ("eigen-based" estimation, Table 1, cost v n p^2):
//   log|V| = sum_k log v_k,  A = X_L'^T diag(1/v) X_L',  c = X_L'^T diag(1/v) y',  R = sum_k r_k^2 / v_k
//   (r = y' - X_L' beta^),  dR/dh = -sum_k r_k^2 (w_k - 1)/v_k^2,  tr(V^-1 dV/dh) = sum_k (w_k - 1)/v_k,
//   dA/dh = -X_L'^T diag((w_k - 1)/v_k^2) X_L'.
// Optimiser (reading E3): grid h_g = g/G, g = 0..G, first argmax, then BISECT_ITERS bisection steps on the sign
// of the derivative in the neighbouring grid interval.
//
// Kernels:
//   est_grid_shared  one CTA per grid point g: the trait-independent log|V_g|, A_g (packed lower) and feasibility
//   est_traits       one CTA per trait: grid likelihoods, argmax, bisection, final (h2^, sigma2^, l)
// All reductions run in a fixed order (per-thread strided partial sums, fixed shuffle tree, warps summed in
// order), so results are bitwise reproducible run to run.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace gw {

constexpr int EST_GRID = 100;        // G of reading E3
constexpr int EST_ITERS = 50;        // bisection steps of reading E3
constexpr int EST_THREADS = 256;
constexpr int EST_NG = 4;            // grid points per pass in est_traits
constexpr double EST_R_REL_MIN = 1e-24;  // reading E1: R <= 1e-24 y'^T V^-1 y' means y in span(X_L) -> error

// per-grid-point record written by est_grid_shared: [0] feasible (1/0), [1] log|V_g|, [2..] A_g packed lower
__host__ __device__ constexpr int est_rec(int p) { return 2 + p * (p + 1) / 2; }

// Block-wide sum of NV per-thread values, fixed order; result valid in thread 0 (returned in `val` there).
template <int NV>
__device__ __forceinline__ void block_sum(double (&val)[NV], double* scratch /* [EST_THREADS/32][NV] */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double x = val[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    val[i] = x;
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) scratch[warp * NV + i] = val[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double s = scratch[i];
      for (int w = 1; w < EST_THREADS / 32; ++w) s += scratch[w * NV + i];
      val[i] = s;
    }
  }
  __syncthreads();
}

// In-register Cholesky of a packed-lower P x P matrix (row-major packed: (f, l) at f(f+1)/2 + l).  Returns false if
// a pivot is not > 0.  logdet receives log|A| = 2 sum log L_ff.
template <int P>
__device__ bool est_chol(const double* Apk, double (&L)[P][P], double* logdet) {
  double ld = 0.0;
  for (int k = 0; k < P; ++k) {
    double d = Apk[k * (k + 1) / 2 + k];
    for (int l = 0; l < k; ++l) d -= L[k][l] * L[k][l];
    if (!(d > 0.0)) return false;
    const double r = sqrt(d);
    L[k][k] = r;
    ld += log(r);
    for (int i = k + 1; i < P; ++i) {
      double s = Apk[i * (i + 1) / 2 + k];
      for (int l = 0; l < k; ++l) s -= L[i][l] * L[k][l];
      L[i][k] = s / r;
    }
  }
  *logdet = 2.0 * ld;
  return true;
}

// x = A^-1 b with A = L L^T
template <int P>
__device__ void est_solve(const double (&L)[P][P], const double* b, double* x) {
  double z[P];
  for (int f = 0; f < P; ++f) {
    double s = b[f];
    for (int l = 0; l < f; ++l) s -= L[f][l] * z[l];
    z[f] = s / L[f][f];
  }
  for (int f = P - 1; f >= 0; --f) {
    double s = z[f];
    for (int l = f + 1; l < P; ++l) s -= L[l][f] * x[l];
    x[f] = s / L[f][f];
  }
}

// One CTA per grid point g = blockIdx.x: feasibility (all v_k > eps_spd, reading E3/A7), log|V_g|, A_g.
// W: eigenvalues (n used), XLp: p rows of kpad doubles (row f = column f of X_L' = Z^T X_L).
template <int P>
__global__ void __launch_bounds__(EST_THREADS) est_grid_shared(const double* __restrict__ W,
                                                               const double* __restrict__ XLp, int n, int kpad,
                                                               double eps_spd, double* __restrict__ rec) {
  constexpr int NA = P * (P + 1) / 2;
  __shared__ double scratch[(EST_THREADS / 32) * (NA + 2)];
  const int g = blockIdx.x;
  const double h = (double)g / (double)EST_GRID;
  double acc[NA + 2];
#pragma unroll
  for (int i = 0; i < NA + 2; ++i) acc[i] = 0.0;
  for (int k = threadIdx.x; k < n; k += EST_THREADS) {
    const double v = h * W[k] + (1.0 - h);
    if (!(v > eps_spd)) acc[0] += 1.0;  // count of infeasible k
    const double u = 1.0 / v;
    acc[1] += log(v);
    double x[P];
#pragma unroll
    for (int f = 0; f < P; ++f) x[f] = XLp[(long long)f * kpad + k];
#pragma unroll
    for (int f = 0; f < P; ++f)
#pragma unroll
      for (int l = 0; l <= f; ++l) acc[2 + f * (f + 1) / 2 + l] += u * x[f] * x[l];
  }
  block_sum<NA + 2>(acc, scratch);
  if (threadIdx.x == 0) {
    double* r = rec + (long long)g * est_rec(P);
    r[0] = acc[0] == 0.0 ? 1.0 : 0.0;
    for (int i = 1; i < NA + 2; ++i) r[i] = acc[i];
  }
}

struct EstOut {
  double* h2;      // [t]
  double* s2;      // [t]
  double* ll;      // [t]
  int* gstar;      // [t] grid argmax (diagnostics)
  unsigned long long* err;  // smallest failing trait (R <= 0, no feasible grid point), init ~0ull
};

// One CTA per trait j = blockIdx.x (two resident per SM: 128 registers, measured 19.9 -> 12.0 ms at C4; three
// spill too much).  method 0 = ML, 1 = REML.  rec: est_grid_shared output.  logdet_xx:
// log|X_L'^T X_L'| (REML constant; equals log|A_0| since v = 1 at h = 0).
template <int P>
__global__ void __launch_bounds__(EST_THREADS, 2) est_traits(const double* __restrict__ W,
                                                          const double* __restrict__ XLp,
                                                          const double* __restrict__ Yp, int n, int kpad, int t,
                                                          int method, const double* __restrict__ rec, EstOut out) {
  constexpr int NA = P * (P + 1) / 2;
  constexpr int NV1 = NA + P + NA + 1;  // derivative pass 1: A, c, A' (REML), sum (w-1)/v; slot NV1: sum log v
  constexpr int NSCR = (NV1 + 1) > EST_NG * (P + 1) ? (NV1 + 1) : EST_NG * (P + 1);
  __shared__ double scratch[(EST_THREADS / 32) * NSCR];
  __shared__ double ll_grid[EST_GRID + 1];
  __shared__ double s_beta[P];
  __shared__ double s_h, s_tr, s_lda, s_lo, s_hi;
  __shared__ int s_ctl, s_gs;
  const int j = blockIdx.x;
  const double* y = Yp + (long long)j * kpad;
  const bool reml = method == 1;
  const double nn = reml ? (double)(n - P) : (double)n;
  const double two_pi = 6.283185307179586476925286766559;
  const double* rec0 = rec;  // g = 0 record: A_0 = X_L'^T X_L'
  double logdet_xx = 0.0;
  if (threadIdx.x == 0 && reml) {
    double L0[P][P];
    if (!est_chol<P>(rec0 + 2, L0, &logdet_xx)) logdet_xx = NAN;
  }

  // ---------------- grid phase: c_g, yy_g for EST_NG grid points per pass
  for (int g0 = 0; g0 <= EST_GRID; g0 += EST_NG) {
    double acc[EST_NG * (P + 1)];
#pragma unroll
    for (int i = 0; i < EST_NG * (P + 1); ++i) acc[i] = 0.0;
    double hg[EST_NG];
#pragma unroll
    for (int q = 0; q < EST_NG; ++q) hg[q] = (double)(g0 + q) / (double)EST_GRID;
    for (int k = threadIdx.x; k < n; k += EST_THREADS) {
      const double wk = W[k], yk = y[k];
      double x[P];
#pragma unroll
      for (int f = 0; f < P; ++f) x[f] = XLp[(long long)f * kpad + k];
#pragma unroll
      for (int q = 0; q < EST_NG; ++q) {
        const double u = 1.0 / (hg[q] * wk + (1.0 - hg[q]));
        const double uy = u * yk;
#pragma unroll
        for (int f = 0; f < P; ++f) acc[q * (P + 1) + f] += uy * x[f];
        acc[q * (P + 1) + P] += uy * yk;
      }
    }
    block_sum<EST_NG * (P + 1)>(acc, scratch);
    if (threadIdx.x == 0) {
      for (int q = 0; q < EST_NG && g0 + q <= EST_GRID; ++q) {
        const double* r = rec + (long long)(g0 + q) * est_rec(P);
        double val = -INFINITY;
        double L[P][P], lda;
        if (r[0] != 0.0 && est_chol<P>(r + 2, L, &lda)) {
          // R = yy - c^T A^-1 c = yy - |L^-1 c|^2
          double z2 = 0.0, z[P];
          for (int f = 0; f < P; ++f) {
            double s = acc[q * (P + 1) + f];
            for (int l = 0; l < f; ++l) s -= L[f][l] * z[l];
            z[f] = s / L[f][f];
            z2 += z[f] * z[f];
          }
          const double yy = acc[q * (P + 1) + P];
          const double R = yy - z2;
          if (R > EST_R_REL_MIN * yy) {
            val = reml ? -0.5 * (nn * log(two_pi * R / nn) + r[1] + lda - logdet_xx + nn)
                       : -0.5 * (nn * log(two_pi * R / nn) + r[1] + nn);
          } else {
            atomicMin(out.err, (unsigned long long)j);
          }
        }
        ll_grid[g0 + q] = val;
      }
    }
    __syncthreads();
  }

  // derivative (and, with want_ll, l and sigma2) at h: two passes (A, c, ... then residuals)
  auto eval = [&](double h, bool want_ll, double* dll, double* llv, double* s2v) {
    double a1[NV1 + 1];
#pragma unroll
    for (int i = 0; i < NV1 + 1; ++i) a1[i] = 0.0;
    for (int k = threadIdx.x; k < n; k += EST_THREADS) {
      const double wk = W[k], yk = y[k];
      const double v = h * wk + (1.0 - h);
      const double u = 1.0 / v, e = wk - 1.0;
      const double eu2 = e * u * u;
      double x[P];
#pragma unroll
      for (int f = 0; f < P; ++f) x[f] = XLp[(long long)f * kpad + k];
#pragma unroll
      for (int f = 0; f < P; ++f) {
#pragma unroll
        for (int l = 0; l <= f; ++l) {
          a1[f * (f + 1) / 2 + l] += u * x[f] * x[l];
          if (reml) a1[NA + P + f * (f + 1) / 2 + l] += eu2 * x[f] * x[l];
        }
        a1[NA + f] += u * x[f] * yk;
      }
      a1[NV1 - 1] += e * u;
      if (want_ll) a1[NV1] += log(v);
    }
    block_sum<NV1 + 1>(a1, scratch);
    if (threadIdx.x == 0) {
      double L[P][P], lda = 0.0;
      double beta[P];
      if (!est_chol<P>(a1, L, &lda)) {
        for (int f = 0; f < P; ++f) beta[f] = NAN;
      } else {
        est_solve<P>(L, a1 + NA, beta);
      }
      for (int f = 0; f < P; ++f) s_beta[f] = beta[f];
      double tr = a1[NV1 - 1];
      if (reml) {  // tr(A^-1 A'), A' = -X'^T diag(e u^2) X'
        for (int l = 0; l < P; ++l) {
          double col[P], xs[P];
          for (int f = 0; f < P; ++f) {
            const int a = f > l ? f : l, b = f > l ? l : f;
            col[f] = -a1[NA + P + a * (a + 1) / 2 + b];
          }
          est_solve<P>(L, col, xs);
          tr += xs[l];
        }
      }
      s_tr = tr;
      s_lda = lda;
      scratch[0] = a1[NV1];  // sum log v (valid if want_ll)
    }
    __syncthreads();
    const double logdetV = scratch[0];
    double beta[P];
#pragma unroll
    for (int f = 0; f < P; ++f) beta[f] = s_beta[f];
    __syncthreads();
    double a2[3] = {0.0, 0.0, 0.0};
    for (int k = threadIdx.x; k < n; k += EST_THREADS) {
      const double wk = W[k];
      const double v = h * wk + (1.0 - h);
      const double u = 1.0 / v, e = wk - 1.0;
      const double yk = y[k];
      a2[2] += u * yk * yk;
      double r = yk;
#pragma unroll
      for (int f = 0; f < P; ++f) r -= XLp[(long long)f * kpad + k] * beta[f];
      const double ur2 = u * r * r;
      a2[0] += ur2;
      a2[1] -= e * u * ur2;
    }
    block_sum<3>(a2, scratch);
    if (threadIdx.x == 0) {
      const double R = a2[0], dR = a2[1];
      if (!(R > EST_R_REL_MIN * a2[2])) atomicMin(out.err, (unsigned long long)j);
      *dll = -0.5 * (nn * dR / R + s_tr);
      if (want_ll) {
        *s2v = R / nn;
        *llv = reml ? -0.5 * (nn * log(two_pi * R / nn) + logdetV + s_lda - logdet_xx + nn)
                    : -0.5 * (nn * log(two_pi * R / nn) + logdetV + nn);
      }
    }
  };

  // ---------------- argmax + bracket
  if (threadIdx.x == 0) {
    int gs = 0;
    double best = ll_grid[0];
    for (int g = 1; g <= EST_GRID; ++g)
      if (ll_grid[g] > best) {  // first maximum (NaN never wins)
        best = ll_grid[g];
        gs = g;
      }
    if (!(best > -INFINITY)) atomicMin(out.err, (unsigned long long)j);
    s_gs = gs;
    s_h = (double)gs / (double)EST_GRID;
  }
  __syncthreads();
  const int gs = s_gs;
  double d0 = 0.0, dummy = 0.0;
  eval((double)gs / (double)EST_GRID, false, &d0, &dummy, &dummy);
  if (threadIdx.x == 0) {
    s_ctl = 0;
    const double* rnext = rec + (long long)(gs + 1) * est_rec(P);
    if (d0 > 0.0 && gs + 1 <= EST_GRID && rnext[0] != 0.0) {
      s_lo = (double)gs / (double)EST_GRID;
      s_hi = (double)(gs + 1) / (double)EST_GRID;
      s_ctl = 1;
    } else if (d0 < 0.0 && gs > 0) {
      s_lo = (double)(gs - 1) / (double)EST_GRID;
      s_hi = (double)gs / (double)EST_GRID;
      s_ctl = 1;
    }
  }
  __syncthreads();
  double h = (double)gs / (double)EST_GRID;
  if (s_ctl) {
    for (int it = 0; it < EST_ITERS; ++it) {
      const double mid = 0.5 * (s_lo + s_hi);
      double dm = 0.0;
      eval(mid, false, &dm, &dummy, &dummy);
      if (threadIdx.x == 0) {
        if (dm > 0.0) s_lo = mid;
        else s_hi = mid;
      }
      __syncthreads();
    }
    h = 0.5 * (s_lo + s_hi);
  }
  double dll = 0.0, llv = 0.0, s2v = 0.0;
  eval(h, true, &dll, &llv, &s2v);
  if (threadIdx.x == 0) {
    out.h2[j] = h;
    out.s2[j] = s2v;
    out.ll[j] = llv;
    out.gstar[j] = gs;
  }
}

}  // namespace gw
