// K3: batched bordered solve by Schur complement (Alg. 4 lines 14-16).
//
// For pair (i, j) the normal equations of X_i = [X_L | g_i] in the M_j^-1 inner product are the bordered
// system
//        [ S_TL_j   a_ij ] [b_L]   [ b_T_j ]        a_ij = X_L'^T D_j x_i'     (p values, C[i, f t + j])
//        [ a_ij^T   c_ij ] [b_g] = [ r_ij  ]        c_ij = x_i'^T D_j x_i'     (C[i, nsq + j])
//                                                   r_ij = x_i'^T D_j y_j'     (C[i, p t + j])
// With S_TL_j = L_j L_j^T and v_j = L_j^-1 b_T_j precomputed in setup:
//        u = L_j^-1 a,  sigma = c - u.u  (Schur complement = last squared Cholesky pivot of S),
//        b_g = (r - u.v_j) / sigma,  Var_gg = 1 / sigma                        (textbook Var, reading A1)
//   full output mode adds q = L_j^-T u,  b_L = S_TL_j^-1 b_T_j - q b_g,  diag Var_L = diag(S_TL_j^-1) + q^2/sigma.
// Collinear SNP (reading A6): sigma <= eps * c -> status 1, NaN payload; non-finite -> status 2.
// HBM-bound: 8(p+2) bytes in, 17 (SNP mode) bytes out per pair.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gw {

struct SchurArgs {
  const double* C;    // cols x ldc (row i = SNP i of the block)
  long long ldc;
  const double* Cy;   // r_ij = Cy[i * ldcy + j] (= C + p t, ldc, unless the low-rank path keeps the y field apart)
  long long ldcy;
  int nsq;            // column offset of the c_ij block
  int cols, t;
  const double* Lpk;  // [e][j], e = f(f+1)/2 + l (packed lower L_TL_j, row-major)
  const double* v;    // [f][j]
  const double* s2;   // [j]
  const double* betaT;  // [f][j] = S_TL_j^-1 b_T_j  (full mode)
  const double* dinv;   // [f][j] = diag(S_TL_j^-1) (full mode)
  double eps_collinear;
  int literal;        // var_convention 1: Var *= sigma2_j
  int full;           // output mode
  int tj;             // threads per block along traits (power of two <= 128); the rest of the block spans SNPs
  int ich;            // SNPs per thread (SCHUR_ICH when t >= 32; 1 for few traits, so a warp reads consecutive rows)
  double* b;
  double* var;
  int8_t* status;
};

constexpr int SCHUR_ICH = 16;  // SNPs per thread: the trait's factors are loaded once per 16 pairs

// One thread per (trait j, chunk of SCHUR_ICH SNPs); with t >= 32 a warp covers 32 consecutive traits, so the C
// reads and the output writes are coalesced, and the per-trait L_TL_j, v_j stay in registers across the chunk.
template <int P>
__global__ void __launch_bounds__(128) schur_solve(SchurArgs s) {
  const int j = blockIdx.x * s.tj + (int)(threadIdx.x % (unsigned)s.tj);
  const int ii = (int)(threadIdx.x / (unsigned)s.tj);
  if (j >= s.t) return;
  const int t = s.t;
  double L[P * (P + 1) / 2], Linv_d[P], v[P];
#pragma unroll
  for (int e = 0; e < P * (P + 1) / 2; ++e) L[e] = __ldg(s.Lpk + (long long)e * t + j);
#pragma unroll
  for (int f = 0; f < P; ++f) {
    Linv_d[f] = 1.0 / L[f * (f + 1) / 2 + f];
    v[f] = __ldg(s.v + (long long)f * t + j);
  }
  const double scale = s.literal ? __ldg(s.s2 + j) : 1.0;
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  const int i0 = (blockIdx.y * (blockDim.x / s.tj) + ii) * s.ich;
  const int i1 = min(s.cols, i0 + s.ich);
  // the P + 2 inputs of the next pair are loaded while the current one is solved (memory-level parallelism:
  // the kernel is HBM-bound, each thread walks its SNP chunk sequentially)
  double nxt[P + 2];
  auto load = [&](int i, double (&x)[P + 2]) {
    const double* row = s.C + (long long)i * s.ldc;
#pragma unroll
    for (int f = 0; f < P; ++f) x[f] = __ldg(row + f * t + j);
    x[P] = __ldg(s.Cy + (long long)i * s.ldcy + j);
    x[P + 1] = __ldg(row + s.nsq + j);
  };
  if (i0 < i1) load(i0, nxt);
  for (int i = i0; i < i1; ++i) {
    double cur[P + 2];
#pragma unroll
    for (int f = 0; f < P + 2; ++f) cur[f] = nxt[f];
    if (i + 1 < i1) load(i + 1, nxt);
    const long long idx = (long long)i * t + j;
    double u[P];
    double uv = 0.0, uu = 0.0;
#pragma unroll
    for (int f = 0; f < P; ++f) {
      double acc = cur[f];
#pragma unroll
      for (int l = 0; l < f; ++l) acc -= L[f * (f + 1) / 2 + l] * u[l];
      u[f] = acc * Linv_d[f];
      uu += u[f] * u[f];
      uv += u[f] * v[f];
    }
    const double r = cur[P];
    const double c = cur[P + 1];
    const double sigma = c - uu;
    int8_t st = 0;
    if (!(isfinite(sigma) && isfinite(c) && isfinite(r) && isfinite(uv))) st = 2;
    else if (!(sigma > s.eps_collinear * c)) st = 1;
    double bg = nan, vg = nan;
    if (st == 0) {
      const double rs = 1.0 / sigma;
      bg = (r - uv) * rs;
      vg = scale * rs;
      if (!(isfinite(bg) && isfinite(vg))) { st = 2; bg = vg = nan; }
    }
    s.status[idx] = st;
    if (!s.full) {
      s.b[idx] = bg;
      s.var[idx] = vg;
      continue;
    }
    // full mode: q = L^-T u (back substitution), then the X_L coefficients
    double q[P];
#pragma unroll
    for (int f = P - 1; f >= 0; --f) {
      double acc = u[f];
#pragma unroll
      for (int l = f + 1; l < P; ++l) acc -= L[l * (l + 1) / 2 + f] * q[l];
      q[f] = acc * Linv_d[f];
    }
    double* bo = s.b + idx * (P + 1);
    double* vo = s.var + idx * (P + 1);
#pragma unroll
    for (int f = 0; f < P; ++f) {
      if (st == 0) {
        bo[f] = __ldg(s.betaT + (long long)f * t + j) - q[f] * bg;
        vo[f] = scale * (__ldg(s.dinv + (long long)f * t + j) + q[f] * q[f] / sigma);
      } else {
        bo[f] = nan;
        vo[f] = nan;
      }
    }
    bo[P] = bg;
    vo[P] = vg;
  }
}

}  // namespace gw
