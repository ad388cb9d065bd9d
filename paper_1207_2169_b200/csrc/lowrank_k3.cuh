// K3 fused with the low-rank recombination (reading L1; SURVEY.md §8(f) NEXT-2 "K3 into K2's
// epilogue").  With D ~ U_r W the K2' product leaves, per SNP i, the r-vectors G_f[i] = X_R'^T (U_r (.) X_L'_f)
// (f < p), G_sq[i] = (X_R'^2)^T U_r and the exact y-term; the per-pair inputs of the bordered solve are
//     a_f(i, j) = sum_rr G_f[i][rr] W[rr][j]   (f < p),     c(i, j) = sum_rr G_sq[i][rr] W[rr][j],
// i.e. p + 1 small products with K = r.  Instead of writing them to HBM and reading them back in K3, each CTA
// computes a 32-SNP x 32-trait tile of all p + 1 fields on the FP64 tensor pipe (mma.sync m8n8k4 -> DMMA) and runs
// the Schur solve of K3 (schur.cuh) on the accumulators: lane (g, q) of warp w holds SNP 8w + g and traits
// 8 ni + 2q + {0, 1} of every field, so each pair's p + 1 values are already in one thread.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "gemm_dmma.cuh"  // dmma_8x8x4
#include "schur.cuh"

namespace gw {

constexpr int LRK3_ROWS = 32, LRK3_COLS = 32, LRK3_THREADS = 128;  // 4 warps x 8 SNPs x 32 traits

struct LowrankK3Args {
  const double* G;   // K2' output rows (ld ldg): fields f < p at columns f r .., y-term at p r + j, squared at nsq_lr ..
  long long ldg;
  int r, nsq_lr;
  const double* Wt;  // t x r (row j: the trait's r mixing weights)
  SchurArgs k3;      // C / nsq unused; Cy = G + p r (ld ldg); factors, outputs, flags as K3
};

template <int P>
__global__ void __launch_bounds__(LRK3_THREADS) lowrank_schur(LowrankK3Args a) {
  constexpr int NA = P * (P + 1) / 2;
  const SchurArgs& s = a.k3;
  const int t = s.t;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int j0 = blockIdx.x * LRK3_COLS, i0 = blockIdx.y * LRK3_ROWS;
  // the tile's per-trait factors, staged once (the pairs of a lane share 8 traits)
  __shared__ double sL[NA][LRK3_COLS], sLinv[P][LRK3_COLS], sv[P][LRK3_COLS], ss2[LRK3_COLS];
  // full mode needs the X_L-coefficient factors, SNP mode the output staging: never both
  union FullOrSnp {
    struct { double bT[P][LRK3_COLS], dinv[P][LRK3_COLS]; } f;
    struct { double vr[LRK3_THREADS / 32][8][LRK3_COLS]; int8_t st[LRK3_THREADS / 32][8][LRK3_COLS]; } o;
  };
  __shared__ FullOrSnp u_;
  auto& sbT = u_.f.bT;
  auto& sdinv = u_.f.dinv;
  for (int idx = threadIdx.x; idx < LRK3_COLS; idx += LRK3_THREADS) {
    const int j = min(j0 + idx, t - 1);
#pragma unroll
    for (int e = 0; e < NA; ++e) sL[e][idx] = __ldg(s.Lpk + (long long)e * t + j);
#pragma unroll
    for (int f = 0; f < P; ++f) {
      sLinv[f][idx] = 1.0 / __ldg(s.Lpk + (long long)(f * (f + 1) / 2 + f) * t + j);
      sv[f][idx] = __ldg(s.v + (long long)f * t + j);
      if (s.full) {
        sbT[f][idx] = __ldg(s.betaT + (long long)f * t + j);
        sdinv[f][idx] = __ldg(s.dinv + (long long)f * t + j);
      }
    }
    ss2[idx] = s.literal ? __ldg(s.s2 + j) : 1.0;
  }
  __syncthreads();

  // ---- p + 1 products with K = r: acc[f][ni] = rows 8w.. x traits 8ni.. of field f
  const int row = i0 + warp * 8 + g;           // A-fragment row of this lane (and its output SNP)
  const bool row_ok = row < s.cols;
  const double* grow = a.G + (long long)(row_ok ? row : 0) * a.ldg;
  double acc[P + 1][4][2];
#pragma unroll
  for (int f = 0; f <= P; ++f)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) acc[f][ni][0] = acc[f][ni][1] = 0.0;
  for (int k0 = 0; k0 < a.r; k0 += 4) {
    double bw[4];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {  // B fragment: k = q, n = g  ->  W[k0 + q][j0 + 8 ni + g]
      const int j = j0 + ni * 8 + g;
      bw[ni] = j < t ? __ldg(a.Wt + (long long)j * a.r + k0 + q) : 0.0;
    }
#pragma unroll
    for (int f = 0; f <= P; ++f) {   // A fragment: row g, k = q
      const int col = (f < P ? f * a.r : a.nsq_lr) + k0 + q;
      const double av = row_ok ? __ldg(grow + col) : 0.0;
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[f][ni], av, bw[ni]);
    }
  }

  // ---- K3 on the accumulators: lane (g, q) owns SNP row 8 w + g of the tile and traits 8 ni + 2 q + e (C fragment
  // of m8n8k4: lane (g, q) holds C[g][2q], C[g][2q + 1]).  The warp's 8 x 32 (SNP, trait) block of y-terms is read,
  // and in SNP mode its b / Var / status written, row by row through shared memory, so every global access is a
  // coalesced run of 32 consecutive traits instead of 2-element pieces of 8 rows.
  __shared__ double sy[LRK3_THREADS / 32][8][LRK3_COLS];   // y-term in, b out (same positions per lane)
  auto& svr = u_.o.vr;
  auto& sst = u_.o.st;
  const int jlane = j0 + lane;
#pragma unroll
  for (int rr = 0; rr < 8; ++rr) {
    const int ri = i0 + warp * 8 + rr;
    sy[warp][rr][lane] = (ri < s.cols && jlane < t) ? __ldg(s.Cy + (long long)ri * s.ldcy + jlane) : 0.0;
  }
  __syncwarp();
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
#pragma unroll
  for (int ni = 0; ni < 4; ++ni) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int jl = ni * 8 + 2 * q + e, j = j0 + jl;
      if (j >= t || !row_ok) continue;
      const long long idx = (long long)row * t + j;
      double u[P];
      double uv = 0.0, uu = 0.0;
#pragma unroll
      for (int f = 0; f < P; ++f) {
        double acc_u = acc[f][ni][e];
#pragma unroll
        for (int l = 0; l < f; ++l) acc_u -= sL[f * (f + 1) / 2 + l][jl] * u[l];
        u[f] = acc_u * sLinv[f][jl];
        uu += u[f] * u[f];
        uv += u[f] * sv[f][jl];
      }
      const double r = sy[warp][g][jl];
      const double c = acc[P][ni][e];
      const double sigma = c - uu;
      int8_t st = 0;
      if (!(isfinite(sigma) && isfinite(c) && isfinite(r) && isfinite(uv))) st = 2;
      else if (!(sigma > s.eps_collinear * c)) st = 1;
      double bg = nan, vg = nan;
      if (st == 0) {
        const double rs = 1.0 / sigma;
        bg = (r - uv) * rs;
        vg = ss2[jl] * rs;
        if (!(isfinite(bg) && isfinite(vg))) { st = 2; bg = vg = nan; }
      }
      if (!s.full) {
        sy[warp][g][jl] = bg;
        svr[warp][g][jl] = vg;
        sst[warp][g][jl] = st;
        continue;
      }
      s.status[idx] = st;
      double qv[P];
#pragma unroll
      for (int f = P - 1; f >= 0; --f) {
        double acc_q = u[f];
#pragma unroll
        for (int l = f + 1; l < P; ++l) acc_q -= sL[l * (l + 1) / 2 + f][jl] * qv[l];
        qv[f] = acc_q * sLinv[f][jl];
      }
      double* bo = s.b + idx * (P + 1);
      double* vo = s.var + idx * (P + 1);
#pragma unroll
      for (int f = 0; f < P; ++f) {
        bo[f] = st == 0 ? sbT[f][jl] - qv[f] * bg : nan;
        vo[f] = st == 0 ? ss2[jl] * (sdinv[f][jl] + qv[f] * qv[f] / sigma) : nan;
      }
      bo[P] = bg;
      vo[P] = vg;
    }
  }
  if (!s.full) {
    __syncwarp();
#pragma unroll
    for (int rr = 0; rr < 8; ++rr) {
      const int ri = i0 + warp * 8 + rr;
      if (ri < s.cols && jlane < t) {
        const long long idx = (long long)ri * t + jlane;
        s.b[idx] = sy[warp][rr][lane];
        s.var[idx] = svr[warp][rr][lane];
        s.status[idx] = sst[warp][rr][lane];
      }
    }
  }
}

}  // namespace gw
