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

#include "ctile.cuh"

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
  int k3_gy;          // schur_solve_tma: CTAs per trait block (aligned row ranges), 0 = flattened ranges
  int tiled;          // C in the trait-tiled layout written by K2 (TILE_T traits x F fields per chunk, see below)
  int tj;             // threads per block along traits (power of two <= 128); the rest of the block spans SNPs
  int ich;            // SNPs per thread (SCHUR_ICH when t >= 32; 1 for few traits, so a warp reads consecutive rows)
  double* b;
  double* var;
  int8_t* status;
};

__device__ __forceinline__ void mbar_init_cta(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(bar)));
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  }
}

constexpr int SCHUR_ICH = 16;  // SNPs per thread: the trait's factors are loaded once per 16 pairs

template <int P, bool TILED = false>
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
  // field f of pair (i, j) is at C[i * ldc + jo + f * fs] (f < P; the y field too when tiled), r_ij at
  // Cy[i * ldcy + jy], c_ij at C[i * ldc + sqo]
  const long long jo = TILED ? ctile_off(j, 0, P + 2) : j;
  const long long fs = TILED ? CTILE_T : t;
  const double* Cy = TILED ? s.C + jo + (long long)P * CTILE_T : s.Cy + j;
  const long long ldcy = TILED ? s.ldc : s.ldcy;
  const long long sqo = TILED ? jo + (long long)(P + 1) * CTILE_T : (long long)s.nsq + j;
  double nxt[P + 2];
  auto load = [&](int i, double (&x)[P + 2]) {
    const double* row = s.C + (long long)i * s.ldc + jo;
#pragma unroll
    for (int f = 0; f < P; ++f) x[f] = __ldg(row + f * fs);
    x[P] = __ldg(Cy + (long long)i * ldcy);
    x[P + 1] = __ldg(s.C + (long long)i * s.ldc + sqo);
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

// ---------------------------------------------------------------------------------------------------------------
// K3 on the trait-tiled C (ctile.cuh): per row, CTILE_T traits x F fields are one contiguous chunk, so one thread
// streams the chunks of R rows per stage into shared memory with bulk copies (cp.async.bulk: the TMA engine, completion
// counted on an mbarrier) through an ST-deep ring, and the CTA's 128 threads (one per trait, factors in registers) solve
// from shared memory.  Work = tiles (trait block jb, R rows), ordered jb-major and split into equal contiguous ranges,
// one per resident CTA (persistent: exactly the SMs' CTA slots, no wave tail whatever t is); a thread reloads its
// factors when its range crosses into the next trait block.  HBM-bound: 8 F bytes read, 17 (SNP mode) written per pair.
constexpr int SCHUR_TMA_R = 4;   // rows per stage
constexpr int SCHUR_TMA_ST = 3;  // stages (ST - 1 tiles in flight while one is solved): 84 KB at p = 5

template <int P, int R = SCHUR_TMA_R, int ST = SCHUR_TMA_ST>
constexpr size_t schur_tma_smem() {
  return (size_t)ST * R * (P + 2) * CTILE_T * sizeof(double) + 64;
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          (uint32_t)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
      : "memory");
}

template <int P, int R = SCHUR_TMA_R, int ST = SCHUR_TMA_ST>
__global__ void __launch_bounds__(CTILE_T) schur_solve_tma(SchurArgs s) {
  constexpr int F = P + 2;
  constexpr uint32_t kChunk = F * CTILE_T * sizeof(double);
  extern __shared__ __align__(128) double sm[];  // [ST][R][F][CTILE_T], then ST mbarriers
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + ST * R * F * CTILE_T);
  const int tid = threadIdx.x;
  const int t = s.t;
  const int ntr = (s.cols + R - 1) / R;                      // row tiles per trait block
  const int gx = (t + CTILE_T - 1) / CTILE_T;
  long long k0;
  int ntile;
  if (s.k3_gy > 0) {  // aligned: k3_gy CTAs per trait block, the same row ranges for every block (DRAM locality)
    const int jb = blockIdx.x % gx, ry = blockIdx.x / gx;
    const int per_r = (ntr + s.k3_gy - 1) / s.k3_gy;
    k0 = (long long)jb * ntr + (long long)ry * per_r;
    ntile = max(0, min(per_r, ntr - ry * per_r));
  } else {            // flattened jb-major ranges (many trait blocks per CTA slot)
    const long long total = (long long)gx * ntr;
    const long long per = (total + gridDim.x - 1) / gridDim.x;
    k0 = (long long)blockIdx.x * per;
    ntile = (int)max(0ll, min(total, k0 + per) - k0);
  }
  if (tid == 0) {
    for (int k = 0; k < ST; ++k) mbar_init_cta(&full[k]);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int k) {  // tile k0 + k -> stage k % ST (thread 0)
    const int st = k % ST;
    const long long tau = k0 + k;
    const int jb = (int)(tau / ntr), i0 = (int)(tau - (long long)jb * ntr) * R;
    const int nr = min(R, s.cols - i0);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&full[st])), "r"(kChunk * nr)
                 : "memory");
    const double* src = s.C + (long long)jb * F * CTILE_T + (long long)i0 * s.ldc;
    for (int r = 0; r < nr; ++r)
      bulk_g2s(sm + (size_t)(st * R + r) * F * CTILE_T, src + (long long)r * s.ldc, kChunk, &full[st]);
  };
  if (tid == 0)
    for (int k = 0; k < ST - 1 && k < ntile; ++k) issue(k);

  double L[P * (P + 1) / 2], Linv_d[P], v[P];
  double scale = 1.0;
  int cur_jb = -1;
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  for (int k = 0; k < ntile; ++k) {
    if (tid == 0 && k + ST - 1 < ntile) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // stage (k-1) % ST was read last iteration
      issue(k + ST - 1);
    }
    const long long tau = k0 + k;
    const int jb = (int)(tau / ntr), i0 = (int)(tau - (long long)jb * ntr) * R;
    const int j = jb * CTILE_T + tid;
    const bool active = j < t;
    if (jb != cur_jb) {  // this thread's trait changed: its L_TL_j, 1/L_ff, v_j, sigma2_j
      cur_jb = jb;
      const int jj = active ? j : t - 1;
#pragma unroll
      for (int e = 0; e < P * (P + 1) / 2; ++e) L[e] = __ldg(s.Lpk + (long long)e * t + jj);
#pragma unroll
      for (int f = 0; f < P; ++f) {
        Linv_d[f] = 1.0 / L[f * (f + 1) / 2 + f];
        v[f] = __ldg(s.v + (long long)f * t + jj);
      }
      scale = s.literal ? __ldg(s.s2 + jj) : 1.0;
    }
    const int st = k % ST;
    mbar_wait_parity(&full[st], (uint32_t)((k / ST) & 1));
    const int nr = min(R, s.cols - i0);
    for (int r = 0; r < nr && active; ++r) {
      const double* cur = sm + (size_t)(st * R + r) * F * CTILE_T + tid;
      const int i = i0 + r;
      const long long idx = (long long)i * t + j;
      double u[P];
      double uv = 0.0, uu = 0.0;
#pragma unroll
      for (int f = 0; f < P; ++f) {
        double acc = cur[f * CTILE_T];
#pragma unroll
        for (int l = 0; l < f; ++l) acc -= L[f * (f + 1) / 2 + l] * u[l];
        u[f] = acc * Linv_d[f];
        uu += u[f] * u[f];
        uv += u[f] * v[f];
      }
      const double rr = cur[P * CTILE_T];
      const double c = cur[(P + 1) * CTILE_T];
      const double sigma = c - uu;
      int8_t stt = 0;
      if (!(isfinite(sigma) && isfinite(c) && isfinite(rr) && isfinite(uv))) stt = 2;
      else if (!(sigma > s.eps_collinear * c)) stt = 1;
      double bg = nan, vg = nan;
      if (stt == 0) {
        const double rs = 1.0 / sigma;
        bg = (rr - uv) * rs;
        vg = scale * rs;
        if (!(isfinite(bg) && isfinite(vg))) { stt = 2; bg = vg = nan; }
      }
      s.status[idx] = stt;
      if (!s.full) {
        s.b[idx] = bg;
        s.var[idx] = vg;
        continue;
      }
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
        if (stt == 0) {
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
    __syncthreads();  // every thread is done with stage st before it is refilled
  }
}

}  // namespace gw
