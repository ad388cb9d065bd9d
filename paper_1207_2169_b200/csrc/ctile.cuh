// Trait-tiled layout of K2's output C (many traits, FP64 exact weights): written by K2's epilogue (gemm_dmma.cuh),
// read by K3 (schur.cuh).
//
// Row i of C holds, for every block jb of CTILE_T consecutive traits, one contiguous chunk of F = p + 2 fields x
// CTILE_T values: C[i][jb][f][j % CTILE_T], with f < p the X_L fields (W_R^T W_L), f = p the y field (W_R^T y_j) and
// f = p + 1 the squared field (W_R^T W_R) of PAPER.md P:146-148.  K3's CTA (CTILE_T threads, one per trait) then reads
// 7 KB contiguous per row (p = 5) instead of 7 strided 1 KB pieces: tools/k3_pattern_bw.cu measured the two access
// patterns, without arithmetic, at 4.90 (strided) vs 6.14 TB/s (tiled) on a B200.
#pragma once

namespace gw {

constexpr int CTILE_T = 128;

__host__ __device__ __forceinline__ long long ctile_off(int j, int f, int F) {  // j >= 0
  const unsigned ju = (unsigned)j;
  return (long long)(ju / CTILE_T) * F * CTILE_T + (long long)f * CTILE_T + (ju % CTILE_T);
}

// Row length (doubles) of the tiled C for t traits and F fields.
__host__ __device__ __forceinline__ long long ctile_ld(int t, int F) {
  return (long long)((t + CTILE_T - 1) / CTILE_T) * F * CTILE_T;
}

}  // namespace gw
