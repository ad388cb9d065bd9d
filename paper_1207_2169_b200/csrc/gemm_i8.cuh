// K1i / K2a: exact integer-sliced products on the 5th-generation tensor cores (tcgen05.mma kind::i8, TMEM),
// the "int8-sliced" mode of SURVEY.md §8(f) NEXT-4.
//
// X_R holds integer dosages (uint8, exact), so for any fp64 matrix B (columns b_c) the product X_R^T B can be
// formed EXACTLY up to the representation of B: each column is scaled by a power of two 2^e_c with
// |b_c| 2^-e_c <= 127/128 and split into S signed 8-bit digits (balanced, round-to-nearest):
//       b_c 2^-e_c = sum_{s<S} d_s 2^{-7(s+1)} + r,   |d_0| <= 127, |d_{s>0}| <= 64, |r| <= 2^{-7S-1}
// Every digit product sum_r g[r,i] d_s[r,c] is an exact int32 on the tensor core (|.| <= 255*127*n < 2^31 for
// n <= 66 000), and the epilogue recombines the S int32 accumulators exactly in two int64 halves, rounds once to
// fp64 and applies 2^e_c.  The representation error is <= 2^-57 (S = 8) or 2^-50 (S = 7) of the column maximum.
//
// Used for B = Z (Alg. 4 line 3: X_R' = Z^T X_R, needed for the W_R^T W_R term) and for the re-associated
// linear terms of lines 13-15: W_R^T W_L = X_R^T (Z D_j X_L') and W_R^T Y_j = X_R^T (Z D_j y'_j),
// i.e. B = B_lin = Z B_op (precomputed once in setup).  Both share the A operand, so one launch covers both:
// output tiles [0, na_tiles) write C_a (X_R'^T), the rest write C_b (the linear block of the K2 output).
//
// Tiles: 128 SNP rows x 64 output columns per CTA.  B rows of a tile are stacked digit-major (row s*64 + j = digit
// s of output column j), so the S*64 (512 or 448) int32 accumulators of the tile fit TMEM's 512 columns x 128
// lanes.  Warp 0: TMA producer into a STAGES ring of BKB-byte K stages; warp 1: TMEM allocation + single-thread
// tcgen05.mma issue (N = 256 for digits 0..3 and N = (S-4)*64 for the rest, K = 32 per instruction),
// tcgen05.commit -> mbarriers; warps 4-7: epilogue (tcgen05.ld 32x32b, exact int64 recombination, fp64 stores or
// the fused squared-term partials).  Two kernels:
//   gemm_i8_sliced_2sm (default): CTA pairs issue cta_group::2 MMAs (M = 256), each CTA staging its 128 A rows and
//     half of the slab, persistent clusters of one or two pairs, 128-byte K stages (128-byte swizzle);
//   gemm_i8_sliced: 1-SM MMAs (M = 128), 2- or 4-CTA clusters multicasting the slab (blocks of <= 128 rows).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "gemm_dmma.cuh"  // smem_u32, mbarrier + TMA helpers

namespace gw {

constexpr int I8_SLICES = 8;       // digits per fp64 value of the exact variant
constexpr int I8_NB = 64;          // output columns per tile
constexpr int I8_BM = 128;         // output rows (SNPs) per tile
constexpr int I8_THREADS = 256;
constexpr size_t I8_SMEM_MAX = 232448;  // 227 KB opt-in shared memory per CTA

// K bytes per pipeline stage, BKB = 64 (64-byte swizzle atoms, the round-1/2 layout) or 128 (128-byte swizzle: each
// TMA box row is one 128-byte request instead of two 64-byte ones, half the TMA row requests per byte).
// Per digit count S (int8_slices = 7 or 8): B rows per tile (S x 64, TMEM columns of the accumulators) and the
// stage ring depth that fits 227 KB of shared memory (A 128 x BKB + B S x 64 x BKB bytes per stage).
template <int S, int BKB>
struct I8Cfg {
  static_assert(S == 7 || S == 8, "int8_slices must be 7 or 8");
  static_assert(BKB == 64 || BKB == 128, "K stage of 64 or 128 bytes");
  static constexpr int BROWS = S * I8_NB;
  static constexpr size_t fixed = 1024 + 256;  // alignment slack + barriers
  static constexpr int STAGES = (int)((I8_SMEM_MAX - fixed - 4608) / ((size_t)(I8_BM + BROWS) * BKB));
  static_assert(STAGES >= 2 && STAGES <= 15, "ring depth");
  static constexpr size_t smem_bytes(size_t epi) { return fixed + (size_t)STAGES * (I8_BM + BROWS) * BKB + epi; }
};
// 2-SM kernel: per CTA a stage holds its 128 A rows and half of each N chunk of the slab (chunk 0 = digits 0..3,
// 256 rows -> 128 per CTA; chunk 1 = digits 4..S-1, (S - 4) x 64 rows -> (S - 4) x 32 per CTA).
template <int S, int BKB>
struct I8Cfg2 {
  static_assert(S == 7 || S == 8, "int8_slices must be 7 or 8");
  static constexpr int NC1 = (S - 4) * 32;  // chunk-1 rows per CTA
  static constexpr int BH_ROWS = 128 + NC1;
  static constexpr size_t fixed = 1024 + 256;
  static constexpr int STAGES = (int)((I8_SMEM_MAX - fixed - 4608) / ((size_t)(I8_BM + BH_ROWS) * BKB));
  static_assert(STAGES >= 2 && STAGES <= 15, "ring depth");
  static constexpr size_t smem_bytes(size_t epi) { return fixed + (size_t)STAGES * (I8_BM + BH_ROWS) * BKB + epi; }
};

struct I8Shape {
  int M;              // rows of A (SNPs of the block)
  int K;              // n
  int tiles_m, tiles_n;
  int na_tiles;       // output tiles [0, na_tiles) -> C_a, the rest -> C_b
  int na, nb;         // valid columns of C_a / C_b
  double* Ca;
  long long lda_c;
  double* Cb;
  long long ldb_c;
  const int* exps;    // 2^e per output column of the concatenated digit matrix (tiles*64 entries)
  int group_m;
  int tri_tiles;      // output tiles [0, tri_tiles) come from a lower-triangular B (CLAK-Chol's L^-1): K < (tn+1)*64
  // K2b fused into the epilogue (ft <= I8_FUSE_T traits; ft = 0: off): the C_a tiles are not
  // stored; each thread accumulates P[tn][row][j] = sum_{c in tile} X_R'[c, row]^2 d_j[c] (d_j = row j of fD, ld fld)
  // for its row, and fused_k2_reduce sums the partials over the C_a tiles in fixed order.
  int dbg;            // debug (GWAS_I8_DBG): 1 = skip TMEM loads in the epilogue, 2 = skip its stores
  unsigned long long* trace;  // debug (GWAS_I8_TRACE): per-CTA %globaltimer stamps of the kernel phases, or null
  int square_a;       // store X_R'^2 in C_a (unfused int8 mode: K2b = (X_R'^2)^T D needs no squaring in its loop)
  int ft;
  const double* fD;
  long long fld;
  double* fP;
  long long fP_stride;
};
constexpr int I8_FUSE_T = 8;

template <int BKB>
__device__ __forceinline__ uint64_t umma_desc_k(uint32_t smem_addr) {
  // K-major, BKB-byte swizzle: 8-row atoms of BKB bytes (SBO = 8 x BKB between atoms), LBO unused (encoded 1),
  // version 1 (sm_100), base offset 0 (tiles are 1024-byte aligned), layout type 4 = SWIZZLE_64B, 2 = SWIZZLE_128B.
  // A K step of 32 bytes inside the atom advances the start address (the swizzle acts on absolute address bits).
  static_assert(BKB == 64 || BKB == 128, "swizzle width");
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(((8 * BKB) >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(BKB == 128 ? 2 : 4) << 61;
  return d;
}
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t smem_addr) { return umma_desc_k<64>(smem_addr); }

// kind::i8 instruction descriptor: D s32, A u8, B s8, both K-major, M = 128, N = n.
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
  return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// Cluster helpers (TMA multicast of the digit slab across CTAs that share it).
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}

__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// Address of the same shared-memory variable in CTA `rank` of the cluster, and a release arrive on it.
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}

// Debug trace (GWAS_I8_TRACE): 16 slots per CTA -- 0..6 %globaltimer phase stamps, 7 smid, 8 clock64 cycles the
// MMA thread waited on full barriers, 9 cycles the producer waited on empty barriers, 10 k-stages.
constexpr int I8_TRACE_SLOTS = 16;
__device__ __forceinline__ void i8_stamp(const I8Shape& s, int slot) {
  if (s.trace && blockIdx.x < 4096) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    s.trace[blockIdx.x * I8_TRACE_SLOTS + slot] = globaltimer_ns();
    s.trace[blockIdx.x * I8_TRACE_SLOTS + 7] = smid;
  }
}
__device__ __forceinline__ void i8_put(const I8Shape& s, int slot, unsigned long long v) {
  if (s.trace && blockIdx.x < 4096) s.trace[blockIdx.x * I8_TRACE_SLOTS + slot] = v;
}

constexpr int EPI_CW = 8;  // output columns per TMEM drain chunk (S x 8 int32 registers in flight)

// Epilogue (warps 4-7): warp w drains TMEM lanes 32 (w % 4) .. +31 (= tile rows), recombines the S digit
// accumulators of each output column (Horner in 2^-7, fp64), scales by 2^(e-7) and stores fp64.
// Per-tile operands of the epilogue, staged in shared memory by the epilogue warps while the MMAs run (each was
// otherwise an L2 round trip inside the drain loop, exposed once per column chunk).
struct I8EpiSmem {
  double scale[I8_NB];  // 2^(e_c - 28) per output column of the tile
  double d[I8_NB][I8_FUSE_T];  // fused D rows, column-major by trait (zero for traits >= ft)
};
constexpr int I8_EPI_SMEM = (int)sizeof(I8EpiSmem);

template <int S>
__device__ __forceinline__ void i8_epilogue(const I8Shape& s, uint32_t tmem_base, uint64_t* tmem_full, int m0, int tn,
                                            int warp, int lane, I8EpiSmem* es, uint32_t parity = 0) {
  // epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31 = tile rows
  const int q = warp & 3;
  const int row = m0 + q * 32 + lane;
  {
    asm volatile("bar.sync 1, 128;\n" ::: "memory");  // (persistent CTAs) the previous tile's reads of es are done
    const int et = threadIdx.x - 128;  // 0..127 over the four epilogue warps
    const int oc = tn * I8_NB;
    if (et < I8_NB) es->scale[et] = scalbn(1.0, __ldg(s.exps + oc + et) - 28);
    if (tn < s.na_tiles && s.ft > 0)
      for (int idx = et; idx < I8_FUSE_T * I8_NB; idx += 128) {
        const int jj = idx / I8_NB, c = idx - jj * I8_NB;
        es->d[c][jj] = (jj < s.ft && oc + c < s.na) ? __ldg(s.fD + jj * s.fld + oc + c) : 0.0;
      }
    asm volatile("bar.sync 1, 128;\n" ::: "memory");  // the four epilogue warps only
  }
  mbar_wait(tmem_full, parity);
  if (threadIdx.x == 128) i8_stamp(s, 4);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tl = tmem_base + ((uint32_t)(q * 32) << 16);
  const int oc0 = tn * I8_NB;  // first output column of the concatenated digit matrix
  const bool in_a = tn < s.na_tiles;
  const bool fuse = in_a && s.ft > 0;
  double part[I8_FUSE_T];
#pragma unroll
  for (int jj = 0; jj < I8_FUSE_T; ++jj) part[jj] = 0.0;
#pragma unroll 1
  for (int j0 = 0; j0 < I8_NB; j0 += EPI_CW) {
    // all S digit planes of EPI_CW columns in flight at once, one wait (the drain is otherwise a chain of S
    // dependent TMEM round trips per chunk, exposed because the accumulators fill TMEM and nothing overlaps them)
    int32_t v[S][EPI_CW];
    if (s.dbg != 1) {
#pragma unroll
      for (int sl = 0; sl < S; ++sl) tmem_ld8(tl + sl * I8_NB + j0, v[sl]);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    } else {
#pragma unroll
      for (int sl = 0; sl < S; ++sl)
#pragma unroll
        for (int c = 0; c < EPI_CW; ++c) v[sl][c] = lane + sl + c + j0;
    }
    // exact integer recombination of the digit accumulators in two halves of <= 4 digits (|.| < 2^53 each, so both
    // convert exactly), one fp64 rounding (the fma), then the exact power-of-two column scale 2^(e - 28):
    //   x = sum_s I_s 2^(-7(s+1)) 2^e = (hi + lo 2^(-7(S-4))) 2^(e - 28),  hi = sum_{s<4} I_s 2^(7(3-s)),
    //   lo = sum_{4<=s<S} I_s 2^(7(S-1-s))
    constexpr double lo_scale = S == 8 ? 0x1p-28 : 0x1p-21;
    double acc[EPI_CW];
#pragma unroll
    for (int c = 0; c < EPI_CW; ++c) {
      const long long hi = (((long long)v[0][c] * 128 + v[1][c]) * 128 + v[2][c]) * 128 + v[3][c];
      long long lo = v[4][c];
#pragma unroll
      for (int sl = 5; sl < S; ++sl) lo = lo * 128 + v[sl][c];
      acc[c] = fma((double)lo, lo_scale, (double)hi) * es->scale[j0 + c];
    }
    if (fuse) {
#pragma unroll
      for (int c = 0; c < EPI_CW; ++c) {
        // the trait loop runs over all I8_FUSE_T slots (zero rows beyond ft, zero columns beyond na): no predicates,
        // and the column's 8 D values arrive as 4 independent 16-byte loads instead of a load->fma chain
        const double x2 = acc[c] * acc[c];
        const double2* dc = reinterpret_cast<const double2*>(es->d[j0 + c]);
#pragma unroll
        for (int jj = 0; jj < I8_FUSE_T; jj += 2) {
          const double2 dd = dc[jj / 2];
          part[jj] = fma(x2, dd.x, part[jj]);
          part[jj + 1] = fma(x2, dd.y, part[jj + 1]);
        }
      }
    } else if (row < s.M && s.dbg != 2) {
      double* crow = in_a ? s.Ca + (long long)row * s.lda_c : s.Cb + (long long)row * s.ldb_c;
      const int cbase = in_a ? oc0 + j0 : (tn - s.na_tiles) * I8_NB + j0;
      const int cmax = in_a ? s.na : s.nb;
#pragma unroll
      for (int c = 0; c < EPI_CW; c += 2) {
        double x0 = acc[c], x1 = acc[c + 1];
        if (in_a && s.square_a) {  // the int8 mode needs X_R' only squared (K2b): store X_R'^2, K2b is then plain
          x0 *= x0;
          x1 *= x1;
        }
        const int col = cbase + c;
        if (col + 1 < cmax) {
          *reinterpret_cast<double2*>(crow + col) = make_double2(x0, x1);
        } else if (col < cmax) {
          crow[col] = x0;
        }
      }
    }
  }
  if (fuse && row < s.M) {
    double* P = s.fP + (long long)tn * s.fP_stride + (long long)row * s.ft;
#pragma unroll
    for (int jj = 0; jj < I8_FUSE_T; ++jj)
      if (jj < s.ft) P[jj] = part[jj];
  }
}

// CL = cluster size along M: the CL CTAs of a cluster compute CL consecutive row tiles of the same output
// column tile, and each loads 1/CL of the shared digit slab and multicasts it to all (L2 reads of the dominant
// B operand / CL).  Stage slots are released cluster-wide: every CTA's MMA completion arrives on every CTA's
// empty barrier (count CL).
template <int CL, int S, int BKB>
__global__ void __launch_bounds__(I8_THREADS, 1)
    gemm_i8_sliced(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, I8Shape s) {
  constexpr int I8_STAGES = I8Cfg<S, BKB>::STAGES;
  constexpr int I8_BKB = BKB;
  constexpr int BROWS = I8Cfg<S, BKB>::BROWS;  // S x 64
  constexpr int A_BYTES = I8_BM * I8_BKB;      // 8 or 16 KB
  constexpr int B_BYTES = BROWS * I8_BKB;      // S x 4 or 8 KB
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = sA + I8_STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + I8_STAGES * B_BYTES);
  uint64_t* empty = full + I8_STAGES;
  uint64_t* tmem_full = empty + I8_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  I8EpiSmem* esm = reinterpret_cast<I8EpiSmem*>(tmem_full + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) i8_stamp(s, 0);
  int tm, tn;
  const uint32_t crank = CL > 1 ? cluster_ctarank() : 0u;
  {
    // grouped rasterisation over (row-tile clusters, column tiles); s.tiles_m is a multiple of CL
    const int pid = blockIdx.x / CL;
    const int tiles_mc = s.tiles_m / CL;
    const int gm = max(1, s.group_m / CL);
    const int per_group = gm * s.tiles_n;
    const int g = pid / per_group;
    const int first_m = g * gm;
    const int gsz = min(tiles_mc - first_m, gm);
    const int r = pid - g * per_group;
    tm = (first_m + r % gsz) * CL + (int)crank;
    tn = r / gsz;
  }
  const int m0 = tm * I8_BM;
  const int brow0 = tn * BROWS;
  const int k_end = tn < s.tri_tiles ? min(s.K, (tn + 1) * I8_NB) : s.K;
  const int KB = (k_end + I8_BKB - 1) / I8_BKB;

  if (threadIdx.x == 0) {
    for (int i = 0; i < I8_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], CL);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {  // whole warp: allocate all 512 TMEM columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if constexpr (CL > 1) cluster_sync_all();  // peers' barriers initialised before any multicast lands
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) i8_stamp(s, 1);

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      unsigned long long wprod = 0;
      for (int kb = 0; kb < KB; ++kb) {
        const int st = kb % I8_STAGES;
        if (kb >= I8_STAGES) {
          const long long c0 = s.trace ? clock64() : 0;
          mbar_wait(&empty[st], ((kb / I8_STAGES) - 1) & 1);
          if (s.trace) wprod += clock64() - c0;
        }
        mbar_expect_tx(&full[st], A_BYTES + B_BYTES);
        tma_load_2d(sA + st * A_BYTES, &tmA, &full[st], kb * I8_BKB, m0);
        if constexpr (CL == 1) {  // two boxes of BROWS/2 rows (the tensor map's box)
          tma_load_2d(sB + st * B_BYTES, &tmB, &full[st], kb * I8_BKB, brow0);
          tma_load_2d(sB + st * B_BYTES + (BROWS / 2) * I8_BKB, &tmB, &full[st], kb * I8_BKB, brow0 + BROWS / 2);
        } else {
          constexpr int QR = BROWS / CL;  // rows of the slab this CTA fetches for the whole cluster
          tma_load_2d_mc(sB + st * B_BYTES + crank * QR * I8_BKB, &tmB, &full[st], kb * I8_BKB,
                         brow0 + (int)crank * QR, (uint16_t)((1u << CL) - 1));
        }
      }
      i8_put(s, 9, wprod);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_i8(256);               // digits 0..3 of the tile's 64 columns
      constexpr uint32_t idesc2 = idesc_i8((S - 4) * I8_NB);  // digits 4..S-1
      unsigned long long wmma = 0;
      for (int kb = 0; kb < KB; ++kb) {
        const int st = kb % I8_STAGES;
        const long long c0 = s.trace ? clock64() : 0;
        mbar_wait(&full[st], (kb / I8_STAGES) & 1);
        if (s.trace && kb > 0) wmma += clock64() - c0;
        if (kb == 0) i8_stamp(s, 2);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t a0 = smem_u32(sA + st * A_BYTES);
        const uint32_t b0 = smem_u32(sB + st * B_BYTES);
#pragma unroll
        for (int kk = 0; kk < I8_BKB / 32; ++kk) {
          const uint64_t ad = umma_desc_k<BKB>(a0 + kk * 32);
          const uint64_t bd0 = umma_desc_k<BKB>(b0 + kk * 32);
          const uint64_t bd1 = umma_desc_k<BKB>(b0 + 256 * I8_BKB + kk * 32);
          const uint32_t acc = (kb | kk) ? 1u : 0u;
          umma_i8(tmem_base, ad, bd0, idesc, acc);
          umma_i8(tmem_base + 256, ad, bd1, idesc2, acc);
        }
        // frees the smem slot (in every CTA of the cluster) when these MMAs have read it
        if constexpr (CL == 1) umma_commit(&empty[st]);
        else umma_commit_mc(&empty[st], (uint16_t)((1u << CL) - 1));
      }
      umma_commit(tmem_full);     // accumulators complete
      i8_stamp(s, 3);
      i8_put(s, 8, wmma);
      i8_put(s, 10, KB);
    }
  } else if (warp >= 4) {
    i8_epilogue<S>(s, tmem_base, tmem_full, m0, tn, warp, lane, esm);
    if (threadIdx.x == 128) i8_stamp(s, 5);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if constexpr (CL > 1) cluster_sync_all();  // no CTA leaves while peers may still signal its barriers
  if (threadIdx.x == 0) i8_stamp(s, 6);
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(512));
  }
}

// ---------------------------------------------------------------------------------------------------------------
// 2-SM variant (tcgen05 cta_group::2): a CTA pair computes a 256 x 64 output tile with M = 256 MMAs issued by the
// pair's leader CTA.  Each CTA stages its own 128 A rows and HALF of each N chunk of the S x 64-row digit slab
// (chunk 0 = digits 0..3: rows rank*128 .. +127; chunk 1 = digits 4..S-1: rows 256 + rank*(S-4)*32 ..); the tensor
// cores of both SMs read both halves, so every slab byte is fetched and written to shared memory once per pair (vs
// once per CTA): per SM (128 + S x 32) x K bytes land per 2 x 128 x S x 64 x K ops instead of (128 + S x 64) x K,
// which relieves the TMA / crossbar bandwidth that bounds the 1-SM kernel.  Each CTA's TMEM holds its own 128 rows x
// S x 64 accumulator columns, drained by its own epilogue warps.  TMA loads of both CTAs signal the leader's full
// barrier; the leader's commits arrive on both CTAs' empty / tmem_full barriers.
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  // the mbarrier operand addresses the LEADER CTA's barrier (peer bit cleared), as for 2-SM UMMA pipelines
  const uint32_t bar_leader = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_leader)
      : "memory");
}

// The same with the slab multicast to the same-role CTA of every pair in the cluster (each destination CTA's bytes
// complete_tx on ITS pair leader's barrier: the peer bit of the barrier address is cleared).
__device__ __forceinline__ void tma_load_2d_2sm_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                   uint16_t mask) {
  const uint32_t bar_leader = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_leader), "h"(mask)
      : "memory");
}

__device__ __forceinline__ void umma_i8_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit_2sm(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__host__ __device__ constexpr uint32_t idesc_i8_m256(int n) {
  return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

// CLP pairs per cluster (1 or 2): with 2, the two pairs compute consecutive 256-row tiles of the same column tile and
// share its digit slab: the CTA of role r in pair q fetches the q-th 1/CLP of its slab half and multicasts it to role r
// of every pair (L2 reads of the slab / CLP); stage slots are then released cluster-wide (empty count CLP, every
// leader's commit multicast to all CTAs).  tmB: box of 128 / CLP slab rows (chunk 0); tmB1: box of (S - 4) x 32 / CLP
// rows (chunk 1).
template <int S, int BKB, int CLP>
__global__ void __launch_bounds__(I8_THREADS, 1)
    gemm_i8_sliced_2sm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const __grid_constant__ CUtensorMap tmB1, I8Shape s) {
  static_assert(CLP == 1 || CLP == 2, "pairs per cluster");
  using Cfg = I8Cfg2<S, BKB>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int R0 = 128 / CLP, R1 = Cfg::NC1 / CLP;  // slab rows this CTA fetches per chunk
  constexpr uint16_t ALL = (uint16_t)((1u << (2 * CLP)) - 1);
  constexpr int NC1 = Cfg::NC1;
  constexpr int A_BYTES = I8_BM * BKB;          // this CTA's 128 rows
  constexpr int BH_BYTES = Cfg::BH_ROWS * BKB;  // this CTA's halves of the two N chunks
  static_assert((2 * STAGES + 4) * 8 <= 256, "barriers + TMEM slot exceed their 256-byte region");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = sA + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * BH_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint64_t* tmem_empty = tmem_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 1);
  I8EpiSmem* esm = reinterpret_cast<I8EpiSmem*>(tmem_empty + 3);  // 16-byte aligned (double2 loads of es->d)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) i8_stamp(s, 0);
  const uint32_t crank = cluster_ctarank();
  const uint32_t rank = crank & 1u, pq = crank >> 1;  // role in the pair, pair index in the cluster
  const bool leader = rank == 0;
  // Persistent clusters: cluster c computes cluster tiles c, c + nclu, ... (grid = every tile: one each).  A cluster
  // tile is CLP consecutive 256-row pair tiles of one 64-column tile, in grouped rasterisation.
  const int nclu = (int)gridDim.x / (2 * CLP);
  const int ctiles = (s.tiles_m / (2 * CLP)) * s.tiles_n;
  auto tile_of = [&](int pid, int& m0, int& tn, int& KB) {
    const int tiles_mc = s.tiles_m / (2 * CLP);
    const int gm = max(1, s.group_m / (2 * CLP));
    const int per_group = gm * s.tiles_n;
    const int g = pid / per_group;
    const int first_m = g * gm;
    const int gsz = min(tiles_mc - first_m, gm);
    const int r = pid - g * per_group;
    m0 = ((first_m + r % gsz) * (2 * CLP) + (int)crank) * I8_BM;
    tn = r / gsz;
    const int k_end = tn < s.tri_tiles ? min(s.K, (tn + 1) * I8_NB) : s.K;
    KB = (k_end + BKB - 1) / BKB;
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], CLP);
    }
    mbar_init(tmem_full, 1);
    mbar_init(tmem_empty, 8);  // the 4 epilogue warps of both CTAs of the pair (used in the leader)
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {  // both CTAs: one warp each, same smem slot
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) i8_stamp(s, 1);

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB1)) : "memory");
      unsigned long long wprod = 0;
      int gk = 0;  // stage counter across this cluster's tiles (the ring runs on into the next tile)
      for (int pid = (int)blockIdx.x / (2 * CLP); pid < ctiles; pid += nclu) {
        int m0, tn, KB;
        tile_of(pid, m0, tn, KB);
        const int brow0 = tn * S * I8_NB;
        for (int kb = 0; kb < KB; ++kb, ++gk) {
          const int st = gk % STAGES;
          if (gk >= STAGES) {
            const long long c0 = s.trace ? clock64() : 0;
            mbar_wait(&empty[st], ((gk / STAGES) - 1) & 1);
            if (s.trace) wprod += clock64() - c0;
          }
          if (leader) mbar_expect_tx(&full[st], 2 * (A_BYTES + BH_BYTES));  // both CTAs' bytes land on it
          tma_load_2d_2sm(sA + st * A_BYTES, &tmA, &full[st], kb * BKB, m0);
          if constexpr (CLP == 1) {
            tma_load_2d_2sm(sB + st * BH_BYTES, &tmB, &full[st], kb * BKB, brow0 + (int)rank * 128);
            tma_load_2d_2sm(sB + st * BH_BYTES + 128 * BKB, &tmB1, &full[st], kb * BKB, brow0 + 256 + (int)rank * NC1);
          } else {
            const uint16_t mc = (uint16_t)((1u << rank) | (1u << (2 + rank)));  // role `rank` of both pairs
            tma_load_2d_2sm_mc(sB + st * BH_BYTES + pq * R0 * BKB, &tmB, &full[st], kb * BKB,
                               brow0 + (int)rank * 128 + (int)pq * R0, mc);
            tma_load_2d_2sm_mc(sB + st * BH_BYTES + (128 + pq * R1) * BKB, &tmB1, &full[st], kb * BKB,
                               brow0 + 256 + (int)rank * NC1 + (int)pq * R1, mc);
          }
        }
      }
      i8_put(s, 9, wprod);
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc0 = idesc_i8_m256(256);      // digits 0..3
      constexpr uint32_t idesc1 = idesc_i8_m256(2 * NC1);  // digits 4..S-1
      unsigned long long wmma = 0;
      int gk = 0, it = 0;
      for (int pid = (int)blockIdx.x / (2 * CLP); pid < ctiles; pid += nclu, ++it) {
        int m0, tn, KB;
        tile_of(pid, m0, tn, KB);
        if (it > 0) {  // the previous tile's accumulators drained by both CTAs' epilogues
          mbar_wait(tmem_empty, (it - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        }
        for (int kb = 0; kb < KB; ++kb, ++gk) {
          const int st = gk % STAGES;
          const long long c0 = s.trace ? clock64() : 0;
          mbar_wait(&full[st], (gk / STAGES) & 1);
          if (s.trace && gk > 0) wmma += clock64() - c0;
          if (gk == 0) i8_stamp(s, 2);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t a0 = smem_u32(sA + st * A_BYTES);
          const uint32_t b0 = smem_u32(sB + st * BH_BYTES);
#pragma unroll
          for (int kk = 0; kk < BKB / 32; ++kk) {
            const uint64_t ad = umma_desc_k<BKB>(a0 + kk * 32);
            const uint32_t acc = (kb | kk) ? 1u : 0u;
            umma_i8_2sm(tmem_base, ad, umma_desc_k<BKB>(b0 + kk * 32), idesc0, acc);
            umma_i8_2sm(tmem_base + 256, ad, umma_desc_k<BKB>(b0 + 128 * BKB + kk * 32), idesc1, acc);
          }
          umma_commit_2sm(&empty[st], ALL);  // every CTA may refill this stage once all pairs' MMAs have read it
        }
        umma_commit_2sm(tmem_full, (uint16_t)(3u << (2 * pq)));  // this pair's accumulators complete
      }
      i8_stamp(s, 3);
      i8_put(s, 8, wmma);
      i8_put(s, 10, gk);
    }
  } else if (warp >= 4) {
    // TMEM drained -> the pair leader's tmem_empty (remote arrive from the peer CTA)
    const uint32_t empty_leader = mapa_shared(smem_u32(tmem_empty), crank & ~1u);
    int it = 0;
    for (int pid = (int)blockIdx.x / (2 * CLP); pid < ctiles; pid += nclu, ++it) {
      int m0, tn, KB;
      tile_of(pid, m0, tn, KB);
      i8_epilogue<S>(s, tmem_base, tmem_full, m0, tn, warp, lane, esm, (uint32_t)(it & 1));
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(empty_leader);
    }
    if (threadIdx.x == 128) i8_stamp(s, 5);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  cluster_sync_all();
  if (threadIdx.x == 0) i8_stamp(s, 6);
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(512));
  }
}

// ---------------------------------------------------------------------------------------------------------------
// Setup helpers for the sliced mode.

// Split rows of an fp64 matrix X (rows x ldx, K-contiguous, n valid entries) into S signed 8-bit digits.
// Row `r` (an output column of the product) goes to digit rows dst_row(r, s) = (r / 64) * 512 + s * 64 + r % 64
// of D (ldd bytes per row, pad zero); exps[r] = e with |X[r, :]| 2^-e <= 127/128.  One CTA per row.
__global__ void digitize_rows(const double* __restrict__ X, long long ldx, int rows, int n, int row_off,
                              int8_t* __restrict__ D, long long ldd, int* __restrict__ exps, int S) {
  const int r = blockIdx.x;
  if (r >= rows) return;
  const double* x = X + (long long)r * ldx;
  __shared__ double red[32];
  double mx = 0.0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) mx = fmax(mx, fabs(x[k]));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    mx = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (threadIdx.x == 0) red[0] = mx;
  }
  __syncthreads();
  mx = red[0];
  // smallest e with mx * 2^-e <= 127/128 (e = 0 for an all-zero row)
  int e = 0;
  if (mx > 0.0) {
    frexp(mx, &e);  // mx = f 2^e, f in [0.5, 1)
    if (ldexp(mx, -e) > 127.0 / 128.0) e += 1;
  }
  const int gr = r + row_off;
  if (threadIdx.x == 0) exps[gr] = e;
  const long long base = (long long)(gr / I8_NB) * (S * I8_NB) + gr % I8_NB;
  for (int k = threadIdx.x; k < ldd; k += blockDim.x) {
    double v = k < n ? ldexp(x[k], -e + 7) : 0.0;  // |v| <= 127
    for (int sl = 0; sl < S; ++sl) {
      const double d = rint(v);
      D[(base + (long long)sl * I8_NB) * ldd + k] = (int8_t)d;
      v = (v - d) * 128.0;  // exact: |v - d| <= 1/2
    }
  }
}

// CLAK-Chol setup (Alg. 3 line 1): M = sigma2 (h2 Phi + (1 - h2) I) in place over a copy of Phi
// (column-major, ld kpad), both triangles from one expression per entry.
__global__ void assemble_m(double* __restrict__ A, int n, int kpad, double sigma2, double h2) {
  for (int c = blockIdx.y; c < n; c += gridDim.y)  // grid-stride in y: n may exceed the 65535 grid limit
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
      const double phi = A[(long long)c * kpad + r];
      A[(long long)c * kpad + r] = sigma2 * (h2 * phi + (r == c ? 1.0 - h2 : 0.0));
    }
}

// Zero the strict upper triangle (and the padding) of a column-major kpad x kpad matrix (dtrtri leaves M there).
__global__ void zero_upper(double* __restrict__ A, int n, int kpad) {
  for (int c = blockIdx.y; c < kpad; c += gridDim.y)
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < kpad; r += gridDim.x * blockDim.x)
      if (r < c || r >= n || c >= n) A[(long long)c * kpad + r] = 0.0;
}

// Out-of-place transpose of a kpad x kpad fp64 matrix (tiled through shared memory).
__global__ void transpose_sq(const double* __restrict__ src, double* __restrict__ dst, int kpad) {
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = by + i, c = bx + threadIdx.x;
    if (r < kpad && c < kpad) tile[i][threadIdx.x] = src[(long long)r * kpad + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = bx + i, c = by + threadIdx.x;
    if (r < kpad && c < kpad) dst[(long long)r * kpad + c] = tile[threadIdx.x][i];
  }
}

}  // namespace gw
