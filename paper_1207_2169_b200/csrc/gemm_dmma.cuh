// K1 / K2: FP64 tensor-core (DMMA) GEMM for sm_100a, C[M x N] = A[M x K] * B[N x K]^T (both K-contiguous).
//
//   K1 (Alg. 4 line 3, "X_R := Z^T X_R"):  A = X_R block (u8 dosages or fp64, one SNP per
//       row of A), B = Z (column k of dsyevd's Z = row k of B), C = X_R'^T (one rotated SNP per row of C).
//   K2 (Alg. 4 lines 13-15, all traits at once):  A = X_R'^T, B = [B_op | D] where
//       B_op[:, f*t+j] = d_j * X_L'[:, f] (f < p), B_op[:, p*t+j] = d_j * y'_j, D[:, j] = d_j; columns >= nsq
//       use A∘A, so C[i, nsq + j] = sum_k X_R'[k,i]^2 d_j[k] = W_R^T W_R (the K of K K^T = D never appears).
//
// Design: FP64 has no tcgen05 kind on sm_100a -- every .f64 mma lowers to
// DMMA.8x8x4 (F2), issued per warp.  Operands are staged by TMA (cp.async.bulk.tensor, 128-byte swizzle for
// fp64 tiles, OOB zero fill for the K / M / N tails) into a STAGES-deep ring guarded by mbarriers; one
// thread issues TMA two tiles behind the slowest consumer, 8 warps each own a 64 x 32 accumulator tile
// (64 doubles / thread) and run m8n8k4 DMMA from swizzled shared memory (conflict-free 64-bit fragment loads).  u8 dosages are
// expanded to fp64 through a 256-entry shared-memory table (exact; no FP64-pipe conversion work).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "ctile.cuh"

namespace gw {

constexpr int GEMM_BK = 16;                 // K elements per stage (one 128-byte fp64 row)
constexpr int GEMM_CONSUMER_WARPS = 8;
constexpr int GEMM_THREADS = GEMM_CONSUMER_WARPS * 32;

struct GemmShape {
  int M, N, K;
  double* C;
  long long ldc;
  int nsq;        // first column using A∘A (>= N: none)
  int tiles_m, tiles_n;
  int group_m;    // rasterisation group along M (L2 reuse of B panels)
  int ksplit;     // K split into ksplit ranges of kt_per_split 16-wide k-tiles (skinny N); partial products of
  int kt_per_split;  // split s go to C + s * split_stride (summed in fixed order by splitk_reduce)
  long long split_stride;
  int tri;        // B lower-triangular in (row, k): row c has no entries at k > c (CLAK-Chol's L^-1), so an output
                  // tile [n0, n0 + BN) only needs k < n0 + BN
  // K2 fused into K1's epilogue (few traits; template FUSE): instead of storing the tile of
  // C = X_R'^T, each CTA contracts it with the fnq K2 operand rows it covers and stores the per-tile partial sums
  // P[tn][i][qq] = sum_{c in tile tn} X_R'[c, i]^e B2[row(qq), c], e = 1 for qq < fnlin (row qq), e = 2 otherwise
  // (row fnsq + qq - fnlin); fused_k2_reduce sums them over tn in fixed order.
  const double* fB;
  long long fldb;
  int fnq, fnlin, fnsq;
  double* fP;
  long long fP_stride;  // doubles per tn
  // C in the trait-tiled layout (ctile.cuh; K2 of the many-trait FP64 path): column col < cnlin is field col / ct,
  // trait col % ct; columns [cnlin, nsq) are padding (not stored); col >= nsq is field cF - 1, trait col - nsq.
  int ctiled, ct, cnlin, cF;
};

constexpr int FUSE_MAX_NQ = 28;  // fused K2 columns t (p + 2) per CTA: reduction buffer + operand slice fit the freed stages

// C[i][col(qq)] = sum_tn P[tn][i][qq], col(qq) = qq (qq < nlin) or nsq + qq - nlin: the fused K2 finished in fixed order.
__global__ void fused_k2_reduce(const double* __restrict__ P, long long stride, int ntiles, int M, int nq, int nlin,
                                int nsq, double* __restrict__ C, long long ldc) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)M * nq) return;
  const int i = (int)(idx / nq), qq = (int)(idx - (long long)i * nq);
  double acc = P[idx];
  for (int tn = 1; tn < ntiles; ++tn) acc += P[tn * stride + idx];
  C[(long long)i * ldc + (qq < nlin ? qq : nsq + qq - nlin)] = acc;
}

// Fixed-order sum of the split-K partial products: C[i][c] = sum_s P_s[i][c] (deterministic, independent of M).
__global__ void splitk_reduce(const double* __restrict__ P, long long split_stride, int ksplit, int M, int N,
                              long long ldp, double* __restrict__ C, long long ldc) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)M * N) return;
  const int i = (int)(idx / N), c = (int)(idx - (long long)i * N);
  double acc = P[(long long)i * ldp + c];
  for (int sp = 1; sp < ksplit; ++sp) acc += P[sp * split_stride + (long long)i * ldp + c];
  C[(long long)i * ldc + c] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// Spin until the phase with the given parity has completed.  A pipeline bug that loses an arrival traps after
// ~10 s of waiting (checked on %globaltimer every 4096 tries) instead of hanging the GPU; the trap surfaces as a
// launch failure on the host.  Legitimate waits are bounded by one tile's compute (milliseconds).
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  uint32_t spins = 0;
  uint64_t t0 = 0;
  while (true) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    if (done) return;
    if ((++spins & 4095u) == 0) {
      const uint64_t t = globaltimer_ns();
      if (t0 == 0) t0 = t;
      else if (t - t0 > 10000000000ull) __trap();
    }
  }
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Byte offset of fp64 element (row r, k) inside a [rows][16] fp64 tile written by TMA with SWIZZLE_128B
// (16-byte chunk index XOR (row & 7); tile base 1024-byte aligned).
__device__ __forceinline__ uint32_t swz128_off(int r, int k) {
  return (uint32_t)(r * 128 + ((((k >> 1) ^ (r & 7)) & 7) << 4) + ((k & 1) << 3));
}

template <typename TA>
struct ATile;
template <>
struct ATile<uint8_t> {
  static constexpr int kBytesPerRow = GEMM_BK;  // 16 dosages, no swizzle (conflict-free: 4 lanes share a word)
};
template <>
struct ATile<double> {
  static constexpr int kBytesPerRow = GEMM_BK * 8;
};

template <typename TA, int BM, int BN>
struct GemmSmem {
  static constexpr int kATile = BM * ATile<TA>::kBytesPerRow;
  static constexpr int kBTile = BN * GEMM_BK * 8;
  static constexpr int kAStride = (kATile + 1023) / 1024 * 1024;
  static constexpr int kBStride = (kBTile + 1023) / 1024 * 1024;
};

template <typename TA>
__device__ __forceinline__ double load_a(const uint8_t* a_tile, const double* lut, int r, int k);

template <>
__device__ __forceinline__ double load_a<uint8_t>(const uint8_t* a_tile, const double* lut, int r, int k) {
  return lut[a_tile[r * GEMM_BK + k]];
}
template <>
__device__ __forceinline__ double load_a<double>(const uint8_t* a_tile, const double* lut, int r, int k) {
  return *reinterpret_cast<const double*>(a_tile + swz128_off(r, k));
}

// One CTA computes a BM x BN tile of C with 8 warps (warp grid 2 x 4 for 128 x 128); thread 0 also issues TMA.
// 64-wide tiles fit two CTAs per SM (smem and <= 128 registers): keep the fused variant there too.
template <typename TA, int BM, int BN, int STAGES, bool SQ, bool FUSE = false>
__global__ void __launch_bounds__(GEMM_THREADS, BN == 64 ? 2 : 1)
    gemm_tn_dmma(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmShape s) {
  constexpr int WARPS_N = BN / 32;  // warp tiles are always 32 columns wide (K2's squaring is per warp)
  constexpr int WARPS_M = GEMM_CONSUMER_WARPS / WARPS_N;
  constexpr int WM = BM / WARPS_M;  // 64 (BN = 128) or 32 (BN = 64)
  constexpr int WN = BN / WARPS_N;  // 32
  static_assert(WN == 32 && WM % 8 == 0, "tile shape");
  constexpr int MI = WM / 8, NI = WN / 8;
  using L = GemmSmem<TA, BM, BN>;

  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment for the 128B-swizzled TMA tiles, by pointer offset (keeps the shared address space
  // visible to the compiler, so fragment reads are LDS, not generic loads)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sB = smem;
  uint8_t* sA = sB + STAGES * L::kBStride;
  uint64_t* full = reinterpret_cast<uint64_t*>(sA + STAGES * L::kAStride);
  uint64_t* empty = full + STAGES;
  double* lut = reinterpret_cast<double*>(empty + STAGES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // grouped rasterisation: consecutive CTAs walk down a group of group_m row tiles, then move along N
  int tm, tn;
  const int split = blockIdx.x % s.ksplit;
  {
    const int pid = blockIdx.x / s.ksplit;
    const int per_group = s.group_m * s.tiles_n;
    const int g = pid / per_group;
    const int first_m = g * s.group_m;
    const int gsz = min(s.tiles_m - first_m, s.group_m);
    const int r = pid - g * per_group;
    tm = first_m + r % gsz;
    tn = r / gsz;
    // lower-triangular B (CLAK-Chol): tile tn needs (tn + 1) k-panels; run the long tiles first so the short ones
    // fill the last wave (longest-processing-time order)
    if (s.tri) tn = s.tiles_n - 1 - tn;
  }
  const int m0 = tm * BM, n0 = tn * BN;
  const int kt_begin = split * s.kt_per_split;
  const int k_end = s.tri ? min(s.K, n0 + BN) : s.K;
  const int KT = min((k_end + GEMM_BK - 1) / GEMM_BK - kt_begin, s.kt_per_split);  // k-tiles of this CTA (>= 1)

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], GEMM_CONSUMER_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (sizeof(TA) == 1) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) lut[i] = (double)i;
  }
  __syncthreads();

  // Producer = thread 0 (also a consumer lane): tiles 0..STAGES-2 up front, then in iteration kt it refills
  // tile kt+STAGES-2 into the slot freed by tile kt-2 (two iterations of slack, so the empty-barrier wait
  // almost never blocks).  No dedicated producer warp: 8 warps keep 255 registers/thread available.
  auto produce = [&](int kf) {
    const int st = kf % STAGES;
    if (kf >= STAGES) mbar_wait(&empty[st], ((kf / STAGES) - 1) & 1);
    mbar_expect_tx(&full[st], L::kATile + L::kBTile);
    tma_load_2d(sA + st * L::kAStride, &tmA, &full[st], (kt_begin + kf) * GEMM_BK, m0);
    tma_load_2d(sB + st * L::kBStride, &tmB, &full[st], (kt_begin + kf) * GEMM_BK, n0);
  };
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int kf = 0; kf < STAGES - 1 && kf < KT; ++kf) produce(kf);
  }

  // ---------------- consumers
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const int g = lane >> 2, q = lane & 3;
  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // K2: this warp's 32 columns take the squared A operand iff they lie in the D block (nsq % 32 == 0)
  const bool warp_sq = SQ && (n0 + wn * WN >= s.nsq);

  // K order inside a 16-wide stage: mma step ks, lane quad-index q reads k = 2 ks + (q & 1) + 8 (q >> 1).
  // Any bijection is valid (A and B use the same one); this one makes every half-warp's 16 64-bit fragment reads
  // hit 16 distinct 8-byte slots of the 128B-swizzled rows (the natural k = 4 ks + q is 2-way bank-conflicted).
  uint32_t off_f64[GEMM_BK / 4], off_u8[GEMM_BK / 4];
#pragma unroll
  for (int ks = 0; ks < GEMM_BK / 4; ++ks) {
    const int k = 2 * ks + (q & 1) + 8 * (q >> 1);
    off_f64[ks] = swz128_off(g, k);
    off_u8[ks] = (uint32_t)(g * GEMM_BK + k);
  }
  const uint32_t a_row0 = (uint32_t)(wm * WM) * ATile<TA>::kBytesPerRow;
  const uint32_t b_row0 = (uint32_t)(wn * WN) * (GEMM_BK * 8);

  // Fragment loads for mma step ks of a stage (A through the u8 -> f64 table or directly; B always f64).
  auto load_frags = [&](double (&a)[MI], double (&b)[NI], int st, int ks) {
    const uint8_t* a_tile = sA + st * L::kAStride + a_row0;
    const uint8_t* b_tile = sB + st * L::kBStride + b_row0;
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      if constexpr (sizeof(TA) == 1) {
        a[i] = lut[a_tile[off_u8[ks] + i * 8 * GEMM_BK]];
      } else {
        a[i] = *reinterpret_cast<const double*>(a_tile + off_f64[ks] + i * 8 * 128);
      }
    }
#pragma unroll
    for (int j = 0; j < NI; ++j) b[j] = *reinterpret_cast<const double*>(b_tile + off_f64[ks] + j * 8 * 128);
  };

  // The mainloop is instantiated twice so the K2 squaring is a warp-uniform choice made once, outside the loop
  // (a per-iteration branch compiles to predicated DMULs that still occupy the shared FP64/DMMA dispatch).
  // Fragments are register double-buffered one mma step ahead, across stage boundaries too: the first step of
  // stage kt+1 is loaded (after its full-barrier wait) while the last step of stage kt is in the DMMA pipe.
  auto mainloop = [&](auto square_tag) {
    constexpr bool SQUARE = decltype(square_tag)::value;
    auto mma_step = [&](double (&a)[MI], double (&b)[NI]) {
      if constexpr (SQUARE) {
#pragma unroll
        for (int i = 0; i < MI; ++i) a[i] = a[i] * a[i];
      }
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma_8x8x4(acc[i][j], a[i], b[j]);
    };
    static_assert(GEMM_BK / 4 == 4, "the step schedule below assumes 4 mma steps per stage");
    double a0[MI], b0[NI], a1[MI], b1[NI];
    mbar_wait(&full[0], 0);
    load_frags(a0, b0, 0, 0);
    for (int kt = 0; kt < KT; ++kt) {
      const int st = kt % STAGES;
      if (threadIdx.x == 0 && kt >= 1 && kt + STAGES - 2 < KT) produce(kt + STAGES - 2);
      __syncwarp();
      load_frags(a1, b1, st, 1);
      mma_step(a0, b0);
      load_frags(a0, b0, st, 2);
      mma_step(a1, b1);
      load_frags(a1, b1, st, 3);
      mma_step(a0, b0);
      if (kt + 1 < KT) {
        const int nst = (kt + 1) % STAGES;
        mbar_wait(&full[nst], ((kt + 1) / STAGES) & 1);
        load_frags(a0, b0, nst, 0);
      }
      mma_step(a1, b1);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
  };
  if (SQ && warp_sq)
    mainloop(std::true_type{});
  else
    mainloop(std::false_type{});

  if constexpr (FUSE) {
    // ---------------- fused K2 epilogue: per-tile partial contractions with the K2 operand rows
    __syncthreads();  // every warp is done with the stage buffers: reuse them for the cross-warp reduction
    const int nq = s.fnq;
    double* red = reinterpret_cast<double*>(smem);  // [WARPS_N][BM][fnq]
    double* bsl = red + WARPS_N * BM * nq;          // [fnq][BN]: the tile's slice of the K2 operand rows
    // one cooperative, coalesced load of the slice (a single L2 round trip instead of one per column)
    for (int idx = threadIdx.x; idx < nq * BN; idx += GEMM_THREADS) {
      const int qq = idx / BN, col = n0 + (idx - qq * BN);
      const int brow = qq < s.fnlin ? qq : s.fnsq + (qq - s.fnlin);
      bsl[idx] = col < s.N ? __ldg(s.fB + (long long)brow * s.fldb + col) : 0.0;
    }
    __syncthreads();
    for (int qq = 0; qq < nq; ++qq) {
      const bool sqc = qq >= s.fnlin;
      double bv[NI][2];
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        const double2 b2 = *reinterpret_cast<const double2*>(bsl + qq * BN + wn * WN + j * 8 + 2 * q);
        bv[j][0] = b2.x;
        bv[j][1] = b2.y;
      }
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        double sum = 0.0;
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          const double a0 = sqc ? acc[i][j][0] * acc[i][j][0] : acc[i][j][0];
          const double a1 = sqc ? acc[i][j][1] * acc[i][j][1] : acc[i][j][1];
          sum = fma(a0, bv[j][0], sum);
          sum = fma(a1, bv[j][1], sum);
        }
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        sum += __shfl_xor_sync(0xffffffffu, sum, 2);
        if (q == 0) red[((long long)wn * BM + wm * WM + i * 8 + g) * nq + qq] = sum;
      }
    }
    __syncthreads();
    double* P = s.fP + (long long)tn * s.fP_stride;
    for (int idx = threadIdx.x; idx < BM * nq; idx += GEMM_THREADS) {
      const int r = idx / nq;
      if (m0 + r >= s.M) continue;
      double v = red[idx];
#pragma unroll
      for (int w2 = 1; w2 < WARPS_N; ++w2) v += red[(long long)w2 * BM * nq + idx];
      P[(long long)(m0 + r) * nq + (idx - r * nq)] = v;
    }
  } else if (s.ctiled) {
    // ---------------- epilogue, trait-tiled C: the lane's 2 NI column offsets are row-independent
    // one integer division per thread: the warp's 32 columns span at most one field boundary (ct >= 32)
    const int cw = n0 + wn * WN;
    const int fb = min(cw, s.cnlin - 1) / s.ct;
    long long coff[NI][2];
#pragma unroll
    for (int j = 0; j < NI; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = cw + j * 8 + 2 * q + e;
        long long o = -1;
        if (col < s.N) {
          if (col < s.cnlin) {
            const int f = fb + (col >= (fb + 1) * s.ct ? 1 : 0);
            o = ctile_off(col - f * s.ct, f, s.cF);
          } else if (col >= s.nsq) {
            o = ctile_off(col - s.nsq, s.cF - 1, s.cF);
          }
        }
        coff[j][e] = o;
      }
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int row = m0 + wm * WM + i * 8 + g;
      if (row >= s.M) continue;
      double* crow = s.C + (long long)row * s.ldc;
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        const long long o0 = coff[j][0], o1 = coff[j][1];
        if (o0 >= 0 && o1 == o0 + 1 && !(o0 & 1)) {
          *reinterpret_cast<double2*>(crow + o0) = make_double2(acc[i][j][0], acc[i][j][1]);
        } else {
          if (o0 >= 0) crow[o0] = acc[i][j][0];
          if (o1 >= 0) crow[o1] = acc[i][j][1];
        }
      }
    }
  } else {
    // ---------------- epilogue: each lane owns C[row][2q, 2q+1] of every 8x8 fragment
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int row = m0 + wm * WM + i * 8 + g;
      if (row >= s.M) continue;
      double* crow = s.C + split * s.split_stride + (long long)row * s.ldc;
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        const int col = n0 + wn * WN + j * 8 + 2 * q;
        if (col + 1 < s.N) {
          *reinterpret_cast<double2*>(crow + col) = make_double2(acc[i][j][0], acc[i][j][1]);
        } else if (col < s.N) {
          crow[col] = acc[i][j][0];
        }
      }
    }
  }
}

}  // namespace gw
