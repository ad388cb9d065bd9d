// libgwas.so -- C-ABI and runtime of the B200-native CLAK-Eig GLS-sequence hot path.
// See include/gwas.h for the contract and DESIGN.md for the design; the kernels live in gemm_dmma.cuh (K1/K2),
// schur.cuh (K3) and setup_kernels.cuh.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cusolverDn.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/gwas.h"
#include "gemm_dmma.cuh"
#include "estimate_launch.cuh"
#include "gemm_i8.cuh"
#include "lowrank_k3.cuh"
#include "schur.cuh"
#include "setup_kernels.cuh"

namespace {

constexpr uint64_t kMagic = 0x4b414c4353415747ull;  // "GWASCLAK"
constexpr int64_t kVersion = 2;  // state layout: 2 adds the low-rank weights and 7-digit int8 fields
constexpr int kPMax = 12;
constexpr int kWideSplitN = 1024;   // widest fp64 product split 2-way along K (int8 K2b; gemm_tn wide_split)
constexpr int kLrMax = 64;          // largest trait-weight rank kept (low-rank mode)
constexpr double kLrTol = 1e-15;    // singular values of D below kLrTol * s_0 are dropped (reading L1)

thread_local std::string g_err;

gwas_status fail(gwas_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CKC(x)                                                                                  \
  do {                                                                                          \
    cudaError_t e__ = (x);                                                                      \
    if (e__ != cudaSuccess) return fail(GWAS_E_CUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e__), \
                                        __FILE__, __LINE__);                                    \
  } while (0)

#define CKS(x)                                                                                     \
  do {                                                                                             \
    cusolverStatus_t s__ = (x);                                                                    \
    if (s__ != CUSOLVER_STATUS_SUCCESS) return fail(GWAS_E_CUDA, "%s: cusolver status %d", #x, (int)s__); \
  } while (0)

#define CKG(x)                              \
  do {                                      \
    gwas_status g__ = (x);                  \
    if (g__ != GWAS_OK) return g__;         \
  } while (0)

// Environment knob set to something other than "" / "0" (include/gwas.h lists the knobs).
inline bool env_flag(const char* name) {
  const char* e = getenv(name);
  return e && e[0] && !(e[0] == '0' && e[1] == 0);
}

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }
inline size_t align256(size_t a) { return (a + 255) / 256 * 256; }

struct StateHeader {
  uint64_t magic;
  int64_t version;
  int64_t n, p, t, kpad, nsq, n2;
  int32_t output_mode, var_convention;
  double eps_collinear;
  int64_t off_Z, off_W, off_B2, off_Lpk, off_v, off_s2, off_betaT, off_dinv, total;
  int32_t int8_slices, algorithm;
  int64_t na_pad, nlin, nlin_pad, off_dig, off_exps;  // int8-sliced mode: digit matrix of [Z | Z B_op] + 2^e
  // low-rank trait weights (opt.trait_rank): D ~ U_r W with r = lr_r (0: exact D); B2 then holds
  // [U_r (.) X_L'_f (p r rows) | d_j (.) y'_j (t rows) | pad to lr_nsq | U_r (r rows)], W^T at off_wt (t x r)
  int32_t trait_rank, lr_r;
  int64_t lr_nsq, lr_nlin, off_wt;
  double lr_s0, lr_sr;  // largest kept / first dropped singular value of D (diagnostics)
};
constexpr size_t kHeaderBytes = 512;
static_assert(sizeof(StateHeader) <= kHeaderBytes, "header");

struct Dims {
  int64_t n, p, t, kpad, nsq, n2, ldc2, lds, kb;
  size_t es;
  int64_t per_pair;                // outputs per pair: 1 (SNP mode) or p + 1 (full mode)
  int i8;                          // int8-sliced mode
  int64_t na_pad, nlin, nlin_pad;  // digit-matrix column blocks (multiples of 64)
  bool lr;                         // low-rank trait weights requested (state reserves room; setup decides r)
  int64_t ldg2;                    // low-rank K2 output row stride (p rmax + t + 32 + rmax)
  bool fuse;                       // K2 fused into K1's epilogue (few traits, opt.fuse_k2)
  bool ctiled;                     // K2 output C in the trait-tiled layout (ctile.cuh): FP64 exact weights, t >= 32
  int64_t fnq, ftiles;             // fused K2 columns per pair-row; max K1 column tiles (partials per block)
};

Dims make_dims(int64_t n, int64_t p, int64_t t, const gwas_options* o) {
  Dims d;
  d.n = n;
  d.p = p;
  d.t = t;
  d.kpad = round_up(n, 16);
  d.nsq = round_up(t * (p + 1), 32);
  d.n2 = d.nsq + t;
  d.ldc2 = round_up(d.n2, 2);
  d.lds = round_up(t * (p + 1), 2);
  d.kb = o->block_cols > 0 ? o->block_cols : 8192;  // 0 (auto): set below, once the product shapes are known
  d.es = o->xr_dtype == GWAS_XR_U8 ? 1 : 8;
  d.i8 = o->int8_slices != 0;
  d.per_pair = o->output_mode == GWAS_OUT_FULL ? p + 1 : 1;
  d.na_pad = round_up(n, gw::I8_NB);
  d.nlin = t * (p + 1);
  d.nlin_pad = round_up(d.nlin, gw::I8_NB);
  // NEXT-2 fusion: FP64 mode contracts all t (p + 2) K2 columns in K1's epilogue, the int8 mode only the t squared
  // columns (its linear K2 terms already come out of K1i)
  d.lr = o->trait_rank != 0 && o->algorithm == GWAS_ALG_EIG;
  d.ldg2 = round_up(p * kLrMax + t + 32 + kLrMax, 2);
  d.fnq = d.i8 ? t : t * (p + 2);
  d.fuse = o->fuse_k2 != 0 && (d.i8 ? t <= gw::I8_FUSE_T : d.fnq <= gw::FUSE_MAX_NQ);
  d.ftiles = d.i8 ? d.na_pad / gw::I8_NB : (n + 63) / 64;
  d.ctiled = !d.i8 && !d.lr && !d.fuse && t >= 32;
  if (d.ctiled) d.ldc2 = gw::ctile_ld((int)t, (int)p + 2);
  return d;
}

StateHeader make_header(const Dims& d, const gwas_options* o) {
  StateHeader h;
  memset(&h, 0, sizeof(h));
  h.magic = kMagic;
  h.version = kVersion;
  h.n = d.n;
  h.p = d.p;
  h.t = d.t;
  h.kpad = d.kpad;
  h.nsq = d.nsq;
  h.n2 = d.n2;
  h.output_mode = o->output_mode;
  h.var_convention = o->var_convention;
  h.eps_collinear = o->eps_collinear;
  size_t off = kHeaderBytes;
  auto take = [&](size_t bytes) {
    size_t r = off;
    off = align256(off + bytes);
    return (int64_t)r;
  };
  h.off_Z = take(sizeof(double) * d.kpad * d.kpad);
  h.off_W = take(sizeof(double) * d.kpad);
  h.off_B2 = take(sizeof(double) * d.n2 * d.kpad);
  const int64_t npk = d.p * (d.p + 1) / 2;
  h.off_Lpk = take(sizeof(double) * npk * d.t);
  h.off_v = take(sizeof(double) * d.p * d.t);
  h.off_s2 = take(sizeof(double) * d.t);
  h.off_betaT = take(sizeof(double) * d.p * d.t);
  h.off_dinv = take(sizeof(double) * d.p * d.t);
  h.int8_slices = o->int8_slices;
  h.algorithm = o->algorithm;
  h.na_pad = d.na_pad;
  h.nlin = d.nlin;
  h.nlin_pad = d.nlin_pad;
  if (d.i8) {
    h.off_dig = take((size_t)((d.na_pad + d.nlin_pad) / gw::I8_NB) * o->int8_slices * gw::I8_NB * d.kpad);
    h.off_exps = take(sizeof(int) * (d.na_pad + d.nlin_pad));
  }
  h.trait_rank = o->trait_rank;
  h.lr_r = 0;            // exact weights until setup decides otherwise
  h.lr_nsq = d.nsq;
  h.lr_nlin = d.nlin;
  if (d.lr) h.off_wt = take(sizeof(double) * d.t * kLrMax);
  h.total = (int64_t)off;
  return h;
}

struct RunLayout {
  size_t stage[2], xrp[2], c2[2], split[2], outb[2], fp[2], g2[2], wsplit[2], total;
  size_t out_bytes;  // per staging set: b, var (8 * per_pair each) + status (1) per pair of a block
};
// overlap mode double-buffers the rotated block and the K2 output so block b+1's K1 can run beside block b's K2/K3
RunLayout run_layout(const Dims& d, bool overlap) {
  RunLayout r;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t x = off;
    off = align256(off + bytes);
    return x;
  };
  r.stage[0] = take(d.es * d.kpad * d.kb);
  r.stage[1] = take(d.es * d.kpad * d.kb);
  r.xrp[0] = take(sizeof(double) * d.kpad * d.kb);
  r.c2[0] = take(sizeof(double) * d.ldc2 * d.kb);
  r.xrp[1] = overlap ? take(sizeof(double) * d.kpad * d.kb) : r.xrp[0];
  r.c2[1] = overlap ? take(sizeof(double) * d.ldc2 * d.kb) : r.c2[0];
  r.split[0] = take(sizeof(double) * 8 * 64 * d.kb);  // split-K partials of skinny K2 products (kSplitMax x kSplitLd)
  r.split[1] = overlap ? take(sizeof(double) * 8 * 64 * d.kb) : r.split[0];
  // host-output mode: each block's b / var / status land here and stream to pinned host memory on the D2H stream
  r.out_bytes = (size_t)d.kb * d.t * (16 * d.per_pair + 1);
  r.outb[0] = take(r.out_bytes);
  r.outb[1] = take(r.out_bytes);
  r.wsplit[0] = r.wsplit[1] = 0;
  if (d.i8 && d.t > 64 && d.t <= kWideSplitN && d.n >= 4096) {  // 2-way K split of K2b (gemm_tn wide_split)
    r.wsplit[0] = take(sizeof(double) * 2 * round_up(d.t, 2) * d.kb);
    r.wsplit[1] = overlap ? take(sizeof(double) * 2 * round_up(d.t, 2) * d.kb) : r.wsplit[0];
  }
  r.g2[0] = r.g2[1] = 0;
  if (d.lr) {  // low-rank K2 output [U_r-projected fields | y | pad | squared]
    r.g2[0] = take(sizeof(double) * d.ldg2 * d.kb);
    r.g2[1] = overlap ? take(sizeof(double) * d.ldg2 * d.kb) : r.g2[0];
  }
  r.fp[0] = r.fp[1] = 0;
  if (d.fuse) {  // per-tile partial sums of the fused K2
    r.fp[0] = take(sizeof(double) * d.ftiles * d.kb * d.fnq);
    r.fp[1] = overlap ? take(sizeof(double) * d.ftiles * d.kb * d.fnq) : r.fp[0];
  }
  r.total = off;
  return r;
}

struct SetupLayout {
  size_t xlpad, ypad, xlp, yp, stl, h2, s2, err, info, est_rec, est_ll, est_gs, work, zt, blin, total;
  size_t lr_a, lr_u, lr_vt, lr_s, lr_work, lr_b2;  // low-rank: SVD of D and the rebuilt operand
};
SetupLayout setup_layout(const Dims& d, int64_t lwork, int64_t lr_lwork = 0) {
  SetupLayout s;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t x = off;
    off = align256(off + bytes);
    return x;
  };
  s.xlpad = take(sizeof(double) * d.p * d.kpad);
  s.ypad = take(sizeof(double) * d.t * d.kpad);
  s.xlp = take(sizeof(double) * d.p * d.kpad);
  s.yp = take(sizeof(double) * d.t * d.kpad);
  s.stl = take(sizeof(double) * d.p * d.lds);
  s.h2 = take(sizeof(double) * d.t);
  s.s2 = take(sizeof(double) * d.t);
  s.err = take(sizeof(unsigned long long) * 4);
  s.info = take(sizeof(int) * 4);
  s.est_rec = take(sizeof(double) * (gw::EST_GRID + 1) * gw::est_rec((int)d.p));
  s.est_ll = take(sizeof(double) * d.t);
  s.est_gs = take(sizeof(int) * d.t);
  s.work = take(sizeof(double) * (size_t)std::max<int64_t>(lwork, 1));
  s.zt = s.blin = 0;
  if (d.i8) {  // Z^T and B_lin = Z B_op (reuse the dsyevd workspace region's tail: allocated after it)
    s.zt = take(sizeof(double) * d.kpad * d.kpad);
    s.blin = take(sizeof(double) * d.nlin * d.kpad);
  }
  s.lr_a = s.lr_u = s.lr_vt = s.lr_s = s.lr_work = s.lr_b2 = 0;
  if (d.lr) {
    s.lr_a = take(sizeof(double) * d.kpad * d.t);
    s.lr_u = take(sizeof(double) * d.kpad * d.t);
    s.lr_vt = take(sizeof(double) * d.t * d.t);
    s.lr_s = take(sizeof(double) * d.t);
    s.lr_work = take(sizeof(double) * std::max<int64_t>(lr_lwork, 1));
    s.lr_b2 = take(sizeof(double) * d.n2 * d.kpad);
  }
  s.total = off;
  return s;
}

gwas_status check_sizes(int64_t n, int64_t p, int64_t t, const gwas_options* o) {
  if (!o) return fail(GWAS_E_ARG, "options is NULL");
  if (p < 1 || p > kPMax) return fail(GWAS_E_ARG, "p = %lld outside [1, %d]", (long long)p, kPMax);
  if (t < 1) return fail(GWAS_E_ARG, "t = %lld < 1", (long long)t);
  if (n < p + 1) return fail(GWAS_E_ARG, "n = %lld < p + 1 = %lld", (long long)n, (long long)p + 1);
  if (n > (1ll << 31) / 16) return fail(GWAS_E_ARG, "n = %lld too large", (long long)n);
  if (o->xr_dtype != GWAS_XR_F64 && o->xr_dtype != GWAS_XR_U8) return fail(GWAS_E_ARG, "bad xr_dtype");
  if (o->output_mode != GWAS_OUT_SNP && o->output_mode != GWAS_OUT_FULL) return fail(GWAS_E_ARG, "bad output_mode");
  if (o->var_convention != GWAS_VAR_TEXTBOOK && o->var_convention != GWAS_VAR_LITERAL)
    return fail(GWAS_E_ARG, "bad var_convention");
  if (o->block_cols < 0 || o->block_cols > (1ll << 20)) return fail(GWAS_E_ARG, "bad block_cols (0 or <= 2^20)");
  if (!(o->eps_spd >= 0) || !(o->eps_collinear >= 0)) return fail(GWAS_E_ARG, "bad eps");
  const int64_t t_p2 = t * (p + 2) + 8;
  if (t_p2 > (1ll << 31) - 1) return fail(GWAS_E_ARG, "t too large");
  if (o->algorithm != GWAS_ALG_EIG && o->algorithm != GWAS_ALG_CHOL) return fail(GWAS_E_ARG, "bad algorithm");
  if (o->trait_rank != 0 && o->trait_rank != -1) return fail(GWAS_E_ARG, "trait_rank must be 0 (exact) or -1 (auto)");
  if (o->algorithm == GWAS_ALG_CHOL && t != 1)
    return fail(GWAS_E_ARG, "CLAK-Chol (Alg. 3) is the single-trait algorithm: t = %lld != 1", (long long)t);
  if (o->int8_slices != 0) {
    if (o->int8_slices != 7 && o->int8_slices != 8)
      return fail(GWAS_E_ARG, "int8_slices = %d unsupported (0, 7 or 8)", o->int8_slices);
    if (o->xr_dtype != GWAS_XR_U8) return fail(GWAS_E_ARG, "int8-sliced mode needs uint8 X_R (exact dosages)");
    if (n > 66000) return fail(GWAS_E_ARG, "int8-sliced mode: n = %lld > 66000 (int32 accumulator bound)", (long long)n);
  }
  return GWAS_OK;
}

// Device workspace (in doubles) of the setup factorisation: dsyevd (CLAK-Eig), or for CLAK-Chol the n x n matrix M
// (kpad x kpad) followed by max(dpotrf, dtrtri) workspace.  *host_bytes: dtrtri's host workspace.
gwas_status solver_lwork(const gwas_options* o, int64_t n, int64_t kpad, int64_t* lwork, size_t* host_bytes) {
  CKC(cudaSetDevice(o->device));
  cusolverDnHandle_t h;
  CKS(cusolverDnCreate(&h));
  *host_bytes = 0;
  cusolverStatus_t s = CUSOLVER_STATUS_SUCCESS;
  if (o->algorithm == GWAS_ALG_CHOL) {
    int lw = 0;
    size_t dev_b = 0, host_b = 0;
    s = cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, (int)n, nullptr, (int)kpad, &lw);
    if (s == CUSOLVER_STATUS_SUCCESS)
      s = cusolverDnXtrtri_bufferSize(h, CUBLAS_FILL_MODE_LOWER, CUBLAS_DIAG_NON_UNIT, n, CUDA_R_64F, nullptr, kpad,
                                      &dev_b, &host_b);
    *lwork = kpad * kpad + std::max<int64_t>(lw, (int64_t)((dev_b + 7) / 8)) + 64;
    *host_bytes = host_b;
  } else {
    int lw = 0;
    s = cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)n, nullptr, (int)kpad,
                                    nullptr, &lw);
    *lwork = lw;
  }
  cusolverDnDestroy(h);
  if (s != CUSOLVER_STATUS_SUCCESS) return fail(GWAS_E_CUDA, "cuSOLVER bufferSize status %d", (int)s);
  return GWAS_OK;
}

// Device workspace (doubles) of cusolverDnDgesvd on the n x t trait-weight matrix D (low-rank mode), 0 if unused.
gwas_status lr_lwork(const gwas_options* o, const Dims& d, int64_t* lwork) {
  *lwork = 0;
  if (!d.lr) return GWAS_OK;
  CKC(cudaSetDevice(o->device));
  cusolverDnHandle_t h;
  CKS(cusolverDnCreate(&h));
  int lw = 0;
  // gesvd needs m >= n: D (n x t) itself, or D^T when t > n
  cusolverStatus_t st = d.t <= d.n ? cusolverDnDgesvd_bufferSize(h, (int)d.n, (int)d.t, &lw)
                                   : cusolverDnDgesvd_bufferSize(h, (int)d.t, (int)d.n, &lw);
  cusolverDnDestroy(h);
  if (st != CUSOLVER_STATUS_SUCCESS) return fail(GWAS_E_CUDA, "cusolverDnDgesvd_bufferSize status %d", (int)st);
  *lwork = lw;
  return GWAS_OK;
}

// ------------------------------------------------------------------ TMA descriptors + GEMM launch
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

gwas_status get_encoder() {
  if (g_encode) return GWAS_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CKC(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (q != cudaDriverEntryPointSuccess || !fn) return fail(GWAS_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return GWAS_OK;
}

// 2-D K-contiguous operand: rows x K elements, leading dimension ld (elements); box = 16 x box_rows.
gwas_status make_map(CUtensorMap* map, const void* ptr, bool u8, int64_t K, int64_t rows, int64_t ld, int box_rows,
                     int box_k = gw::GEMM_BK, int swizzle = -1) {
  CKG(get_encoder());
  const size_t es = u8 ? 1 : 8;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * es)};
  cuuint32_t box[2] = {(cuuint32_t)box_k, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || ((ld * es) & 15))
    return fail(GWAS_E_ARG, "operand not 16-byte aligned (ptr %p, ld %lld)", ptr, (long long)ld);
  CUresult r = g_encode(map, u8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                        const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle >= 0 ? (CUtensorMapSwizzle)swizzle
                                     : (u8 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B),
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(GWAS_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return GWAS_OK;
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device (per-context) setting: remember, per kernel
// instantiation, the devices it has been set on (bit d of `mask`).  Setting it twice (two threads racing on a
// fresh device) is harmless: the call is idempotent.
template <typename Kern>
gwas_status ensure_smem_attr(Kern kern, size_t smem, std::atomic<uint64_t>& mask) {
  int dev = 0;
  CKC(cudaGetDevice(&dev));
  const uint64_t bit = 1ull << (dev & 63);
  if (mask.load(std::memory_order_acquire) & bit) return GWAS_OK;
  CKC(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  mask.fetch_or(bit, std::memory_order_acq_rel);
  return GWAS_OK;
}

constexpr int kBM = 128;
constexpr int kStagesU8 = 8, kStagesF64 = 6, kStagesF64N64 = 8;

template <typename TA, int BN, int STAGES>
constexpr size_t gemm_smem_bytes() {
  using L = gw::GemmSmem<TA, kBM, BN>;
  return 1024 + STAGES * (L::kAStride + L::kBStride) + 2 * STAGES * sizeof(uint64_t) + 256 * sizeof(double);
}

template <typename TA, int BN, int STAGES, bool SQ, bool FUSE = false>
gwas_status launch_gemm_t(const CUtensorMap& ma, const CUtensorMap& mb, const gw::GemmShape& s, cudaStream_t st) {
  static std::atomic<uint64_t> attr_devs{0};  // per instantiation, per device
  constexpr size_t smem = gemm_smem_bytes<TA, BN, STAGES>();
  static_assert(!FUSE || (size_t)((BN / 32) * kBM + BN) * gw::FUSE_MAX_NQ * 8 <=
                             (size_t)STAGES * (gw::GemmSmem<TA, kBM, BN>::kAStride + gw::GemmSmem<TA, kBM, BN>::kBStride),
                "fused-K2 reduction buffer must fit in the stage buffers");
  auto kern = gw::gemm_tn_dmma<TA, kBM, BN, STAGES, SQ, FUSE>;
  CKG(ensure_smem_attr(kern, smem, attr_devs));
  const int grid = s.tiles_m * s.tiles_n * s.ksplit;
  kern<<<grid, gw::GEMM_THREADS, smem, st>>>(ma, mb, s);
  CKC(cudaGetLastError());
  return GWAS_OK;
}

// Output-tile width (128 or 64 columns) of the DMMA kernel for an M x N product.
//   - 64 wide when 128 x 128 tiles would give fewer than 4 waves on 148 SMs (e.g. K2b, N = t): the wave tail
//     dominates there, not the extra fragment loads of the narrower warp tiles (GWAS_BN64_WAVES overrides the
//     4-wave threshold; 0 = always 128 wide; tuning knob).
//   - fp64 A (one CTA per SM either way): whole waves compared, a 64-wide tile doing half the work of a 128-wide
//     one at ~93 % of its efficiency (measured on K2b, C4: 5.36 ms at 128 vs 5.04 ms at 64 wide).
//   - fused K2: the per-tile partials are summed over the column tiles, so the tile width fixes the rounding of the
//     K2 terms.  It is chosen from N alone -- the width a full 8192-column block would get -- so results stay bitwise
//     invariant to the block size and to shard edges (a short tail block gets the same tiles).
//   - wide_split (medium-width fp64 products with a long K: the int8 mode's K2b at t <= 1024, n >= 4096): 128-wide
//     tiles split 2-way along K (fixed halves, chosen from N and K only) instead of 64-wide tiles.
int bn64_waves() {
  static const int w = [] {
    const char* e = getenv("GWAS_BN64_WAVES");
    return e ? atoi(e) : 4;
  }();
  return w;
}

int choose_bn(bool a_u8, int64_t M, int64_t N, bool fuse, bool wide_split) {
  if (wide_split) return 128;
  if (N <= 64) return 64;
  if (fuse) return (8192 / kBM) * ((N + 127) / 128) < (int64_t)bn64_waves() * 148 ? 64 : 128;
  const int64_t tiles128 = ((M + kBM - 1) / kBM) * ((N + 127) / 128);
  if (!a_u8 && !getenv("GWAS_BN64_WAVES")) {
    const int64_t tiles64 = ((M + kBM - 1) / kBM) * ((N + 63) / 64);
    const double cost128 = (double)((tiles128 + 147) / 148), cost64 = (double)((tiles64 + 147) / 148) * 0.5 / 0.93;
    return cost64 < cost128 ? 64 : 128;
  }
  return tiles128 < (int64_t)bn64_waves() * 148 ? 64 : 128;
}

// Relative time of one M-row DMMA product of width N on `sms` SMs: whole waves of CTAs, a wave costing the CTA slots
// it occupies (a 64-wide tile is half a 128-wide one, at ~93 % of its efficiency; u8-A 64-wide tiles run two per SM).
double dmma_wave_cost(bool a_u8, int64_t M, int64_t N, bool fuse, int sms) {
  const int bn = choose_bn(a_u8, M, N, fuse, false);
  const int per_sm = (a_u8 && bn == 64) ? 2 : 1;
  const int64_t tiles = ((M + kBM - 1) / kBM) * ((N + bn - 1) / bn);
  const int64_t slots = (int64_t)sms * per_sm;
  const double waves = (double)((tiles + slots - 1) / slots);
  return waves * (double)slots * bn / 128.0 / (double)per_sm / (bn == 64 ? 0.93 : 1.0);
}

// block_cols = 0 (auto): the k in [4096, 16384] (a multiple of 128) that minimises the wave-quantised time per SNP
// column of the block's DMMA products -- K1 (M = k, N = n, u8 or fp64 A, with K2 fused when it is) and the unfused
// K2 (M = k, N = t(p+2) rounded as in the state, fp64 A) -- both with K = n.  Ties go to the k closest to 8192.
// The int8-sliced mode keeps 8192.  Results do not depend on k (fixed K order, no split chosen from M).
int64_t auto_block_cols(const Dims& d, const gwas_options* o) {
  if (d.i8) return 8192;
  int sms = 148;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, o->device) != cudaSuccess || sms <= 0) {
    cudaGetLastError();
    sms = 148;
  }
  const bool u8 = d.es == 1;
  int64_t best = 8192;
  double best_cost = 1e300;
  for (int64_t k = 4096; k <= 16384; k += kBM) {
    double cost = dmma_wave_cost(u8, k, d.n, d.fuse, sms);
    if (!d.fuse) cost += dmma_wave_cost(false, k, d.n2, false, sms);
    cost /= (double)k;
    const bool better = cost < best_cost * (1.0 - 1e-9) ||
                        (cost <= best_cost * (1.0 + 1e-9) && std::llabs(k - 8192) < std::llabs(best - 8192));
    if (better) {
      best = k;
      best_cost = cost;
    }
  }
  return best;
}

Dims make_dims_kb(int64_t n, int64_t p, int64_t t, const gwas_options* o) {
  Dims d = make_dims(n, p, t, o);
  if (o->block_cols == 0) d.kb = auto_block_cols(d, o);
  return d;
}

// C[M x N] (row-major, ldc) = A[M x K] (rows K-contiguous, lda) * B[N x K]^T (rows K-contiguous, ldb)
// group_m: rasterisation group along M (consecutive CTAs sweep group_m row tiles, then move along N): large for
// K1 (the u8 X_R panels of a whole block stay in L2 while Z streams through once), small for K2.
// split_scratch (optional, >= kSplitMax * M * kSplitLd doubles): skinny products (N <= 64, one column tile, K >= 256)
// are split along K into fixed ranges (independent of M, so results stay bitwise invariant to the block size)
// and summed in fixed order.
constexpr int kSplitMax = 8, kSplitLd = 64;
// fuse (optional): K2 fused into the epilogue (GemmShape's f* fields; C is then not written, see gemm_dmma.cuh).
gwas_status gemm_tn(bool a_u8, const void* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                    int64_t M, int64_t N, int64_t K, int64_t nsq, cudaStream_t st, int group_m = 16,
                    double* split_scratch = nullptr, bool tri = false, const gw::GemmShape* fuse = nullptr,
                    int* tiles_n_out = nullptr, double* wide_split_scratch = nullptr,
                    const gw::GemmShape* ctile = nullptr) {
  if (M <= 0 || N <= 0) return GWAS_OK;
  if (K <= 0) return fail(GWAS_E_ARG, "gemm K = %lld", (long long)K);
  if ((ldc & 1) || (reinterpret_cast<uintptr_t>(C) & 15)) return fail(GWAS_E_ARG, "C not 16-byte aligned / ldc odd");
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return fail(GWAS_E_ARG, "gemm dims too large");
  // 128 x 64 tiles when 128 x 128 tiles would give fewer than 4 waves on 148 SMs (e.g. K2b, N = t):
  // the wave tail dominates there, not the extra fragment loads of the narrower warp tiles
  // GWAS_BN64_WAVES overrides the 4-wave threshold (0 = always 128 wide; tuning knob).
  const int kt_all0 = (int)((K + gw::GEMM_BK - 1) / gw::GEMM_BK);
  const bool wide_split = wide_split_scratch && !fuse && !a_u8 && N > 64 && N <= kWideSplitN && kt_all0 >= 256;
  const int bn = choose_bn(a_u8, M, N, fuse, wide_split);
  CUtensorMap ma, mb;
  CKG(make_map(&ma, A, a_u8, K, M, lda, kBM));
  CKG(make_map(&mb, B, false, K, N, ldb, bn));
  gw::GemmShape s;
  s.M = (int)M;
  s.N = (int)N;
  s.K = (int)K;
  s.C = C;
  s.ldc = ldc;
  s.nsq = (int)std::min<int64_t>(nsq, N);
  s.tiles_m = (int)((M + kBM - 1) / kBM);
  s.tiles_n = (int)((N + bn - 1) / bn);
  if (tiles_n_out) *tiles_n_out = s.tiles_n;
  s.group_m = std::max(1, group_m);
  const int kt_all = (int)((K + gw::GEMM_BK - 1) / gw::GEMM_BK);
  s.ksplit = 1;
  s.kt_per_split = kt_all;
  s.split_stride = 0;
  s.tri = tri ? 1 : 0;
  s.fB = nullptr;
  s.fldb = 0;
  s.fnq = s.fnlin = s.fnsq = 0;
  s.fP = nullptr;
  s.fP_stride = 0;
  s.ctiled = 0;
  s.ct = s.cnlin = s.cF = 0;
  if (ctile) {  // C in the trait-tiled layout (ctile.cuh); no split along K for these (wide) products
    if (fuse || N <= kSplitLd || wide_split) return fail(GWAS_E_ARG, "trait-tiled C needs a plain wide product");
    s.ctiled = 1;
    s.ct = ctile->ct;
    s.cnlin = ctile->cnlin;
    s.cF = ctile->cF;
  }
  if (fuse) {
    if (nsq < N || fuse->fnq > gw::FUSE_MAX_NQ || fuse->fnq < 1) return fail(GWAS_E_ARG, "bad fused-K2 shape");
    s.fB = fuse->fB;
    s.fldb = fuse->fldb;
    s.fnq = fuse->fnq;
    s.fnlin = fuse->fnlin;
    s.fnsq = fuse->fnsq;
    s.fP = fuse->fP;
    s.fP_stride = fuse->fP_stride;
  }
  double* c_final = C;
  int64_t ldc_final = ldc;
  int64_t split_ld = kSplitLd;
  if (split_scratch && !fuse && N <= kSplitLd && kt_all >= 16) {
    s.kt_per_split = std::max(8, (kt_all + kSplitMax - 1) / kSplitMax);
    s.ksplit = (kt_all + s.kt_per_split - 1) / s.kt_per_split;
    s.C = split_scratch;
    s.ldc = kSplitLd;
    s.split_stride = (long long)M * kSplitLd;
  } else if (wide_split) {
    split_ld = round_up(N, 2);
    s.kt_per_split = (kt_all + 1) / 2;
    s.ksplit = 2;
    s.C = wide_split_scratch;
    s.ldc = split_ld;
    s.split_stride = (long long)M * split_ld;
  }
  const bool sq = nsq < N;
  if (sq && (nsq % 32)) return fail(GWAS_E_ARG, "nsq must be a multiple of 32");
  auto launch = [&]() -> gwas_status {
    if (fuse) {
      if (bn == 64) {
        if (a_u8) return launch_gemm_t<uint8_t, 64, kStagesU8, false, true>(ma, mb, s, st);
        return launch_gemm_t<double, 64, kStagesF64N64, false, true>(ma, mb, s, st);
      }
      if (a_u8) return launch_gemm_t<uint8_t, 128, kStagesU8, false, true>(ma, mb, s, st);
      return launch_gemm_t<double, 128, kStagesF64, false, true>(ma, mb, s, st);
    }
    if (bn == 64) {
      if (a_u8) {
        if (sq) return launch_gemm_t<uint8_t, 64, kStagesU8, true>(ma, mb, s, st);
        return launch_gemm_t<uint8_t, 64, kStagesU8, false>(ma, mb, s, st);
      }
      if (sq) return launch_gemm_t<double, 64, kStagesF64N64, true>(ma, mb, s, st);
      return launch_gemm_t<double, 64, kStagesF64N64, false>(ma, mb, s, st);
    }
    if (a_u8) {
      if (sq) return launch_gemm_t<uint8_t, 128, kStagesU8, true>(ma, mb, s, st);
      return launch_gemm_t<uint8_t, 128, kStagesU8, false>(ma, mb, s, st);
    }
    if (sq) return launch_gemm_t<double, 128, kStagesF64, true>(ma, mb, s, st);
    return launch_gemm_t<double, 128, kStagesF64, false>(ma, mb, s, st);
  };
  CKG(launch());
  if (s.ksplit > 1) {
    const long long total = M * N;
    gw::splitk_reduce<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(s.C, s.split_stride, s.ksplit, (int)M, (int)N,
                                                                       split_ld, c_final, ldc_final);
    CKC(cudaGetLastError());
  }
  return GWAS_OK;
}

// K3 fused with the low-rank recombination (lowrank_k3.cuh): grid of 32-trait x 64-SNP tiles.
gwas_status launch_lowrank_schur(const gw::LowrankK3Args& a, int p, cudaStream_t st) {
  if ((long long)a.k3.cols * a.k3.t == 0) return GWAS_OK;
  const dim3 grid((unsigned)((a.k3.t + gw::LRK3_COLS - 1) / gw::LRK3_COLS),
                  (unsigned)((a.k3.cols + gw::LRK3_ROWS - 1) / gw::LRK3_ROWS));
  switch (p) {
#define CASE_P(P) \
  case P: gw::lowrank_schur<P><<<grid, gw::LRK3_THREADS, 0, st>>>(a); break;
    CASE_P(1) CASE_P(2) CASE_P(3) CASE_P(4) CASE_P(5) CASE_P(6)
    CASE_P(7) CASE_P(8) CASE_P(9) CASE_P(10) CASE_P(11) CASE_P(12)
#undef CASE_P
    default:
      return fail(GWAS_E_ARG, "p = %d unsupported", p);
  }
  CKC(cudaGetLastError());
  return GWAS_OK;
}

// K3 on the trait-tiled C: bulk-copy (TMA) streamed persistent kernel, one CTA per resident slot.  Two shapes
// (measured per 15104-SNP C4 block / 8192-SNP block at n = 1e3, t = 1e4): 2 rows x 4 stages with the same row ranges
// for every trait block when that fills >= 90 % of the CTA slots (C4: 0.178 ms, 6.2 TB/s), else 4 rows x 3 stages
// over flattened trait-block-major ranges (t = 1e4: 0.99 ms, 6.0 TB/s).
template <int P, int R, int ST>
gwas_status launch_schur_tma_rs(const gw::SchurArgs& a, cudaStream_t st, bool need_aligned, bool* launched) {
  constexpr size_t smem = gw::schur_tma_smem<P, R, ST>();
  static std::atomic<uint64_t> attr_devs{0};
  *launched = false;
  CKG(ensure_smem_attr(gw::schur_solve_tma<P, R, ST>, smem, attr_devs));
  int dev = 0, sms = 148, occ = 1;
  CKC(cudaGetDevice(&dev));
  CKC(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CKC(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gw::schur_solve_tma<P, R, ST>, gw::CTILE_T, smem));
  const int gx = (a.t + gw::CTILE_T - 1) / gw::CTILE_T;
  const long long ntr = (a.cols + R - 1) / R;
  const long long slots = (long long)std::max(occ, 1) * sms;
  gw::SchurArgs b = a;
  long long grid;
  const long long gy = std::min<long long>(slots / gx, ntr);
  if (gy >= 1 && gx * gy >= (slots * 9) / 10) {  // aligned row ranges fill >= 90 % of the CTA slots
    b.k3_gy = (int)gy;
    grid = gx * gy;
  } else {
    if (need_aligned) return GWAS_OK;
    b.k3_gy = 0;
    grid = std::max<long long>(1, std::min<long long>((long long)gx * ntr, slots));
  }
  gw::schur_solve_tma<P, R, ST><<<(unsigned)grid, gw::CTILE_T, smem, st>>>(b);
  CKC(cudaGetLastError());
  *launched = true;
  return GWAS_OK;
}

template <int P>
gwas_status launch_schur_tma(const gw::SchurArgs& a, cudaStream_t st) {
  bool done = false;
  CKG((launch_schur_tma_rs<P, 2, 4>(a, st, true, &done)));
  if (!done) CKG((launch_schur_tma_rs<P, 4, 3>(a, st, false, &done)));
  return GWAS_OK;
}

gwas_status launch_schur(const gw::SchurArgs& a, int p, cudaStream_t st) {
  const long long np = (long long)a.cols * a.t;
  if (np == 0) return GWAS_OK;
  static const bool k3_plain = env_flag("GWAS_K3_PLAIN");
  if (a.tiled && !k3_plain) {
    switch (p) {
#define CASE_P(P) \
  case P: return launch_schur_tma<P>(a, st);
      CASE_P(1) CASE_P(2) CASE_P(3) CASE_P(4) CASE_P(5) CASE_P(6)
      CASE_P(7) CASE_P(8) CASE_P(9) CASE_P(10) CASE_P(11) CASE_P(12)
#undef CASE_P
      default:
        return fail(GWAS_E_ARG, "p = %d unsupported", p);
    }
  }
  const int threads = 128;
  gw::SchurArgs args = a;
  args.tj = 1;
  while (args.tj < a.t && args.tj < threads) args.tj *= 2;
  args.ich = a.t >= 32 ? gw::SCHUR_ICH : 1;
  const int snps_per_block = (threads / args.tj) * args.ich;
  const dim3 grid((unsigned)((a.t + args.tj - 1) / args.tj), (unsigned)((a.cols + snps_per_block - 1) / snps_per_block));
  switch (p) {
#define CASE_P(P) \
  case P:                                                                  \
    if (args.tiled) gw::schur_solve<P, true><<<grid, threads, 0, st>>>(args); \
    else gw::schur_solve<P, false><<<grid, threads, 0, st>>>(args);          \
    break;
    CASE_P(1) CASE_P(2) CASE_P(3) CASE_P(4) CASE_P(5) CASE_P(6)
    CASE_P(7) CASE_P(8) CASE_P(9) CASE_P(10) CASE_P(11) CASE_P(12)
#undef CASE_P
    default:
      return fail(GWAS_E_ARG, "p = %d unsupported", p);
  }
  CKC(cudaGetLastError());
  return GWAS_OK;
}

// K1i/K2a: C_a[i][c] (c < na) and C_b[i][c'] (c' < nb) from the u8 A block and the stacked digit matrix.
// Launch of the S-digit kernel with cluster size CL (1 = plain launch) and BKB-byte K stages.
template <int S, int BKB>
gwas_status launch_i8_s(int CL, const CUtensorMap& ma, const CUtensorMap& mb, const gw::I8Shape& s, unsigned grid,
                        cudaStream_t st) {
  constexpr size_t smem = gw::I8Cfg<S, BKB>::smem_bytes(gw::I8_EPI_SMEM);
  static std::atomic<uint64_t> attr1{0}, attr2{0}, attr4{0};
  CKG(ensure_smem_attr(gw::gemm_i8_sliced<1, S, BKB>, smem, attr1));
  CKG(ensure_smem_attr(gw::gemm_i8_sliced<2, S, BKB>, smem, attr2));
  CKG(ensure_smem_attr(gw::gemm_i8_sliced<4, S, BKB>, smem, attr4));
  if (CL == 1) {
    gw::gemm_i8_sliced<1, S, BKB><<<grid, gw::I8_THREADS, smem, st>>>(ma, mb, s);
    CKC(cudaGetLastError());
    return GWAS_OK;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(gw::I8_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (CL == 2) CKC(cudaLaunchKernelEx(&cfg, gw::gemm_i8_sliced<2, S, BKB>, ma, mb, s));
  else CKC(cudaLaunchKernelEx(&cfg, gw::gemm_i8_sliced<4, S, BKB>, ma, mb, s));
  return GWAS_OK;
}

// The 2-SM kernel (CTA pairs, cta_group::2 MMAs of M = 256), CLP pairs per cluster.
template <int S, int BKB, int CLP>
gwas_status launch_i8_2sm(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mb1,
                          const gw::I8Shape& s, unsigned grid, cudaStream_t st) {
  constexpr size_t smem = gw::I8Cfg2<S, BKB>::smem_bytes(gw::I8_EPI_SMEM);
  static std::atomic<uint64_t> attr{0};
  CKG(ensure_smem_attr(gw::gemm_i8_sliced_2sm<S, BKB, CLP>, smem, attr));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(gw::I8_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeClusterDimension;
  la[0].val.clusterDim.x = 2 * CLP;
  la[0].val.clusterDim.y = 1;
  la[0].val.clusterDim.z = 1;
  cfg.attrs = la;
  cfg.numAttrs = 1;
  // Persistent clusters (GWAS_I8_PERSIST=0: one cluster per cluster tile): as many as can be co-resident, each
  // looping over cluster tiles, so a tile's first stages load while the previous tile's accumulators drain.
  static const int persist = getenv("GWAS_I8_PERSIST") ? atoi(getenv("GWAS_I8_PERSIST")) : 1;
  if (persist) {
    int nclu = 0;  // per call: cheap beside a multi-ms launch, and correct for whichever device is current
    CKC(cudaOccupancyMaxActiveClusters(&nclu, gw::gemm_i8_sliced_2sm<S, BKB, CLP>, &cfg));
    const unsigned ctiles = grid / (2 * CLP);
    if (nclu > 0 && (unsigned)nclu < ctiles) cfg.gridDim = dim3((unsigned)nclu * 2 * CLP);
  }
  CKC(cudaLaunchKernelEx(&cfg, gw::gemm_i8_sliced_2sm<S, BKB, CLP>, ma, mb, mb1, s));
  return GWAS_OK;
}

gwas_status launch_i8(int S, const void* A, int64_t lda, int64_t M, int64_t K, const int8_t* dig, int64_t ldd,
                      int64_t tiles_n, int64_t na_tiles, const int* exps, double* Ca, int64_t ldca, int64_t na,
                      double* Cb, int64_t ldcb, int64_t nb, cudaStream_t st, int64_t tri_tiles = 0,
                      int ft = 0, const double* fD = nullptr, int64_t fld = 0, double* fP = nullptr,
                      int64_t fP_stride = 0) {
  if (M <= 0) return GWAS_OK;
  if (S != 7 && S != 8) return fail(GWAS_E_ARG, "int8 digits %d", S);
  // Kernel choice (measured at C4, K1i per 8192-SNP block, 5 passes; profiles/ncu_int8_c4_r02.md):
  //                                                        7 digits   8 digits
  //   2-SM pairs, 128-byte K stages, persistent clusters:
  //     two pairs per cluster sharing the slab              5.39 ms    6.04 ms   (7-digit default)
  //     one pair per cluster                                5.48 ms    5.91 ms   (8-digit default)
  //   the same, one cluster per tile (GWAS_I8_PERSIST=0)    5.60/5.43  6.26/5.99
  //   2-SM, 64-byte K stages (GWAS_I8_BK=64)                7.87 ms    8.47 ms
  //   1-SM, 2-CTA slab multicast, 128/64-byte stages        6.19/6.94  8.94/7.57 (used when the block has <= 128 rows)
  // GWAS_I8_KERNEL=1sm|2sm, GWAS_I8_CLUSTER=1|2|4, GWAS_I8_BK=64|128 and GWAS_I8_PERSIST=0|1 override the choice.
  static int mode_env = [] {
    const char* e = getenv("GWAS_I8_KERNEL");
    return (e && std::string(e) == "1sm") ? 1 : 2;
  }();
  static int cl_env = [] {
    const char* e = getenv("GWAS_I8_CLUSTER");
    const int v = e ? atoi(e) : 0;
    return (v == 1 || v == 2 || v == 4) ? v : 0;
  }();
  static int bk_env = [] {
    const char* e = getenv("GWAS_I8_BK");
    return e ? (atoi(e) == 64 ? 64 : 128) : 0;
  }();
  const bool two_sm = mode_env == 2 && M > gw::I8_BM;
  const int cl_want = cl_env ? cl_env : (two_sm ? (S == 7 ? 4 : 2) : 2);
  // 2-SM: a cluster of 4 (two pairs sharing the slab) needs more than two row tiles
  const int CL = two_sm ? ((cl_want == 4 && M > 2 * gw::I8_BM) ? 4 : 2)
                        : ((M >= (int64_t)cl_want * gw::I8_BM) ? cl_want : 1);
  const int CLP = two_sm ? CL / 2 : 1;
  // 128-byte stages except the 1-SM 8-digit kernel, whose 80 KB stages would leave a 2-deep ring (8.94 vs 7.57 ms)
  const int bk = bk_env ? bk_env : (!two_sm && S == 8 ? 64 : 128);
  const int brows = S * gw::I8_NB;  // digit rows per 64-column tile
  const int swz = bk == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  CUtensorMap ma, mb, mb1;
  CKG(make_map(&ma, A, true, K, M, lda, gw::I8_BM, bk, swz));
  const int box_b = two_sm ? 128 / CLP : (CL == 1 ? brows / 2 : brows / CL);
  CKG(make_map(&mb, dig, true, K, tiles_n * brows, ldd, box_b, bk, swz));
  if (two_sm) CKG(make_map(&mb1, dig, true, K, tiles_n * brows, ldd, (S - 4) * 32 / CLP, bk, swz));
  gw::I8Shape s;
  s.M = (int)M;
  s.K = (int)K;
  s.tiles_m = (int)round_up((M + gw::I8_BM - 1) / gw::I8_BM, CL);
  s.tiles_n = (int)tiles_n;
  s.na_tiles = (int)na_tiles;
  s.na = (int)na;
  s.nb = (int)nb;
  s.Ca = Ca;
  s.lda_c = ldca;
  s.Cb = Cb;
  s.ldb_c = ldcb;
  s.exps = exps;
  // rasterisation group (row tiles per sweep of the digit slabs): 32 keeps the group's X_R rows (41 MB at n = 1e4)
  // L2-resident while the slabs stream; 64 (the whole 8192-SNP block) re-read X_R from DRAM every wave
  // (C4, 7 digits: DRAM read 10.3 -> 3.3 GB per launch, 7.31 -> 7.04 ms).  GWAS_I8_GROUP overrides (tuning).
  static const int i8_group = getenv("GWAS_I8_GROUP") ? atoi(getenv("GWAS_I8_GROUP")) : 32;
  s.group_m = std::max(CL, i8_group);
  s.tri_tiles = (int)tri_tiles;
  if (ft < 0 || ft > gw::I8_FUSE_T) return fail(GWAS_E_ARG, "bad fused-K2b trait count");
  // GWAS_I8_TRACE=<file>: debug phase stamps of the first 4096 CTAs of every launch, appended to <file>
  static const char* trace_path = getenv("GWAS_I8_TRACE");
  static unsigned long long* trace_dev = nullptr;
  if (trace_path && !trace_dev) CKC(cudaMalloc(&trace_dev, sizeof(unsigned long long) * 4096 * gw::I8_TRACE_SLOTS));
  s.trace = trace_path ? trace_dev : nullptr;
  if (trace_dev) CKC(cudaMemsetAsync(trace_dev, 0, sizeof(unsigned long long) * 4096 * gw::I8_TRACE_SLOTS, st));
  static const int dbg_env = getenv("GWAS_I8_DBG") ? atoi(getenv("GWAS_I8_DBG")) : 0;
  s.dbg = dbg_env;
  s.square_a = ft == 0 ? 1 : 0;
  s.ft = ft;
  s.fD = fD;
  s.fld = fld;
  s.fP = fP;
  s.fP_stride = fP_stride;
  const unsigned grid = (unsigned)(s.tiles_m * s.tiles_n);
  if (two_sm) {
    auto f = S == 8 ? (bk == 128 ? (CLP == 2 ? launch_i8_2sm<8, 128, 2> : launch_i8_2sm<8, 128, 1>)
                                 : (CLP == 2 ? launch_i8_2sm<8, 64, 2> : launch_i8_2sm<8, 64, 1>))
                    : (bk == 128 ? (CLP == 2 ? launch_i8_2sm<7, 128, 2> : launch_i8_2sm<7, 128, 1>)
                                 : (CLP == 2 ? launch_i8_2sm<7, 64, 2> : launch_i8_2sm<7, 64, 1>));
    CKG(f(ma, mb, mb1, s, grid, st));
  } else if (S == 8) {
    CKG((bk == 128 ? launch_i8_s<8, 128>(CL, ma, mb, s, grid, st) : launch_i8_s<8, 64>(CL, ma, mb, s, grid, st)));
  } else {
    CKG((bk == 128 ? launch_i8_s<7, 128>(CL, ma, mb, s, grid, st) : launch_i8_s<7, 64>(CL, ma, mb, s, grid, st)));
  }
  CKC(cudaGetLastError());
  if (trace_dev) {
    std::vector<unsigned long long> h(4096 * gw::I8_TRACE_SLOTS);
    CKC(cudaStreamSynchronize(st));
    CKC(cudaMemcpy(h.data(), trace_dev, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost));
    if (FILE* f = fopen(trace_path, "ab")) {
      fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
      fclose(f);
    }
  }
  return GWAS_OK;
}

// Variance-component estimation kernels (estimate.cuh), dispatched on the compile-time p (est_p*.cu).
gwas_status launch_estimate(int p, const double* W, const double* xlp, const double* yp, int n, int kpad, int t,
                            int method, double eps_spd, double* rec, gw::EstOut eo, cudaStream_t st) {
  if (p < 1 || p > 12) return fail(GWAS_E_ARG, "estimation: p = %d unsupported", p);
  auto f = p <= 3 ? gw::est_launch_p1_3 : p <= 6 ? gw::est_launch_p4_6 : p <= 9 ? gw::est_launch_p7_9 : gw::est_launch_p10_12;
  CKC(f(p, W, xlp, yp, n, kpad, t, method, eps_spd, rec, eo, st));
  return GWAS_OK;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

bool is_pinned_host(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

}  // namespace

// ------------------------------------------------------------------ context
struct gwas_ctx {
  gwas_options opt;
  Dims d;
  StateHeader h;
  uint8_t* state = nullptr;
  uint8_t* work = nullptr;
  size_t work_bytes = 0;
  RunLayout rl;
  cudaStream_t cs = nullptr, ps = nullptr;
  cudaStream_t aux = nullptr;  // overlap mode: K2 + K3 of block b beside K1 of block b+1 (owned by the context)
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
  cudaEvent_t ev_k1[2] = {nullptr, nullptr}, ev_set_free[2] = {nullptr, nullptr}, ev_join = nullptr;
  cudaStream_t dstream = nullptr;  // D2H of results when the caller's outputs are pinned host memory
  cudaEvent_t ev_out_ready[2] = {nullptr, nullptr}, ev_out_free[2] = {nullptr, nullptr}, ev_djoin = nullptr;
  int stage_next = 0;
  bool stage_zeroed = false;
  float ms_eig = 0.f, ms_pre = 0.f, ms_est = 0.f;
  std::vector<int32_t> est_gstar;  // estimation: first grid argmax per trait (reading E3), copied at setup
  // per-kernel event timers
  struct Pending {
    int kind;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> pool;
  double ms_acc[GWAS_NUM_TIMERS] = {0, 0, 0, 0};
  int64_t launches[GWAS_NUM_TIMERS] = {0, 0, 0, 0};

  double* Z() const { return reinterpret_cast<double*>(state + h.off_Z); }
  double* W() const { return reinterpret_cast<double*>(state + h.off_W); }
  double* B2() const { return reinterpret_cast<double*>(state + h.off_B2); }
  double* Lpk() const { return reinterpret_cast<double*>(state + h.off_Lpk); }
  double* v() const { return reinterpret_cast<double*>(state + h.off_v); }
  double* s2() const { return reinterpret_cast<double*>(state + h.off_s2); }
  double* betaT() const { return reinterpret_cast<double*>(state + h.off_betaT); }
  double* dinv() const { return reinterpret_cast<double*>(state + h.off_dinv); }
  int8_t* dig() const { return reinterpret_cast<int8_t*>(state + h.off_dig); }
  int* exps() const { return reinterpret_cast<int*>(state + h.off_exps); }

  cudaEvent_t ev() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
  gwas_status tic(int kind, cudaStream_t st, cudaEvent_t* out) {
    *out = nullptr;
    if (!opt.timing) return GWAS_OK;
    *out = ev();
    CKC(cudaEventRecord(*out, st));
    pending.push_back({kind, *out, nullptr});
    return GWAS_OK;
  }
  gwas_status toc(cudaStream_t st) {
    if (!opt.timing) return GWAS_OK;
    cudaEvent_t e = ev();
    CKC(cudaEventRecord(e, st));
    pending.back().b = e;
    return GWAS_OK;
  }
  gwas_status drain() {
    for (auto& pd : pending) {
      CKC(cudaEventSynchronize(pd.b));
      float ms = 0.f;
      CKC(cudaEventElapsedTime(&ms, pd.a, pd.b));
      ms_acc[pd.kind] += ms;
      launches[pd.kind] += 1;
      pool.push_back(pd.a);
      pool.push_back(pd.b);
    }
    pending.clear();
    return GWAS_OK;
  }
};

namespace {

gwas_status ctx_init(gwas_ctx* c, const gwas_options* o, const Dims& d, const StateHeader& h, void* state,
                     void* work, size_t work_bytes) {
  c->opt = *o;
  c->d = d;
  c->h = h;
  c->state = static_cast<uint8_t*>(state);
  c->work = static_cast<uint8_t*>(work);
  c->work_bytes = work_bytes;
  c->rl = run_layout(d, o->overlap != 0);
  c->cs = static_cast<cudaStream_t>(o->compute_stream);
  c->ps = o->copy_stream ? static_cast<cudaStream_t>(o->copy_stream) : c->cs;
  for (int i = 0; i < 2; ++i) {
    CKC(cudaEventCreateWithFlags(&c->ev_in[i], cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&c->ev_free[i], cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&c->ev_k1[i], cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&c->ev_set_free[i], cudaEventDisableTiming));
  }
  CKC(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  CKC(cudaEventCreateWithFlags(&c->ev_djoin, cudaEventDisableTiming));
  for (int i = 0; i < 2; ++i) {
    CKC(cudaEventCreateWithFlags(&c->ev_out_ready[i], cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&c->ev_out_free[i], cudaEventDisableTiming));
  }
  CKC(cudaStreamCreateWithFlags(&c->dstream, cudaStreamNonBlocking));
  if (o->overlap) CKC(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
  return GWAS_OK;
}

}  // namespace

extern "C" {

}  // extern "C"

namespace {
// Low-rank recombination (reading L1): c2[:, f t + j] = sum_r g2[:, f r + rr] W[rr, j] for the p X_L fields and
// c2[:, nsq + j] = sum_r g2[:, lr_nsq + rr] W[rr, j] for the squared term (DMMA products with K = r).
gwas_status lowrank_recombine(gwas_ctx* c, const double* g2, double* c2, int64_t cols, cudaStream_t st) {
  const Dims& d = c->d;
  const int64_t r = c->h.lr_r;
  const double* wt = reinterpret_cast<const double*>(c->state + c->h.off_wt);
  for (int64_t f = 0; f < d.p; ++f)
    CKG(gemm_tn(false, g2 + f * r, d.ldg2, wt, r, c2 + f * d.t, d.ldc2, cols, d.t, r, d.t, st, 16));
  CKG(gemm_tn(false, g2 + c->h.lr_nsq, d.ldg2, wt, r, c2 + d.nsq, d.ldc2, cols, d.t, r, d.t, st, 16));
  return GWAS_OK;
}
}  // namespace

extern "C" {

void gwas_default_options(gwas_options* o) {
  if (!o) return;
  memset(o, 0, sizeof(*o));
  o->device = 0;
  o->xr_dtype = GWAS_XR_U8;
  o->output_mode = GWAS_OUT_SNP;
  o->var_convention = GWAS_VAR_TEXTBOOK;
  o->block_cols = 8192;
  o->eps_spd = 1e-10;
  o->eps_collinear = 1e-10;
  o->compute_stream = nullptr;
  o->copy_stream = nullptr;
  o->timing = 0;
  o->fuse_k2 = 1;
}

const char* gwas_last_error(void) { return g_err.c_str(); }
const char* gwas_version(void) {
  return "gwas-clak-eig-b200 2 (sm_100a: FP64 DMMA, int8-sliced tcgen05, low-rank trait weights, ML/REML estimation)";
}

size_t gwas_state_bytes(int64_t n, int64_t p, int64_t t, const gwas_options* o) {
  if (check_sizes(n, p, t, o) != GWAS_OK) return 0;
  Dims d = make_dims_kb(n, p, t, o);
  return (size_t)make_header(d, o).total;
}

size_t gwas_workspace_bytes(int64_t n, int64_t p, int64_t t, const gwas_options* o) {
  if (check_sizes(n, p, t, o) != GWAS_OK) return 0;
  Dims d = make_dims_kb(n, p, t, o);
  int64_t lwork = 0;
  size_t host_ws = 0;
  if (solver_lwork(o, n, d.kpad, &lwork, &host_ws) != GWAS_OK) return 0;
  int64_t lrw = 0;
  if (lr_lwork(o, d, &lrw) != GWAS_OK) return 0;
  return std::max(setup_layout(d, lwork, lrw).total, run_layout(d, o->overlap != 0).total);
}

}  // extern "C"

namespace {
// gwas_setup (est_method < 0: h2 / sigma2 given) and gwas_setup_estimate (est_method = GWAS_EST_ML / _REML: h2 and
// sigma2 estimated in the eigenbasis after Alg. 4 lines 1, 2, 4, then the same per-trait precompute).
gwas_status setup_impl(const gwas_options* o, int64_t n, int64_t p, int64_t t, const double* phi, const double* XL,
                       const double* Y, const double* h2, const double* sigma2, int est_method, double* h2_out,
                       double* s2_out, double* ll_out, void* state_dev, size_t state_bytes, void* work_dev,
                       size_t work_bytes, gwas_ctx** out) {
  g_err.clear();
  CKG(check_sizes(n, p, t, o));
  const bool est = est_method >= 0;
  if (!out || !phi || !XL || !Y || (!est && (!h2 || !sigma2)) || !state_dev || !work_dev)
    return fail(GWAS_E_ARG, "NULL pointer argument");
  *out = nullptr;
  CKC(cudaSetDevice(o->device));
  Dims d = make_dims_kb(n, p, t, o);
  StateHeader h = make_header(d, o);
  int64_t lwork = 0;
  size_t host_ws = 0;
  CKG(solver_lwork(o, n, d.kpad, &lwork, &host_ws));
  int64_t lrw = 0;
  CKG(lr_lwork(o, d, &lrw));
  SetupLayout sl = setup_layout(d, lwork, lrw);
  RunLayout rl = run_layout(d, o->overlap != 0);
  if (state_bytes < (size_t)h.total) return fail(GWAS_E_NOMEM, "state %zu < %lld bytes", state_bytes, (long long)h.total);
  if (work_bytes < std::max(sl.total, rl.total))
    return fail(GWAS_E_NOMEM, "workspace %zu < %zu bytes", work_bytes, std::max(sl.total, rl.total));
  if (!is_device_ptr(state_dev) || !is_device_ptr(work_dev)) return fail(GWAS_E_ARG, "state/work must be device memory");

  // validate (h2, sigma2) on the host
  std::vector<double> hh(t), ss(t);
  if (!est) {
    CKC(cudaMemcpy(hh.data(), h2, sizeof(double) * t, cudaMemcpyDefault));
    CKC(cudaMemcpy(ss.data(), sigma2, sizeof(double) * t, cudaMemcpyDefault));
  } else {
    std::fill(hh.begin(), hh.end(), 0.5);
    std::fill(ss.begin(), ss.end(), 1.0);
  }
  for (int64_t j = 0; j < t; ++j) {
    if (!(hh[j] >= 0.0 && hh[j] <= 1.0)) return fail(GWAS_E_ARG, "h2[%lld] = %g outside [0, 1]", (long long)j, hh[j]);
    if (!(ss[j] > 0.0) || !std::isfinite(ss[j])) return fail(GWAS_E_ARG, "sigma2[%lld] = %g not > 0", (long long)j, ss[j]);
  }

  gwas_ctx* c = new gwas_ctx();
  gwas_status st = ctx_init(c, o, d, h, state_dev, work_dev, work_bytes);
  if (st != GWAS_OK) {
    gwas_destroy(c);
    return st;
  }
  cudaStream_t cs = c->cs;
  uint8_t* w = c->work;
  double* xlpad = reinterpret_cast<double*>(w + sl.xlpad);
  double* ypad = reinterpret_cast<double*>(w + sl.ypad);
  double* xlp = reinterpret_cast<double*>(w + sl.xlp);
  double* yp = reinterpret_cast<double*>(w + sl.yp);
  double* stl = reinterpret_cast<double*>(w + sl.stl);
  double* dh2 = reinterpret_cast<double*>(w + sl.h2);
  double* ds2 = reinterpret_cast<double*>(w + sl.s2);
  unsigned long long* derr = reinterpret_cast<unsigned long long*>(w + sl.err);
  int* dinfo = reinterpret_cast<int*>(w + sl.info);
  double* dwork = reinterpret_cast<double*>(w + sl.work);

  auto body = [&]() -> gwas_status {
    cudaEvent_t e0, e1, e2, e3;
    CKC(cudaEventCreate(&e0));
    CKC(cudaEventCreate(&e1));
    CKC(cudaEventCreate(&e2));
    CKC(cudaEventCreate(&e3));
    CKC(cudaEventRecord(e0, cs));
    // header + Phi into Z (ld kpad, zero padding), W zero
    CKC(cudaMemcpyAsync(c->state, &c->h, sizeof(StateHeader), cudaMemcpyHostToDevice, cs));
    CKC(cudaMemsetAsync(c->Z(), 0, sizeof(double) * d.kpad * d.kpad, cs));
    CKC(cudaMemsetAsync(c->W(), 0, sizeof(double) * d.kpad, cs));
    CKC(cudaMemcpy2DAsync(c->Z(), sizeof(double) * d.kpad, phi, sizeof(double) * n, sizeof(double) * n, n,
                          cudaMemcpyDefault, cs));
    if (!est) {
      CKC(cudaMemcpyAsync(dh2, h2, sizeof(double) * t, cudaMemcpyDefault, cs));
      CKC(cudaMemcpyAsync(ds2, sigma2, sizeof(double) * t, cudaMemcpyDefault, cs));
      CKC(cudaMemcpyAsync(c->s2(), sigma2, sizeof(double) * t, cudaMemcpyDefault, cs));
    }
    CKC(cudaMemcpy2DAsync(xlpad, sizeof(double) * d.kpad, XL, sizeof(double) * n, sizeof(double) * n, p,
                          cudaMemcpyDefault, cs));
    CKC(cudaMemcpy2DAsync(ypad, sizeof(double) * d.kpad, Y, sizeof(double) * n, sizeof(double) * n, t,
                          cudaMemcpyDefault, cs));
    CKC(cudaMemsetAsync(derr, 0xff, sizeof(unsigned long long) * 4, cs));
    CKC(cudaEventRecord(e1, cs));
    cusolverDnHandle_t hs;
    CKS(cusolverDnCreate(&hs));
    cusolverStatus_t ss2 = cusolverDnSetStream(hs, cs);
    const bool chol = o->algorithm == GWAS_ALG_CHOL;
    std::vector<uint8_t> host_ws_buf(std::max<size_t>(host_ws, 1));
    if (!chol) {
      // Alg. 4 line 1: Phi = Z W Z^T, in place (Z overwrites Phi)
      if (ss2 == CUSOLVER_STATUS_SUCCESS)
        ss2 = cusolverDnDsyevd(hs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)n, c->Z(), (int)d.kpad,
                               c->W(), dwork, (int)lwork, dinfo);
    } else {
      // Alg. 3 lines 1-2: M = sigma2 (h2 Phi + (1 - h2) I) = L L^T, then L^-1 (dtrtri) so that
      // line 4, X_R := L^-1 X_R, is a (lower-triangular) product; the state's rotation R = L^-1 stored by rows.
      double* Mw = dwork;
      double* sw = dwork + d.kpad * d.kpad;
      const int64_t slw = lwork - d.kpad * d.kpad;
      CKC(cudaMemcpy2DAsync(Mw, sizeof(double) * d.kpad, c->Z(), sizeof(double) * d.kpad, sizeof(double) * d.kpad,
                            d.kpad, cudaMemcpyDeviceToDevice, cs));
      gw::assemble_m<<<dim3((unsigned)std::min<int64_t>((n + 255) / 256, 64), (unsigned)std::min<int64_t>(n, 65535)),
                        256, 0, cs>>>(
          Mw, (int)n, (int)d.kpad, ss[0], hh[0]);
      CKC(cudaGetLastError());
      if (ss2 == CUSOLVER_STATUS_SUCCESS)
        ss2 = cusolverDnDpotrf(hs, CUBLAS_FILL_MODE_LOWER, (int)n, Mw, (int)d.kpad, sw, (int)slw, dinfo);
      CKC(cudaStreamSynchronize(cs));
      int pinfo = 0;
      CKC(cudaMemcpy(&pinfo, dinfo, sizeof(int), cudaMemcpyDeviceToHost));
      if (ss2 == CUSOLVER_STATUS_SUCCESS && pinfo != 0) {
        cusolverDnDestroy(hs);
        return fail(GWAS_E_NOT_SPD, "trait 0: M = sigma2 (h2 Phi + (1 - h2) I) not positive definite (dpotrf info %d)",
                    pinfo);
      }
      if (ss2 == CUSOLVER_STATUS_SUCCESS)
        ss2 = cusolverDnXtrtri(hs, CUBLAS_FILL_MODE_LOWER, CUBLAS_DIAG_NON_UNIT, n, CUDA_R_64F, Mw, d.kpad, sw,
                               (size_t)slw * sizeof(double), host_ws_buf.data(), host_ws, dinfo);
      gw::zero_upper<<<dim3((unsigned)std::min<int64_t>((d.kpad + 255) / 256, 64),
                            (unsigned)std::min<int64_t>(d.kpad, 65535)), 256, 0, cs>>>(
          Mw, (int)n, (int)d.kpad);
      CKC(cudaGetLastError());
      gw::transpose_sq<<<dim3((unsigned)((d.kpad + 31) / 32), (unsigned)((d.kpad + 31) / 32)), dim3(32, 8), 0, cs>>>(
          Mw, c->Z(), (int)d.kpad);
      CKC(cudaGetLastError());
      // D = I: the trait's M^-1 is applied through L^-1 already (K2 weights d = 1 via h2 = 0, sigma2 = 1)
      CKC(cudaMemsetAsync(dh2, 0, sizeof(double) * t, cs));
      const double one = 1.0;
      CKC(cudaMemcpyAsync(ds2, &one, sizeof(double), cudaMemcpyHostToDevice, cs));
    }
    CKC(cudaEventRecord(e2, cs));
    CKC(cudaStreamSynchronize(cs));
    cusolverDnDestroy(hs);
    if (ss2 != CUSOLVER_STATUS_SUCCESS)
      return fail(GWAS_E_CUDA, "cuSOLVER %s status %d", chol ? "dpotrf/dtrtri" : "dsyevd", (int)ss2);
    int info = 0;
    CKC(cudaMemcpy(&info, dinfo, sizeof(int), cudaMemcpyDeviceToHost));
    if (info != 0) return fail(GWAS_E_EIG, "%s info = %d", chol ? "dtrtri" : "dsyevd", info);
    // Alg. 4 lines 2, 4: X_L' = Z^T X_L, Y' = Z^T Y  (K1 kernel, fp64 A)
    CKG(gemm_tn(false, xlpad, d.kpad, c->Z(), d.kpad, xlp, d.kpad, p, n, n, n, cs));
    CKG(gemm_tn(false, ypad, d.kpad, c->Z(), d.kpad, yp, d.kpad, t, n, n, n, cs));
    cudaEvent_t ee0 = nullptr, ee1 = nullptr;
    if (est) {
      // the paper's first step, eigen-based: per-trait (h2, sigma2) by ML / REML (readings E1-E4)
      CKC(cudaEventCreate(&ee0));
      CKC(cudaEventCreate(&ee1));
      CKC(cudaEventRecord(ee0, cs));
      gw::EstOut eo{dh2, ds2, reinterpret_cast<double*>(w + sl.est_ll), reinterpret_cast<int*>(w + sl.est_gs),
                    derr + 2};
      CKG(launch_estimate((int)p, c->W(), xlp, yp, (int)n, (int)d.kpad, (int)t, est_method, o->eps_spd,
                          reinterpret_cast<double*>(w + sl.est_rec), eo, cs));
      CKC(cudaMemcpyAsync(c->s2(), ds2, sizeof(double) * t, cudaMemcpyDeviceToDevice, cs));
      CKC(cudaEventRecord(ee1, cs));
    }
    // Alg. 4 lines 6, 8, 9: D_j and the D_j-scaled operand B2 = [B_op | D]
    {
      dim3 grid((unsigned)std::min<int64_t>((d.kpad + 255) / 256, 64), (unsigned)std::min<int64_t>(d.n2, 65535));
      gw::build_b2<<<grid, 256, 0, cs>>>(xlp, yp, c->W(), dh2, ds2, (int)n, (int)p, (int)t, (int)d.kpad, (int)d.nsq,
                                         (int)d.n2, o->eps_spd, c->B2(), derr);
      CKC(cudaGetLastError());
    }
    // Alg. 4 lines 10-11: S_TL_j = X_L'^T D_j X_L', b_T_j = X_L'^T D_j y'_j for all j (K2 kernel)
    CKG(gemm_tn(false, xlp, d.kpad, c->B2(), d.kpad, stl, d.lds, p, t * (p + 1), n, d.n2, cs));
    gw::trait_factor<kPMax><<<(unsigned)((t + 127) / 128), 128, 0, cs>>>(stl, d.lds, (int)p, (int)t,
                                                                         o->eps_collinear, c->Lpk(), c->v(),
                                                                         c->betaT(), c->dinv(), derr + 1);
    CKC(cudaGetLastError());
    // Low-rank trait weights (opt.trait_rank = -1, reading L1): D = U S V^T (gesvd), keep the r singular triplets
    // above kLrTol s_0 (r rounded up to 8), and rebuild the K2 operand from U_r (p r + t + r rows instead of
    // t (p + 2)); the run recombines with W = S_r V_r^T.  Skipped when it would not shrink the products.
    c->h.lr_r = 0;
    c->h.lr_nsq = d.nsq;
    c->h.lr_nlin = d.nlin;
    if (d.lr && t >= 16) {
      double* A = reinterpret_cast<double*>(w + sl.lr_a);
      double* U = reinterpret_cast<double*>(w + sl.lr_u);
      double* VT = reinterpret_cast<double*>(w + sl.lr_vt);
      double* S = reinterpret_cast<double*>(w + sl.lr_s);
      const bool tall = t <= n;  // gesvd needs m >= n: factor D (n x t), else D^T (t x n)
      const int64_t ns = std::min<int64_t>(n, t);
      if (tall) {
        CKC(cudaMemcpy2DAsync(A, sizeof(double) * d.kpad, c->B2() + d.nsq * d.kpad, sizeof(double) * d.kpad,
                              sizeof(double) * n, t, cudaMemcpyDeviceToDevice, cs));
      } else {
        gw::rows_to_colmajor<<<(unsigned)((t * n + 255) / 256), 256, 0, cs>>>(c->B2() + d.nsq * d.kpad, d.kpad,
                                                                               (int)t, (int)n, A, t);
        CKC(cudaGetLastError());
      }
      cusolverDnHandle_t hv;
      CKS(cusolverDnCreate(&hv));
      cusolverStatus_t sv = cusolverDnSetStream(hv, cs);
      if (sv == CUSOLVER_STATUS_SUCCESS) {
        double* lw_ptr = reinterpret_cast<double*>(w + sl.lr_work);
        const int lw_n = (int)std::max<int64_t>(lrw, 1);
        sv = tall ? cusolverDnDgesvd(hv, 'S', 'S', (int)n, (int)t, A, (int)d.kpad, S, U, (int)d.kpad, VT, (int)t,
                                     lw_ptr, lw_n, nullptr, dinfo)
                  : cusolverDnDgesvd(hv, 'S', 'S', (int)t, (int)n, A, (int)t, S, U, (int)t, VT, (int)n, lw_ptr,
                                     lw_n, nullptr, dinfo);
      }
      std::vector<double> hs(ns);
      CKC(cudaMemcpyAsync(hs.data(), S, sizeof(double) * ns, cudaMemcpyDeviceToHost, cs));
      int sinfo = 0;
      CKC(cudaMemcpyAsync(&sinfo, dinfo, sizeof(int), cudaMemcpyDeviceToHost, cs));
      CKC(cudaStreamSynchronize(cs));
      cusolverDnDestroy(hv);
      if (sv != CUSOLVER_STATUS_SUCCESS || sinfo != 0)
        return fail(GWAS_E_EIG, "gesvd of the trait weights: status %d info %d", (int)sv, sinfo);
      int64_t r = 0;
      while (r < ns && hs[r] > kLrTol * hs[0]) ++r;
      r = std::max<int64_t>(8, round_up(r, 8));
      if (r <= kLrMax && 2 * r < t) {
        const int64_t nsq_lr = round_up(p * r + t, 32);
        double* nb2 = reinterpret_cast<double*>(w + sl.lr_b2);
        dim3 grid((unsigned)std::min<int64_t>((d.kpad + 255) / 256, 64), (unsigned)std::min<int64_t>(nsq_lr + r, 65535));
        // D = U S V^T: tall -> U (n x t, ld kpad), V^T (t x t, ld t); wide -> D^T = U' S V'^T, i.e. U = V'
        // (rows of VT, ld n) and V = U' (t x n, ld t)
        const long long su_k = tall ? 1 : n, su_r = tall ? d.kpad : 1;
        const long long sv_j = tall ? t : 1, sv_r = tall ? 1 : t;
        gw::build_lowrank_b2<<<grid, 256, 0, cs>>>(tall ? U : VT, su_k, su_r, xlp, c->B2(), (int)n, (int)p, (int)t,
                                                   (int)d.kpad, (int)r, (int)nsq_lr, nb2);
        CKC(cudaGetLastError());
        CKC(cudaMemcpyAsync(c->B2(), nb2, sizeof(double) * (nsq_lr + r) * d.kpad, cudaMemcpyDeviceToDevice, cs));
        gw::build_lowrank_wt<<<(unsigned)((t * r + 255) / 256), 256, 0, cs>>>(
            S, tall ? VT : U, sv_j, sv_r, (int)t, (int)r, reinterpret_cast<double*>(c->state + c->h.off_wt));
        CKC(cudaGetLastError());
        c->h.lr_r = (int32_t)r;
        c->h.lr_nsq = nsq_lr;
        c->h.lr_nlin = p * r + t;
        c->h.lr_s0 = hs[0];
        c->h.lr_sr = r < ns ? hs[r] : 0.0;
      }
      CKC(cudaMemcpyAsync(c->state, &c->h, sizeof(StateHeader), cudaMemcpyHostToDevice, cs));
      CKC(cudaStreamSynchronize(cs));
    }
    const int64_t nlin_eff = c->h.lr_nlin, nlin_pad_eff = round_up(nlin_eff, gw::I8_NB);
    if (d.i8) {
      // sliced mode: B_lin = Z B_op (n x t(p+1), rows = output columns), then S-digit split of [Z | B_lin]
      double* zt = reinterpret_cast<double*>(w + sl.zt);
      double* blin = reinterpret_cast<double*>(w + sl.blin);
      gw::transpose_sq<<<dim3((unsigned)((d.kpad + 31) / 32), (unsigned)((d.kpad + 31) / 32)), dim3(32, 8), 0, cs>>>(
          c->Z(), zt, (int)d.kpad);
      CKC(cudaGetLastError());
      CKG(gemm_tn(false, c->B2(), d.kpad, zt, d.kpad, blin, d.kpad, nlin_eff, n, n, n, cs));
      const size_t dig_bytes = (size_t)((d.na_pad + nlin_pad_eff) / gw::I8_NB) * o->int8_slices * gw::I8_NB * d.kpad;
      CKC(cudaMemsetAsync(c->dig(), 0, dig_bytes, cs));
      CKC(cudaMemsetAsync(c->exps(), 0, sizeof(int) * (d.na_pad + nlin_pad_eff), cs));
      gw::digitize_rows<<<(unsigned)n, 256, 0, cs>>>(c->Z(), d.kpad, (int)n, (int)n, 0, c->dig(), d.kpad, c->exps(),
                                                     o->int8_slices);
      CKC(cudaGetLastError());
      gw::digitize_rows<<<(unsigned)nlin_eff, 256, 0, cs>>>(blin, d.kpad, (int)nlin_eff, (int)n, (int)d.na_pad,
                                                             c->dig(), d.kpad, c->exps(), o->int8_slices);
      CKC(cudaGetLastError());
    }
    CKC(cudaEventRecord(e3, cs));
    unsigned long long herr[3];
    CKC(cudaMemcpyAsync(herr, derr, sizeof(herr), cudaMemcpyDeviceToHost, cs));
    CKC(cudaStreamSynchronize(cs));
    if (est) {
      float ms = 0.f;
      CKC(cudaEventElapsedTime(&ms, ee0, ee1));
      c->ms_est = ms;
      cudaEventDestroy(ee0);
      cudaEventDestroy(ee1);
      if (herr[2] != ~0ull)
        return fail(GWAS_E_NOT_SPD, "trait %lld: estimation failed (y_j in the span of X_L, or no feasible h2)",
                    (long long)herr[2]);
      if (h2_out) CKC(cudaMemcpy(h2_out, dh2, sizeof(double) * t, cudaMemcpyDefault));
      if (s2_out) CKC(cudaMemcpy(s2_out, ds2, sizeof(double) * t, cudaMemcpyDefault));
      if (ll_out) CKC(cudaMemcpy(ll_out, w + sl.est_ll, sizeof(double) * t, cudaMemcpyDefault));
      c->est_gstar.resize(t);
      CKC(cudaMemcpy(c->est_gstar.data(), w + sl.est_gs, sizeof(int32_t) * t, cudaMemcpyDeviceToHost));
    }
    float ms_all = 0.f, ms_eig = 0.f;
    CKC(cudaEventElapsedTime(&ms_all, e0, e3));
    CKC(cudaEventElapsedTime(&ms_eig, e1, e2));
    c->ms_eig = ms_eig;
    c->ms_pre = ms_all - ms_eig;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    cudaEventDestroy(e3);
    if (herr[0] != ~0ull) {
      const long long j = (long long)(herr[0] / (unsigned long long)n), k = (long long)(herr[0] % (unsigned long long)n);
      double wk = 0.0;
      CKC(cudaMemcpy(&wk, c->W() + k, sizeof(double), cudaMemcpyDeviceToHost));
      return fail(GWAS_E_NOT_SPD, "trait %lld: sigma2 (h2 w_k + 1 - h2) <= eps_spd at eigen-index k = %lld (w_k = %g)",
                  j, k, wk);
    }
    if (herr[1] != ~0ull)
      return fail(GWAS_E_NOT_SPD, "trait %lld: S_TL = X_L'^T D_j X_L' not positive definite (X_L rank-deficient?)",
                  (long long)herr[1]);
    return GWAS_OK;
  };
  st = body();
  if (st != GWAS_OK) {
    gwas_destroy(c);
    return st;
  }
  *out = c;
  return GWAS_OK;
}
}  // namespace

extern "C" {

gwas_status gwas_setup(const gwas_options* o, int64_t n, int64_t p, int64_t t, const double* phi, const double* XL,
                       const double* Y, const double* h2, const double* sigma2, void* state_dev, size_t state_bytes,
                       void* work_dev, size_t work_bytes, gwas_ctx** out) {
  return setup_impl(o, n, p, t, phi, XL, Y, h2, sigma2, -1, nullptr, nullptr, nullptr, state_dev, state_bytes,
                    work_dev, work_bytes, out);
}

gwas_status gwas_setup_estimate(const gwas_options* o, int64_t n, int64_t p, int64_t t, const double* phi,
                                const double* XL, const double* Y, int32_t method, double* h2_out, double* sigma2_out,
                                double* loglik_out, void* state_dev, size_t state_bytes, void* work_dev,
                                size_t work_bytes, gwas_ctx** out) {
  g_err.clear();
  if (!o) return fail(GWAS_E_ARG, "options is NULL");
  if (method != GWAS_EST_ML && method != GWAS_EST_REML) return fail(GWAS_E_ARG, "bad estimation method %d", method);
  if (o->algorithm != GWAS_ALG_EIG)
    return fail(GWAS_E_ARG, "estimation runs in the eigenbasis: use GWAS_ALG_EIG (then pass the estimates to a "
                            "GWAS_ALG_CHOL context's gwas_setup)");
  if (method == GWAS_EST_REML && n <= p) return fail(GWAS_E_ARG, "REML needs n > p");
  return setup_impl(o, n, p, t, phi, XL, Y, nullptr, nullptr, method, h2_out, sigma2_out, loglik_out, state_dev,
                    state_bytes, work_dev, work_bytes, out);
}

gwas_status gwas_trait_rank(gwas_ctx* c, int32_t* r, double* s0, double* s_r) {
  g_err.clear();
  if (!c || !r) return fail(GWAS_E_ARG, "NULL argument");
  *r = c->h.lr_r;
  if (s0) *s0 = c->h.lr_s0;
  if (s_r) *s_r = c->h.lr_sr;
  return GWAS_OK;
}

gwas_status gwas_run_info(gwas_ctx* c, int64_t* block_cols, int32_t* fused_k2) {
  g_err.clear();
  if (!c) return fail(GWAS_E_STATE, "NULL context");
  if (block_cols) *block_cols = c->d.kb;
  if (fused_k2) *fused_k2 = c->d.fuse ? 1 : 0;
  return GWAS_OK;
}

gwas_status gwas_estimate_grid_argmax(gwas_ctx* c, int32_t* g_star) {
  g_err.clear();
  if (!c || !g_star) return fail(GWAS_E_ARG, "NULL argument");
  if (c->est_gstar.size() != (size_t)c->d.t) return fail(GWAS_E_STATE, "context was not created by gwas_setup_estimate");
  std::copy(c->est_gstar.begin(), c->est_gstar.end(), g_star);
  return GWAS_OK;
}

gwas_status gwas_estimate_ms(gwas_ctx* c, double* ms) {
  g_err.clear();
  if (!c || !ms) return fail(GWAS_E_ARG, "NULL argument");
  *ms = c->ms_est;
  return GWAS_OK;
}

gwas_status gwas_attach(const gwas_options* o, int64_t n, int64_t p, int64_t t, void* state_dev, size_t state_bytes,
                        void* work_dev, size_t work_bytes, gwas_ctx** out) {
  g_err.clear();
  CKG(check_sizes(n, p, t, o));
  if (!out || !state_dev || !work_dev) return fail(GWAS_E_ARG, "NULL pointer argument");
  *out = nullptr;
  CKC(cudaSetDevice(o->device));
  Dims d = make_dims_kb(n, p, t, o);
  StateHeader want = make_header(d, o);
  if (state_bytes < (size_t)want.total) return fail(GWAS_E_NOMEM, "state buffer too small");
  RunLayout rl = run_layout(d, o->overlap != 0);
  if (work_bytes < rl.total) return fail(GWAS_E_NOMEM, "workspace %zu < %zu bytes", work_bytes, rl.total);
  StateHeader got;
  CKC(cudaMemcpy(&got, state_dev, sizeof(got), cudaMemcpyDeviceToHost));
  if (got.magic != kMagic || got.version != kVersion || got.n != n || got.p != p || got.t != t ||
      got.total != want.total || got.output_mode != o->output_mode || got.var_convention != o->var_convention ||
      got.int8_slices != o->int8_slices || got.algorithm != o->algorithm || got.trait_rank != o->trait_rank)
    return fail(GWAS_E_STATE, "state header does not match (n, p, t, options)");
  gwas_ctx* c = new gwas_ctx();
  gwas_status st = ctx_init(c, o, d, got, state_dev, work_dev, work_bytes);
  if (st != GWAS_OK) {
    gwas_destroy(c);
    return st;
  }
  *out = c;
  return GWAS_OK;
}

gwas_status gwas_run(gwas_ctx* c, int64_t ncols, const void* XR, int64_t ldx, double* b, double* var, int8_t* status) {
  g_err.clear();
  if (!c) return fail(GWAS_E_STATE, "NULL context");
  if (ncols < 0) return fail(GWAS_E_ARG, "ncols < 0");
  if (ncols == 0) return GWAS_OK;
  if (!XR || !b || !var || !status) return fail(GWAS_E_ARG, "NULL pointer argument");
  const Dims& d = c->d;
  if (ldx < d.n) return fail(GWAS_E_ARG, "ldx = %lld < n = %lld", (long long)ldx, (long long)d.n);
  CKC(cudaSetDevice(c->opt.device));
  const bool dev = is_device_ptr(XR);
  if (!dev && !is_pinned_host(XR)) return fail(GWAS_E_ARG, "X_R host buffer is not page-locked (use pinned memory)");
  if (dev && (((ldx * (int64_t)d.es) & 15) || (reinterpret_cast<uintptr_t>(XR) & 15)))
    return fail(GWAS_E_ARG, "device X_R: ldx * elem_size must be a multiple of 16 and XR 16-byte aligned");
  const bool out_dev = is_device_ptr(b);
  if (is_device_ptr(var) != out_dev || is_device_ptr(status) != out_dev)
    return fail(GWAS_E_ARG, "b, var and status must all be device memory or all pinned host memory");
  if (!out_dev && !(is_pinned_host(b) && is_pinned_host(var) && is_pinned_host(status)))
    return fail(GWAS_E_ARG, "host outputs must be page-locked (pinned)");
  const bool u8 = c->opt.xr_dtype == GWAS_XR_U8;
  const bool chol = c->opt.algorithm == GWAS_ALG_CHOL;
  const int64_t lr_r = c->h.lr_r, lr_nsq = c->h.lr_nsq, lr_nlin = c->h.lr_nlin;
  // low-rank: K3 fused with the K = r recombination (GWAS_LR_UNFUSED=1: separate products + K3, for comparison)
  static const bool lr_unfused_env = env_flag("GWAS_LR_UNFUSED");
  const bool lr_fused = lr_r > 0 && (!lr_unfused_env || (d.t & 1));  // the separate products need even t (alignment)
  const int64_t w = d.p + 1;
  const int64_t per_pair = c->opt.output_mode == GWAS_OUT_FULL ? w : 1;
  cudaStream_t cs = c->cs, ps = c->ps;
  const bool ovl = c->aux != nullptr;
  cudaStream_t cs2 = ovl ? c->aux : cs;  // stream of K2 + K3
  cudaEvent_t dummy;
  if (ovl) {  // the aux stream starts after everything already enqueued on compute_stream
    CKC(cudaEventRecord(c->ev_join, cs));
    CKC(cudaStreamWaitEvent(cs2, c->ev_join, 0));
  }
  int64_t bi = 0;
  for (int64_t blk = 0; blk < ncols; blk += d.kb, ++bi) {
    const int64_t cols = std::min<int64_t>(d.kb, ncols - blk);
    const int set = ovl ? (int)(bi & 1) : 0;
    double* xrp = reinterpret_cast<double*>(c->work + c->rl.xrp[set]);
    double* c2 = reinterpret_cast<double*>(c->work + c->rl.c2[set]);
    double* splitbuf = reinterpret_cast<double*>(c->work + c->rl.split[set]);
    double* g2 = d.lr ? reinterpret_cast<double*>(c->work + c->rl.g2[set]) : nullptr;
    if (ovl) CKC(cudaStreamWaitEvent(cs, c->ev_set_free[set], 0));  // K2/K3 of block bi-2 done with this set
    const uint8_t* src = static_cast<const uint8_t*>(XR) + blk * ldx * (int64_t)d.es;
    const void* A = src;
    int64_t lda = ldx;
    int s = -1;
    if (!dev) {
      // H1 staging (P:158, P:210 double buffering -> host->HBM on the copy stream)
      s = c->stage_next;
      c->stage_next ^= 1;
      void* stage = c->work + c->rl.stage[s];
      CKC(cudaStreamWaitEvent(ps, c->ev_free[s], 0));
      CKG(c->tic(GWAS_H2D, ps, &dummy));
      if (ldx == d.kpad) {
        CKC(cudaMemcpyAsync(stage, src, (size_t)((cols - 1) * ldx + d.n) * d.es, cudaMemcpyHostToDevice, ps));
      } else {
        CKC(cudaMemcpy2DAsync(stage, (size_t)d.kpad * d.es, src, (size_t)ldx * d.es, (size_t)d.n * d.es, (size_t)cols,
                              cudaMemcpyHostToDevice, ps));
      }
      CKG(c->toc(ps));
      CKC(cudaEventRecord(c->ev_in[s], ps));
      CKC(cudaStreamWaitEvent(cs, c->ev_in[s], 0));
      A = stage;
      lda = d.kpad;
    }
    double* fpart = d.fuse ? reinterpret_cast<double*>(c->work + c->rl.fp[set]) : nullptr;
    const int64_t fstride = d.kb * d.fnq;
    if (!d.i8) {
      // K1 (Alg. 4 line 3): X_R'^T = X_R^T Z  (row i of xrp = Z^T g_i)
      gw::GemmShape fz{};
      int k1_tiles = 0;
      if (d.fuse) {  // NEXT-2: K2 contracted in K1's epilogue, per column tile; X_R' never leaves the SM
        fz.fB = c->B2();
        fz.fldb = d.kpad;
        fz.fnq = (int)d.fnq;
        fz.fnlin = (int)(d.t * (d.p + 1));
        fz.fnsq = (int)d.nsq;
        fz.fP = fpart;
        fz.fP_stride = fstride;
      }
      CKG(c->tic(GWAS_K1, cs, &dummy));
      // rasterisation group of K1: 32 row tiles (half of an 8192-column block's X_R panel, ~41 MB) per sweep of the
      // Z column panels: ncu DRAM read per C4 block 3.29 GB vs 3.89 GB at 64, 4.22 GB at 16 (time unchanged, DMMA-bound)
      static const int k1_group = getenv("GWAS_K1_GROUP") ? atoi(getenv("GWAS_K1_GROUP")) : 32;
      CKG(gemm_tn(u8, A, lda, c->Z(), d.kpad, xrp, d.kpad, cols, d.n, d.n, d.n, cs, k1_group, nullptr, chol,
                  d.fuse ? &fz : nullptr, &k1_tiles));
      CKG(c->toc(cs));
      if (s >= 0) CKC(cudaEventRecord(c->ev_free[s], cs));
      if (ovl) {
        CKC(cudaEventRecord(c->ev_k1[set], cs));
        CKC(cudaStreamWaitEvent(cs2, c->ev_k1[set], 0));
      }
      // K2 (Alg. 4 lines 13-15): all traits' W_R^T W_L, W_R^T y_j, W_R^T W_R in one product
      CKG(c->tic(GWAS_K2, cs2, &dummy));
      if (d.fuse) {
        const long long tot = cols * d.fnq;
        gw::fused_k2_reduce<<<(unsigned)((tot + 255) / 256), 256, 0, cs2>>>(
            fpart, fstride, k1_tiles, (int)cols, (int)d.fnq, (int)(d.t * (d.p + 1)), (int)d.nsq, c2, d.ldc2);
        CKC(cudaGetLastError());
      } else if (lr_r > 0) {  // low-rank trait weights: the products against U_r, then the recombination with W
        CKG(gemm_tn(false, xrp, d.kpad, c->B2(), d.kpad, g2, d.ldg2, cols, lr_nsq + lr_r, d.n, lr_nsq, cs2, 16,
                    splitbuf));
        if (!lr_fused) CKG(lowrank_recombine(c, g2, c2, cols, cs2));
      } else {
        static const int k2_group = getenv("GWAS_K2_GROUP") ? atoi(getenv("GWAS_K2_GROUP")) : 16;
        gw::GemmShape ct{};
        ct.ct = (int)d.t;
        ct.cnlin = (int)(d.t * (d.p + 1));
        ct.cF = (int)(d.p + 2);
        CKG(gemm_tn(false, xrp, d.kpad, c->B2(), d.kpad, c2, d.ldc2, cols, d.n2, d.n, d.nsq, cs2, k2_group,
                    splitbuf, false, nullptr, nullptr, nullptr, d.ctiled ? &ct : nullptr));
      }
      CKG(c->toc(cs2));
    } else {
      // K1i + K2a (int8-sliced, exact): X_R'^T = X_R^T Z and C[:, 0:t(p+1)] = X_R^T (Z B_op) in one launch
      CKG(c->tic(GWAS_K1, cs, &dummy));
      CKG(launch_i8(c->opt.int8_slices, A, lda, cols, d.n, c->dig(), d.kpad, (d.na_pad + round_up(lr_nlin, gw::I8_NB)) / gw::I8_NB,
                    d.na_pad / gw::I8_NB, c->exps(), xrp, d.kpad, d.n, lr_r > 0 ? g2 : c2,
                    lr_r > 0 ? d.ldg2 : d.ldc2, lr_nlin, cs, chol ? d.na_pad / gw::I8_NB : 0,
                    d.fuse ? (int)d.t : 0, c->B2() + d.nsq * d.kpad, d.kpad, fpart, fstride));
      CKG(c->toc(cs));
      if (s >= 0) CKC(cudaEventRecord(c->ev_free[s], cs));
      if (ovl) {
        CKC(cudaEventRecord(c->ev_k1[set], cs));
        CKC(cudaStreamWaitEvent(cs2, c->ev_k1[set], 0));
      }
      // K2b (DMMA): C[:, nsq + j] = sum_k X_R'[k,i]^2 d_j[k]  (W_R^T W_R, the term that needs the rotation)
      CKG(c->tic(GWAS_K2, cs2, &dummy));
      if (d.fuse) {  // NEXT-2: the squared term was contracted in K1i's epilogue; finish it in fixed order
        const long long tot = cols * d.t;
        gw::fused_k2_reduce<<<(unsigned)((tot + 255) / 256), 256, 0, cs2>>>(
            fpart, fstride, (int)(d.na_pad / gw::I8_NB), (int)cols, (int)d.t, 0, (int)d.nsq, c2, d.ldc2);
        CKC(cudaGetLastError());
      } else if (lr_r > 0) {  // low-rank: X_R'^2 against the r columns of U_r, then the recombination with W
        CKG(gemm_tn(false, xrp, d.kpad, c->B2() + lr_nsq * d.kpad, d.kpad, g2 + lr_nsq, d.ldg2, cols, lr_r, d.n,
                    lr_r, cs2, 16, splitbuf));
        if (!lr_fused) CKG(lowrank_recombine(c, g2, c2, cols, cs2));
      } else {
        // xrp holds X_R'^2 (squared in K1i's epilogue), so this is a plain product (nsq = N: no squaring)
        double* wsb = c->rl.wsplit[set] ? reinterpret_cast<double*>(c->work + c->rl.wsplit[set]) : nullptr;
        CKG(gemm_tn(false, xrp, d.kpad, c->B2() + d.nsq * d.kpad, d.kpad, c2 + d.nsq, d.ldc2, cols, d.t, d.n, d.t,
                    cs2, 16, splitbuf, false, nullptr, nullptr, wsb));
      }
      CKG(c->toc(cs2));
    }
    // K3 (Alg. 4 line 16): b_ij := S^-1 b_ij by Schur complement
    gw::SchurArgs a;
    a.C = c2;
    a.ldc = d.ldc2;
    a.Cy = lr_r > 0 ? g2 + d.p * lr_r : c2 + d.p * d.t;  // r_ij: the y field (kept apart in low-rank mode)
    a.ldcy = lr_r > 0 ? d.ldg2 : d.ldc2;
    a.nsq = (int)d.nsq;
    a.cols = (int)cols;
    a.t = (int)d.t;
    a.Lpk = c->Lpk();
    a.v = c->v();
    a.s2 = c->s2();
    a.betaT = c->betaT();
    a.dinv = c->dinv();
    a.eps_collinear = c->opt.eps_collinear;
    a.literal = c->opt.var_convention == GWAS_VAR_LITERAL;
    a.full = c->opt.output_mode == GWAS_OUT_FULL;
    a.tiled = (d.ctiled && lr_r == 0) ? 1 : 0;
    const int oset = (int)(bi & 1);
    uint8_t* ob = c->work + c->rl.outb[oset];
    if (out_dev) {
      a.b = b + blk * d.t * per_pair;
      a.var = var + blk * d.t * per_pair;
      a.status = status + blk * d.t;
    } else {  // results of block bi-2 must have left this staging set
      CKC(cudaStreamWaitEvent(cs2, c->ev_out_free[oset], 0));
      a.b = reinterpret_cast<double*>(ob);
      a.var = a.b + cols * d.t * per_pair;
      a.status = reinterpret_cast<int8_t*>(a.var + cols * d.t * per_pair);
    }
    CKG(c->tic(GWAS_K3, cs2, &dummy));
    if (lr_fused) {  // the recombination products and K3 in one kernel (lowrank_k3.cuh)
      gw::LowrankK3Args la;
      la.G = g2;
      la.ldg = d.ldg2;
      la.r = (int)lr_r;
      la.nsq_lr = (int)lr_nsq;
      la.Wt = reinterpret_cast<const double*>(c->state + c->h.off_wt);
      la.k3 = a;
      CKG(launch_lowrank_schur(la, (int)d.p, cs2));
    } else {
      CKG(launch_schur(a, (int)d.p, cs2));
    }
    CKG(c->toc(cs2));
    if (ovl) CKC(cudaEventRecord(c->ev_set_free[set], cs2));
    if (!out_dev) {  // stream this block's results to the caller's pinned host buffers, overlapped with compute
      CKC(cudaEventRecord(c->ev_out_ready[oset], cs2));
      CKC(cudaStreamWaitEvent(c->dstream, c->ev_out_ready[oset], 0));
      const size_t nb = sizeof(double) * cols * d.t * per_pair;
      CKC(cudaMemcpyAsync(b + blk * d.t * per_pair, a.b, nb, cudaMemcpyDeviceToHost, c->dstream));
      CKC(cudaMemcpyAsync(var + blk * d.t * per_pair, a.var, nb, cudaMemcpyDeviceToHost, c->dstream));
      CKC(cudaMemcpyAsync(status + blk * d.t, a.status, (size_t)cols * d.t, cudaMemcpyDeviceToHost, c->dstream));
      CKC(cudaEventRecord(c->ev_out_free[oset], c->dstream));
    }
  }
  if (ovl) {  // join: the call completes on compute_stream
    CKC(cudaEventRecord(c->ev_join, cs2));
    CKC(cudaStreamWaitEvent(cs, c->ev_join, 0));
  }
  if (!out_dev) {
    CKC(cudaEventRecord(c->ev_djoin, c->dstream));
    CKC(cudaStreamWaitEvent(cs, c->ev_djoin, 0));
  }
  return GWAS_OK;
}

gwas_status gwas_timings(gwas_ctx* c, double* ms_eig, double* ms_pre, double* ms_run) {
  if (!c) return fail(GWAS_E_STATE, "NULL context");
  CKG(c->drain());
  if (ms_eig) *ms_eig = c->ms_eig;
  if (ms_pre) *ms_pre = c->ms_pre;
  if (ms_run) *ms_run = c->ms_acc[0] + c->ms_acc[1] + c->ms_acc[2] + c->ms_acc[3];
  return GWAS_OK;
}

gwas_status gwas_kernel_times(gwas_ctx* c, double* ms, int64_t* launches, int32_t reset) {
  if (!c) return fail(GWAS_E_STATE, "NULL context");
  CKG(c->drain());
  for (int k = 0; k < GWAS_NUM_TIMERS; ++k) {
    if (ms) ms[k] = c->ms_acc[k];
    if (launches) launches[k] = c->launches[k];
    if (reset) {
      c->ms_acc[k] = 0;
      c->launches[k] = 0;
    }
  }
  return GWAS_OK;
}

gwas_status gwas_gemm_tn(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int32_t a_u8, const double* B,
                         int64_t ldb, double* C, int64_t ldc, int64_t nsq, void* stream) {
  g_err.clear();
  if (!A || !B || !C) return fail(GWAS_E_ARG, "NULL pointer argument");
  if (lda < K || ldb < K || ldc < N) return fail(GWAS_E_ARG, "leading dimension too small");
  return gemm_tn(a_u8 != 0, A, lda, B, ldb, C, ldc, M, N, K, nsq, static_cast<cudaStream_t>(stream));
}

void gwas_destroy(gwas_ctx* c) {
  if (!c) return;
  c->drain();
  for (auto e : c->pool) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i) {
    if (c->ev_in[i]) cudaEventDestroy(c->ev_in[i]);
    if (c->ev_free[i]) cudaEventDestroy(c->ev_free[i]);
    if (c->ev_k1[i]) cudaEventDestroy(c->ev_k1[i]);
    if (c->ev_set_free[i]) cudaEventDestroy(c->ev_set_free[i]);
  }
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->ev_djoin) cudaEventDestroy(c->ev_djoin);
  for (int i = 0; i < 2; ++i) {
    if (c->ev_out_ready[i]) cudaEventDestroy(c->ev_out_ready[i]);
    if (c->ev_out_free[i]) cudaEventDestroy(c->ev_out_free[i]);
  }
  if (c->dstream) {
    cudaStreamSynchronize(c->dstream);
    cudaStreamDestroy(c->dstream);
  }
  if (c->aux) {
    cudaStreamSynchronize(c->aux);
    cudaStreamDestroy(c->aux);
  }
  delete c;
}

}  // extern "C"
