/* gwas.h -- C-ABI of the B200-native CLAK-Eig hot path (libgwas.so).
 *
 * The library solves the 2-D sequence of generalised least-squares problems of PAPER.md Eq. probDef
 * (P:26-40): for every SNP i (1..m) and trait j (1..t), with X_i = [X_L | g_i] (n x w, w = p + 1),
 *
 *     b_ij   = (X_i^T M_j^-1 X_i)^-1 X_i^T M_j^-1 y_j,     M_j = sigma2_j (h2_j Phi + (1 - h2_j) I)
 *     Var_ij = (X_i^T M_j^-1 X_i)^-1                       (var_convention 0; reading A1)
 *            = sigma2_j (X_i^T M_j^-1 X_i)^-1              (var_convention 1; P:31 as printed)
 *
 * by CLAK-Eig for multi-trait analysis (Alg. 4):
 *     gwas_setup  = Alg. 4 lines 1, 2, 4 and the per-trait block 6-11: Phi = Z W Z^T
 *                   (cuSOLVER dsyevd, timed separately), X_L' = Z^T X_L, Y' = Z^T Y, D_j, and the
 *                   Cholesky-factored top-left blocks S_TL_j = X_L'^T D_j X_L', b_T_j = X_L'^T D_j y'_j;
 *     gwas_run    = Alg. 4 line 3 (X_R := Z^T X_R) streamed in column blocks, and the inner loop
 *                   lines 13-16 for every (i, j) of the block.
 *
 * Conventions (all calls):
 *   - Matrices are column-major fp64 unless stated; sizes are int64_t; "ld" = leading dimension in elements.
 *   - The caller owns every buffer (state, workspace, outputs) and the compute / copy streams; the library
 *     allocates no device memory (a cuSOLVER handle is created inside gwas_setup only).  Each context creates
 *     and owns two internal streams: the overlap-mode auxiliary stream and the D2H stream for host outputs.
 *   - Pointers documented "host or device" are classified with cudaPointerGetAttributes.
 *   - Calls enqueue on options.compute_stream (and options.copy_stream for staging) and return without
 *     synchronising, except gwas_setup / gwas_attach, which synchronise to report errors.
 *   - On error a call returns a non-zero gwas_status and gwas_last_error() (thread-local) names the cause
 *     (for GWAS_E_NOT_SPD: the trait j and, for D_j, the eigen-index k).
 *   - Per-pair numerical failures never fail a call: status[i][j] = 1 (SNP collinear with X_L: Schur
 *     complement sigma_ij <= eps_collinear * c_ij, reading A6) or 2 (non-finite), with NaN payload.
 */
/* Environment knobs (tuning / debugging only; results are bitwise unaffected unless stated):
 *   GWAS_I8_KERNEL=1sm      the 1-SM int8 kernel (M = 128 MMAs) for every block; default: the 2-SM (cta_group::2,
 *                           M = 256) kernel for blocks of more than 128 SNP rows, the 1-SM one otherwise
 *   GWAS_I8_CLUSTER=1|2|4   int8 cluster size: 1-SM kernel, CTAs multicasting the digit slab (default 2); 2-SM
 *                           kernel, 2 = one pair, 4 = two pairs sharing the slab (default 4 at 7 digits, 2 at 8)
 *   GWAS_I8_BK=64|128       int8 K bytes per pipeline stage (64- or 128-byte swizzle); default 128 (64 for the 1-SM
 *                           8-digit kernel, whose 128-byte stages would leave a 2-deep ring)
 *   GWAS_I8_PERSIST=0|1     2-SM int8 kernel: persistent clusters looping over tiles (default 1) or one per tile
 *   GWAS_BN64_WAVES=w       force the 128/64-wide tile choice of the DMMA kernel by a w-wave threshold
 *   GWAS_I8_GROUP=g         int8 kernel rasterisation group (row tiles per sweep of the digit slabs), default 32
 *   GWAS_K1_GROUP=g         K1 rasterisation group (row tiles per sweep of the Z panels), default 32
 *   GWAS_K2_GROUP=g         K2 rasterisation group, default 16 (DRAM read per 8192-SNP C4 block: 4 -> 10.9,
 *                           8 -> 7.9, 16 -> 6.8, 32 -> 9.8, 64 -> 17.5 GB; per 15104-SNP block 8 / 16 / 32 -> 19.3 /
 *                           15.5 / 22.5 GB; time unchanged: DMMA-bound)
 *   GWAS_I8_TRACE=<file>    append the int8 kernel's debug trace to <file>: per CTA 16 slots -- %globaltimer phase
 *                           stamps, SM id, clock64 cycles waited on full / empty barriers, k-stages (tools/i8_trace.py;
 *                           allocates a 512 KB device buffer and synchronises after every launch)
 *   GWAS_I8_DBG=1|2         int8 epilogue without TMEM loads / stores (timing experiments; results invalid)
 *   GWAS_K3_PLAIN=1         K3 on the trait-tiled C with the register-prefetch kernel instead of the bulk-copy
 *                           (TMA) streamed one (comparison only; bitwise identical results)
 *   GWAS_LR_UNFUSED=1       low-rank mode: separate K = r recombination products + K3 instead of the fused kernel
 *                           (even t only; results equal up to rounding) */
#ifndef GWAS_H
#define GWAS_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define GWAS_API __attribute__((visibility("default")))
#else
#define GWAS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gwas_ctx gwas_ctx; /* opaque, bound to one CUDA device */

typedef enum {
  GWAS_OK = 0,
  GWAS_E_ARG = 1,      /* bad pointer / shape / range: n < p + 1, p < 1, t < 1, h2 outside [0,1], sigma2 <= 0,
                          non-finite inputs, unaligned ld, unpinned host X_R, ... */
  GWAS_E_NOT_SPD = 2,  /* some sigma2_j (h2_j w_k + 1 - h2_j) <= eps_spd (reading A7), or S_TL_j not SPD
                          (X_L rank-deficient); message names j (and k) */
  GWAS_E_EIG = 3,      /* cusolverDnDsyevd (or, for GWAS_ALG_CHOL, dtrtri) reported info != 0 */
  GWAS_E_CUDA = 4,     /* a CUDA / cuSOLVER runtime error */
  GWAS_E_NOMEM = 5,    /* caller-provided state or workspace smaller than gwas_state_bytes / _workspace_bytes */
  GWAS_E_STATE = 6     /* wrong call order, or a state buffer whose header does not match (gwas_attach) */
} gwas_status;

enum { GWAS_XR_F64 = 0, GWAS_XR_U8 = 1 };          /* X_R element type: fp64, or uint8 dosages (exact) */
enum { GWAS_OUT_SNP = 0, GWAS_OUT_FULL = 1 };      /* outputs per pair: (b_g, Var_gg) or w entries of b, diag Var */
enum { GWAS_VAR_TEXTBOOK = 0, GWAS_VAR_LITERAL = 1 };
enum { GWAS_PAIR_OK = 0, GWAS_PAIR_COLLINEAR = 1, GWAS_PAIR_NONFINITE = 2 };
enum { GWAS_K1 = 0, GWAS_K2 = 1, GWAS_K3 = 2, GWAS_H2D = 3, GWAS_NUM_TIMERS = 4 };
enum { GWAS_ALG_EIG = 0, GWAS_ALG_CHOL = 1 };
enum { GWAS_EST_ML = 0, GWAS_EST_REML = 1 };         /* variance-component estimator (gwas_setup_estimate) */

typedef struct {
  int32_t device;          /* CUDA ordinal the context binds to */
  int32_t xr_dtype;        /* GWAS_XR_F64 or GWAS_XR_U8 */
  int32_t output_mode;     /* GWAS_OUT_SNP (default) or GWAS_OUT_FULL */
  int32_t var_convention;  /* GWAS_VAR_TEXTBOOK (default) or GWAS_VAR_LITERAL */
  int64_t block_cols;      /* SNP columns per streamed block k ("user-configurable"); default 8192.
                              0 = auto: FP64 mode picks the k in [4096, 16384] (multiple of 128) whose K1 / K2 tile
                              grids quantise best into whole waves on the device's SMs (int8-sliced mode: 8192);
                              gwas_run_info reports the choice.  Results are bitwise independent of k. */
  double eps_spd;          /* default 1e-10 */
  double eps_collinear;    /* default 1e-10, relative Schur-complement threshold (reading A6) */
  void* compute_stream;    /* cudaStream_t for kernels (NULL = legacy default stream) */
  void* copy_stream;       /* cudaStream_t for host->HBM staging of X_R blocks (NULL = compute_stream) */
  int32_t timing;          /* 1 = bracket every K1/K2/K3/H2D launch with CUDA events (gwas_kernel_times) */
  int32_t int8_slices;     /* 0 (default): K1/K2 on the FP64 DMMA tensor pipe.  8 or 7: integer-sliced mode
                              (requires xr_dtype = GWAS_XR_U8 and n <= 66000): X_R^T Z and
                              the linear K2 terms X_R^T (Z D_j [X_L' | y'_j]) run as int8 tcgen05 products against
                              S signed digits of each fp64 column (exact int32 accumulation in TMEM), the
                              W_R^T W_R term stays on DMMA.  Representation error of a column: <= 2^-57 (S = 8, below
                              fp64 rounding) or 2^-50 (S = 7, 12 % less tensor work; below the error of Z itself)
                              of its largest entry.  Fixed at setup (part of the state). */
  int32_t overlap;         /* 1 = pipeline blocks over two streams: block b's K2 + K3 run on an internal auxiliary
                              stream while block b+1's K1 runs on compute_stream (double-buffered intermediates;
                              the stream is created and owned by the context).  gwas_run still completes on
                              compute_stream.  Per-kernel event times then overlap.  Default 0. */
  int32_t algorithm;       /* GWAS_ALG_EIG (default): CLAK-Eig, Alg. 4, any t.
                              GWAS_ALG_CHOL: CLAK-Chol single-trait analysis, Alg. 3, t == 1 only:
                              M = sigma2 (h2 Phi + (1 - h2) I) = L L^T (cuSOLVER dpotrf) and L^-1 (dtrtri) replace
                              the eigendecomposition; K1 becomes X_R := L^-1 X_R on the lower triangle only
                              (half the flops of Z^T X_R), K2/K3 run with D = I.  Fixed at setup (state). */
  int32_t fuse_k2;         /* 1 (default): for few traits (FP64 mode t (p + 2) <= 28; int8-sliced mode t <= 8) K2 is
                              contracted inside K1's epilogue per column tile, so X_R' never
                              goes to HBM; a fixed-order reduction finishes it.  0: separate K2 product.  A run-time
                              choice (not part of the state); results differ from the unfused path only by rounding. */
  int32_t trait_rank;      /* 0 (default): the exact per-trait weights D_j of Alg. 4 line 6 in K2 (the paper's design).
                              -1: low-rank trait weights (reading L1, CLAK-Eig only, t >= 16): setup
                              factors D = [d_1 .. d_t] = U S V^T (cuSOLVER gesvd, of D^T when t > n), keeps the r <= 64 singular
                              triplets above 1e-15 s_0 (r rounded up to 8) and K2 contracts X_R' against the p r + t + r
                              columns [U_r (.) X_L'_f | d_j (.) y'_j | U_r] instead of t (p + 2); a K = r product with
                              W = S_r V_r^T restores the per-trait terms.  Error vs the exact weights ~ 1e-13 relative.
                              Kept exact when it would not shrink the products (2 r >= t).  Part of the state. */
} gwas_options;

/* Fills the defaults listed above (device 0, u8 X_R). */
GWAS_API void gwas_default_options(gwas_options* opt);

/* Bytes of the replicated state buffer (header + Z + W + B_op/D operand + per-trait factors).  The buffer is
 * position-independent: rank 0 fills it in gwas_setup, other ranks receive it byte-for-byte (one NCCL
 * broadcast) and call gwas_attach.  Returns 0 on invalid sizes. */
GWAS_API size_t gwas_state_bytes(int64_t n, int64_t p, int64_t t, const gwas_options* opt);

/* Bytes of per-device scratch: max(setup needs incl. the dsyevd workspace, run needs = 2 staging buffers +
 * the rotated block X_R' + the block's reductions).  Queries cuSOLVER on opt->device.  0 on error. */
GWAS_API size_t gwas_workspace_bytes(int64_t n, int64_t p, int64_t t, const gwas_options* opt);

/* Alg. 4 lines 1-2, 4, 6-11; with GWAS_ALG_CHOL, Alg. 3 lines 1-3, 5-7.
 *   phi    n x n symmetric (col-major, ld = n), host or device, read-only
 *   XL     n x p (col-major, ld = n), column 0 is the intercept (any full-column-rank X_L is accepted)
 *   Y      n x t (col-major, ld = n)
 *   h2, sigma2   t values each (host or device); h2 in [0,1], sigma2 > 0
 *   state_dev / work_dev   caller-owned device buffers of at least the sizes above
 * On success *out is a new context (free with gwas_destroy) and state_dev holds the replicated state.
 * Synchronises; setup time is reported by gwas_timings (eig and precompute separately). */
GWAS_API gwas_status gwas_setup(const gwas_options* opt, int64_t n, int64_t p, int64_t t,
                       const double* phi, const double* XL, const double* Y,
                       const double* h2, const double* sigma2,
                       void* state_dev, size_t state_bytes, void* work_dev, size_t work_bytes,
                       gwas_ctx** out);

/* The paper's first step ("the reduced model (with X = [1 | L]) is fit to the data, thus obtaining the
 * estimates {sigma2^, h2^}"; eigen-based ML (GenABEL, FaST-LMM) or REML (EMMAX), cost 10/3 n^3 + O(v n p^2))
 * followed by gwas_setup with those estimates, sharing one eigendecomposition.  After Alg. 4 lines 1, 2, 4 every
 * trait's profile log-likelihood l_j(h) (beta and sigma2 profiled out; reading E1) is evaluated in the
 * eigenbasis on the grid h = g/100, g = 0..100 (points with some h w_k + 1 - h <= eps_spd are infeasible), and
 * the first grid maximum is refined by 50 bisection steps on the sign of dl/dh in the neighbouring grid interval
 * (readings E2, E3).  sigma2_j = R/n (ML) or R/(n - p) (REML) at h2_j.  Requires opt->algorithm = GWAS_ALG_EIG.
 *   method        GWAS_EST_ML or GWAS_EST_REML
 *   h2_out, sigma2_out, loglik_out   t doubles each, host or device, may be NULL; written before returning
 *   other arguments as gwas_setup (without h2 / sigma2).
 * Errors: GWAS_E_ARG (bad method / algorithm), GWAS_E_NOT_SPD naming the first trait whose residual R is not > 0
 * (y_j in the span of X_L) or that has no feasible grid point; otherwise as gwas_setup.  The estimation time
 * (kernels only) is reported by gwas_estimate_ms. */
GWAS_API gwas_status gwas_setup_estimate(const gwas_options* opt, int64_t n, int64_t p, int64_t t,
                                const double* phi, const double* XL, const double* Y, int32_t method,
                                double* h2_out, double* sigma2_out, double* loglik_out,
                                void* state_dev, size_t state_bytes, void* work_dev, size_t work_bytes,
                                gwas_ctx** out);

/* Low-rank trait weights chosen at setup: *r = kept rank (0 = exact weights), *s0 / *s_r = largest singular value
 * of D and the first dropped one (either may be NULL). */
GWAS_API gwas_status gwas_trait_rank(gwas_ctx* ctx, int32_t* r, double* s0, double* s_r);

/* Estimation diagnostics: g_star[j] = index g of the first grid maximum h = g/100 of trait j's profile likelihood
 * (reading E3), t int32 values written to host memory.  GWAS_E_STATE for a context not made by gwas_setup_estimate. */
GWAS_API gwas_status gwas_estimate_grid_argmax(gwas_ctx* ctx, int32_t* g_star);

/* Run configuration fixed at setup / attach: *block_cols = k actually used (resolves block_cols = 0), *fused_k2 =
 * 1 if K2 is contracted in K1's epilogue for this shape (opt.fuse_k2 and few traits).  Either may be NULL. */
GWAS_API gwas_status gwas_run_info(gwas_ctx* ctx, int64_t* block_cols, int32_t* fused_k2);

/* Event time (ms) of the estimation kernels of gwas_setup_estimate (0 for a gwas_setup context). */
GWAS_API gwas_status gwas_estimate_ms(gwas_ctx* ctx, double* ms);

/* For ranks != 0 after state_dev was broadcast from a gwas_setup rank: validates the state header against
 * (n, p, t, opt) and creates a context.  Synchronises. */
GWAS_API gwas_status gwas_attach(const gwas_options* opt, int64_t n, int64_t p, int64_t t,
                        void* state_dev, size_t state_bytes, void* work_dev, size_t work_bytes,
                        gwas_ctx** out);

/* Alg. 4 line 3 + lines 13-16 for ncols SNP columns.
 *   XR     n x ncols, column-major with leading dimension ldx (elements, >= n), element type opt.xr_dtype.
 *          Device pointer: ldx * sizeof(elem) must be a multiple of 16 and the address 16-byte aligned.
 *          Host pointer: must be page-locked (cudaHostAlloc / cudaHostRegister); blocks of block_cols
 *          columns are staged to HBM on copy_stream, double-buffered against compute (any ldx >= n).
 *   b, var, status: all device memory, or all page-locked host memory (then each block's results are staged in
 *          the workspace and copied to the host on an internal D2H stream while later blocks compute -- the
 *          output side of the paper's double buffering).
 *   b, var ncols x t row-major ([i][j], trait fastest) in GWAS_OUT_SNP mode, or
 *          ncols x t x w ([i][j][e], e = 0..p-1 the X_L coefficients, e = p the SNP) in GWAS_OUT_FULL mode;
 *          var holds Var_gg (SNP mode) or the diagonal of Var (full mode).
 *   status ncols x t int8 (GWAS_PAIR_*).
 * Asynchronous on compute_stream; XR and the outputs must stay valid until it completes. */
GWAS_API gwas_status gwas_run(gwas_ctx* ctx, int64_t ncols, const void* XR, int64_t ldx,
                     double* b, double* var, int8_t* status);

/* Event-based times (ms): eigendecomposition, the rest of setup, and the sum of gwas_run calls' kernels
 * (ms_run = K1 + K2 + K3 + H2D event sums; requires opt.timing).  Synchronises the compute stream. */
GWAS_API gwas_status gwas_timings(gwas_ctx* ctx, double* ms_eig, double* ms_precompute, double* ms_run);

/* Per-kernel event sums since the last reset (requires opt.timing): ms[GWAS_K1..GWAS_H2D] and launch counts.
 * reset != 0 clears them after reading.  Synchronises the compute and copy streams. */
GWAS_API gwas_status gwas_kernel_times(gwas_ctx* ctx, double* ms, int64_t* launches, int32_t reset);

/* Unit-test entry to the K1/K2 kernel itself (no context):  C[i][c] = sum_r A(r, i) * B(r, c) for
 * i < M, c < N, r < K, with A column-major K x M (ld lda; uint8 if a_u8 else fp64) and B column-major K x N
 * (ld ldb), C row-major M x N (ld ldc); columns c >= nsq use A(r,i)^2 (K2's squared block; pass
 * nsq >= N for a plain product; otherwise nsq % 32 == 0).  All device pointers; lda*elem and ldb*8 multiples of 16, ldc even. */
GWAS_API gwas_status gwas_gemm_tn(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int32_t a_u8,
                         const double* B, int64_t ldb, double* C, int64_t ldc, int64_t nsq, void* stream);

GWAS_API void gwas_destroy(gwas_ctx* ctx);      /* frees the context only, nothing caller-owned */
GWAS_API const char* gwas_last_error(void);     /* thread-local message of the last failing call ("" if none) */
GWAS_API const char* gwas_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GWAS_H */
