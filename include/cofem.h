/* cofem.h — C ABI of the B200-native covariance-free EM (CoFEM) hot path.
 *
 * Paper: covariance-free expectation-maximization (CoFEM) for sparse Bayesian
 * learning, arXiv 2202.12808 (/root/reference/PAPER.md, cited as P:<line>).
 *
 * The library implements Algorithm 1: for each EM iteration it
 * solves  A X = B,  A = beta Phi^T Phi + diag(alpha)  (Eq. 7) for the
 * K+1 right-hand sides B = [b0 | p_1 .. p_K] with b0 = beta Phi^T y (Eq. 5,
 * P:60-63) and K Rademacher probes p_k (Alg. 1 l.5) by U iterations of
 * column-independent Jacobi-preconditioned conjugate gradient batched into
 * matrix-matrix applies (§3.2; readings R3-R6), then
 *     mu = x_0,   s = (1/K) sum_k p_k o x_k        (Eq. 6; Alg. 1 l.7)
 *     alpha_new = 1 / (mu o mu + s)                 (Eq. 8; floor/clamp R7)
 *
 * Conventions (all entry points):
 *  - Vector arguments (alpha, mu, s, y, Phi, obs_idx, taps) may be HOST or
 *    DEVICE pointers; the library detects which (cudaPointerGetAttributes)
 *    and stages host buffers through its own device workspace with
 *    cudaMemcpyAsync on the context's stream.  Device pointers must be on the
 *    context's device.  The caller owns every buffer it passes.
 *  - Phi (DENSE) is never modified.  A DEVICE Phi is borrowed (zero-copy, row
 *    stride ld; the tensor-core path needs ld % 4 == 0) and must outlive the
 *    context; a HOST Phi is copied to a library-owned device buffer at setup.
 *  - Every call enqueues on the context's CUDA stream and returns after one
 *    stream synchronisation (needed to report numerical breakdown).
 *  - A context serves one stream and is not thread-safe.
 *  - Invalid arguments return COFEM_ERR_INVALID and leave the context
 *    unchanged; cofem_last_error() returns a message.
 *  - CG that does not converge within U iterations is NOT an error;
 *    a NaN/Inf met in a recurrence freezes that column and the call returns
 *    COFEM_ERR_NUMERIC with the column and iteration in cofem_last_report()
 *    (S:107).  The M-step never fails (floor/clamp).
 *  - Layout: every D-vector is contiguous, element d = coefficient index d.
 *    DCT2 coefficient vectors are row-major images, d = r * cols + c.
 */
#ifndef COFEM_H
#define COFEM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cofem_ctx_s* cofem_ctx;

typedef enum {
  COFEM_OK = 0,
  COFEM_ERR_INVALID = 1,     /* bad argument / dimension mismatch */
  COFEM_ERR_CUDA = 2,        /* CUDA runtime error */
  COFEM_ERR_NCCL = 3,        /* NCCL unavailable or a library-owned collective failed (sharded modes) */
  COFEM_ERR_NUMERIC = 4,     /* NaN/Inf in the CG recurrence */
  COFEM_ERR_OOM = 5,         /* device allocation failed */
  COFEM_ERR_UNSUPPORTED = 6  /* valid but not implemented (e.g. DCT grid not a power of two) */
} cofem_status;

typedef enum {
  COFEM_OP_DENSE = 0,        /* Phi: N x D matrix, row-major fp32 (§4.1) */
  COFEM_OP_DCT2_MASKED = 1,  /* Phi = S C2^T: orthonormal 2D inverse DCT, then N masked pixels (§4.2; R11) */
  COFEM_OP_CIRCCONV = 2      /* (Phi x)_i = sum_{j<T} h_j x_{(i-j) mod D}, N = D (R12) */
} cofem_op_kind;

typedef struct {
  int32_t kind;              /* cofem_op_kind */
  int64_t N, D;              /* Phi is N x D */
  /* DENSE */
  const float* phi;          /* N x D row-major fp32, row stride ld (>= D) elements; host or device */
  int64_t ld;
  /* DCT2_MASKED */
  int32_t rows, cols;        /* grid, rows * cols == D, each a power of two in [16, 1024] */
  const int64_t* obs_idx;    /* N pixel indices (r * cols + c), sorted, distinct, in [0, D); host or device */
  int32_t convention;        /* 0: Phi = S C2^T (paper, default; 1024 x 1024 fast path); 1: Phi = S C2 (BASELINE config 4 literally; generic passes) */
  /* CIRCCONV */
  const float* taps;         /* ntaps fp32 filter taps h_j; host or device */
  int32_t ntaps;             /* 1 <= ntaps <= 64, ntaps <= D */
  /* DENSE column-sharded mode: this rank holds Phi's columns
   * [d_offset, d_offset + D) of D_global (phi is N x D local, y the full N); alpha, mu, s
   * are the matching D-slices.  d_offset must be a multiple of 128 (probe counters,
   * reading R8).  D_global = 0: unsharded. */
  int64_t d_offset;
  int64_t D_global;
} cofem_operator;

typedef struct {
  int32_t cg_iters;          /* U >= 1: fixed CG iteration count (BASELINE north_star; R5) */
  int32_t precond;           /* 1: Jacobi z = r / (beta colsq + alpha) (default, R6); 0: plain CG */
  double den_floor;          /* M-step floor on mu^2 + s (default 1e-12) */
  double alpha_max;          /* M-step clamp (default 1e12) */
  int32_t probe_precision;   /* 0: probe columns in fp32 (fast); 1: fp64 (parity mode). The mean column is always fp64. */
  int32_t max_probes;        /* K capacity of the workspaces (>= any K passed later) */
  /* Column-sharded dense mode: NCCL rank / world and the 128-byte ncclUniqueId from
   * cofem_get_unique_id (broadcast by the caller).  nccl_id = NULL: single GPU.  World 1 with
   * an id runs the sharded code path on a 1-rank communicator (tests). */
  int32_t rank, world;
  const uint8_t* nccl_id;
  /* NEXT-1, the paper's stopping rule ("||A X - B||_F / ||B||_F < eps"), reading R19:
   * cg_rtol = eps > 0 freezes column j once rho_j <= eps^2 rho_j(0), rho = r^T M^-1 r (with
   * precond = 0 exactly ||r_j|| <= eps ||b_j||); when every column has frozen the Frobenius
   * criterion holds and the remaining iterations launch but do no column work.  U stays the cap.
   * 0 (default): fixed U iterations (BASELINE north_star, R5).  Must be in [0, 1). */
  double cg_rtol;
  /* Operator path (tests, comparisons): 0 = auto, the fastest eligible kernels (dense: the whole
   * CG loop in thread-block clusters (one launch) when Phi fits a cluster's shared memory -- config 1 --, else
   * tcgen05 3xTF32 for fp32 probes; DCT2 1024 x 1024: the warp-per-line FFT path; CIRCCONV:
   * overlap-save FFT); 1 = the general kernels (dense FP32 SIMT, generic DCT passes, direct 127-tap
   * stencil); 2 = as 0 without the cluster CG loop (small dense problems on the per-iteration
   * tensor-core kernels). */
  int32_t apply_path;
  /* Concurrent probe-column groups, 0 = auto.  1024 x 1024 DCT path: that many groups on their own
   * streams (auto 2, range 0..4).  Dense cluster CG loop: that many thread-block
   * clusters in one launch, each solving a contiguous share of the probes (cluster 0 also the mean;
   * DESIGN.md §7.2.1; auto max(min(4, K), ceil(K/4)), at most K and 8).  Ignored elsewhere. */
  int32_t probe_groups;
  /* 1 (default): each E-step is captured once into a CUDA graph and replayed; 0: launched directly. */
  int32_t use_graph;
  /* Multi-GPU mode; rank, world and nccl_id as above.
   *  0: single GPU, or (nccl_id set) the sharded mode the operator implies: column-sharded DENSE /
   *     D-sharded CIRCCONV (d_offset, D_global);
   *  1: probe-parallel (BASELINE north_star "probe-parallel when Phi fits on one GPU"): every rank
   *     holds the whole operator; cofem_estep / cofem_em take the GLOBAL K and this library splits
   *     the probes over the ranks (global Philox indices, R8; rank 0 also solves the mean system
   *     with fewer probes), then sums s over ranks (one NCCL all-reduce of D fp64 per E-step) and
   *     broadcasts mu = x0 from rank 0; every rank returns the same mu, s and alpha.  max_probes is
   *     the per-rank capacity (>= ceil(K / world) + 1). */
  int32_t dist_mode;
  /* NEXT-1 (reading R20, P:98 leaves the initial guess open): 1 =
   * inside cofem_em, every E-step after the call's first starts the mean system's CG from the
   * previous E-step's mu (x0 = mu_prev, r0 = b0 - A mu_prev: one extra mean-column apply per
   * E-step), the probes from zero (they are fresh); the freeze threshold stays relative to
   * b0^T M^-1 b0.  0 (default): X0 = 0 every E-step (R4).  Not in the sharded modes. */
  int32_t warm_start;
  /* NEXT-2 CG variant ("any" CG method; reading R23 in DESIGN.md).  1: the standard
   * preconditioned CG of Algorithm 1 (two reductions per iteration, gamma = p^T A p and
   * rho' = r'^T M^-1 r', in the oracle's order).  2: single-reduction CG -- after the apply one
   * reduction gives gamma, rho = r^T M^-1 r (recomputed, so no drift), delta1 = q^T M^-1 r and
   * delta2 = q^T M^-1 q; a = rho / gamma as in Algorithm 1, and rho' = rho - 2 a delta1 + a^2 delta2
   * (exact algebra for r' = r - a q) gives b = rho' / rho; the update then needs no reduction.
   * In the column-sharded dense mode this merges the gamma and rho' NCCL all-reduces into one
   * (with the two W all-reduces grouped into one NCCL launch: two collective launches per CG
   * iteration instead of four).  Only the column-sharded dense mode
   * implements 2 (COFEM_ERR_UNSUPPORTED elsewhere).  0 (default): auto = 2 in the column-sharded
   * dense mode, 1 everywhere else. */
  int32_t cg_variant;
} cofem_options;

/* NCCL unique id for cofem_options.nccl_id (call on one rank, broadcast the 128 bytes).
 * Returns COFEM_ERR_NCCL if libnccl.so.2 cannot be loaded. */
cofem_status cofem_get_unique_id(uint8_t id[128]);

/* Fill *opt with the defaults above (U = 100, precond = 1, max_probes = 32, apply_path = 0,
 * probe_groups = 0, use_graph = 1, single GPU). */
void cofem_default_options(cofem_options* opt);

/* Build a context: validate, copy/derive the operator (dense Phi copy; DCT
 * mask and twiddle tables; conv Gram stencil g = autocorr(h)), compute
 * b0 = beta Phi^T y (fp64, Eq. 5) and colsq = diag(Phi^T Phi) (fp64), and
 * allocate all workspaces for K <= opt->max_probes.
 *   y:           N fp32 observations, host or device
 *   beta:        noise precision > 0 (Alg. 1 signature)
 *   cuda_stream: cudaStream_t to enqueue on (NULL = legacy default stream)
 * Errors: COFEM_ERR_INVALID (dims, beta <= 0, mask unsorted, ntaps out of
 * range), COFEM_ERR_UNSUPPORTED, COFEM_ERR_OOM, COFEM_ERR_CUDA. */
cofem_status cofem_setup(cofem_ctx* out, const cofem_operator* op, const float* y,
                         double beta, const cofem_options* opt, void* cuda_stream);

/* One simplified E-step (Alg. 1 lines 3-7; Eq. 6-7) at precision alpha:
 *   alpha:     D fp64, every entry > 0 and finite
 *   K:         number of probes this call solves, 1 <= K <= max_probes
 *   seed, t:   probe stream: p_k[d] from Philox4x32-10 with key = seed and
 *              counter (d/128, k_offset + k, t, 0x50524F42) (R8)
 *   k_offset:  global index of this call's first probe (probe-parallel ranks)
 *   K_total:   the K of Eq. 6's 1/K (== K on one GPU; the global K when the
 *              probes are split over ranks: s is then this rank's partial sum)
 *   mu, s:     out, D fp64 each
 * Returns COFEM_OK or COFEM_ERR_NUMERIC (mu/s still written). */
cofem_status cofem_estep(cofem_ctx ctx, const double* alpha, int32_t K, uint64_t seed, int32_t t,
                         int32_t k_offset, int32_t K_total, double* mu, double* s);

/* The same E-step for the probe columns only (probe-parallel ranks that do not own the mean
 * system): column 0 (b0 = beta Phi^T y) is frozen at once and none of its work is
 * launched; s is this rank's partial sum as in cofem_estep; mu is not computed (the owner rank
 * broadcasts it).  Arguments and errors as cofem_estep. */
cofem_status cofem_estep_probes(cofem_ctx ctx, const double* alpha, int32_t K, uint64_t seed, int32_t t,
                                int32_t k_offset, int32_t K_total, double* s);

/* One batched Gram apply (the CG matrix-matrix product of §3.2; Eq. 7):
 *   q0 = A x0,  Q_k = A X_k  (k < K),   A = beta Phi^T Phi + diag(alpha),
 * through exactly the kernels the E-step uses (mean column in fp64; probe columns in
 * probe precision: fp32, or fp64 with probe_precision = 1), plus gamma_j = x_j^T (A x_j).
 *   alpha:  D fp64 (> 0, finite)          x0, q0: D fp64 (mean column)
 *   X, Q:   K x D, row k = column k + 1 of the block, contiguous (row stride D), float
 *           (probe_precision 0) or double (1)
 *   gamma:  K + 1 fp64 out (column 0 first), may be NULL
 * Host or device pointers; 1 <= K <= max_probes.  Errors: COFEM_ERR_INVALID. */
cofem_status cofem_apply(cofem_ctx ctx, const double* alpha, int32_t K, const double* x0, const void* X,
                         double* q0, void* Q, double* gamma);

/* M-step (Eq. 8): alpha_out_d = min(1 / max(mu_d^2 + s_d, den_floor), alpha_max). Never fails. */
cofem_status cofem_mstep(cofem_ctx ctx, const double* mu, const double* s, double* alpha_out);

/* Algorithm 1: `iters` EM iterations with fresh probes each (probe counter
 * t = t0 + i), starting from alpha_init (NULL: all ones, Alg. 1 l.1).
 * Outputs alpha after the last M-step and mu, s of the last E-step (R9);
 * any output may be NULL.  cofem_em(ctx, 1, K, seed, 0, NULL, ...) equals
 * cofem_estep(alpha = 1, t = 0) followed by cofem_mstep. */
cofem_status cofem_em(cofem_ctx ctx, int32_t iters, int32_t K, uint64_t seed, int32_t t0,
                      const double* alpha_init, double* alpha_out, double* mu_out, double* s_out);

/* NEXT-4 multi-task SBL (P:179 names the extension; reading R22 in DESIGN.md): L tasks
 * y_l = Phi z_l + noise share Phi, beta and the prior precisions alpha.  Sigma is then shared, so
 * the E-step solves A x = beta Phi^T y_l for every task mean and the K probes give one s; the
 * M-step is alpha = 1 / (mean_l mu_l o mu_l + s) (floor / clamp as Eq. 8).  `iters` EM iterations
 * (probe counter t0 + i) from alpha_init (NULL: ones).
 *   Y:      L x N fp32, row l = task l's observations (host or device)
 *   MU_out: L x D fp64, row l = task l's mu (last E-step); alpha_out, s_out: D fp64; any may be NULL
 * L = 1 is cofem_em.  The context's own y (cofem_setup) is unchanged afterwards.
 * Errors: COFEM_ERR_INVALID (L < 1, K), COFEM_ERR_UNSUPPORTED (sharded / probe-parallel contexts,
 * warm_start). */
cofem_status cofem_em_multi(cofem_ctx ctx, int32_t L, const float* Y, int32_t iters, int32_t K, uint64_t seed,
                            int32_t t0, const double* alpha_init, double* alpha_out, double* MU_out, double* s_out);

typedef struct {
  int32_t cols;                   /* K + 1 columns of the last E-step (column 0 = mean, R2) */
  int32_t cg_iters;               /* U */
  const int32_t* frozen_at;       /* [cols] iteration at which a column froze, -1 if never (R5) */
  const double* rho;              /* [cols] final recursive M^-1-norm residual^2 r^T z */
  const double* rho0;             /* [cols] initial r^T z */
  int32_t bad_col, bad_iter;      /* first column that met NaN/Inf, -1 if none */
  double estep_ms_last;           /* device time of the last E-step (CUDA events) */
  int64_t launches;               /* kernels launched by this context so far */
  /* Support certificate of the last E-step's mu (BASELINE north_star: recovered support
   * |mu_d| > 1e-3 max|mu|, reading R16; SURVEY §8(c) "fragility"): support_count coordinates are
   * in the support; support_adjacent of them or of the rest lie within support_delta of the
   * threshold, | |mu_d| / max|mu| - 1e-3 | < support_delta -- the only coordinates whose membership
   * a relative perturbation of mu below support_delta (e.g. fp32 probe columns vs fp64) can flip;
   * support_min_margin is the smallest such margin over all d.  support_delta = 1e-6. */
  int64_t support_count, support_adjacent;
  double support_max_abs_mu, support_min_margin, support_delta;
  int64_t collectives;            /* NCCL launches by this context so far (a grouped call counts once;
                                   * 0 on a single GPU) */
} cofem_report;

/* The probe-parallel owner split (dist_mode 1) of a global K over `world` ranks, a host-only
 * utility (no GPU): rank 0 owns the mean system and K0 = max(1, min(K - (world - 1),
 * floor((K + mean_cost) / world - mean_cost + 1/2))) probes; ranks 1.. split the remaining K - K0
 * contiguously.  mean_cost = the mean system's cost in probe columns (the library uses 2 on the
 * 1024 x 1024 DCT and FFT-convolution paths, 0 on the dense tensor-core path).  Writes the first
 * global probe index, the count and whether the rank solves the mean system.
 * Errors: COFEM_ERR_INVALID when K < world or rank is out of range. */
cofem_status cofem_probe_split(int32_t K, int32_t world, int32_t rank, double mean_cost, int32_t* k_offset,
                               int32_t* K_local, int32_t* owns_mean);

/* Report of the last E-step; the pointers stay valid until the next call on ctx. */
cofem_status cofem_last_report(cofem_ctx ctx, cofem_report* out);

/* Per-kernel-class device timing (CUDA events around each launch of the
 * classes in `mask` on the context stream; bit i = class i, see
 * cofem_kernel_class_name).  cofem_profile_read syncs and returns, for class
 * i, the summed milliseconds and launch count since the last reset. */
cofem_status cofem_profile_enable(cofem_ctx ctx, uint32_t mask);
cofem_status cofem_profile_read(cofem_ctx ctx, int32_t cls, double* total_ms, int64_t* count, int32_t reset);
/* Busy time of class i since its last reset: the measure of the union of its launch intervals, so
 * launches of the class that ran concurrently (probe-column groups on separate streams) count
 * once.  <= total_ms.  Reset together with cofem_profile_read(..., reset = 1). */
cofem_status cofem_profile_busy(cofem_ctx ctx, int32_t cls, double* busy_ms);
const char* cofem_kernel_class_name(int32_t cls);   /* NULL past the last class */

const char* cofem_last_error(cofem_ctx ctx);        /* message of the last failing call ("" if none); ctx may be NULL */
const char* cofem_version(void);
void cofem_destroy(cofem_ctx ctx);

#ifdef __cplusplus
}
#endif
#endif /* COFEM_H */
