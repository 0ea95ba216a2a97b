// internal.cuh — shared declarations of the CoFEM CUDA library (sm_100a).
// Product code: nothing here is shared with, or derived from, oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/cofem.h"

namespace cofem {

// ---------------------------------------------------------------- constants
constexpr int MAXM = 129;              // max columns (K + 1) supported by the fused vector kernels
constexpr int VEC_THREADS = 256;       // vector kernels: threads per CTA
constexpr int VEC_ELEMS = 8;           // elements per thread per tile
constexpr int VEC_TILE = VEC_THREADS * VEC_ELEMS;   // 2048 d per tile
constexpr double FREEZE_TAU = 1e-30;   // reading R5
constexpr uint32_t PROBE_TAG = 0x50524F42u;

enum KernelClass : int {
  KC_PROBES = 0, KC_INIT, KC_DIR, KC_UPDATE, KC_FINAL,
  KC_DENSE_PHI_P, KC_DENSE_PHIT_W,
  KC_DCT_ROWS_INV, KC_DCT_COLS, KC_DCT_ROWS_FWD,
  KC_CONV_APPLY, KC_MEAN, KC_SETUP, KC_DCT_FLOW, KC_DENSE_CLUSTER, KC_COUNT
};

// Per-column CG scalars (device).  Column 0 = mean system (R2).
struct ColState {
  double rho, rho0, gamma, a, b;
  int frozen;       // 1 once a freeze rule fired (R5)
  int frozen_at;    // iteration index, -1 if never
  int nonfinite;    // the freeze was caused by NaN/Inf
  int pad;
  double tau;       // freeze when !(rho > tau rho0): FREEZE_TAU (R5) or cg_rtol^2 (reading R19)
};

template <typename T> struct cplx { T x, y; };

// ---------------------------------------------------------------- context
struct Ctx {
  int kind = 0;
  double freeze_tau = FREEZE_TAU;   // max(FREEZE_TAU, cg_rtol^2)
  // k_update over (D tile x probe-column chunk) when the D tiles alone underfill the SMs
  int upd_chunks = 1, upd_grid = 0;
  double* s_part = nullptr;          // [upd_chunks][Dp] partial s of each chunk
  unsigned* tile_cnt = nullptr;      // [D tiles] arrival tickets (last chunk sums s_part in order)
  int64_t N = 0, D = 0, Dp = 0;        // Dp: D padded to a multiple of VEC_TILE (zero padding)
  double beta = 0;
  cofem_options opt{};
  cudaStream_t stream = nullptr;
  int device = 0;
  int num_sms = 148;
  bool probe64 = false;                 // probe columns in fp64
  int Kcap = 0, m_cap = 0;              // workspace capacity (columns = Kcap + 1)

  // operator data
  float* phi = nullptr; int64_t ld = 0; // DENSE Phi on the device, row-major N x ld
  bool phi_owned = false;               // true: the library's copy of a host Phi; false: borrowed
  int rows = 0, cols = 0, conv = 0;     // DCT2
  uint8_t* mask_vvT = nullptr;          // DCT2: mask in v-order, transposed [cols][rows]
  uint32_t* maskL = nullptr;            // DCT2 1024 fast path: lane-packed mask (op_dct1k.cu)
  void* maskH = nullptr;                // its half-warp column pass: [line][16] uint64 mask (fft512h.cuh layout)
  void* twh = nullptr;                  //   and the W_512^{t k1} tables
  void* tab1k32 = nullptr; void* tab1k64 = nullptr;   // its twiddle tables (float / double)
  bool fast1k = false;                  // DCT2 1024 x 1024: fast path, mean column on `side`
  void* flow_state = nullptr;           // k1k_flow (dataflow probe kernel): dispenser / counters
  void* flow_part2 = nullptr;           //   and its rho' partials [m_cap][D tiles]
  cudaStream_t side = nullptr;          // second stream (mean column of the fast DCT path)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // fast DCT path: probe-column groups 1..3 on their own streams with their own s accumulators
  static constexpr int MAXG = 8;
  int probe_groups = 1;                 // groups of the E-step being enqueued (launch sizing)
  cudaStream_t gstream[MAXG] = {};
  cudaEvent_t gjoin[MAXG] = {};
  double* gs[MAXG] = {};
  cudaStream_t work = nullptr;          // capturable stream the E-step graph runs on
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  void* dparams = nullptr;              // device ProbeParams of the current E-step
  int* bad_flag = nullptr;              // validate_alpha: device flag
  int* bad_host = nullptr;              //   and its pinned host mirror
  void* sup_stats = nullptr; void* sup_host = nullptr;   // support certificate (device / pinned host)
  int64_t sup_count = 0, sup_adjacent = 0;
  double sup_max = 0, sup_min_margin = 0;
  // captured E-steps (cofem.cu estep_device), a small LRU cache keyed by the launch shape (the
  // multi-task EM alternates mean-only and full E-steps)
  struct GraphSlot { cudaGraphExec_t exec = nullptr; int K = -1, Kt = -1, skip = -1, warm = -1; int64_t launches = 0, colls = 0; uint64_t used = 0; };
  static constexpr int NGRAPH = 4;
  GraphSlot gslot[NGRAPH];
  uint64_t gclock = 0;
  bool warm_now = false;                // this E-step starts the mean column from x0 (R20)
  bool skip_mean = false;          // cofem_estep_probes: column 0 frozen from the start (mean owned elsewhere)
  // multi-task EM (cofem_em_multi, reading R22): beta Phi^T y_l and mu_l of every task
  double* mt_b0 = nullptr; double* mt_mu = nullptr; double* b0_saved = nullptr; int mt_cap = 0;
  int64_t* obs_dev = nullptr;           // DCT2: mask indices kept on the device (b0 of other y)
  double conv_sumsq = 0;                // CIRCCONV: sum h^2 (b0 of other y)
  void* dct_tab32 = nullptr;            // DCT2 twiddle tables (float), see op_dct.cu
  void* dct_tab64 = nullptr;            // (double)
  int ntaps = 0;                        // CIRCCONV
  float* taps = nullptr;                // fp32 h (device)
  double* g64 = nullptr;                // Gram stencil g_l, l = -(T-1)..(T-1), fp64
  float* g32 = nullptr;                 // same, fp32

  double* b0 = nullptr;                 // beta Phi^T y (fp64, Dp)
  double* colsq = nullptr;              // diag(Phi^T Phi) (fp64, Dp)

  // E-step state
  double* alpha = nullptr;              // fp64 Dp
  double* dinv64 = nullptr;             // 1 / diag(A) fp64
  void* dinvp = nullptr;                // same in probe precision
  void* alphap = nullptr;               // alpha in probe precision (probe-column applies)
  void* Pb = nullptr; double* p0b = nullptr;   // CIRCCONV FFT path: ping-pong p buffers (overlapping windows)
  void* conv_tab32 = nullptr; void* conv_tab64 = nullptr;   // its FFT / spectrum tables
  bool fast_conv = false;               // CIRCCONV: overlap-save FFT apply (op_conv_fft.cu)
  double *x0 = nullptr, *r0 = nullptr, *p0 = nullptr, *q0 = nullptr;  // mean column (fp64)
  void *R = nullptr, *P = nullptr, *Q = nullptr;                       // probe block [Kcap][Dp]
  double* s = nullptr;                  // accumulated (1/K) sum p_k o x_k  (fp64 Dp)
  double* mu_out = nullptr;             // staging for outputs
  double* s_out = nullptr;
  double* alpha_out = nullptr;
  uint32_t* bits = nullptr;             // probe signs [Kcap][Dp/32]
  ColState* cs = nullptr;               // [m_cap]
  double* part = nullptr;               // per-CTA partial sums [m_cap][part_stride]
  int part_stride = 0;
  unsigned* counters = nullptr;         // last-block counters [m_cap + 1]
  int vec_grid = 0;                     // CTAs of the fused vector kernels

  // operator scratch
  void* ws1 = nullptr; void* ws2 = nullptr;   // probe-precision scratch (dense W partials / DCT T1,T2)
  double* ws1d = nullptr; double* ws2d = nullptr;   // mean-column scratch
  int dense_splits = 1;
  void* dense_tc = nullptr;             // tensor-core dense path state (op_dense_tc.cu), NULL: SIMT
  bool dense_cluster = false;           // small dense: the CG loop in one thread-block cluster (op_dense_cluster.cu)
  // column-sharded dense mode (comm.cu): per-column sums go through colsum + an NCCL all-reduce
  bool sharded = false;
  bool pp = false;                      // probe-parallel mode (dist_mode 1): probes split over ranks
  double pp_mean_cost = 0;              // the mean system's cost in probe columns (owner split)
  int64_t d_offset = 0, D_global = 0;
  void* comm = nullptr;                 // ncclComm_t
  double* colsum = nullptr;             // [4 MAXM] per-column totals of this rank (gamma; single-reduction CG:
                                        // + rho at [m, 2m), delta1 at [2m, 3m), delta2 at [3m, 4m))
  bool sr = false;                      // single-reduction CG (cg_variant 2, reading R23)
  bool p_presplit = false;              // k_dir wrote the tf32 halves of P: the next tensor-core apply skips k_tc_split_p
  double* sr_part = nullptr;            // k_sr_dots CTA partials [3 MAXM][part_stride]
  unsigned* sr_cnt = nullptr;           // k_sr_dots last-CTA tickets [MAXM]
  int rank = 0, world = 1;
  // D-sharded convolution (op_conv_fft.cu): per column [side][r | p | dinv][64] halo records
  void* halo_send = nullptr; void* halo_recv = nullptr;        // probe precision, [K][2][3][64]
  double* halo_send0 = nullptr; double* halo_recv0 = nullptr;  // mean column (fp64), [2][3][64]

  // host mirrors for the report
  std::vector<ColState> cs_host;
  std::vector<int32_t> frozen_host;
  std::vector<double> rho_host, rho0_host;
  int last_cols = 0;
  int bad_col = -1, bad_iter = -1;
  double estep_ms = 0;
  int64_t launches = 0;
  int64_t collectives = 0;              // NCCL launches (report; a group counts once)
  int comm_depth = 0;                   // open comm_group nesting
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;

  // profiling
  uint32_t prof_mask = 0;
  struct Rec { int cls; cudaEvent_t a, b; cudaStream_t st; };
  std::vector<Rec> prof_recs;
  std::vector<cudaEvent_t> ev_pool;
  double prof_ms[KC_COUNT] = {0};
  int64_t prof_cnt[KC_COUNT] = {0};
  double prof_busy[KC_COUNT] = {0};    // union of the class's launch intervals (concurrent launches once)

  std::string err;
};

// launch bookkeeping: call around every kernel launch
void launch_begin(Ctx* c, int cls, cudaStream_t st = nullptr);   // st = nullptr: the context stream
void launch_end(Ctx* c, int cls, cudaStream_t st = nullptr);
cudaError_t check_launch(Ctx* c, const char* what);

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Philox4x32-10 (Salmon et al. SC'11), product-side implementation.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u; k.y += 0xBB67AE85u;
  }
  return c;
}

// Finish a per-column reduction of `n` CTA partials in fixed order (deterministic).
// Called by one full warp.
__device__ __forceinline__ double reduce_partials(const double* __restrict__ p, int n) {
  double v = 0.0;
  for (int i = threadIdx.x & 31; i < n; i += 32) v += __ldcg(p + i);   // L2: written by other CTAs
  return warp_sum(v);
}

// Freeze rule + step length after gamma_j is known (R5): executed by one thread.
__device__ __forceinline__ void finish_gamma(ColState& c, double gamma, int iter) {
  if (c.frozen) return;
  c.gamma = gamma;
  bool finite = isfinite(gamma) && isfinite(c.rho);
  bool ok = finite && (gamma > 0.0) && (c.rho > c.tau * c.rho0);
  if (!ok) {
    c.frozen = 1; c.frozen_at = iter; c.nonfinite = finite ? 0 : 1; c.a = 0.0;
  } else {
    c.a = c.rho / gamma;
  }
}

// Per-column reduction of one CTA value v (already CTA-reduced, valid in thread 0):
// part[j][bx] = v; the last CTA of column j (grid.x CTAs) reduces in fixed order and
// calls fin(sum) from one thread.  Requires blockDim.x >= 32 and all threads present.
template <typename Fin>
__device__ __forceinline__ void column_finish(double v, int j, double* part, int stride, unsigned* counters,
                                              Fin fin) {
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    part[(int64_t)j * stride + blockIdx.x] = v;
    __threadfence();
    s_last = (atomicAdd(counters + j, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x < 32) {
    double tot = reduce_partials(part + (int64_t)j * stride, gridDim.x);
    if (threadIdx.x == 0) { fin(tot); counters[j] = 0u; }
  }
}

// As column_finish, for persistent kernels: CTA work item `slot` of `count` per column.
template <typename Fin>
__device__ __forceinline__ void column_finish_n(double v, int j, int slot, int count, double* part, int stride,
                                                unsigned* counters, Fin fin) {
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
    part[(int64_t)j * stride + slot] = v;
    __threadfence();
    s_last = (atomicAdd(counters + j, 1u) == (unsigned)count - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x < 32) {
    double tot = reduce_partials(part + (int64_t)j * stride, count);
    if (threadIdx.x == 0) { fin(tot); counters[j] = 0u; }
  }
}

// CTA-wide sum of one double per thread (result valid in thread 0). blockDim.x <= 1024.
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double s_w[32];
  v = warp_sum(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (lane == 0) s_w[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = lane < nw ? s_w[lane] : 0.0;
    r = warp_sum(r);
  }
  return r;
}

// ---------------------------------------------------------------- operator launchers
// every apply computes Q = A P for all active columns and finishes gamma_j / a_j.
cofem_status dense_setup(Ctx* c, const float* y_dev);
cofem_status dense_apply(Ctx* c, int m, int iter);
bool dense_cluster_eligible(const Ctx* c);
cofem_status dense_cluster_setup(Ctx* c);
cofem_status dense_cluster_cg(Ctx* c, int K, double invK);
void dense_tc_p_split(Ctx* c, float** ph, float** pl);   // the tensor-core path's P_hi / P_lo (or null)
cofem_status dense_tc_setup(Ctx* c);
cofem_status dense_tc_apply(Ctx* c, int m, int iter);
void dense_tc_free(Ctx* c);
cofem_status dct_setup(Ctx* c, const float* y_dev, const int64_t* obs_dev);
cofem_status dct_apply(Ctx* c, int m, int iter, bool dir);   // direction update fused into pass A
cofem_status conv_setup(Ctx* c, const float* y_dev, const float* taps_host);
cofem_status conv_apply(Ctx* c, int m, int iter);
cofem_status dense_b0(Ctx* c, const float* y_dev, double* out);   // beta Phi^T y of another y (R22)
cofem_status dct_b0(Ctx* c, const float* y_dev, double* out);
cofem_status conv_b0(Ctx* c, const float* y_dev, double* out);

bool dct1k_eligible(const Ctx* c);
cofem_status dct1k_setup(Ctx* c);
cofem_status dct1k_apply(Ctx* c, int j0, int j1, int iter, bool dir, cudaStream_t st);
cofem_status dct1k_flow(Ctx* c, int K, int K_total, cudaStream_t st);   // all U iterations of the fp32 probes
int dct1k_flow_groups(const Ctx* c, int K);                             // its column groups
bool conv_fft_eligible(const Ctx* c);
cofem_status conv_fft_setup(Ctx* c, const std::vector<double>& g);
cofem_status conv_fft_apply(Ctx* c, int j0, int j1, int iter, bool dir, cudaStream_t st);
cofem_status conv_halo_exchange(Ctx* c, int K);

cofem_status comm_init(Ctx* c, int rank, int world, const uint8_t* id);
void comm_destroy(Ctx* c);
cofem_status comm_allreduce(Ctx* c, void* buf, size_t count, int dtype);
// NCCL group around several collectives (one fused launch): comm_group(c, true) ... comm_group(c, false)
cofem_status comm_group(Ctx* c, bool begin);
// single-reduction CG (R23): rho_j = r_j^T M^-1 r_j, delta1_j = q_j^T M^-1 r_j, delta2_j = q_j^T M^-1 q_j
// of this rank's rows into colsum[m + j], colsum[2m + j], colsum[3m + j]
cofem_status sr_dots(Ctx* c, int m);
cofem_status comm_bcast(Ctx* c, void* buf, size_t count, int dtype, int root);
cofem_status comm_halo(Ctx* c, const void* send_left, const void* send_right, void* recv_left, void* recv_right,
                       size_t count, int dtype);
// after a per-column reduction written to c->colsum: sum over ranks, then apply it (mode:
// 0 = rho0 (init), 1 = gamma -> freeze rule / step length, 2 = rho' -> b)
cofem_status sharded_finish(Ctx* c, int m, int mode, int iter);

// cudaFuncAttributeMaxDynamicSharedMemorySize belongs to the function, not to a context: only ever
// raise it, so that a context set up later with a smaller need (max_probes, N, D) does not break the
// launches of an earlier one
inline cudaError_t raise_smem_attr(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> cur;
  std::lock_guard<std::mutex> lock(mu);
  size_t& c = cur[fn];
  if (bytes <= c) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) c = bytes;
  return e;
}

// vector kernels (cofem.cu)
cofem_status launch_dir(Ctx* c, int m);

}  // namespace cofem
