// op_dense.cu — dense dictionary Phi (N x D, fp32 row-major): setup and the batched
// Gram apply  Q = beta Phi^T (Phi P) + alpha o P  (Eq. 7; reading R1).
//
// v1 path: FP32 SIMT with shared-memory staging for the probe columns and
// fp64 accumulation (fp32 Phi promoted exactly) for the mean column 0
// (fp32 rounding of the mean system lands in null(Phi) where A's
// eigenvalue is alpha, so mu needs fp64).
//   K1 k_dense_phiP   : W = Phi P            split over d (deterministic 2-stage)
//   K2 k_dense_phiTW  : Q = beta Phi^T W + alpha o P, gamma_j = p_j^T q_j (+ freeze / a_j)
#include <algorithm>

#include "internal.cuh"

namespace cofem {

constexpr int DK1_ROWS = 32;      // n rows per CTA (K1)
constexpr int DK1_BK = 32;        // d chunk per smem stage (K1)
constexpr int DK2_COLS = 64;      // d outputs per CTA (K2)
constexpr int DK2_BN = 16;        // n chunk per smem stage (K2)
constexpr int DMAXK = 128;

// ---------------------------------------------------------------- setup: b0, colsq
__global__ void k_dense_setup(const float* __restrict__ phi, int64_t N, int64_t D, int64_t ld,
                              const float* __restrict__ y, double beta, double* __restrict__ b0,
                              double* __restrict__ colsq) {
  for (int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; d < D; d += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0, sq = 0.0;
    for (int64_t n = 0; n < N; ++n) {
      double v = (double)phi[n * ld + d];
      acc += v * (double)y[n];
      sq += v * v;
    }
    b0[d] = beta * acc;     // Eq. 5: b0 = beta Phi^T y
    colsq[d] = sq;          // diag(Phi^T Phi)
  }
}

// ---------------------------------------------------------------- K1: W = Phi P
template <typename TP>
__global__ void __launch_bounds__(256) k_dense_phiP(const float* __restrict__ phi, int64_t N, int64_t D, int64_t ld,
                                                    const double* __restrict__ p0, const TP* __restrict__ P,
                                                    int64_t Dp, int K, int64_t chunk,
                                                    TP* __restrict__ Wpart, double* __restrict__ W0part) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* phs = reinterpret_cast<float*>(smem_raw);                    // [32][33]
  double* p0s = reinterpret_cast<double*>(phs + DK1_ROWS * 33 + 1);   // [32] (8B aligned below)
  p0s = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(p0s) + 15) & ~uintptr_t(15));
  TP* ps = reinterpret_cast<TP*>(p0s + DK1_BK);                        // [K][33]
  const int tid = threadIdx.x;
  const int nl = tid >> 3, jg = tid & 7;
  const int64_t n0 = (int64_t)blockIdx.x * DK1_ROWS;
  const int split = blockIdx.y;
  const int64_t dbeg = split * chunk, dend = D < dbeg + chunk ? D : dbeg + chunk;
  constexpr int NACC = DMAXK / 8;
  TP acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = (TP)0;
  double acc0 = 0.0;
  for (int64_t d0 = dbeg; d0 < dend; d0 += DK1_BK) {
    {   // Phi tile 32 x 32
      const int r = tid >> 3, c4 = (tid & 7) * 4;
      const int64_t n = n0 + r;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t d = d0 + c4 + e;
        phs[r * 33 + c4 + e] = (n < N && d < dend) ? phi[n * ld + d] : 0.0f;
      }
    }
    for (int i = tid; i < K * DK1_BK; i += 256) {
      const int k = i / DK1_BK, c = i % DK1_BK;
      const int64_t d = d0 + c;
      ps[k * 33 + c] = d < dend ? P[(int64_t)k * Dp + d] : (TP)0;
    }
    if (tid < DK1_BK) p0s[tid] = (d0 + tid < dend) ? p0[d0 + tid] : 0.0;
    __syncthreads();
#pragma unroll 4
    for (int c = 0; c < DK1_BK; ++c) {
      const float a = phs[nl * 33 + c];
#pragma unroll
      for (int i = 0; i < NACC; ++i) {
        const int k = jg + 8 * i;
        if (k < K) acc[i] += (TP)a * ps[k * 33 + c];
      }
      if (jg == 0) acc0 += (double)a * p0s[c];
    }
    __syncthreads();
  }
  const int64_t n = n0 + nl;
  if (n < N) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      const int k = jg + 8 * i;
      if (k < K) Wpart[((int64_t)split * N + n) * K + k] = acc[i];
    }
    if (jg == 0) W0part[(int64_t)split * N + n] = acc0;
  }
}

// Sum the split-K partials in fixed order (deterministic) into partial slot 0.
template <typename TP>
__global__ void k_dense_reduce_w(int64_t N, int K, int splits, TP* __restrict__ Wpart, double* __restrict__ W0part) {
  const int64_t total = N * K;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total + N; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < total) {
      TP v = Wpart[i];
      for (int sp = 1; sp < splits; ++sp) v += Wpart[(int64_t)sp * total + i];
      Wpart[i] = v;
    } else {
      const int64_t n = i - total;
      double v = W0part[n];
      for (int sp = 1; sp < splits; ++sp) v += W0part[(int64_t)sp * N + n];
      W0part[n] = v;
    }
  }
}

// ---------------------------------------------------------------- K2: Q = beta Phi^T W + alpha o P
template <typename TP>
__global__ void __launch_bounds__(256) k_dense_phiTW(const float* __restrict__ phi, int64_t N, int64_t D, int64_t ld,
                                                     const TP* __restrict__ W, const double* __restrict__ W0,
                                                     int K, int64_t Dp, double beta, const double* __restrict__ alpha,
                                                     const double* __restrict__ p0, double* __restrict__ q0,
                                                     const TP* __restrict__ P, TP* __restrict__ Q,
                                                     ColState* cs, double* part, int stride, unsigned* counter,
                                                     int iter) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* phs = reinterpret_cast<float*>(smem_raw);                 // [16][64]
  double* w0s = reinterpret_cast<double*>(phs + DK2_BN * DK2_COLS); // [16]
  TP* ws = reinterpret_cast<TP*>(w0s + DK2_BN);                     // [16][K]
  __shared__ double red[8][MAXM];
  __shared__ bool s_last;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int dl = tid & 63, jg = tid >> 6;
  const int64_t d0 = (int64_t)blockIdx.x * DK2_COLS;
  constexpr int NACC = DMAXK / 4;
  TP acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = (TP)0;
  double acc0 = 0.0;
  for (int i = tid; i < 8 * MAXM; i += 256) (&red[0][0])[i] = 0.0;
  for (int64_t nb = 0; nb < N; nb += DK2_BN) {
    for (int i = tid; i < DK2_BN * DK2_COLS; i += 256) {
      const int r = i / DK2_COLS, c = i % DK2_COLS;
      const int64_t n = nb + r, d = d0 + c;
      phs[i] = (n < N && d < D) ? phi[n * ld + d] : 0.0f;
    }
    for (int i = tid; i < DK2_BN * K; i += 256) {
      const int r = i / K, k = i % K;
      const int64_t n = nb + r;
      ws[r * K + k] = n < N ? W[n * K + k] : (TP)0;
    }
    if (tid < DK2_BN) w0s[tid] = (nb + tid < N) ? W0[nb + tid] : 0.0;
    __syncthreads();
#pragma unroll 4
    for (int r = 0; r < DK2_BN; ++r) {
      const float a = phs[r * DK2_COLS + dl];
#pragma unroll
      for (int i = 0; i < NACC; ++i) {
        const int k = jg + 4 * i;
        if (k < K) acc[i] += (TP)a * ws[r * K + k];
      }
      if (jg == 0) acc0 += (double)a * w0s[r];
    }
    __syncthreads();
  }
  // epilogue: q = beta acc + alpha o p, gamma partials
  const int64_t d = d0 + dl;
  const bool valid = d < D;
  const double al = valid ? alpha[d] : 0.0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) {
    const int k = jg + 4 * i;
    if (k < K) {                         // warp-uniform (jg is per warp)
      double g = 0.0;
      if (valid) {
        const TP p = P[(int64_t)k * Dp + d];
        const TP q = (TP)beta * acc[i] + (TP)al * p;
        Q[(int64_t)k * Dp + d] = q;
        g = (double)p * (double)q;
      }
      g = warp_sum(g);
      if (lane == 0) red[warp][k + 1] = g;
    }
  }
  if (jg == 0) {
    double g = 0.0;
    if (valid) {
      const double p = p0[d];
      const double q = beta * acc0 + al * p;
      q0[d] = q;
      g = p * q;
    }
    g = warp_sum(g);
    if (lane == 0) red[warp][0] = g;
  }
  __syncthreads();
  const int m = K + 1;
  for (int j = tid; j < m; j += 256) {
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v += red[w][j];
    part[(int64_t)j * stride + blockIdx.x] = v;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int j = warp; j < m; j += 8) {
    const double v = reduce_partials(part + (int64_t)j * stride, gridDim.x);
    if (lane == 0) { ColState c = cs[j]; finish_gamma(c, v, iter); cs[j] = c; }
  }
  if (tid == 0) *counter = 0u;
}

// ---------------------------------------------------------------- host
static size_t k1_smem(int K, size_t tp) { return DK1_ROWS * 33 * 4 + 4 + 16 + DK1_BK * 8 + (size_t)K * 33 * tp + 16; }
static size_t k2_smem(int K, size_t tp) { return DK2_BN * DK2_COLS * 4 + DK2_BN * 8 + (size_t)DK2_BN * K * tp; }

cofem_status dense_setup(Ctx* c, const float* y_dev) {
  if (c->Kcap > DMAXK) { c->err = "DENSE: max_probes must be <= 128"; return COFEM_ERR_INVALID; }
  launch_begin(c, KC_SETUP);
  k_dense_setup<<<(unsigned)((c->D + 255) / 256), 256, 0, c->stream>>>(c->phi, c->N, c->D, c->ld, y_dev, c->beta, c->b0, c->colsq);
  launch_end(c, KC_SETUP);
  if (check_launch(c, "k_dense_setup")) return COFEM_ERR_CUDA;
  // split-K for W = Phi P: about 2 waves of CTAs, >= 256 d per split
  const int64_t ntile = (c->N + DK1_ROWS - 1) / DK1_ROWS;
  int splits = (int)std::max<int64_t>(1, (2 * c->num_sms + ntile - 1) / ntile);
  splits = (int)std::min<int64_t>(splits, std::max<int64_t>(1, c->D / 256));
  c->dense_splits = splits;
  const size_t tp = c->probe64 ? 8 : 4;
  if (cudaMalloc(&c->ws1, (size_t)splits * c->N * c->Kcap * tp) != cudaSuccess ||
      cudaMalloc(&c->ws1d, (size_t)splits * c->N * sizeof(double)) != cudaSuccess) {
    c->err = "cudaMalloc dense workspace"; return COFEM_ERR_OOM;
  }
  const int k2grid = (int)((c->D + DK2_COLS - 1) / DK2_COLS);
  c->part_stride = std::max(c->part_stride, k2grid);
  size_t s1 = k1_smem(c->Kcap, tp), s2 = k2_smem(c->Kcap, tp);
  if (c->probe64) {
    raise_smem_attr((const void*)k_dense_phiP<double>, s1);
    raise_smem_attr((const void*)k_dense_phiTW<double>, s2);
  } else {
    raise_smem_attr((const void*)k_dense_phiP<float>, s1);
    raise_smem_attr((const void*)k_dense_phiTW<float>, s2);
  }
  cofem_status st = dense_tc_setup(c);
  if (st == COFEM_OK && dense_cluster_eligible(c)) st = dense_cluster_setup(c);
  return st;
}

template <typename TP>
static cofem_status dense_apply_t(Ctx* c, int m, int iter) {
  const int K = m - 1;
  const size_t tp = sizeof(TP);
  const int64_t ntile = (c->N + DK1_ROWS - 1) / DK1_ROWS;
  const int splits = c->dense_splits;
  int64_t chunk = (c->D + splits - 1) / splits;
  chunk = (chunk + DK1_BK - 1) / DK1_BK * DK1_BK;
  TP* W = (TP*)c->ws1;
  launch_begin(c, KC_DENSE_PHI_P);
  k_dense_phiP<TP><<<dim3((unsigned)ntile, splits), 256, k1_smem(K, tp), c->stream>>>(
      c->phi, c->N, c->D, c->ld, c->p0, (const TP*)c->P, c->Dp, K, chunk, W, c->ws1d);
  launch_end(c, KC_DENSE_PHI_P);
  if (check_launch(c, "k_dense_phiP")) return COFEM_ERR_CUDA;
  if (splits > 1) {
    launch_begin(c, KC_DENSE_PHI_P);
    k_dense_reduce_w<TP><<<c->num_sms * 2, 256, 0, c->stream>>>(c->N, K, splits, W, c->ws1d);
    launch_end(c, KC_DENSE_PHI_P);
    if (check_launch(c, "k_dense_reduce_w")) return COFEM_ERR_CUDA;
  }
  const int k2grid = (int)((c->D + DK2_COLS - 1) / DK2_COLS);
  launch_begin(c, KC_DENSE_PHIT_W);
  k_dense_phiTW<TP><<<k2grid, 256, k2_smem(K, tp), c->stream>>>(
      c->phi, c->N, c->D, c->ld, W, c->ws1d, K, c->Dp, c->beta, c->alpha, c->p0, c->q0,
      (const TP*)c->P, (TP*)c->Q, c->cs, c->part, c->part_stride, c->counters + MAXM, iter);
  launch_end(c, KC_DENSE_PHIT_W);
  if (check_launch(c, "k_dense_phiTW")) return COFEM_ERR_CUDA;
  return COFEM_OK;
}

// b0 = beta Phi^T y for another observation vector (multi-task EM, R22); colsq is recomputed as is
cofem_status dense_b0(Ctx* c, const float* y_dev, double* out) {
  launch_begin(c, KC_SETUP);
  k_dense_setup<<<(unsigned)((c->D + 255) / 256), 256, 0, c->stream>>>(c->phi, c->N, c->D, c->ld, y_dev, c->beta, out, c->colsq);
  launch_end(c, KC_SETUP);
  return check_launch(c, "dense_b0") == cudaSuccess ? COFEM_OK : COFEM_ERR_CUDA;
}

cofem_status dense_apply(Ctx* c, int m, int iter) {
  if (c->dense_tc) return dense_tc_apply(c, m, iter);     // tcgen05 3xTF32 path (op_dense_tc.cu)
  return c->probe64 ? dense_apply_t<double>(c, m, iter) : dense_apply_t<float>(c, m, iter);
}

}  // namespace cofem
