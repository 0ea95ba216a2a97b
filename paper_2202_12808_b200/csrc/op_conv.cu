// op_conv.cu — circular-convolution dictionary (BASELINE config 5; reading R12):
//   (Phi x)_i = sum_{j<T} h_j x_{(i-j) mod D},   N = D.
// Phi^T Phi is circulant with the symmetric (2T-1)-tap stencil g_l = sum_k h_k h_{k+l}
// (autocorrelation of h), so the Gram apply is one stencil pass per column:
//   q_i = beta sum_{|l|<T} g_l p_{(i+l) mod D} + alpha_i p_i        (Eq. 7 with A = beta Phi^T Phi + diag alpha)
// Mathematically identical to applying Phi then Phi^T (half the FMAs, one HBM pass).
// v1: direct stencil from a shared-memory tile with a (T-1) halo on each side.
#include <algorithm>
#include <vector>

#include "internal.cuh"

namespace cofem {

constexpr int CONV_THREADS = 256;
constexpr int CONV_PER_THREAD = 8;
constexpr int CONV_TILE = CONV_THREADS * CONV_PER_THREAD;
constexpr int CONV_MAXH = 63;

// b0_i = beta (Phi^T y)_i = beta sum_j h_j y_{(i+j) mod D}  (Eq. 5), colsq_i = sum_j h_j^2
__global__ void k_conv_setup(const float* __restrict__ h, int T, const float* __restrict__ y, int64_t D, int64_t Dwrap,
                             double beta, double sumsq, double* __restrict__ b0, double* __restrict__ colsq) {
  // Dwrap: period of y's indexing (D; D-sharded: D + 64, y extended by the right halo)
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < D; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < T; ++j) {
      int64_t idx = i + j;
      if (idx >= Dwrap) idx -= Dwrap;
      acc += (double)h[j] * (double)y[idx];
    }
    b0[i] = beta * acc;
    colsq[i] = sumsq;
  }
}

template <typename T>
__device__ double conv_body(int64_t D, int H, const T* __restrict__ g, const T* __restrict__ p,
                            T* __restrict__ q, const double* __restrict__ alpha, double beta, T* sm) {
  T* gs = sm;                    // [2H+1]
  T* xs = sm + 2 * CONV_MAXH + 2; // [TILE + 2H]
  const int64_t t0 = (int64_t)blockIdx.x * CONV_TILE;
  for (int l = threadIdx.x; l < 2 * H + 1; l += CONV_THREADS) gs[l] = g[l];
  for (int e = threadIdx.x; e < CONV_TILE + 2 * H; e += CONV_THREADS) {
    int64_t idx = t0 - H + e;
    idx %= D;
    if (idx < 0) idx += D;
    xs[e] = p[idx];
  }
  __syncthreads();
  T acc[CONV_PER_THREAD];
#pragma unroll
  for (int e = 0; e < CONV_PER_THREAD; ++e) acc[e] = (T)0;
  for (int l = 0; l <= 2 * H; ++l) {
    const T gl = gs[l];
#pragma unroll
    for (int e = 0; e < CONV_PER_THREAD; ++e) acc[e] += gl * xs[threadIdx.x + CONV_THREADS * e + l];
  }
  double g2 = 0.0;
  const T bt = (T)beta;
#pragma unroll
  for (int e = 0; e < CONV_PER_THREAD; ++e) {
    const int64_t i = t0 + threadIdx.x + CONV_THREADS * e;
    if (i < D) {
      const T pi = xs[threadIdx.x + CONV_THREADS * e + H];
      const T qi = bt * acc[e] + (T)alpha[i] * pi;
      q[i] = qi;
      g2 += (double)pi * (double)qi;
    }
  }
  return g2;
}

template <typename TP>
__global__ void __launch_bounds__(CONV_THREADS) k_conv_apply(int64_t D, int64_t Dp, int H, const double* __restrict__ g64,
                                                             const TP* __restrict__ gp, const double* __restrict__ p0,
                                                             double* __restrict__ q0, const TP* __restrict__ P,
                                                             TP* __restrict__ Q, const double* __restrict__ alpha,
                                                             double beta, ColState* cs, double* part, int stride,
                                                             unsigned* counters, int iter) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int j = blockIdx.y;
  if (cs[j].frozen) return;
  double g = j == 0 ? conv_body<double>(D, H, g64, p0, q0, alpha, beta, reinterpret_cast<double*>(smem_raw))
                    : conv_body<TP>(D, H, gp, P + (int64_t)(j - 1) * Dp, Q + (int64_t)(j - 1) * Dp, alpha, beta,
                                    reinterpret_cast<TP*>(smem_raw));
  g = block_sum(g);
  column_finish(g, j, part, stride, counters, [cs, j, iter](double tot) {
    ColState c = cs[j]; finish_gamma(c, tot, iter); cs[j] = c;
  });
}

static size_t conv_smem() { return (size_t)(2 * CONV_MAXH + 2 + CONV_TILE + 2 * CONV_MAXH) * sizeof(double); }

// b0 = beta Phi^T y for another observation vector (multi-task EM, R22; unsharded)
cofem_status conv_b0(Ctx* c, const float* y_dev, double* out) {
  launch_begin(c, KC_SETUP);
  k_conv_setup<<<c->num_sms * 8, 256, 0, c->stream>>>(c->taps, c->ntaps, y_dev, c->D, c->D, c->beta, c->conv_sumsq, out,
                                                      c->colsq);
  launch_end(c, KC_SETUP);
  return check_launch(c, "conv_b0") == cudaSuccess ? COFEM_OK : COFEM_ERR_CUDA;
}

cofem_status conv_setup(Ctx* c, const float* y_dev, const float* taps_host) {
  const int T = c->ntaps, H = T - 1;
  std::vector<double> g(2 * H + 1);
  double sumsq = 0.0;
  for (int k = 0; k < T; ++k) sumsq += (double)taps_host[k] * (double)taps_host[k];
  for (int l = 0; l <= H; ++l) {
    double v = 0.0;
    for (int k = 0; k + l < T; ++k) v += (double)taps_host[k] * (double)taps_host[k + l];
    g[H + l] = v; g[H - l] = v;
  }
  std::vector<float> g32(g.begin(), g.end());
  if (cudaMalloc(&c->g64, g.size() * 8) != cudaSuccess || cudaMalloc(&c->g32, g.size() * 4) != cudaSuccess ||
      cudaMalloc(&c->taps, T * 4) != cudaSuccess) { c->err = "cudaMalloc conv"; return COFEM_ERR_OOM; }
  cudaMemcpy(c->g64, g.data(), g.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(c->g32, g32.data(), g.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(c->taps, taps_host, T * 4, cudaMemcpyHostToDevice);
  if (c->probe64) {   // parity mode: fp64 stencil for the probe columns too
    double* gp; cudaMalloc(&gp, g.size() * 8); cudaMemcpy(gp, g.data(), g.size() * 8, cudaMemcpyHostToDevice);
    cudaFree(c->g32); c->g32 = reinterpret_cast<float*>(gp);
  }
  c->conv_sumsq = sumsq;
  const float* y_use = y_dev;
  float* y_ext = nullptr;
  int64_t Dwrap = c->D;
  if (c->sharded) {   // D-sharded: b0_i needs y up to i + 63 -> the right neighbour's first 64 samples
    if (c->D < 2048 || c->ntaps > 64) { c->err = "D-sharded convolution: local D >= 2048 and ntaps <= 64"; return COFEM_ERR_UNSUPPORTED; }
    float* sbuf;
    if (cudaMalloc(&y_ext, (c->D + 64) * sizeof(float)) != cudaSuccess || cudaMalloc(&sbuf, 128 * sizeof(float)) != cudaSuccess) {
      c->err = "cudaMalloc y halo"; return COFEM_ERR_OOM;
    }
    cudaMemcpyAsync(y_ext, y_dev, c->D * sizeof(float), cudaMemcpyDeviceToDevice, c->stream);
    cudaMemcpyAsync(sbuf, y_dev, 64 * sizeof(float), cudaMemcpyDeviceToDevice, c->stream);
    cudaMemcpyAsync(sbuf + 64, y_dev + c->D - 64, 64 * sizeof(float), cudaMemcpyDeviceToDevice, c->stream);
    float* left_unused;
    cudaMalloc(&left_unused, 64 * sizeof(float));
    cofem_status hs = comm_halo(c, sbuf, sbuf + 64, left_unused, y_ext + c->D, 64, 0);
    cudaStreamSynchronize(c->stream);
    cudaFree(sbuf); cudaFree(left_unused);
    if (hs != COFEM_OK) { cudaFree(y_ext); return hs; }
    y_use = y_ext; Dwrap = c->D + 64;
  }
  launch_begin(c, KC_SETUP);
  k_conv_setup<<<c->num_sms * 8, 256, 0, c->stream>>>(c->taps, T, y_use, c->D, Dwrap, c->beta, sumsq, c->b0, c->colsq);
  launch_end(c, KC_SETUP);
  if (y_ext) { cudaStreamSynchronize(c->stream); cudaFree(y_ext); }
  if (check_launch(c, "k_conv_setup")) return COFEM_ERR_CUDA;
  const int grid = (int)((c->D + CONV_TILE - 1) / CONV_TILE);
  c->part_stride = std::max(c->part_stride, grid);
  if (conv_fft_eligible(c)) {        // overlap-save FFT apply, mean column on the side stream
    const size_t tp = c->probe64 ? 8 : 4;
    if (cudaMalloc(&c->Pb, (size_t)c->Kcap * c->Dp * tp) != cudaSuccess || cudaMalloc(&c->p0b, c->Dp * 8) != cudaSuccess) {
      c->err = "cudaMalloc conv p buffers"; return COFEM_ERR_OOM;
    }
    cudaMemset(c->Pb, 0, (size_t)c->Kcap * c->Dp * tp); cudaMemset(c->p0b, 0, c->Dp * 8);
    cofem_status st = conv_fft_setup(c, g);
    if (st != COFEM_OK) return st;
    c->fast_conv = true;
  }
  if (c->probe64) cudaFuncSetAttribute(k_conv_apply<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)conv_smem());
  else cudaFuncSetAttribute(k_conv_apply<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)conv_smem());
  return COFEM_OK;
}

cofem_status conv_apply(Ctx* c, int m, int iter) {
  const int H = c->ntaps - 1;
  dim3 grid((unsigned)((c->D + CONV_TILE - 1) / CONV_TILE), m);
  launch_begin(c, KC_CONV_APPLY);
  if (c->probe64)
    k_conv_apply<double><<<grid, CONV_THREADS, conv_smem(), c->stream>>>(
        c->D, c->Dp, H, c->g64, reinterpret_cast<const double*>(c->g32), c->p0, c->q0, (const double*)c->P,
        (double*)c->Q, c->alpha, c->beta, c->cs, c->part, c->part_stride, c->counters, iter);
  else
    k_conv_apply<float><<<grid, CONV_THREADS, conv_smem(), c->stream>>>(
        c->D, c->Dp, H, c->g64, c->g32, c->p0, c->q0, (const float*)c->P, (float*)c->Q, c->alpha, c->beta, c->cs,
        c->part, c->part_stride, c->counters, iter);
  launch_end(c, KC_CONV_APPLY);
  return check_launch(c, "k_conv_apply") == cudaSuccess ? COFEM_OK : COFEM_ERR_CUDA;
}

}  // namespace cofem
