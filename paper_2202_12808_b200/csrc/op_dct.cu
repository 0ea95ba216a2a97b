// op_dct.cu — masked orthonormal 2D DCT dictionary (§4.2; reading R11):
//   Phi = S C2^T  (2D inverse DCT, then keep the N masked pixels),
//   Phi^T Phi P = C2 (M o (C2^T P)),  so  Q = beta C2 (M o C2^T P) + alpha o P.
//
// The apply is three HBM passes over the (K+1) coefficient images (rows x cols,
// row-major), each a batch of length-L DCTs computed as an L/2-point complex
// FFT (Makhoul's even/odd packing) in shared memory:
//   pass A  k_dct_rows_inv : [fused CG direction p = M^-1 r + b p]; DCT-III along each row
//   pass B  k_dct_cols     : per column strip: DCT-III along the column, mask, DCT-II
//   pass C  k_dct_rows_fwd : DCT-II along each row; q = beta X + alpha o p; gamma = p^T q
// Intermediates T1/T2 keep pixel columns (and pass B keeps pixel rows internally)
// in "v-order", m -> 2m (m < L/2), 2(L-1-m)+1 (m >= L/2): the DCT's even/odd
// shuffle then cancels between the inverse and the forward transform, so no pass
// ever permutes data.  Column 0 (mean system) runs the same code in
// fp64 (CTA-uniform branch); probe columns run in fp32 (or fp64 in parity mode).
#include <math.h>

#include <algorithm>
#include <vector>

#include "fft_common.cuh"

namespace cofem {

// ---------------------------------------------------------------- Stockham FFT (team of M/8 threads)
// pass with stride NS (> 1): radix R = min(8, M/NS); each thread does 8/R butterflies.
template <typename T, int M, int SIGN, int NS>
struct FftPass {
  static __device__ __forceinline__ void run(cplx<T>* buf, cplx<T> (&v)[8], int t, const cplx<T>* __restrict__ tw) {
    constexpr int R = (M / NS) >= 8 ? 8 : (M / NS);
    constexpr int BPT = 8 / R;
    constexpr int NB = M / R;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < BPT; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r) v[u * R + r] = buf[(t * BPT + u) + r * NB];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < BPT; ++u) {
      const int b = t * BPT + u;
      const int bm = b & (NS - 1);
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const cplx<T> w = tw[r * bm * (M / (NS * R))];
        v[u * R + r] = SIGN < 0 ? cmul(v[u * R + r], w) : cmulc(v[u * R + r], w);
      }
      dftR<R, SIGN>(&v[u * R]);
      const int idxD = (b / NS) * NS * R + bm;
#pragma unroll
      for (int r = 0; r < R; ++r) buf[idxD + r * NS] = v[u * R + r];
    }
    FftPass<T, M, SIGN, NS * R>::run(buf, v, t, tw);
  }
};
template <typename T, int M, int SIGN>
struct FftPass<T, M, SIGN, M> {
  static __device__ __forceinline__ void run(cplx<T>*, cplx<T> (&)[8], int, const cplx<T>*) {}
};

// Length-M DFT (SIGN -1) / unnormalised inverse DFT (SIGN +1).  On entry v[r] = w[t + r*M/8]
// (thread t of the team); buf may still be being read by the caller's gather.  On exit the
// natural-order result is in buf (after a CTA barrier).  All CTA threads must call it.
template <typename T, int M, int SIGN>
__device__ __forceinline__ void fft_team(cplx<T>* buf, cplx<T> (&v)[8], int t, const cplx<T>* __restrict__ tw) {
  dft8<SIGN>(v);
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 8; ++r) buf[t * 8 + r] = v[r];
  FftPass<T, M, SIGN, 8>::run(buf, v, t, tw);
  __syncthreads();
}

// DCT-III (inverse of the orthonormal DCT-II) pre-processing: from the natural-order
// coefficient vector X (stride xs) build the packed spectrum W[k] = Ve + i Vo for
// k = t + r*M/8, with the 1/M IFFT normalisation and 1/s_k folded in.
template <typename T, int L>
__device__ __forceinline__ void dct3_gather(const T* X, int xs, int t, cplx<T> (&v)[8], DctTab<T> tb) {
  constexpr int M = L / 2, NT = M / 8;
  const T sc0 = (T)(sqrt((double)L) / M), sc = (T)(sqrt((double)L / 2.0) / M);
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int k = t + r * NT;
    const T xk = X[k * xs] * (k == 0 ? sc0 : sc);
    const T xLk = k == 0 ? (T)0 : X[(L - k) * xs] * sc;
    const T xkM = X[(k + M) * xs] * sc;
    const T xMk = X[(M - k) * xs] * (M - k == 0 ? sc0 : sc);
    // V(kk) = exp(i pi kk / 2L) (Xu[kk] - i Xu[L-kk])
    const cplx<T> V1 = cmulc(cplx<T>{xk, -xLk}, tb.tq[k]);
    const cplx<T> V2 = cmulc(cplx<T>{xkM, -xMk}, tb.tq[k + M]);
    const cplx<T> Ve = {(V1.x + V2.x) * (T)0.5, (V1.y + V2.y) * (T)0.5};
    const cplx<T> Vo = cmulc(cplx<T>{(V1.x - V2.x) * (T)0.5, (V1.y - V2.y) * (T)0.5}, tb.th[k]);
    v[r] = {Ve.x - Vo.y, Ve.y + Vo.x};      // Ve + i Vo
  }
}

// DCT-II post-processing from the natural-order FFT output W (in smem) to orthonormal
// coefficients X[k], X[k+M] for k = t + r*M/8.
template <typename T, int L>
__device__ __forceinline__ void dct2_post(const cplx<T>* W, int t, T (&lo)[8], T (&hi)[8], DctTab<T> tb) {
  constexpr int M = L / 2, NT = M / 8;
  const T s0 = (T)sqrt(1.0 / L), s = (T)sqrt(2.0 / L);
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int k = t + r * NT;
    const cplx<T> Wk = W[k], Wm = W[(M - k) & (M - 1)];
    const cplx<T> Ve = {(Wk.x + Wm.x) * (T)0.5, (Wk.y - Wm.y) * (T)0.5};   // (Wk + conj Wm)/2
    const cplx<T> Vo = {(Wk.y + Wm.y) * (T)0.5, (Wm.x - Wk.x) * (T)0.5};   // -i (Wk - conj Wm)/2
    const cplx<T> tt = cmul(tb.th[k], Vo);
    const cplx<T> V1 = cadd(Ve, tt), V2 = csub(Ve, tt);
    const cplx<T> q1 = tb.tq[k], q2 = tb.tq[k + M];
    lo[r] = (q1.x * V1.x - q1.y * V1.y) * (k == 0 ? s0 : s);
    hi[r] = (q2.x * V2.x - q2.y * V2.y) * s;
  }
}

// v-order permutation m -> natural index (Makhoul's even/odd shuffle)
__host__ __device__ __forceinline__ int vperm(int m, int L) { return m < L / 2 ? 2 * m : 2 * (L - 1 - m) + 1; }

// Convention 1 (Phi = S C2, reading R11: BASELINE config 4's literal "rows of DCT-II"): the forward
// transform comes first.  DCT-II of a natural-order sequence X (stride xs): the packed input of the
// M-point FFT, z[i] = X[vperm(2i)] + i X[vperm(2i+1)] for i = t + r M/8 (thread t of the team).
template <typename T, int L>
__device__ __forceinline__ void dct2_gather(const T* X, int xs, int t, cplx<T> (&v)[8]) {
  constexpr int M = L / 2, NT = M / 8;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = t + r * NT;
    v[r] = {X[vperm(2 * i, L) * xs], X[vperm(2 * i + 1, L) * xs]};
  }
}

constexpr int DCT_THREADS = 256;
constexpr int ROW_ITERS = 2;
template <int L> struct RowGeom {
  static constexpr int M = L / 2, NT = M / 8, TEAMS = DCT_THREADS / NT, RPC = TEAMS * ROW_ITERS;
};

// ---------------------------------------------------------------- pass A
template <typename T, int L, int CONV>
__device__ void rows_inv_body(const DctArgs& a, int j, bool dir, double bcoef, T* sm) {
  using G = RowGeom<L>;
  const int team = threadIdx.x / G::NT, t = threadIdx.x % G::NT;
  T* row = sm + team * L;
  cplx<T>* buf = reinterpret_cast<cplx<T>*>(row);
  const DctCol<T> c = col_of<T>(a, j);
  const DctTab<T> tb = tab_c<T>(a);
  const T b = (T)bcoef;
  for (int it = 0; it < ROW_ITERS; ++it) {
    const int r = blockIdx.x * G::RPC + it * G::TEAMS + team;
    const bool active = r < a.rows;
    if (active) {
      const int64_t base = (int64_t)r * L;
      for (int e = t; e < L; e += G::NT) {
        T p = c.p[base + e];
        if (dir) { p = c.dinv[base + e] * c.r[base + e] + b * p; c.p[base + e] = p; }
        row[e] = p;
      }
    }
    __syncthreads();
    cplx<T> v[8];
    if constexpr (CONV == 0) {         // DCT-III along the row -> v-order pixel columns
      dct3_gather<T, L>(row, 1, t, v, tb);
      fft_team<T, G::M, +1>(buf, v, t, tb.tw);
    } else {                           // DCT-II along the row -> natural-order pixel columns
      dct2_gather<T, L>(row, 1, t, v);
      fft_team<T, G::M, -1>(buf, v, t, tb.tw);
      T lo[8], hi[8];
      dct2_post<T, L>(buf, t, lo, hi, tb);
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 8; ++q) { row[t + q * G::NT] = lo[q]; row[t + q * G::NT + G::M] = hi[q]; }
      __syncthreads();
    }
    if (active) {
      const int64_t base = (int64_t)r * L;
      for (int e = t; e < L; e += G::NT) c.t1[base + e] = row[e];
    }
    __syncthreads();
  }
}

template <typename TP, int L, int CONV>
__global__ void __launch_bounds__(DCT_THREADS) k_dct_rows_inv(DctArgs a, int dir) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int j = blockIdx.y;
  const ColState st = a.cs[j];
  if (st.frozen) return;
  if (j == 0) rows_inv_body<double, L, CONV>(a, 0, dir, st.b, reinterpret_cast<double*>(smem_raw));
  else rows_inv_body<TP, L, CONV>(a, j, dir, st.b, reinterpret_cast<TP*>(smem_raw));
}

// ---------------------------------------------------------------- pass B
template <typename T> struct StripW { static constexpr int W = sizeof(T) == 8 ? 8 : 16; };

template <typename T, int L, int CONV>
__device__ void cols_body(const DctArgs& a, int j, T* sm) {
  constexpr int M = L / 2, NT = M / 8, TEAMS = DCT_THREADS / NT, W = StripW<T>::W, WS = W + 1;
  const int c0 = blockIdx.x * W;
  if (c0 >= a.cols) return;                      // CTA-uniform
  const int team = threadIdx.x / NT, t = threadIdx.x % NT;
  T* strip = sm;                                 // [L][W+1]
  cplx<T>* buf = reinterpret_cast<cplx<T>*>(sm + L * WS + (L * WS) % 2) + team * M;
  const DctCol<T> c = col_of<T>(a, j);
  const DctTab<T> tb = tab_r<T>(a);
  for (int e = threadIdx.x; e < L * W; e += DCT_THREADS) {
    const int r = e / W, cc = e % W;
    strip[r * WS + cc] = c.t1[(int64_t)r * a.cols + c0 + cc];
  }
  __syncthreads();
  constexpr int NIT = (W + TEAMS - 1) / TEAMS;
  for (int it = 0; it < NIT; ++it) {
    const int cc = it * TEAMS + team;
    const bool active = cc < W;
    const int ccs = active ? cc : 0;
    cplx<T> v[8];
    if constexpr (CONV == 1) {
      // DCT-II along the column (natural-order pixel rows), mask, DCT-III back (v-order output rows)
      dct2_gather<T, L>(strip + ccs, WS, t, v);
      fft_team<T, M, -1>(buf, v, t, tb.tw);
      T lo[8], hi[8];
      dct2_post<T, L>(buf, t, lo, hi, tb);
      const uint8_t* mk = a.maskT + (int64_t)(c0 + ccs) * a.rows;   // natural-order mask, [cols][rows]
      __syncthreads();                           // every team has read its column
      if (active) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int k = t + r * NT;
          strip[k * WS + cc] = mk[k] ? lo[r] : (T)0;
          strip[(k + M) * WS + cc] = mk[k + M] ? hi[r] : (T)0;
        }
      }
      __syncthreads();
      dct3_gather<T, L>(strip + ccs, WS, t, v, tb);
      fft_team<T, M, +1>(buf, v, t, tb.tw);      // v-order rows, complex-packed
      if (active) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const int i = t + r * NT;
          const cplx<T> w = buf[i];
          strip[(2 * i) * WS + cc] = w.x;
          strip[(2 * i + 1) * WS + cc] = w.y;
        }
      }
      __syncthreads();
      continue;
    }
    dct3_gather<T, L>(strip + ccs, WS, t, v, tb);
    fft_team<T, M, +1>(buf, v, t, tb.tw);        // v-order pixel column (complex-packed)
    const uint8_t* mk = a.maskT + (int64_t)(c0 + ccs) * a.rows;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int idx = t + r * NT;
      const uchar2 m2 = *reinterpret_cast<const uchar2*>(mk + 2 * idx);
      const cplx<T> w = buf[idx];
      v[r] = {m2.x ? w.x : (T)0, m2.y ? w.y : (T)0};
    }
    fft_team<T, M, -1>(buf, v, t, tb.tw);
    T lo[8], hi[8];
    dct2_post<T, L>(buf, t, lo, hi, tb);
    if (active) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int k = t + r * NT;
        strip[k * WS + cc] = lo[r];
        strip[(k + M) * WS + cc] = hi[r];
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < L * W; e += DCT_THREADS) {
    const int r = e / W, cc = e % W;
    c.t2[(int64_t)r * a.cols + c0 + cc] = strip[r * WS + cc];
  }
}

template <typename TP, int L, int CONV>
__global__ void __launch_bounds__(DCT_THREADS) k_dct_cols(DctArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int j = blockIdx.y;
  if (a.cs[j].frozen) return;
  if (j == 0) cols_body<double, L, CONV>(a, 0, reinterpret_cast<double*>(smem_raw));
  else cols_body<TP, L, CONV>(a, j, reinterpret_cast<TP*>(smem_raw));
}

// ---------------------------------------------------------------- pass C
template <typename T, int L, int CONV>
__device__ double rows_fwd_body(const DctArgs& a, int j, T* sm) {
  using G = RowGeom<L>;
  const int team = threadIdx.x / G::NT, t = threadIdx.x % G::NT;
  T* row = sm + team * L;
  cplx<T>* buf = reinterpret_cast<cplx<T>*>(row);
  const DctCol<T> c = col_of<T>(a, j);
  const DctTab<T> tb = tab_c<T>(a);
  const T beta = (T)a.beta;
  double g = 0.0;
  for (int it = 0; it < ROW_ITERS; ++it) {
    const int r = blockIdx.x * G::RPC + it * G::TEAMS + team;
    const bool active = r < a.rows;
    // conv. 1: T2 row r holds coefficient row vperm(r) (pass B left the rows in v-order)
    const int64_t base = (int64_t)(CONV == 0 || !active ? r : vperm(r, a.rows)) * L, base_in = (int64_t)r * L;
    if (active)
      for (int e = t; e < L; e += G::NT) row[e] = c.t2[base_in + e];
    __syncthreads();
    cplx<T> v[8];
    if constexpr (CONV == 0) {         // DCT-II along the row (packed v-order input) -> natural coefficients
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = buf[t + q * G::NT];
      fft_team<T, G::M, -1>(buf, v, t, tb.tw);
      T lo[8], hi[8];
      dct2_post<T, L>(buf, t, lo, hi, tb);
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 8; ++q) { row[t + q * G::NT] = lo[q]; row[t + q * G::NT + G::M] = hi[q]; }
    } else {                           // DCT-III along the row (natural input) -> v-order, un-shuffled
      dct3_gather<T, L>(row, 1, t, v, tb);
      fft_team<T, G::M, +1>(buf, v, t, tb.tw);
      cplx<T> w[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) w[q] = buf[t + q * G::NT];
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int i = t + q * G::NT;
        row[vperm(2 * i, L)] = w[q].x;
        row[vperm(2 * i + 1, L)] = w[q].y;
      }
    }
    __syncthreads();
    if (active) {
      for (int e = t; e < L; e += G::NT) {
        const T p = c.p[base + e];
        const T qv = beta * row[e] + (T)a.alpha[base + e] * p;
        c.q[base + e] = qv;
        g += (double)p * (double)qv;
      }
    }
    __syncthreads();
  }
  return g;
}

template <typename TP, int L, int CONV>
__global__ void __launch_bounds__(DCT_THREADS) k_dct_rows_fwd(DctArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int j = blockIdx.y;
  if (a.cs[j].frozen) return;
  double g = j == 0 ? rows_fwd_body<double, L, CONV>(a, 0, reinterpret_cast<double*>(smem_raw))
                    : rows_fwd_body<TP, L, CONV>(a, j, reinterpret_cast<TP*>(smem_raw));
  g = block_sum(g);
  ColState* cs = a.cs;
  const int iter = a.iter;
  column_finish(g, j, a.part, a.stride, a.counters, [cs, j, iter](double tot) {
    ColState c = cs[j]; finish_gamma(c, tot, iter); cs[j] = c;
  });
}

// ---------------------------------------------------------------- setup kernels

__global__ void k_mask_scatter(const int64_t* __restrict__ obs, int64_t N, uint8_t* __restrict__ mask) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    mask[obs[i]] = 1;
}
__global__ void k_mask_vvT(const uint8_t* __restrict__ mask, int rows, int cols, uint8_t* __restrict__ maskT) {
  const int64_t total = (int64_t)rows * cols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / rows), mr = (int)(i % rows);
    maskT[i] = mask[(int64_t)vperm(mr, rows) * cols + vperm(c, cols)];
  }
}
__global__ void k_y_scatter(const int64_t* __restrict__ obs, int64_t N, const float* __restrict__ y, double* __restrict__ img) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    img[obs[i]] = (double)y[i];
}
__global__ void k_mask_T(const uint8_t* __restrict__ mask, int rows, int cols, uint8_t* __restrict__ maskT) {
  const int64_t total = (int64_t)rows * cols;     // natural order, transposed [cols][rows] (convention 1)
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / rows), r = (int)(i % rows);
    maskT[i] = mask[(int64_t)r * cols + c];
  }
}
__global__ void k_mask_to_double(const uint8_t* __restrict__ m, int64_t n, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (double)m[i];
}

// C = alpha * op(A) * op(B), fp64, 16x16 tiles (setup only).  op(X) = X or X^T.
__global__ void k_gemm64(int M, int Nn, int Kk, const double* __restrict__ A, int lda, int ta,
                         const double* __restrict__ B, int ldb, int tb, double* __restrict__ C, int ldc, double alpha) {
  __shared__ double As[16][17], Bs[16][17];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int row = blockIdx.y * 16 + ty, col = blockIdx.x * 16 + tx;
  double acc = 0.0;
  for (int k0 = 0; k0 < Kk; k0 += 16) {
    const int ka = k0 + tx, kb = k0 + ty;
    As[ty][tx] = (row < M && ka < Kk) ? (ta ? A[(int64_t)ka * lda + row] : A[(int64_t)row * lda + ka]) : 0.0;
    Bs[ty][tx] = (kb < Kk && col < Nn) ? (tb ? B[(int64_t)col * ldb + kb] : B[(int64_t)kb * ldb + col]) : 0.0;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) acc += As[ty][k] * Bs[k][tx];
    __syncthreads();
  }
  if (row < M && col < Nn) C[(int64_t)row * ldc + col] = alpha * acc;
}

// ---------------------------------------------------------------- host
template <typename T> static void fill_tab(std::vector<cplx<T>>& h, int L) {
  const int M = L / 2;
  const double PI = 3.14159265358979323846;
  for (int k = 0; k < M; ++k) h.push_back({(T)cos(-2 * PI * k / M), (T)sin(-2 * PI * k / M)});
  for (int k = 0; k < L; ++k) h.push_back({(T)cos(-PI * k / (2.0 * L)), (T)sin(-PI * k / (2.0 * L))});
  for (int k = 0; k < M; ++k) h.push_back({(T)cos(-2 * PI * k / L), (T)sin(-2 * PI * k / L)});
}
template <typename T> static DctTab<T> tab_at(const cplx<T>* base, int L) {
  const int M = L / 2;
  return {base, base + M, base + M + L};
}

static void gemm64(Ctx* c, int M, int Nn, int Kk, const double* A, int lda, int ta, const double* B, int ldb, int tb,
                   double* C, int ldc, double alpha) {
  dim3 grid((Nn + 15) / 16, (M + 15) / 16), blk(16, 16);
  launch_begin(c, KC_SETUP);
  k_gemm64<<<grid, blk, 0, c->stream>>>(M, Nn, Kk, A, lda, ta, B, ldb, tb, C, ldc, alpha);
  launch_end(c, KC_SETUP);
}

static void dct_matrix(std::vector<double>& C, int L, bool square) {   // C[k][n] (or its square)
  C.resize((size_t)L * L);
  const double PI = 3.14159265358979323846;
  for (int k = 0; k < L; ++k)
    for (int n = 0; n < L; ++n) {
      double v = cos(PI * (2.0 * n + 1.0) * k / (2.0 * L)) * (k == 0 ? sqrt(1.0 / L) : sqrt(2.0 / L));
      C[(size_t)k * L + n] = square ? v * v : v;
    }
}

template <typename TP> static void set_smem_attrs(int rows, int cols);

template <int L> static size_t row_smem() { return (size_t)RowGeom<L>::TEAMS * L * sizeof(double); }
template <int L> static size_t col_smem() {
  constexpr int M = L / 2, NT = M / 8, TEAMS = DCT_THREADS / NT;
  size_t d = (size_t)L * (StripW<double>::W + 1) * 8 + 16 + (size_t)TEAMS * M * 16;
  size_t f = (size_t)L * (StripW<float>::W + 1) * 4 + 16 + (size_t)TEAMS * M * 8;
  return std::max(d, f);
}

#define DCT_LENGTHS(X) X(16) X(32) X(64) X(128) X(256) X(512) X(1024)

template <typename TP>
static cofem_status set_attrs(Ctx* c) {
#define SET_ROW(L)                                                                                                  \
  if (c->cols == L) {                                                                                               \
    cudaFuncSetAttribute(k_dct_rows_inv<TP, L, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)row_smem<L>()); \
    cudaFuncSetAttribute(k_dct_rows_fwd<TP, L, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)row_smem<L>()); \
    cudaFuncSetAttribute(k_dct_rows_inv<TP, L, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)row_smem<L>()); \
    cudaFuncSetAttribute(k_dct_rows_fwd<TP, L, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)row_smem<L>()); \
  }
#define SET_COL(L)                                                                                                  \
  if (c->rows == L) {                                                                                               \
    cudaFuncSetAttribute(k_dct_cols<TP, L, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)col_smem<L>());     \
    cudaFuncSetAttribute(k_dct_cols<TP, L, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)col_smem<L>());     \
  }
  DCT_LENGTHS(SET_ROW)
  DCT_LENGTHS(SET_COL)
#undef SET_ROW
#undef SET_COL
  return check_launch(c, "dct attrs") == cudaSuccess ? COFEM_OK : COFEM_ERR_CUDA;
}

// b0 = beta Phi^T y (Eq. 5): scatter y into a zero image, then the forward 2D DCT C_r Y C_c^T
// (convention 1: Phi^T = C2^T S^T, C_r^T Y C_c), fp64 -- at setup and for the further observation
// vectors of the multi-task EM (R22)
cofem_status dct_b0(Ctx* c, const float* y_dev, double* out) {
  const int rows = c->rows, cols = c->cols;
  const int64_t D = c->D;
  double *Cr = nullptr, *Cc = nullptr, *tmp = nullptr, *img = nullptr;
  if (cudaMalloc(&tmp, D * 8) != cudaSuccess || cudaMalloc(&img, D * 8) != cudaSuccess ||
      cudaMalloc(&Cr, (size_t)rows * rows * 8) != cudaSuccess || cudaMalloc(&Cc, (size_t)cols * cols * 8) != cudaSuccess) {
    c->err = "cudaMalloc dct b0"; return COFEM_ERR_OOM;
  }
  cudaMemsetAsync(img, 0, D * 8, c->stream);
  launch_begin(c, KC_SETUP);
  k_y_scatter<<<c->num_sms * 4, 256, 0, c->stream>>>(c->obs_dev, c->N, y_dev, img);
  launch_end(c, KC_SETUP);
  std::vector<double> h;
  dct_matrix(h, rows, false); cudaMemcpyAsync(Cr, h.data(), h.size() * 8, cudaMemcpyHostToDevice, c->stream); cudaStreamSynchronize(c->stream);
  dct_matrix(h, cols, false); cudaMemcpyAsync(Cc, h.data(), h.size() * 8, cudaMemcpyHostToDevice, c->stream); cudaStreamSynchronize(c->stream);
  const int tcv = c->conv ? 0 : 1, tr = c->conv ? 1 : 0;
  gemm64(c, rows, cols, cols, img, cols, 0, Cc, cols, tcv, tmp, cols, 1.0);
  gemm64(c, rows, cols, rows, Cr, rows, tr, tmp, cols, 0, out, cols, c->beta);
  cudaStreamSynchronize(c->stream);
  cudaFree(tmp); cudaFree(img); cudaFree(Cr); cudaFree(Cc);
  return check_launch(c, "dct_b0") == cudaSuccess ? COFEM_OK : COFEM_ERR_CUDA;
}

cofem_status dct_setup(Ctx* c, const float* y_dev, const int64_t* obs_dev) {
  const int rows = c->rows, cols = c->cols;
  const int64_t D = c->D;
  // twiddle tables: [rows-length | cols-length], float and double
  {
    std::vector<cplx<float>> h32; std::vector<cplx<double>> h64;
    fill_tab(h32, rows); fill_tab(h32, cols); fill_tab(h64, rows); fill_tab(h64, cols);
    if (cudaMalloc(&c->dct_tab32, h32.size() * sizeof(cplx<float>)) != cudaSuccess ||
        cudaMalloc(&c->dct_tab64, h64.size() * sizeof(cplx<double>)) != cudaSuccess) { c->err = "cudaMalloc tables"; return COFEM_ERR_OOM; }
    cudaMemcpy(c->dct_tab32, h32.data(), h32.size() * sizeof(cplx<float>), cudaMemcpyHostToDevice);
    cudaMemcpy(c->dct_tab64, h64.data(), h64.size() * sizeof(cplx<double>), cudaMemcpyHostToDevice);
  }
  uint8_t* mask = nullptr;
  double *md = nullptr, *Cr = nullptr, *Cc = nullptr, *tmp = nullptr, *img = nullptr;
  const size_t tp = c->probe64 ? 8 : 4;
  if (cudaMalloc(&mask, D) != cudaSuccess || cudaMalloc(&c->mask_vvT, D) != cudaSuccess ||
      cudaMalloc(&md, D * 8) != cudaSuccess || cudaMalloc(&tmp, D * 8) != cudaSuccess ||
      cudaMalloc(&img, D * 8) != cudaSuccess || cudaMalloc(&Cr, (size_t)rows * rows * 8) != cudaSuccess ||
      cudaMalloc(&Cc, (size_t)cols * cols * 8) != cudaSuccess ||
      cudaMalloc(&c->ws1, (size_t)c->Kcap * c->Dp * tp) != cudaSuccess ||
      cudaMalloc(&c->ws2, (size_t)c->Kcap * c->Dp * tp) != cudaSuccess ||
      cudaMalloc(&c->ws1d, c->Dp * 8) != cudaSuccess || cudaMalloc(&c->ws2d, c->Dp * 8) != cudaSuccess) {
    c->err = "cudaMalloc dct setup"; return COFEM_ERR_OOM;
  }
  cudaMemsetAsync(mask, 0, D, c->stream);
  cudaMemsetAsync(img, 0, D * 8, c->stream);
  launch_begin(c, KC_SETUP);
  k_mask_scatter<<<c->num_sms * 4, 256, 0, c->stream>>>(obs_dev, c->N, mask);
  if (c->conv == 0) k_mask_vvT<<<c->num_sms * 4, 256, 0, c->stream>>>(mask, rows, cols, c->mask_vvT);
  else k_mask_T<<<c->num_sms * 4, 256, 0, c->stream>>>(mask, rows, cols, c->mask_vvT);
  k_mask_to_double<<<c->num_sms * 4, 256, 0, c->stream>>>(mask, D, md);
  launch_end(c, KC_SETUP);
  // colsq = Q_r M Q_c^T with Q = C o C (diag of C2 M C2^T)
  std::vector<double> h;
  dct_matrix(h, rows, true); cudaMemcpyAsync(Cr, h.data(), h.size() * 8, cudaMemcpyHostToDevice, c->stream); cudaStreamSynchronize(c->stream);
  dct_matrix(h, cols, true); cudaMemcpyAsync(Cc, h.data(), h.size() * 8, cudaMemcpyHostToDevice, c->stream); cudaStreamSynchronize(c->stream);
  // convention 1 (Phi = S C2, Phi[n, d] = C2[obs_n, d]): colsq = Q_r^T M Q_c
  const int tcv = c->conv ? 0 : 1, tr = c->conv ? 1 : 0;
  gemm64(c, rows, cols, cols, md, cols, 0, Cc, cols, tcv, tmp, cols, 1.0);        // M Q_c^T  (conv. 1: M Q_c)
  gemm64(c, rows, cols, rows, Cr, rows, tr, tmp, cols, 0, c->colsq, cols, 1.0);   // Q_r (.)  (conv. 1: Q_r^T (.))
  cudaStreamSynchronize(c->stream);
  cudaFree(mask); cudaFree(md); cudaFree(tmp); cudaFree(img); cudaFree(Cr); cudaFree(Cc);
  // the mask indices stay on the device (b0 of further observation vectors, multi-task EM)
  if (cudaMalloc(&c->obs_dev, c->N * sizeof(int64_t)) != cudaSuccess) { c->err = "cudaMalloc obs"; return COFEM_ERR_OOM; }
  cudaMemcpyAsync(c->obs_dev, obs_dev, c->N * sizeof(int64_t), cudaMemcpyDeviceToDevice, c->stream);
  {
    cofem_status sb = dct_b0(c, y_dev, c->b0);
    if (sb != COFEM_OK) return sb;
  }
  if (check_launch(c, "dct setup")) return COFEM_ERR_CUDA;
  // partial-sum stride: pass C grid.x
  int rpc = 1;
#define RPC_OF(L) if (cols == L) rpc = RowGeom<L>::RPC;
  DCT_LENGTHS(RPC_OF)
#undef RPC_OF
  const int gridA = (rows + rpc - 1) / rpc;
  c->part_stride = std::max(c->part_stride, gridA);
  cofem_status st = c->probe64 ? set_attrs<double>(c) : set_attrs<float>(c);
  if (st == COFEM_OK && dct1k_eligible(c) && c->opt.apply_path != 1 && c->conv == 0) {   // apply_path 1 / conv. 1: generic
    st = dct1k_setup(c);
    c->fast1k = st == COFEM_OK;
    for (int g = 1; c->fast1k && g < Ctx::MAXG; ++g)      // probe groups' s accumulators (cofem.cu)
      if (cudaMalloc(&c->gs[g], c->Dp * sizeof(double)) != cudaSuccess) { c->gs[g] = nullptr; cudaGetLastError(); break; }
  }
  return st;
}

DctArgs dct_args(Ctx* c, int m, int iter) {
  DctArgs a;
  a.rows = c->rows; a.cols = c->cols; a.Dp = c->Dp; a.K = m - 1;
  a.beta = c->beta; a.alpha = c->alpha;
  a.p0 = c->p0; a.r0 = c->r0; a.dinv64 = c->dinv64; a.t1d = c->ws1d; a.t2d = c->ws2d; a.q0 = c->q0;
  a.P = c->P; a.R = c->R; a.dinvp = c->dinvp; a.t1 = c->ws1; a.t2 = c->ws2; a.Q = c->Q;
  a.maskT = c->mask_vvT;
  const cplx<float>* b32 = (const cplx<float>*)c->dct_tab32;
  const cplx<double>* b64 = (const cplx<double>*)c->dct_tab64;
  const int lr = 2 * c->rows;   // table entries for the rows length: M + L + M = 2L
  a.tr32 = tab_at(b32, c->rows); a.tc32 = tab_at(b32 + lr, c->cols);
  a.tr64 = tab_at(b64, c->rows); a.tc64 = tab_at(b64 + lr, c->cols);
  a.cs = c->cs; a.part = c->part; a.stride = c->part_stride; a.counters = c->counters; a.iter = iter;
  a.ticket = c->counters + MAXM + 2;
  a.maskL = c->maskL; a.alphap = c->alphap; a.tab1k32 = c->tab1k32; a.tab1k64 = c->tab1k64;
  return a;
}

template <typename TP>
static cofem_status dct_apply_t(Ctx* c, int m, int iter, bool dir) {
  DctArgs a = dct_args(c, m, iter);
  bool launched = false;
#define LAUNCH_ROWS(L)                                                                                   \
  if (c->cols == L) {                                                                                    \
    dim3 g((c->rows + RowGeom<L>::RPC - 1) / RowGeom<L>::RPC, m);                                        \
    launch_begin(c, KC_DCT_ROWS_INV);                                                                    \
    if (c->conv) k_dct_rows_inv<TP, L, 1><<<g, DCT_THREADS, row_smem<L>(), c->stream>>>(a, dir ? 1 : 0);  \
    else k_dct_rows_inv<TP, L, 0><<<g, DCT_THREADS, row_smem<L>(), c->stream>>>(a, dir ? 1 : 0);          \
    launch_end(c, KC_DCT_ROWS_INV);                                                                      \
    launched = true;                                                                                     \
  }
  DCT_LENGTHS(LAUNCH_ROWS)
#undef LAUNCH_ROWS
  if (!launched || check_launch(c, "k_dct_rows_inv")) return COFEM_ERR_CUDA;
  launched = false;
#define LAUNCH_COLS(L)                                                                                   \
  if (c->rows == L) {                                                                                    \
    dim3 g(c->cols / StripW<double>::W, m);                                                              \
    launch_begin(c, KC_DCT_COLS);                                                                        \
    if (c->conv) k_dct_cols<TP, L, 1><<<g, DCT_THREADS, col_smem<L>(), c->stream>>>(a);                  \
    else k_dct_cols<TP, L, 0><<<g, DCT_THREADS, col_smem<L>(), c->stream>>>(a);                          \
    launch_end(c, KC_DCT_COLS);                                                                          \
    launched = true;                                                                                     \
  }
  DCT_LENGTHS(LAUNCH_COLS)
#undef LAUNCH_COLS
  if (!launched || check_launch(c, "k_dct_cols")) return COFEM_ERR_CUDA;
  launched = false;
#define LAUNCH_FWD(L)                                                                                    \
  if (c->cols == L) {                                                                                    \
    dim3 g((c->rows + RowGeom<L>::RPC - 1) / RowGeom<L>::RPC, m);                                        \
    launch_begin(c, KC_DCT_ROWS_FWD);                                                                    \
    if (c->conv) k_dct_rows_fwd<TP, L, 1><<<g, DCT_THREADS, row_smem<L>(), c->stream>>>(a);               \
    else k_dct_rows_fwd<TP, L, 0><<<g, DCT_THREADS, row_smem<L>(), c->stream>>>(a);                       \
    launch_end(c, KC_DCT_ROWS_FWD);                                                                      \
    launched = true;                                                                                     \
  }
  DCT_LENGTHS(LAUNCH_FWD)
#undef LAUNCH_FWD
  if (!launched || check_launch(c, "k_dct_rows_fwd")) return COFEM_ERR_CUDA;
  return COFEM_OK;
}

cofem_status dct_apply(Ctx* c, int m, int iter, bool dir) {
  return c->probe64 ? dct_apply_t<double>(c, m, iter, dir) : dct_apply_t<float>(c, m, iter, dir);
}

}  // namespace cofem
