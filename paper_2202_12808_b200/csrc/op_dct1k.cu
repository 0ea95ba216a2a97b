// op_dct1k.cu — fast path of the masked 2D DCT Gram apply for 1024 x 1024 grids,
// the BASELINE headline workload (config 4, D = 2^20; §4.2; reading R11):
//   Q = beta C2 (M o (C2^T P)) + alpha o P,  C2 = C_r (x) C_c orthonormal 2D DCT-II.
//
// One warp owns one line (1024 reals = a 512-point complex FFT after Makhoul's
// even/odd packing), 16 complex points per lane, three radix-8 Stockham stages
// with two warp-synchronous shared-memory exchanges whose padded layouts are
// bank-conflict-free.  Lane l owns butterflies {l, 64-l} (lane 0:
// {0, 32}) in the first and last stage, so the DCT's k <-> M-k pairing (pre- and
// post-processing) never leaves the lane, and every lane loads/stores exactly its
// 32 "canonical" positions {ja, jb, 512+ja, 512+jb} + 64 r of the line, coalesced.
//
//   pass A  k1k_rows_inv : fused CG direction p = M^-1 r + b p (a6); DCT-III along each
//                          image row; write T^T (columns become contiguous lines)
//   pass B  k1k_cols     : on each T^T line: DCT-III, mask, DCT-II, in place
//   pass C  k1k_rows_fwd : transposed read of T^T; DCT-II along each row;
//                          q = beta X + alpha o p; gamma_j = p_j^T q_j (a3 + a4)
// Intermediates keep the transformed axes in "v-order" (m -> 2m, 2(L-1-m)+1): the
// inverse transform's packed output is the forward transform's packed input, so
// pass B never leaves registers between its IFFT and FFT and no pass permutes data.
// Probe columns run in fp32 (8 rows per CTA); the fp64 mean column (4 rows per
// CTA) runs on a second stream concurrently (cofem.cu).
#include <math.h>

#include <algorithm>
#include <vector>

#include "fft_common.cuh"

namespace cofem {
namespace d1k {

constexpr int L = 1024, M = 512;
constexpr int XS1 = 68, XS2 = 72;      // exchange row strides: pads 4 and 8 words (conflict-free)
constexpr int XPL = 8 * XS2;           // elements per plane of the exchange buffer
constexpr int WREG = 2 * XPL;          // per-warp smem region (elements of T): exchange planes / one tile row (>= L)
template <typename T> struct Geo { static constexpr int RT = sizeof(T) == 8 ? 4 : 8; };   // rows (warps) per CTA

// Twiddle tables, host-built in fp64 and rounded to T, copied to shared memory by every CTA
// in layouts that make each warp access conflict-free (lanes read consecutive entries):
//   w2[r*8 + k]  = W_64^{r k}      (stage 2, k = lane & 7)
//   w3[r*64 + j] = W_512^{r j}     (stage 3, j = butterfly)
//   tq[k] = exp(-i pi k / 2L) (k < L),  th[k] = exp(-2 pi i k / L) (k < M)   (Makhoul pre/post)
constexpr int TW2 = 0, TW3 = 64, TTQ = TW3 + 512, TTH = TTQ + L, TTOT = TTH + M;   // offsets in complex entries
template <typename T> struct Tw { const cplx<T>* w2; const cplx<T>* w3; const cplx<T>* tq; const cplx<T>* th; };

template <typename T>
__device__ __forceinline__ Tw<T> load_tables(const cplx<T>* __restrict__ g, cplx<T>* sm) {
  for (int i = threadIdx.x; i < TTOT; i += blockDim.x) sm[i] = g[i];
  __syncthreads();
  return {sm + TW2, sm + TW3, sm + TTQ, sm + TTH};
}

template <typename T, int SIGN>
__device__ __forceinline__ void twid(cplx<T>& v, cplx<T> w) { v = SIGN < 0 ? cmul(v, w) : cmulc(v, w); }

// 512-point DFT (SIGN -1) / unnormalised inverse (SIGN +1) by one warp.
// In:  va[r] = x[ja + 64 r], vb[r] = x[jb + 64 r].  Out: va[r] = X[ja + 64 r], vb[r] = X[jb + 64 r].
// Stockham radix-8: stage s reads x[j + 64 r], twiddles by W_{8 Ns}^{r (j mod Ns)}, DFT8,
// writes y[(j / Ns) 8 Ns + (j mod Ns) + r Ns]; Ns = 1, 8, 64.  Exchanges store [r][j].
template <typename T, int SIGN>
__device__ __forceinline__ void fft512(cplx<T> (&va)[8], cplx<T> (&vb)[8], int lane, T* __restrict__ re,
                                       T* __restrict__ im, const Tw<T>& tw) {
  const int ja = lane, jb = lane ? 64 - lane : 32;
  dft8<SIGN>(va); dft8<SIGN>(vb);                       // stage 1 (Ns = 1): butterflies ja, jb
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    re[r * XS1 + ja] = va[r].x; im[r * XS1 + ja] = va[r].y;
    re[r * XS1 + jb] = vb[r].x; im[r * XS1 + jb] = vb[r].y;
  }
  __syncwarp();
  {   // stage 2 (Ns = 8): butterflies lane, lane + 32; y[i] lives at [(i & 7)][i >> 3]
    const int base = (lane & 7) * XS1 + (lane >> 3);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      va[r] = {re[base + 8 * r], im[base + 8 * r]};
      vb[r] = {re[base + 4 + 8 * r], im[base + 4 + 8 * r]};
    }
    const int k = lane & 7;
#pragma unroll
    for (int r = 1; r < 8; ++r) {
      const cplx<T> w = tw.w2[r * 8 + k];
      twid<T, SIGN>(va[r], w); twid<T, SIGN>(vb[r], w);
    }
  }
  dft8<SIGN>(va); dft8<SIGN>(vb);
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    re[r * XS2 + lane] = va[r].x; im[r * XS2 + lane] = va[r].y;
    re[r * XS2 + lane + 32] = vb[r].x; im[r * XS2 + lane + 32] = vb[r].y;
  }
  __syncwarp();
  {   // stage 3 (Ns = 64): butterflies ja, jb; y'[i] written by j2 = 8 (i >> 6) + (i & 7), r2 = (i >> 3) & 7
    const int ba = (ja >> 3) * XS2 + (ja & 7), bb = (jb >> 3) * XS2 + (jb & 7);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      va[r] = {re[ba + 8 * r], im[ba + 8 * r]};
      vb[r] = {re[bb + 8 * r], im[bb + 8 * r]};
    }
#pragma unroll
    for (int r = 1; r < 8; ++r) {
      twid<T, SIGN>(va[r], tw.w3[r * 64 + ja]);
      twid<T, SIGN>(vb[r], tw.w3[r * 64 + jb]);
    }
  }
  dft8<SIGN>(va); dft8<SIGN>(vb);
  __syncwarp();                                         // exchange region free again
}

// DCT-III (orthonormal inverse) pre-processing for one k (Makhoul): packed spectrum W[k]
// from X[k], X[L-k], X[k+M], X[M-k]; the 1/M IFFT normalisation and 1/s_k are folded in.
template <typename T>
__device__ __forceinline__ cplx<T> dct3_pre(int k, T Xk, T XLk, T XkM, T XMk, const Tw<T>& tb) {
  const T sc0 = (T)0.0625, sc = (T)0.044194173824159216;   // sqrt(L)/M, sqrt(L/2)/M
  const T xk = Xk * (k == 0 ? sc0 : sc);
  const T xLk = k == 0 ? (T)0 : XLk * sc;
  const T xkM = XkM * sc, xMk = XMk * sc;
  const cplx<T> V1 = cmulc(cplx<T>{xk, -xLk}, tb.tq[k]);
  const cplx<T> V2 = cmulc(cplx<T>{xkM, -xMk}, tb.tq[k + M]);
  const cplx<T> Ve = {(V1.x + V2.x) * (T)0.5, (V1.y + V2.y) * (T)0.5};
  const cplx<T> Vo = cmulc(cplx<T>{(V1.x - V2.x) * (T)0.5, (V1.y - V2.y) * (T)0.5}, tb.th[k]);
  return {Ve.x - Vo.y, Ve.y + Vo.x};
}

// DCT-II post-processing for one k from W[k], W[(M-k) mod M]: orthonormal X[k], X[k+M].
template <typename T>
__device__ __forceinline__ void dct2_post(int k, cplx<T> Wk, cplx<T> Wm, const Tw<T>& tb, T& lo, T& hi) {
  const T s0 = (T)0.03125, s = (T)0.044194173824159216;    // sqrt(1/L), sqrt(2/L)
  const cplx<T> Ve = {(Wk.x + Wm.x) * (T)0.5, (Wk.y - Wm.y) * (T)0.5};
  const cplx<T> Vo = {(Wk.y + Wm.y) * (T)0.5, (Wm.x - Wk.x) * (T)0.5};
  const cplx<T> tt = cmul(tb.th[k], Vo);
  const cplx<T> V1 = cadd(Ve, tt), V2 = csub(Ve, tt);
  const cplx<T> q1 = tb.tq[k], q2 = tb.tq[k + M];
  lo = (q1.x * V1.x - q1.y * V1.y) * (k == 0 ? s0 : s);
  hi = (q2.x * V2.x - q2.y * V2.y) * s;
}

// Canonical positions of a lane in a line: slot A r -> ja + 64r, B -> jb + 64r,
// C -> 512 + ja + 64r, E -> 512 + jb + 64r (r = 0..7): 32 distinct positions per lane,
// together the whole line; each load/store instruction is coalesced.
__device__ __forceinline__ void canon(int lane, int r, int (&o)[4]) {
  const int ja = lane, jb = lane ? 64 - lane : 32;
  o[0] = ja + 64 * r; o[1] = jb + 64 * r; o[2] = M + ja + 64 * r; o[3] = M + jb + 64 * r;
}

// Packed spectra of the DCT-III of a line held canonically in A, B, C, E.
template <typename T>
__device__ __forceinline__ void pre_all(int lane, const T (&A)[8], const T (&B)[8], const T (&C)[8], const T (&E)[8],
                                        cplx<T> (&va)[8], cplx<T> (&vb)[8], const Tw<T>& tb) {
  const int ja = lane, jb = lane ? 64 - lane : 32;
  const bool l0 = lane == 0;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    // slot a, k = ja + 64 r: X[M-k], X[L-k]
    const T aMk = l0 ? (r ? A[(8 - r) & 7] : C[0]) : B[7 - r];
    const T aLk = l0 ? (r ? C[(8 - r) & 7] : (T)0) : E[7 - r];
    va[r] = dct3_pre<T>(ja + 64 * r, A[r], aLk, C[r], aMk, tb);
    // slot b, k = jb + 64 r
    const T bMk = l0 ? B[7 - r] : A[7 - r];
    const T bLk = l0 ? E[7 - r] : C[7 - r];
    vb[r] = dct3_pre<T>(jb + 64 * r, B[r], bLk, E[r], bMk, tb);
  }
}

// DCT-II outputs of a line from its FFT (va, vb) into canonical A, B, C, E.
template <typename T>
__device__ __forceinline__ void post_all(int lane, const cplx<T> (&va)[8], const cplx<T> (&vb)[8], T (&A)[8], T (&B)[8],
                                         T (&C)[8], T (&E)[8], const Tw<T>& tb) {
  const int ja = lane, jb = lane ? 64 - lane : 32;
  const bool l0 = lane == 0;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const cplx<T> wa = l0 ? va[(8 - r) & 7] : vb[7 - r];
    dct2_post<T>(ja + 64 * r, va[r], wa, tb, A[r], C[r]);
    const cplx<T> wb = l0 ? vb[7 - r] : va[7 - r];
    dct2_post<T>(jb + 64 * r, vb[r], wb, tb, B[r], E[r]);
  }
}

template <typename T> __device__ __forceinline__ const T* alpha_of(const DctArgs& a, int j) {
  if constexpr (sizeof(T) == 8) { if (j == 0) return a.alpha; }
  return (const T*)a.alphap;
}

// RT consecutive elements (32 bytes) <-> registers
template <typename T, int N> __device__ __forceinline__ void st32B(T* p, const T (&v)[N]) {
  static_assert(N * sizeof(T) == 32, "32-byte segment");
  if constexpr (sizeof(T) == 4) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  } else {
    reinterpret_cast<double2*>(p)[0] = make_double2(v[0], v[1]);
    reinterpret_cast<double2*>(p)[1] = make_double2(v[2], v[3]);
  }
}
template <typename T, int N> __device__ __forceinline__ void ld32B(const T* p, T (&v)[N]) {
  static_assert(N * sizeof(T) == 32, "32-byte segment");
  if constexpr (sizeof(T) == 4) {
    const float4 x = reinterpret_cast<const float4*>(p)[0], y = reinterpret_cast<const float4*>(p)[1];
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w; v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
  } else {
    const double2 x = reinterpret_cast<const double2*>(p)[0], y = reinterpret_cast<const double2*>(p)[1];
    v[0] = x.x; v[1] = x.y; v[2] = y.x; v[3] = y.y;
  }
}

template <typename T> __device__ __forceinline__ const cplx<T>* tab1k(const DctArgs& a) {
  if constexpr (sizeof(T) == 8) return (const cplx<T>*)a.tab1k64; else return (const cplx<T>*)a.tab1k32;
}

// ---------------------------------------------------------------- pass A
// Shared memory: [RT warps][WREG] (FFT exchange / output tile row) then the twiddle tables.
template <typename T>
__global__ void __launch_bounds__(Geo<T>::RT * 32) k1k_rows_inv(DctArgs a, int j0, int dir) {
  constexpr int RT = Geo<T>::RT;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int j = j0 + blockIdx.y;
  const ColState st = a.cs[j];
  if (st.frozen) return;
  T* sm = reinterpret_cast<T*>(smraw);
  const Tw<T> tb = load_tables<T>(tab1k<T>(a), reinterpret_cast<cplx<T>*>(sm + RT * WREG));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = blockIdx.x * RT;
  const DctCol<T> c = col_of<T>(a, j);
  const int64_t rb = (int64_t)(row0 + warp) * L;
  T A[8], B[8], C[8], E[8];
  {
    T* __restrict__ pr = c.p + rb;
    const T* __restrict__ rr = c.r + rb;
    const T* __restrict__ dv = c.dinv + rb;
    const T bb = (T)st.b;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      int o[4];
      canon(lane, r, o);
      A[r] = pr[o[0]]; B[r] = pr[o[1]]; C[r] = pr[o[2]]; E[r] = pr[o[3]];
    }
    if (dir) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {    // a6: p = M^-1 r + b p  (all loads before any store)
        int o[4];
        canon(lane, r, o);
        A[r] = dv[o[0]] * rr[o[0]] + bb * A[r];
        B[r] = dv[o[1]] * rr[o[1]] + bb * B[r];
        C[r] = dv[o[2]] * rr[o[2]] + bb * C[r];
        E[r] = dv[o[3]] * rr[o[3]] + bb * E[r];
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        int o[4];
        canon(lane, r, o);
        pr[o[0]] = A[r]; pr[o[1]] = B[r]; pr[o[2]] = C[r]; pr[o[3]] = E[r];
      }
    }
  }
  cplx<T> va[8], vb[8];
  pre_all<T>(lane, A, B, C, E, va, vb, tb);
  T* reg = sm + warp * WREG;
  fft512<T, +1>(va, vb, lane, reg, reg + XPL, tb);
  const int ja = lane, jb = lane ? 64 - lane : 32;
#pragma unroll
  for (int r = 0; r < 8; ++r) {     // packed v-order output w[n] = v[2n] + i v[2n+1]
    *reinterpret_cast<cplx<T>*>(reg + 2 * (ja + 64 * r)) = va[r];
    *reinterpret_cast<cplx<T>*>(reg + 2 * (jb + 64 * r)) = vb[r];
  }
  __syncthreads();
  T* __restrict__ out = c.t1;       // T^T[cv][row], line length L
#pragma unroll
  for (int it = 0; it < L / (RT * 32); ++it) {
    const int cv = it * RT * 32 + threadIdx.x;
    T v[RT];
#pragma unroll
    for (int i = 0; i < RT; ++i) v[i] = sm[i * WREG + cv];
    st32B<T, RT>(out + (int64_t)cv * L + row0, v);
  }
}

// ---------------------------------------------------------------- pass B
template <typename T>
__global__ void __launch_bounds__(Geo<T>::RT * 32) k1k_cols(DctArgs a, int j0) {
  constexpr int RT = Geo<T>::RT;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int j = j0 + blockIdx.y;
  if (a.cs[j].frozen) return;
  T* sm = reinterpret_cast<T*>(smraw);
  const Tw<T> tb = load_tables<T>(tab1k<T>(a), reinterpret_cast<cplx<T>*>(sm + RT * WREG));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int line = blockIdx.x * RT + warp;          // v-order image column cv
  const DctCol<T> c = col_of<T>(a, j);
  T* __restrict__ ln = c.t1 + (int64_t)line * L;
  const uint32_t mb = a.maskL[line * 32 + lane];    // bits (2r, 2r+1): slot a; (16+2r, 17+2r): slot b
  T A[8], B[8], C[8], E[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    int o[4];
    canon(lane, r, o);
    A[r] = ln[o[0]]; B[r] = ln[o[1]]; C[r] = ln[o[2]]; E[r] = ln[o[3]];
  }
  cplx<T> va[8], vb[8];
  pre_all<T>(lane, A, B, C, E, va, vb, tb);
  T* reg = sm + warp * WREG;
  fft512<T, +1>(va, vb, lane, reg, reg + XPL, tb);
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    if (!((mb >> (2 * r)) & 1u)) va[r].x = (T)0;
    if (!((mb >> (2 * r + 1)) & 1u)) va[r].y = (T)0;
    if (!((mb >> (16 + 2 * r)) & 1u)) vb[r].x = (T)0;
    if (!((mb >> (17 + 2 * r)) & 1u)) vb[r].y = (T)0;
  }
  fft512<T, -1>(va, vb, lane, reg, reg + XPL, tb);
  post_all<T>(lane, va, vb, A, B, C, E, tb);
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    int o[4];
    canon(lane, r, o);
    ln[o[0]] = A[r]; ln[o[1]] = B[r]; ln[o[2]] = C[r]; ln[o[3]] = E[r];
  }
}

// ---------------------------------------------------------------- pass C
template <typename T>
__global__ void __launch_bounds__(Geo<T>::RT * 32) k1k_rows_fwd(DctArgs a, int j0) {
  constexpr int RT = Geo<T>::RT;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int j = j0 + blockIdx.y;
  if (a.cs[j].frozen) return;
  T* sm = reinterpret_cast<T*>(smraw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = blockIdx.x * RT;
  const DctCol<T> c = col_of<T>(a, j);
  {
    const T* __restrict__ tin = c.t1;
    T v[L / (RT * 32)][RT];
#pragma unroll
    for (int it = 0; it < L / (RT * 32); ++it)
      ld32B<T, RT>(tin + (int64_t)(it * RT * 32 + threadIdx.x) * L + row0, v[it]);
#pragma unroll
    for (int it = 0; it < L / (RT * 32); ++it)
#pragma unroll
      for (int i = 0; i < RT; ++i) sm[i * WREG + it * RT * 32 + threadIdx.x] = v[it][i];
  }
  const Tw<T> tb = load_tables<T>(tab1k<T>(a), reinterpret_cast<cplx<T>*>(sm + RT * WREG));   // + barrier
  T* reg = sm + warp * WREG;
  const int ja = lane, jb = lane ? 64 - lane : 32;
  cplx<T> va[8], vb[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    va[r] = *reinterpret_cast<const cplx<T>*>(reg + 2 * (ja + 64 * r));
    vb[r] = *reinterpret_cast<const cplx<T>*>(reg + 2 * (jb + 64 * r));
  }
  fft512<T, -1>(va, vb, lane, reg, reg + XPL, tb);
  T A[8], B[8], C[8], E[8];
  post_all<T>(lane, va, vb, A, B, C, E, tb);
  const int64_t rb = (int64_t)(row0 + warp) * L;
  const T* __restrict__ pp = c.p + rb;
  const T* __restrict__ al = alpha_of<T>(a, j) + rb;
  T* __restrict__ qq = c.q + rb;
  const T beta = (T)a.beta;
  double g = 0.0;
#pragma unroll
  for (int r = 0; r < 8; ++r) {     // a3: q = beta Phi^T Phi p + alpha o p  (loads first)
    int o[4];
    canon(lane, r, o);
    const T p0 = pp[o[0]], p1 = pp[o[1]], p2 = pp[o[2]], p3 = pp[o[3]];
    A[r] = beta * A[r] + al[o[0]] * p0;
    B[r] = beta * B[r] + al[o[1]] * p1;
    C[r] = beta * C[r] + al[o[2]] * p2;
    E[r] = beta * E[r] + al[o[3]] * p3;
    g += (double)p0 * (double)A[r] + (double)p1 * (double)B[r] + (double)p2 * (double)C[r] +
         (double)p3 * (double)E[r];      // a4: gamma partial
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    int o[4];
    canon(lane, r, o);
    qq[o[0]] = A[r]; qq[o[1]] = B[r]; qq[o[2]] = C[r]; qq[o[3]] = E[r];
  }
  g = block_sum(g);
  ColState* cs = a.cs;
  const int iter = a.iter;
  column_finish(g, j, a.part, a.stride, a.counters, [cs, j, iter](double tot) {
    ColState cc = cs[j]; finish_gamma(cc, tot, iter); cs[j] = cc;
  });
}

// ---------------------------------------------------------------- setup: lane-packed mask
// maskL[cv][lane] bit 2r / 2r+1 = mask at v-order rows 2n, 2n+1, n = ja + 64 r; bits 16+2r, 17+2r
// likewise for n = jb + 64 r.  maskT is the v-order mask transposed, [cols][rows].
__global__ void k1k_mask_lanes(const uint8_t* __restrict__ maskT, uint32_t* __restrict__ maskL) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= L * 32) return;
  const int line = idx >> 5, lane = idx & 31;
  const int ja = lane, jb = lane ? 64 - lane : 32;
  const uint8_t* m = maskT + (int64_t)line * L;
  uint32_t w = 0;
  for (int r = 0; r < 8; ++r) {
    const int na = ja + 64 * r, nb = jb + 64 * r;
    w |= (uint32_t)(m[2 * na] != 0) << (2 * r);
    w |= (uint32_t)(m[2 * na + 1] != 0) << (2 * r + 1);
    w |= (uint32_t)(m[2 * nb] != 0) << (16 + 2 * r);
    w |= (uint32_t)(m[2 * nb + 1] != 0) << (17 + 2 * r);
  }
  maskL[idx] = w;
}

template <typename T> static size_t smem_bytes() {
  return (size_t)Geo<T>::RT * WREG * sizeof(T) + (size_t)TTOT * sizeof(cplx<T>);
}

template <typename T> static void set_attrs() {
  const int s = (int)smem_bytes<T>();
  cudaFuncSetAttribute(k1k_rows_inv<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, s);
  cudaFuncSetAttribute(k1k_cols<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, s);
  cudaFuncSetAttribute(k1k_rows_fwd<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, s);
}

}  // namespace d1k

bool dct1k_eligible(const Ctx* c) { return c->kind == COFEM_OP_DCT2_MASKED && c->rows == 1024 && c->cols == 1024; }

template <typename T> static std::vector<cplx<T>> build_tables() {
  using namespace d1k;
  const double PI = 3.14159265358979323846;
  std::vector<cplx<T>> h(TTOT);
  auto e = [&](double ang) { return cplx<T>{(T)cos(ang), (T)sin(ang)}; };
  for (int r = 0; r < 8; ++r)
    for (int k = 0; k < 8; ++k) h[TW2 + r * 8 + k] = e(-2 * PI * r * k / 64.0);
  for (int r = 0; r < 8; ++r)
    for (int jj = 0; jj < 64; ++jj) h[TW3 + r * 64 + jj] = e(-2 * PI * r * jj / 512.0);
  for (int k = 0; k < L; ++k) h[TTQ + k] = e(-PI * k / (2.0 * L));
  for (int k = 0; k < M; ++k) h[TTH + k] = e(-2 * PI * k / L);
  return h;
}

cofem_status dct1k_setup(Ctx* c) {
  using namespace d1k;
  {
    auto h32 = build_tables<float>();
    auto h64 = build_tables<double>();
    if (cudaMalloc(&c->tab1k32, h32.size() * sizeof(h32[0])) != cudaSuccess ||
        cudaMalloc(&c->tab1k64, h64.size() * sizeof(h64[0])) != cudaSuccess) { c->err = "cudaMalloc dct1k tables"; return COFEM_ERR_OOM; }
    cudaMemcpy(c->tab1k32, h32.data(), h32.size() * sizeof(h32[0]), cudaMemcpyHostToDevice);
    cudaMemcpy(c->tab1k64, h64.data(), h64.size() * sizeof(h64[0]), cudaMemcpyHostToDevice);
  }
  if (cudaMalloc(&c->maskL, (size_t)L * 32 * sizeof(uint32_t)) != cudaSuccess) { c->err = "cudaMalloc maskL"; return COFEM_ERR_OOM; }
  launch_begin(c, KC_SETUP);
  k1k_mask_lanes<<<L * 32 / 256, 256, 0, c->stream>>>(c->mask_vvT, c->maskL);
  launch_end(c, KC_SETUP);
  set_attrs<float>();
  set_attrs<double>();
  c->part_stride = std::max(c->part_stride, L / Geo<double>::RT);
  return check_launch(c, "dct1k setup") == cudaSuccess ? COFEM_OK : COFEM_ERR_CUDA;
}

DctArgs dct_args(Ctx* c, int m, int iter);

// Apply to columns [j0, j1) (all of one precision: the mean column alone, or probes) on `st`.
template <typename T>
static cofem_status dct1k_apply_t(Ctx* c, int j0, int j1, int iter, bool dir, cudaStream_t st) {
  using namespace d1k;
  DctArgs a = dct_args(c, j1, iter);
  constexpr int RT = Geo<T>::RT;
  const dim3 g(L / RT, j1 - j0), blk(RT * 32);
  const size_t sm = smem_bytes<T>();
  const bool mean = j0 == 0;        // the fp64 mean column is timed as its own class
  launch_begin(c, mean ? KC_MEAN : KC_DCT_ROWS_INV, st);
  k1k_rows_inv<T><<<g, blk, sm, st>>>(a, j0, dir ? 1 : 0);
  launch_end(c, mean ? KC_MEAN : KC_DCT_ROWS_INV, st);
  launch_begin(c, mean ? KC_MEAN : KC_DCT_COLS, st);
  k1k_cols<T><<<g, blk, sm, st>>>(a, j0);
  launch_end(c, mean ? KC_MEAN : KC_DCT_COLS, st);
  launch_begin(c, mean ? KC_MEAN : KC_DCT_ROWS_FWD, st);
  k1k_rows_fwd<T><<<g, blk, sm, st>>>(a, j0);
  launch_end(c, mean ? KC_MEAN : KC_DCT_ROWS_FWD, st);
  return check_launch(c, "dct1k apply") == cudaSuccess ? COFEM_OK : COFEM_ERR_CUDA;
}

cofem_status dct1k_apply(Ctx* c, int j0, int j1, int iter, bool dir, cudaStream_t st) {
  if (j0 == 0 || c->probe64) return dct1k_apply_t<double>(c, j0, j1, iter, dir, st);
  return dct1k_apply_t<float>(c, j0, j1, iter, dir, st);
}

}  // namespace cofem
