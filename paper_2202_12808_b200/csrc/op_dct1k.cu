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
#include <stdlib.h>

#include <algorithm>
#include <complex>
#include <vector>

#include "fft512.cuh"

namespace cofem {
namespace d1k {

// DCT-III (orthonormal inverse) pre-processing for one k: W[k] = u1 P_k + u2 Q_k.
template <typename T>
__device__ __forceinline__ cplx<T> dct3_pre(int k, T Xk, T XLk, T XkM, T XMk, const Tw<T>& tb) {
  const cplx<T> P = tb.base[TP + k], Q = tb.base[TQ + k];
  // (Xk - i XLk) P + (XkM - i XMk) Q
  return {Xk * P.x + XLk * P.y + XkM * Q.x + XMk * Q.y, Xk * P.y - XLk * P.x + XkM * Q.y - XMk * Q.x};
}

// DCT-II post-processing for one k from W[k], W[(M-k) mod M]: orthonormal X[k], X[k+M].
template <typename T>
__device__ __forceinline__ void dct2_post(int k, cplx<T> Wk, cplx<T> Wm, const Tw<T>& tb, T& lo, T& hi) {
  const cplx<T> R1 = tb.base[TR1 + k], R2 = tb.base[TR2 + k], R3 = tb.base[TR3 + k], R4 = tb.base[TR4 + k];
  lo = Wk.x * R1.x - Wk.y * R1.y + Wm.x * R2.x + Wm.y * R2.y;
  hi = Wk.x * R3.x - Wk.y * R3.y + Wm.x * R4.x + Wm.y * R4.y;
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

// L2 prefetch of one warp's next 4 KB line of an fp32 image (one 128-byte line per lane), issued
// before the current item's work so the next item's loads hit L2 (COFEM_1K_NOPF disables, A/B)
template <typename T> __device__ __forceinline__ void pf_line(const T* line) {
#ifndef COFEM_1K_NOPF
  if constexpr (sizeof(T) == 4)
    asm volatile("prefetch.global.L2 [%0];" ::"l"(line + 32 * (threadIdx.x & 31)));
#endif
}

#ifndef COFEM_1K_PFD
#define COFEM_1K_PFD 1       // prefetch distance in items of the warp
#endif

template <typename T> __device__ __forceinline__ const cplx<T>* tab1k(const DctArgs& a) {
  if constexpr (sizeof(T) == 8) return (const cplx<T>*)a.tab1k64; else return (const cplx<T>*)a.tab1k32;
}

// ---------------------------------------------------------------- pass A
// Shared memory: [RT warps][WREG] (FFT exchange / output tile row) then the twiddle tables.
// Persistent kernels: work item w = (column j0 + w / NTILE, tile w % NTILE), grid-strided.
template <typename T> struct Work { static constexpr int NTILE = L / Geo<T>::RT; };

template <typename T>
__device__ __forceinline__ void rows_inv_item(const DctArgs& a, int j, int tile, int dir, double bcoef, T* sm,
                                              const Tw<T>& tb);

template <typename T>
#ifndef COFEM_1K_INV_MINB
#define COFEM_1K_INV_MINB 1   // explicit: nvcc then takes 96 registers (2 CTAs per SM): 47.7 -> 47.1 ms; 3: 47.6, 4: 48.4
#endif
__global__ void __launch_bounds__(Geo<T>::RT * 32, sizeof(T) == 4 ? COFEM_1K_INV_MINB : 1) k1k_rows_inv(DctArgs a, int j0, int ncols, int dir) {
  constexpr int RT = Geo<T>::RT, NT = Work<T>::NTILE;
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sm = reinterpret_cast<T*>(smraw);
  __shared__ ColFlags ci;
  load_colinfo(ci, a.cs, j0, ncols);
  if (!any_active(ci, ncols)) return;
  if (blockIdx.x < ncols * NT && !ci.frozen[blockIdx.x / NT]) {   // the first item's rows, before the tables
    const DctCol<T> cn = col_of<T>(a, j0 + blockIdx.x / NT);
    const int64_t rn = (int64_t)((blockIdx.x % NT) * RT + (threadIdx.x >> 5)) * L;
    pf_line(cn.p + rn);
    if (dir) pf_line(cn.r + rn);
  }
  // pass A needs the FFT twiddles and the DCT-III pre tables only: the [0, TR1) prefix (12.8 KB in fp32)
  const Tw<T> tb = load_tables<T>(tab1k<T>(a), reinterpret_cast<cplx<T>*>(sm + RT * WREG), TR1);   // + barrier
  for (int w = blockIdx.x; w < ncols * NT; w += gridDim.x) {
    const int jj = w / NT;
    if (ci.frozen[jj]) continue;
    if (w + COFEM_1K_PFD * (int)gridDim.x < ncols * NT) {   // a later item of this warp: p and r rows
      const int wn = w + COFEM_1K_PFD * gridDim.x, jn = wn / NT;
      if (!ci.frozen[jn]) {
        const DctCol<T> cn = col_of<T>(a, j0 + jn);
        const int64_t rn = (int64_t)((wn % NT) * RT + (threadIdx.x >> 5)) * L;
        pf_line(cn.p + rn);
        if (dir) pf_line(cn.r + rn);
#ifdef COFEM_1K_PF_SHARED
        if (dir) pf_line(cn.dinv + rn);
#endif
      }
    }
    rows_inv_item<T>(a, j0 + jj, w % NT, dir, ci.b[jj], sm, tb);
    __syncthreads();                 // smem tile reuse
  }
}

template <typename T>
__device__ __forceinline__ void rows_inv_item(const DctArgs& a, int j, int tile, int dir, double bcoef, T* sm,
                                              const Tw<T>& tb) {
  constexpr int RT = Geo<T>::RT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = tile * RT;
  const DctCol<T> c = col_of<T>(a, j);
  const int64_t rb = (int64_t)(row0 + warp) * L;
  T A[8], B[8], C[8], E[8];
  if constexpr (sizeof(T) == 4) {
    // fp32: the row moves as 16-byte vectors (lane l: elements 4 l + 128 i), the direction
    // update a6 is elementwise there, and the warp's exchange region turns the row into the
    // canonical per-lane positions (8 LDG.128 per array instead of 32 scalar loads)
    float4* __restrict__ pr = reinterpret_cast<float4*>(c.p + rb);
    const float4* __restrict__ rr = reinterpret_cast<const float4*>(c.r + rb);
    const float4* __restrict__ dv = reinterpret_cast<const float4*>(c.dinv + rb);
    float4* r4 = reinterpret_cast<float4*>(sm + warp * WREG);
    const float bb = (float)bcoef;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float4 pv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) pv[i] = pr[lane + 32 * (4 * h + i)];
      if (dir) {
        float4 rv[4], dd[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) { rv[i] = rr[lane + 32 * (4 * h + i)]; dd[i] = dv[lane + 32 * (4 * h + i)]; }
#pragma unroll
        for (int i = 0; i < 4; ++i) {    // a6: p = M^-1 r + b p
          pv[i].x = dd[i].x * rv[i].x + bb * pv[i].x; pv[i].y = dd[i].y * rv[i].y + bb * pv[i].y;
          pv[i].z = dd[i].z * rv[i].z + bb * pv[i].z; pv[i].w = dd[i].w * rv[i].w + bb * pv[i].w;
          pr[lane + 32 * (4 * h + i)] = pv[i];
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) r4[lane + 32 * (4 * h + i)] = pv[i];
    }
    __syncwarp();
    const T* reg = sm + warp * WREG;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      int o[4];
      canon(lane, r, o);
      A[r] = reg[o[0]]; B[r] = reg[o[1]]; C[r] = reg[o[2]]; E[r] = reg[o[3]];
    }
    __syncwarp();                    // fft512 reuses the region
  } else {
    T* __restrict__ pr = c.p + rb;
    const T* __restrict__ rr = c.r + rb;
    const T* __restrict__ dv = c.dinv + rb;
    const T bb = (T)bcoef;
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
  fft512<T, +1>(va, vb, lane, reinterpret_cast<cplx<T>*>(reg), tb);
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
__device__ __forceinline__ void cols_item(const DctArgs& a, int j, int tile, T* sm, const Tw<T>& tb);

template <typename T>
__global__ void __launch_bounds__(Geo<T>::RT * 32) k1k_cols(DctArgs a, int j0, int ncols) {
  constexpr int RT = Geo<T>::RT, NT = Work<T>::NTILE;
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sm = reinterpret_cast<T*>(smraw);
  __shared__ ColFlags ci;
  load_colinfo(ci, a.cs, j0, ncols);
  if (!any_active(ci, ncols)) return;
  if (blockIdx.x < ncols * NT && !ci.frozen[blockIdx.x / NT])     // the first item's line, before the tables
    pf_line(col_of<T>(a, j0 + blockIdx.x / NT).t1 + (int64_t)((blockIdx.x % NT) * RT + (threadIdx.x >> 5)) * L);
  const Tw<T> tb = load_tables<T>(tab1k<T>(a), reinterpret_cast<cplx<T>*>(sm + RT * WREG));   // + barrier
  for (int w = blockIdx.x; w < ncols * NT; w += gridDim.x) {
    const int jj = w / NT;
    if (ci.frozen[jj]) continue;
    if (w + COFEM_1K_PFD * (int)gridDim.x < ncols * NT) {   // a later item of this warp: its T^T line
      const int wn = w + COFEM_1K_PFD * gridDim.x, jn = wn / NT;
      if (!ci.frozen[jn]) pf_line(col_of<T>(a, j0 + jn).t1 + (int64_t)((wn % NT) * RT + (threadIdx.x >> 5)) * L);
    }
    cols_item<T>(a, j0 + jj, w % NT, sm, tb);
  }
}

template <typename T>
__device__ __forceinline__ void cols_item(const DctArgs& a, int j, int tile, T* sm, const Tw<T>& tb) {
  constexpr int RT = Geo<T>::RT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int line = tile * RT + warp;                // v-order image column cv
  const DctCol<T> c = col_of<T>(a, j);
  const T* __restrict__ ln = c.t1 + (int64_t)line * L;
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
  fft512<T, +1>(va, vb, lane, reinterpret_cast<cplx<T>*>(reg), tb);
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    if (!((mb >> (2 * r)) & 1u)) va[r].x = (T)0;
    if (!((mb >> (2 * r + 1)) & 1u)) va[r].y = (T)0;
    if (!((mb >> (16 + 2 * r)) & 1u)) vb[r].x = (T)0;
    if (!((mb >> (17 + 2 * r)) & 1u)) vb[r].y = (T)0;
  }
  fft512<T, -1>(va, vb, lane, reinterpret_cast<cplx<T>*>(reg), tb);
  post_all<T>(lane, va, vb, A, B, C, E, tb);
#pragma unroll
  for (int r = 0; r < 8; ++r) {     // natural-order column values -> tile row (the exchange region is free)
    int o[4];
    canon(lane, r, o);
    reg[o[0]] = A[r]; reg[o[1]] = B[r]; reg[o[2]] = C[r]; reg[o[3]] = E[r];
  }
  __syncthreads();
  T* __restrict__ out = c.t2;       // T2[row][cv] row-major: 32-byte segments of RT v-order columns
#pragma unroll
  for (int it = 0; it < L / (RT * 32); ++it) {
    const int row = it * RT * 32 + threadIdx.x;
    T v[RT];
#pragma unroll
    for (int i = 0; i < RT; ++i) v[i] = sm[i * WREG + row];
    st32B<T, RT>(out + (int64_t)row * L + tile * RT, v);
  }
  __syncthreads();
}

// ---------------------------------------------------------------- pass C
template <typename T>
__device__ __forceinline__ double rows_fwd_item(const DctArgs& a, int j, int tile, T* sm, const Tw<T>& tb);

template <typename T>
__global__ void __launch_bounds__(Geo<T>::RT * 32) k1k_rows_fwd(DctArgs a, int j0, int ncols) {
  constexpr int RT = Geo<T>::RT, NT = Work<T>::NTILE;
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sm = reinterpret_cast<T*>(smraw);
  __shared__ ColFlags ci;
  load_colinfo(ci, a.cs, j0, ncols);
  if (!any_active(ci, ncols)) return;
  if (blockIdx.x < ncols * NT && !ci.frozen[blockIdx.x / NT]) {   // the first item's rows, before the tables
    const DctCol<T> cn = col_of<T>(a, j0 + blockIdx.x / NT);
    const int64_t rn = (int64_t)((blockIdx.x % NT) * RT + (threadIdx.x >> 5)) * L;
    pf_line(cn.t2 + rn); pf_line(cn.p + rn);
  }
  const Tw<T> tb = load_tables<T>(tab1k<T>(a), reinterpret_cast<cplx<T>*>(sm + RT * WREG));   // + barrier
  const int warp = threadIdx.x >> 5;
  for (int w = blockIdx.x; w < ncols * NT; w += gridDim.x) {
    const int jj = w / NT;
    if (ci.frozen[jj]) continue;
    if (w + COFEM_1K_PFD * (int)gridDim.x < ncols * NT) {   // a later item of this warp: T2 and p rows
      const int wn = w + COFEM_1K_PFD * gridDim.x, jn = wn / NT;
      if (!ci.frozen[jn]) {
        const DctCol<T> cn = col_of<T>(a, j0 + jn);
        const int64_t rn = (int64_t)((wn % NT) * RT + (threadIdx.x >> 5)) * L;
        pf_line(cn.t2 + rn);
        pf_line(cn.p + rn);
#ifdef COFEM_1K_PF_SHARED
        pf_line(alpha_of<T>(a, j0 + jn) + rn);
#endif
      }
    }
    const double gw = rows_fwd_item<T>(a, j0 + jj, w % NT, sm, tb);   // warp-reduced, valid in lane 0
    // a4 partial of image row (tile RT + warp): part[j][row].  One slot per row, whatever the grid,
    // so gamma (and mu, s) do not depend on the launch size, K, max_probes or the probe groups
    if ((threadIdx.x & 31) == 0) a.part[(int64_t)(j0 + jj) * a.stride + (w % NT) * RT + warp] = gw;
  }
  // a4: gamma_j = p_j^T q_j.  The last CTA reduces the L row partials of every column in fixed
  // order and applies the freeze rule / step length (R5).
  __threadfence();
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int jj = warp; jj < ncols; jj += RT) {
    const int j = j0 + jj;
    const double tot = reduce_partials(a.part + (int64_t)j * a.stride, L);
    if ((threadIdx.x & 31) == 0 && !ci.frozen[jj]) {
      ColState cc = a.cs[j]; finish_gamma(cc, tot, a.iter); a.cs[j] = cc;
    }
  }
  if (threadIdx.x == 0) *a.ticket = 0u;
}

template <typename T>
__device__ __forceinline__ double rows_fwd_item(const DctArgs& a, int j, int tile, T* sm, const Tw<T>& tb) {
  constexpr int RT = Geo<T>::RT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = tile * RT;
  const DctCol<T> c = col_of<T>(a, j);
  const int64_t rb = (int64_t)(row0 + warp) * L;
  T* reg = sm + warp * WREG;
  const int ja = lane, jb = lane ? 64 - lane : 32;
  cplx<T> va[8], vb[8];
  {
    const cplx<T>* __restrict__ rowc = reinterpret_cast<const cplx<T>*>(c.t2 + rb);   // packed v-order z[n]
#pragma unroll
    for (int r = 0; r < 8; ++r) { va[r] = rowc[ja + 64 * r]; vb[r] = rowc[jb + 64 * r]; }
  }
  fft512<T, -1>(va, vb, lane, reinterpret_cast<cplx<T>*>(reg), tb);
  T A[8], B[8], C[8], E[8];
  post_all<T>(lane, va, vb, A, B, C, E, tb);
  double g = 0.0;
  if constexpr (sizeof(T) == 4) {
    // fp32: canonical values -> the warp's exchange region -> 16-byte vectors (lane l: elements
    // 4 l + 128 i), so p, alpha and q move as LDG/STG.128
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      int o[4];
      canon(lane, r, o);
      reg[o[0]] = A[r]; reg[o[1]] = B[r]; reg[o[2]] = C[r]; reg[o[3]] = E[r];
    }
    __syncwarp();
    const float4* r4 = reinterpret_cast<const float4*>(reg);
    const float4* __restrict__ pp = reinterpret_cast<const float4*>(c.p + rb);
    const float4* __restrict__ al = reinterpret_cast<const float4*>(alpha_of<T>(a, j) + rb);
    float4* __restrict__ qq = reinterpret_cast<float4*>(c.q + rb);
    const float beta = (float)a.beta;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float4 pv[4], av[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { pv[i] = pp[lane + 32 * (4 * h + i)]; av[i] = al[lane + 32 * (4 * h + i)]; }
#pragma unroll
      for (int i = 0; i < 4; ++i) {   // a3: q = beta Phi^T Phi p + alpha o p; a4: gamma partial
        const float4 x = r4[lane + 32 * (4 * h + i)];
        float4 q;
        q.x = beta * x.x + av[i].x * pv[i].x; q.y = beta * x.y + av[i].y * pv[i].y;
        q.z = beta * x.z + av[i].z * pv[i].z; q.w = beta * x.w + av[i].w * pv[i].w;
        g += (double)pv[i].x * (double)q.x + (double)pv[i].y * (double)q.y + (double)pv[i].z * (double)q.z +
             (double)pv[i].w * (double)q.w;
        qq[lane + 32 * (4 * h + i)] = q;
      }
    }
    __syncwarp();                    // the next item's FFT reuses the region
    return warp_sum(g);
  }
  const T* __restrict__ pp = c.p + rb;
  const T* __restrict__ al = alpha_of<T>(a, j) + rb;
  T* __restrict__ qq = c.q + rb;
  const T beta = (T)a.beta;
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
  return warp_sum(g);
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

template <typename T> static size_t smem_bytes(int ntab = TTOT) {
  return (size_t)Geo<T>::RT * WREG * sizeof(T) + (size_t)ntab * sizeof(cplx<T>);
}

template <typename T> static void set_attrs() {
  const int s = (int)smem_bytes<T>();
  cudaFuncSetAttribute(k1k_rows_inv<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<T>(TR1));
  cudaFuncSetAttribute(k1k_cols<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, s);
  cudaFuncSetAttribute(k1k_rows_fwd<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, s);
}

}  // namespace d1k

bool dct1k_eligible(const Ctx* c) { return c->kind == COFEM_OP_DCT2_MASKED && c->rows == 1024 && c->cols == 1024; }

// Derivation (Makhoul, orthonormal): with q1 = e^{-i pi k/2L}, q2 = e^{-i pi (k+M)/2L},
// h = e^{-2 pi i k/L}, the DCT-III spectrum is W = [V1 + V2]/2 + i conj(h) [V1 - V2]/2 with
// V1 = sc_k u1 conj(q1), V2 = sc u2 conj(q2), so P = sc_k conj(q1)(1 + i conj h)/2,
// Q = sc conj(q2)(1 - i conj h)/2 (sc = sqrt(L/2)/M, sc_0 = sqrt(L)/M).  The DCT-II outputs
// X[k] = s_k Re(q1 V1'), X[k+M] = s Re(q2 V2'), V1' = W_k (1 - i h)/2 + conj(W_m)(1 + i h)/2,
// V2' = W_k (1 + i h)/2 + conj(W_m)(1 - i h)/2, so R1 = s_k q1 (1 - i h)/2, R2 = s_k q1 (1 + i h)/2,
// R3 = s q2 (1 + i h)/2, R4 = s q2 (1 - i h)/2 (s = sqrt(2/L), s_0 = sqrt(1/L)); the device
// evaluates Re(conj(w) b) as w.x b.x + w.y b.y.
template <typename T> static std::vector<cplx<T>> build_tables() {
  using namespace d1k;
  typedef std::complex<double> C;
  const double PI = 3.14159265358979323846;
  std::vector<cplx<T>> h(TTOT);
  auto put = [&](int i, C z) { h[i] = cplx<T>{(T)z.real(), (T)z.imag()}; };
  auto e = [](double ang) { return C(cos(ang), sin(ang)); };
  for (int r = 0; r < 8; ++r)
    for (int k = 0; k < 8; ++k) put(TW2 + r * 8 + k, e(-2 * PI * r * k / 64.0));
  for (int r = 0; r < 8; ++r)
    for (int jj = 0; jj < 64; ++jj) put(TW3 + r * 64 + jj, e(-2 * PI * r * jj / 512.0));
  const C I(0, 1);
  const double sc = sqrt(L / 2.0) / M, sc0 = sqrt((double)L) / M, s = sqrt(2.0 / L), s0 = sqrt(1.0 / L);
  for (int k = 0; k < M; ++k) {
    const C q1 = e(-PI * k / (2.0 * L)), q2 = e(-PI * (k + M) / (2.0 * L)), hh = e(-2 * PI * k / L);
    const double sck = k == 0 ? sc0 : sc, sk = k == 0 ? s0 : s;
    put(TP + k, sck * std::conj(q1) * (1.0 + I * std::conj(hh)) / 2.0);
    put(TQ + k, sc * std::conj(q2) * (1.0 - I * std::conj(hh)) / 2.0);
    const C r1 = sk * q1 * (1.0 - I * hh) / 2.0, r2 = sk * q1 * (1.0 + I * hh) / 2.0;
    const C r3 = s * q2 * (1.0 + I * hh) / 2.0, r4 = s * q2 * (1.0 - I * hh) / 2.0;
    // lo = Re(Wk r1) + Re(conj(Wm) r2) = Wk.x r1.x - Wk.y r1.y + Wm.x r2.x + Wm.y r2.y
    put(TR1 + k, r1); put(TR2 + k, r2); put(TR3 + k, r3); put(TR4 + k, r4);
  }
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
  c->part_stride = std::max(c->part_stride, std::max(L, c->num_sms * 8));   // >= L row partials (pass C), grids
  return check_launch(c, "dct1k setup") == cudaSuccess ? COFEM_OK : COFEM_ERR_CUDA;
}

DctArgs dct_args(Ctx* c, int m, int iter);

// Apply to columns [j0, j1) (all of one precision: the mean column alone, or probes) on `st`.
template <typename T>
static cofem_status dct1k_apply_t(Ctx* c, int j0, int j1, int iter, bool dir, cudaStream_t st) {
  using namespace d1k;
  DctArgs a = dct_args(c, j1, iter);
  a.ticket = j0 == 0 ? c->counters + MAXM + 3 : j0 == 1 ? c->counters + MAXM + 2 : c->counters + 2 * MAXM + j0;
  constexpr int RT = Geo<T>::RT;
  const int ncols = j1 - j0;
  const size_t sm = smem_bytes<T>();
  // persistent grids at full occupancy (measured best: tools/sweep_slots.sh)
#ifndef COFEM_1K_SLOTS
#define COFEM_1K_SLOTS -1   // tuning build switch: CTAs per SM of the persistent grids (-1 = occupancy, 0 = one per item)
#endif
  constexpr int slots_env = COFEM_1K_SLOTS;
  // the concurrent fp64 mean column is confined to a fraction of the SMs (COFEM_1K_MEAN_SMS),
  // shrinking as the probe work grows (tools/time_estep.py, C4 at a fixed alpha, with the
  // concurrent probe groups): an eighth at >= 32 probes (57.3 vs 57.5 ms for a quarter), a
  // quarter at >= 16 (33.1 vs 33.3 for an eighth), half below (21.1 vs 24.0 at 8 probes)
#ifndef COFEM_1K_MEAN_SMS
#define COFEM_1K_MEAN_SMS -1   // tuning build switch: SMs of the mean column (-1 = the rule above)
#endif
  constexpr int mean_sms_env = COFEM_1K_MEAN_SMS;
  auto grid_of = [&](const void* fn, size_t smb) {
    const int items = ncols * Work<T>::NTILE;
    if (slots_env == 0) return items;                  // one CTA per work item
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, RT * 32, smb);
    const int per_sm = slots_env > 0 ? std::min(slots_env, occ) : occ;
    int g = std::min(std::min(c->num_sms * per_sm, items), c->part_stride);
    if (j0 == 0 && c->fast1k) {
      const int msms = mean_sms_env > 0 ? mean_sms_env
                                        : std::max(1, c->num_sms / (c->Kcap >= 32 ? 8 : c->Kcap >= 16 ? 4 : 2));
      if (mean_sms_env != 0) g = std::min(g, msms * per_sm);
    }
    // with concurrent probe groups each probe launch takes ~80 % of the SMs (C4: 120 of 148 best,
    // 16.70 vs 16.51 EM it/s uncapped; tools/time_estep.py sweep 74..148)
#ifndef COFEM_1K_GROUP_SMS
#define COFEM_1K_GROUP_SMS -1   // tuning build switch: SMs of each probe-group launch (-1 = 120/148)
#endif
    constexpr int group_sms_env = COFEM_1K_GROUP_SMS;
    const int gsms = group_sms_env >= 0 ? group_sms_env : (c->probe_groups > 1 ? (c->num_sms * 120) / 148 : 0);
    if (j0 > 0 && gsms > 0) g = std::min(g, gsms * per_sm);
    return g;
  };
  const dim3 blk(RT * 32);
  const bool mean = j0 == 0;        // the fp64 mean column is timed as its own class
  launch_begin(c, mean ? KC_MEAN : KC_DCT_ROWS_INV, st);
  k1k_rows_inv<T><<<grid_of((const void*)k1k_rows_inv<T>, smem_bytes<T>(TR1)), blk, smem_bytes<T>(TR1), st>>>(
      a, j0, ncols, dir ? 1 : 0);
  launch_end(c, mean ? KC_MEAN : KC_DCT_ROWS_INV, st);
  launch_begin(c, mean ? KC_MEAN : KC_DCT_COLS, st);
  k1k_cols<T><<<grid_of((const void*)k1k_cols<T>, sm), blk, sm, st>>>(a, j0, ncols);
  launch_end(c, mean ? KC_MEAN : KC_DCT_COLS, st);
  launch_begin(c, mean ? KC_MEAN : KC_DCT_ROWS_FWD, st);
  k1k_rows_fwd<T><<<grid_of((const void*)k1k_rows_fwd<T>, sm), blk, sm, st>>>(a, j0, ncols);
  launch_end(c, mean ? KC_MEAN : KC_DCT_ROWS_FWD, st);
  return check_launch(c, "dct1k apply") == cudaSuccess ? COFEM_OK : COFEM_ERR_CUDA;
}

cofem_status dct1k_apply(Ctx* c, int j0, int j1, int iter, bool dir, cudaStream_t st) {
  if (j0 == 0 || c->probe64) return dct1k_apply_t<double>(c, j0, j1, iter, dir, st);
  return dct1k_apply_t<float>(c, j0, j1, iter, dir, st);
}

}  // namespace cofem
