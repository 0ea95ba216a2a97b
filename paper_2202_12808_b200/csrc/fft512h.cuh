// fft512h.cuh — half-warp 512-point complex FFT pair for the 1024 x 1024 DCT column pass
// (op_dct1k.cu k1k_cols_h).  Product code, sm_100a.
//
// Sixteen lanes own one line (32 complex points per lane, two lines per warp) and the FFT is
// radix-16 x 32 with ONE shared-memory exchange (the one-warp fft512.cuh is radix-8^3 with two):
//   k = k1 + 32 k2 (k1 < 32, k2 < 16),  n = t + 16 m (t < 16, m < 32),
//   W_512^{nk} = W_512^{t k1} W_16^{t k2} W_32^{m k1}.
// k-layout: lane u holds k1 in {ka, kb} = {u, 32 - u} (lane 0: {0, 16}) for every k2, so the DCT's
// k <-> 512 - k pairing stays in the lane (as the one-warp FFT's {l, 64 - l} ownership does).
// n-layout: lane t holds n = t + 16 m for every m.
//   inverse (k -> n): DFT-16 over k2 (in registers), twiddle W^{+t k1}, exchange, DFT-32 over k1
//   forward (n -> k): DFT-32 over m (in registers), twiddle W^{-t k1}, exchange, DFT-16 over t
// The inverse's n-layout output is the forward's input, so the mask between them (the column
// pass) stays in registers: one exchange per transform, two per line instead of four.
#pragma once
#include "fft_common.cuh"

namespace cofem {
namespace d1kh {

constexpr int M = 512, L = 1024;
constexpr int XS = 17;                   // exchange row stride (complex entries, odd: conflict-free)
constexpr int XREG = 32 * XS;            // complex entries of one half-warp's exchange region

// in-register DFT of size R1 R2 (natural order in and out): n = n1 + R1 n2, k = k2 + R2 k1;
// step 1: DFT-R2 over n2 for each n1; twiddle W_N^{n1 k2}; step 2: DFT-R1 over n1 for each k2
template <int SIGN, typename T>
__device__ __forceinline__ void dft16(cplx<T> (&v)[16]) {
  cplx<T> y[16];
#pragma unroll
  for (int n1 = 0; n1 < 4; ++n1) {
    cplx<T> s[4] = {v[n1], v[n1 + 4], v[n1 + 8], v[n1 + 12]};
    dft4<SIGN>(s);
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) y[n1 * 4 + k2] = s[k2];
  }
#pragma unroll
  for (int n1 = 1; n1 < 4; ++n1)
#pragma unroll
    for (int k2 = 1; k2 < 4; ++k2) {
      const double ang = SIGN * 2.0 * 3.14159265358979323846 * (n1 * k2) / 16.0;
      y[n1 * 4 + k2] = cmul(y[n1 * 4 + k2], cplx<T>{(T)cos(ang), (T)sin(ang)});
    }
#pragma unroll
  for (int k2 = 0; k2 < 4; ++k2) {
    cplx<T> s[4] = {y[k2], y[4 + k2], y[8 + k2], y[12 + k2]};
    dft4<SIGN>(s);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) v[k2 + 4 * k1] = s[k1];
  }
}

template <int SIGN, typename T>
__device__ __forceinline__ void dft32(cplx<T> (&v)[32]) {
  cplx<T> y[32];
#pragma unroll
  for (int n1 = 0; n1 < 4; ++n1) {            // R1 = 4, R2 = 8
    cplx<T> s[8];
#pragma unroll
    for (int n2 = 0; n2 < 8; ++n2) s[n2] = v[n1 + 4 * n2];
    dft8<SIGN>(s);
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) y[n1 * 8 + k2] = s[k2];
  }
#pragma unroll
  for (int n1 = 1; n1 < 4; ++n1)
#pragma unroll
    for (int k2 = 1; k2 < 8; ++k2) {
      const double ang = SIGN * 2.0 * 3.14159265358979323846 * (n1 * k2) / 32.0;
      y[n1 * 8 + k2] = cmul(y[n1 * 8 + k2], cplx<T>{(T)cos(ang), (T)sin(ang)});
    }
#pragma unroll
  for (int k2 = 0; k2 < 8; ++k2) {
    cplx<T> s[4] = {y[k2], y[8 + k2], y[16 + k2], y[24 + k2]};
    dft4<SIGN>(s);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) v[k2 + 8 * k1] = s[k1];
  }
}

// twiddle tables (device, staged in shared memory by the kernel):
//   wk[k1 * 16 + t] = W_512^{t k1}  (for the n-layout lanes: fixed k1, lanes t consecutive)
//   wt[t * 32 + k1] = W_512^{t k1}  (for the k-layout lanes: fixed t, lanes k1 consecutive)
constexpr int TWK = 0, TWT = 512, TWTOT = 1024;

__device__ __forceinline__ int kb_of(int u) { return u ? 32 - u : 16; }

// inverse FFT (SIGN +1, unnormalised): va[k2] = W[ka + 32 k2], vb[k2] = W[kb + 32 k2] in the k-layout
// -> v[m] = y[t + 16 m] in the n-layout.  x: this half-warp's exchange region (XREG entries).
template <typename T>
__device__ __forceinline__ void ifft_k2n(cplx<T> (&va)[16], cplx<T> (&vb)[16], cplx<T> (&v)[32], int t,
                                         cplx<T>* __restrict__ x, const cplx<T>* __restrict__ tw) {
  const int ka = t, kb = kb_of(t);
  dft16<+1>(va); dft16<+1>(vb);                       // Z[k1][t'] = sum_k2 W[k1 + 32 k2] W_16^{t' k2}
  __syncwarp();
#pragma unroll
  for (int tp = 0; tp < 16; ++tp) {                    // twiddle W^{+t' k1} (conj of the table), exchange [k1][t']
    const cplx<T> wa = tw[TWT + tp * 32 + ka], wb = tw[TWT + tp * 32 + kb];
    x[ka * XS + tp] = cmulc(va[tp], wa);
    x[kb * XS + tp] = cmulc(vb[tp], wb);
  }
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < 32; ++k1) v[k1] = x[k1 * XS + t];
  dft32<+1>(v);                                        // y[t + 16 m] = sum_k1 Z'[k1][t] W_32^{m k1}
  __syncwarp();
}

// forward FFT (SIGN -1): v[m] = y[t + 16 m] (n-layout) -> va[k2] = X[ka + 32 k2], vb[k2] = X[kb + 32 k2]
template <typename T>
__device__ __forceinline__ void fft_n2k(cplx<T> (&v)[32], cplx<T> (&va)[16], cplx<T> (&vb)[16], int t,
                                        cplx<T>* __restrict__ x, const cplx<T>* __restrict__ tw) {
  const int ka = t, kb = kb_of(t);
  dft32<-1>(v);                                        // A[t][k1] = sum_m y[t + 16 m] W_32^{-m k1}
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < 32; ++k1) x[k1 * XS + t] = cmul(v[k1], tw[TWK + k1 * 16 + t]);   // x W^{-t k1}
  __syncwarp();
#pragma unroll
  for (int tp = 0; tp < 16; ++tp) { va[tp] = x[ka * XS + tp]; vb[tp] = x[kb * XS + tp]; }
  dft16<-1>(va); dft16<-1>(vb);                        // X[k1 + 32 k2] = sum_t' A'[t'][k1] W_16^{-t' k2}
  __syncwarp();
}

}  // namespace d1kh
}  // namespace cofem
