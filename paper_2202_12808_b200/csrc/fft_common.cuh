// fft_common.cuh — complex arithmetic, radix-2/4/8 DFT kernels and DCT twiddle
// tables shared by the DCT kernels (op_dct.cu generic path, op_dct1k.cu 1024 fast path).
// Product code (sm_100a); nothing here is shared with oracle/.
#pragma once
#include "internal.cuh"

namespace cofem {

// ---------------------------------------------------------------- complex helpers
template <typename T> __device__ __forceinline__ cplx<T> cadd(cplx<T> a, cplx<T> b) { return {a.x + b.x, a.y + b.y}; }
template <typename T> __device__ __forceinline__ cplx<T> csub(cplx<T> a, cplx<T> b) { return {a.x - b.x, a.y - b.y}; }
template <typename T> __device__ __forceinline__ cplx<T> cmul(cplx<T> a, cplx<T> b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
template <typename T> __device__ __forceinline__ cplx<T> cmulc(cplx<T> a, cplx<T> b) {   // a * conj(b)
  return {a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y};
}
// multiply by SIGN * i
template <int SIGN, typename T> __device__ __forceinline__ cplx<T> mul_si(cplx<T> a) {
  return SIGN > 0 ? cplx<T>{-a.y, a.x} : cplx<T>{a.y, -a.x};
}

template <int SIGN, typename T> __device__ __forceinline__ void dft2(cplx<T>* v) {
  cplx<T> a = v[0], b = v[1];
  v[0] = cadd(a, b); v[1] = csub(a, b);
}
template <int SIGN, typename T> __device__ __forceinline__ void dft4(cplx<T>* v) {
  cplx<T> s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
  cplx<T> s13 = cadd(v[1], v[3]), d13 = mul_si<SIGN>(csub(v[1], v[3]));
  v[0] = cadd(s02, s13); v[2] = csub(s02, s13);
  v[1] = cadd(d02, d13); v[3] = csub(d02, d13);
}
// X_k = E_k + W^k O_k, X_{k+4} = E_k - W^k O_k, W = exp(SIGN 2 pi i / 8)
template <int SIGN, typename T> __device__ __forceinline__ void dft8(cplx<T>* v) {
  cplx<T> e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
  dft4<SIGN>(e); dft4<SIGN>(o);
  const T h = (T)0.70710678118654752440;
  cplx<T> w1 = {h, (T)SIGN * h}, w3 = {-h, (T)SIGN * h};
  cplx<T> t0 = o[0], t1 = cmul(o[1], w1), t2 = mul_si<SIGN>(o[2]), t3 = cmul(o[3], w3);
  v[0] = cadd(e[0], t0); v[4] = csub(e[0], t0);
  v[1] = cadd(e[1], t1); v[5] = csub(e[1], t1);
  v[2] = cadd(e[2], t2); v[6] = csub(e[2], t2);
  v[3] = cadd(e[3], t3); v[7] = csub(e[3], t3);
}
template <int R, int SIGN, typename T> __device__ __forceinline__ void dftR(cplx<T>* v) {
  if constexpr (R == 8) dft8<SIGN>(v);
  else if constexpr (R == 4) dft4<SIGN>(v);
  else dft2<SIGN>(v);
}

// Twiddle tables for one transform length L (M = L/2):
//   tw[k] = exp(-2 pi i k / M)     (k < M)   FFT
//   tq[k] = exp(-i pi k / (2L))    (k < L)   DCT post/pre twiddle
//   th[k] = exp(-2 pi i k / L)     (k < M)   even/odd split of the packed real FFT
template <typename T> struct DctTab { const cplx<T>* tw; const cplx<T>* tq; const cplx<T>* th; };

template <typename T> struct DctCol {   // one column's arrays (all Dp-strided images)
  T* p; const T* r; const T* dinv; T* t1; T* t2; T* q;
};

struct DctArgs {
  int rows, cols; int64_t Dp; int K;
  double beta; const double* alpha;
  // mean column (fp64)
  double *p0; const double* r0; const double* dinv64; double* t1d; double* t2d; double* q0;
  // probe block
  void* P; const void* R; const void* dinvp; void* t1; void* t2; void* Q;
  const uint8_t* maskT;      // v-order mask, [cols][rows]
  const uint32_t* maskL;     // 1024 fast path: lane-packed v-order mask [cols][32] (op_dct1k.cu)
  const void* alphap;        // alpha in probe precision (probe columns)
  const void* tab1k32; const void* tab1k64;   // 1024 fast path twiddle tables (op_dct1k.cu)
  DctTab<float> tr32, tc32;  // rows-length / cols-length tables
  DctTab<double> tr64, tc64;
  ColState* cs; double* part; int stride; unsigned* counters; int iter;
  unsigned* ticket;   // this launch's last-CTA ticket (distinct per concurrently running column group)
};

template <typename T> __device__ __forceinline__ DctCol<T> col_of(const DctArgs& a, int j) {
  if constexpr (sizeof(T) == 8) {
    if (j == 0) return {a.p0, a.r0, a.dinv64, a.t1d, a.t2d, a.q0};
  }
  const int64_t o = (int64_t)(j - 1) * a.Dp;
  return {(T*)a.P + o, (const T*)a.R + o, (const T*)a.dinvp, (T*)a.t1 + o, (T*)a.t2 + o, (T*)a.Q + o};
}
template <typename T> __device__ __forceinline__ DctTab<T> tab_r(const DctArgs& a);
template <> __device__ __forceinline__ DctTab<float> tab_r<float>(const DctArgs& a) { return a.tr32; }
template <> __device__ __forceinline__ DctTab<double> tab_r<double>(const DctArgs& a) { return a.tr64; }
template <typename T> __device__ __forceinline__ DctTab<T> tab_c(const DctArgs& a);
template <> __device__ __forceinline__ DctTab<float> tab_c<float>(const DctArgs& a) { return a.tc32; }
template <> __device__ __forceinline__ DctTab<double> tab_c<double>(const DctArgs& a) { return a.tc64; }

}  // namespace cofem
