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
#include "fft512h.cuh"

namespace cofem {
namespace d1k {

#ifdef COFEM_1K_TAB6
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
#else
// With Ahat = sc q1 (1 - i h)/2 and Bhat = sc q2 (1 + i h)/2 (build_tables), the six round-1 tables
// are P = conj(Ahat) (x sqrt 2 at k = 0), Q = conj(Bhat), R1 = Ahat, R2 = e^{i pi/4} Bhat, R3 = Bhat,
// R4 = e^{-i pi/4} Ahat (x 1/sqrt 2 on R1, R2 at k = 0), since q2 = e^{-i pi/4} q1 and s / sc = 2M/L = 1:
// two shared-memory loads per k instead of six; the k = 0 factors are applied by the caller.
// DCT-III (orthonormal inverse) pre-processing for one k: W[k] = (Xk - i XLk) P + (XkM - i XMk) Q.
template <typename T> __device__ __forceinline__ void ld_ab(const Tw<T>& tb, int k, cplx<T>& A, cplx<T>& B) {
#ifdef COFEM_1K_AB_INTERLEAVE
  if constexpr (sizeof(T) == 4) {
    const float4 v = *reinterpret_cast<const float4*>(tb.base + TAB2 + 2 * k);
    A = {v.x, v.y}; B = {v.z, v.w};
    return;
  }
#endif
  A = tb.base[TAB2 + ia(k)]; B = tb.base[TAB2 + ib(k)];
}
template <typename T>
__device__ __forceinline__ cplx<T> dct3_pre(int k, T Xk, T XLk, T XkM, T XMk, const Tw<T>& tb) {
  cplx<T> A, B;
  ld_ab(tb, k, A, B);
  return {Xk * A.x - XLk * A.y + XkM * B.x - XMk * B.y, -Xk * A.y - XLk * A.x - XkM * B.y - XMk * B.x};
}

// DCT-II post-processing for one k from W[k], W[(M-k) mod M]: orthonormal X[k], X[k+M].
template <typename T>
__device__ __forceinline__ void dct2_post(int k, cplx<T> Wk, cplx<T> Wm, const Tw<T>& tb, T& lo, T& hi) {
  cplx<T> A, B;
  ld_ab(tb, k, A, B);
  const T h = (T)0.70710678118654752440;
  const T u = h * (Wm.x + Wm.y), v = h * (Wm.x - Wm.y);     // e^{-i pi/4} Wm = (u, -v), e^{i pi/4} Wm = (v, u)
  lo = Wk.x * A.x - Wk.y * A.y + u * B.x - v * B.y;
  hi = Wk.x * B.x - Wk.y * B.y + v * A.x + u * A.y;
}
#endif

#ifndef COFEM_1K_TAB6
// Computed factors (COFEM_1K_CTAB, fft512.cuh): Ahat, Bhat of k = k0 + 64 r from the lane's bases
// u = u_{k0}, v = v_{k0}; the rotations e^{-i pi r/32}, e^{-5 i pi r/32} are compile-time constants.
template <typename T>
__device__ __forceinline__ void ab_comp(cplx<T> u, cplx<T> v, int r, cplx<T>& A, cplx<T>& B) {
  constexpr double c1[8] = {1.0, 0.99518472667219692873, 0.98078528040323043058, 0.95694033573220882438,
                            0.92387953251128673848, 0.88192126434835504956, 0.83146961230254523567, 0.77301045336273699338};
  constexpr double s1[8] = {0.0, 0.09801714032956060363, 0.19509032201612824808, 0.29028467725446233105,
                            0.38268343236508978178, 0.47139673682599764204, 0.55557023301960217765, 0.63439328416364548779};
  constexpr double c5[8] = {1.0, 0.88192126434835504956, 0.55557023301960228867, 0.09801714032956077016,
                            -0.38268343236508972627, -0.77301045336273699338, -0.98078528040323043058, -0.95694033573220893540};
  constexpr double s5[8] = {0.0, 0.47139673682599764204, 0.83146961230254523567, 0.99518472667219681771,
                            0.92387953251128673848, 0.63439328416364548779, 0.19509032201612860891, -0.29028467725446210901};
  cplx<T> U = u, V = v;
  if (r) {   // U = u e^{-i pi r/32}, V = v e^{-5 i pi r/32}
    const T c = (T)c1[r], s = (T)s1[r], cc = (T)c5[r], ss = (T)s5[r];
    U = {u.x * c + u.y * s, u.y * c - u.x * s};
    V = {v.x * cc + v.y * ss, v.y * cc - v.x * ss};
  }
  const T h = (T)0.70710678118654752440;
  A = {U.x + V.y, U.y - V.x};                              // U - i V
  const T tx = U.x - V.y, ty = U.y + V.x;                  // U + i V
  B = {h * (tx + ty), h * (ty - tx)};                      // e^{-i pi/4} (U + i V)
}
template <typename T>
__device__ __forceinline__ cplx<T> dct3_pre_ab(cplx<T> A, cplx<T> B, T Xk, T XLk, T XkM, T XMk) {
  return {Xk * A.x - XLk * A.y + XkM * B.x - XMk * B.y, -Xk * A.y - XLk * A.x - XkM * B.y - XMk * B.x};
}
template <typename T>
__device__ __forceinline__ void dct2_post_ab(cplx<T> A, cplx<T> B, cplx<T> Wk, cplx<T> Wm, T& lo, T& hi) {
  const T h = (T)0.70710678118654752440;
  const T u = h * (Wm.x + Wm.y), v = h * (Wm.x - Wm.y);
  lo = Wk.x * A.x - Wk.y * A.y + u * B.x - v * B.y;
  hi = Wk.x * B.x - Wk.y * B.y + v * A.x + u * A.y;
}
#endif

// Packed spectra of the DCT-III of a line held canonically in A, B, C, E.
// CT: Makhoul factors computed from the per-lane bases (fft512.cuh) instead of read from the tables.
template <typename T, bool CT = false>
__device__ __forceinline__ void pre_all(int lane, const T (&A)[8], const T (&B)[8], const T (&C)[8], const T (&E)[8],
                                        cplx<T> (&va)[8], cplx<T> (&vb)[8], const Tw<T>& tb) {
  const int ja = lane, jb = lane ? 64 - lane : 32;
  const bool l0 = lane == 0;
#ifndef COFEM_1K_TAB6
  if constexpr (CT) {
    const cplx<T> ua = tb.base[TBAS + lane], wa = tb.base[TBAS + 32 + lane];
    const cplx<T> ub = tb.base[TBAS + 64 + lane], wb = tb.base[TBAS + 96 + lane];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const T aMk = l0 ? (r ? A[(8 - r) & 7] : C[0]) : B[7 - r];
      const T aLk = l0 ? (r ? C[(8 - r) & 7] : (T)0) : E[7 - r];
      cplx<T> Af, Bf;
      ab_comp<T>(ua, wa, r, Af, Bf);
      va[r] = dct3_pre_ab<T>(Af, Bf, (l0 && r == 0) ? A[0] * (T)1.41421356237309504880 : A[r], aLk, C[r], aMk);
      const T bMk = l0 ? B[7 - r] : A[7 - r];
      const T bLk = l0 ? E[7 - r] : C[7 - r];
      ab_comp<T>(ub, wb, r, Af, Bf);
      vb[r] = dct3_pre_ab<T>(Af, Bf, B[r], bLk, E[r], bMk);
    }
    return;
  }
#endif
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    // slot a, k = ja + 64 r: X[M-k], X[L-k]
    const T aMk = l0 ? (r ? A[(8 - r) & 7] : C[0]) : B[7 - r];
    const T aLk = l0 ? (r ? C[(8 - r) & 7] : (T)0) : E[7 - r];
#ifdef COFEM_1K_TAB6
    va[r] = dct3_pre<T>(ja + 64 * r, A[r], aLk, C[r], aMk, tb);
#else
    va[r] = dct3_pre<T>(ja + 64 * r, (l0 && r == 0) ? A[0] * (T)1.41421356237309504880 : A[r], aLk, C[r], aMk, tb);
#endif
    // slot b, k = jb + 64 r
    const T bMk = l0 ? B[7 - r] : A[7 - r];
    const T bLk = l0 ? E[7 - r] : C[7 - r];
    vb[r] = dct3_pre<T>(jb + 64 * r, B[r], bLk, E[r], bMk, tb);
  }
}

// DCT-II outputs of a line from its FFT (va, vb) into canonical A, B, C, E.
template <typename T, bool CT = false>
__device__ __forceinline__ void post_all(int lane, const cplx<T> (&va)[8], const cplx<T> (&vb)[8], T (&A)[8], T (&B)[8],
                                         T (&C)[8], T (&E)[8], const Tw<T>& tb) {
  const int ja = lane, jb = lane ? 64 - lane : 32;
  const bool l0 = lane == 0;
#ifndef COFEM_1K_TAB6
  if constexpr (CT) {
    const cplx<T> ua = tb.base[TBAS + lane], wa0 = tb.base[TBAS + 32 + lane];
    const cplx<T> ub = tb.base[TBAS + 64 + lane], wb0 = tb.base[TBAS + 96 + lane];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      cplx<T> Af, Bf;
      const cplx<T> wa = l0 ? va[(8 - r) & 7] : vb[7 - r];
      ab_comp<T>(ua, wa0, r, Af, Bf);
      dct2_post_ab<T>(Af, Bf, va[r], wa, A[r], C[r]);
      if (l0 && r == 0) A[0] *= (T)0.70710678118654752440;     // k = 0: s0 / s = 1 / sqrt 2
      const cplx<T> wb = l0 ? vb[7 - r] : va[7 - r];
      ab_comp<T>(ub, wb0, r, Af, Bf);
      dct2_post_ab<T>(Af, Bf, vb[r], wb, B[r], E[r]);
    }
    return;
  }
#endif
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const cplx<T> wa = l0 ? va[(8 - r) & 7] : vb[7 - r];
    dct2_post<T>(ja + 64 * r, va[r], wa, tb, A[r], C[r]);
#ifndef COFEM_1K_TAB6
    if (l0 && r == 0) A[0] *= (T)0.70710678118654752440;     // k = 0: s0 / s = 1 / sqrt 2
#endif
    const cplx<T> wb = l0 ? vb[7 - r] : va[7 - r];
    dct2_post<T>(jb + 64 * r, vb[r], wb, tb, B[r], E[r]);
  }
}

// Loads of arrays other CTAs of the same launch may have rewritten (the dataflow kernel k1k_flow:
// p, r, T^T, T2, q change between its items): CG = true reads through L2 (ld.global.cg), never a
// stale L1 line.  The per-pass kernels (one pass per launch) read normally.
template <bool CG, typename V> __device__ __forceinline__ V ldx(const V* p) {
  if constexpr (CG) return __ldcg(p); else return *p;
}
template <bool CG> __device__ __forceinline__ cplx<float> ldc(const cplx<float>* p) {
  const float2 v = ldx<CG>(reinterpret_cast<const float2*>(p));
  return {v.x, v.y};
}
template <bool CG> __device__ __forceinline__ cplx<double> ldc(const cplx<double>* p) {
  const double2 v = ldx<CG>(reinterpret_cast<const double2*>(p));
  return {v.x, v.y};
}

template <typename T> __device__ __forceinline__ const T* alpha_of(const DctArgs& a, int j) {
  if constexpr (sizeof(T) == 8) { if (j == 0) return a.alpha; }
  return (const T*)a.alphap;
}

// Barrier of the RT warps that process an item: barrier 1 over RT * 32 threads.  In the per-pass
// kernels that is the whole CTA (= __syncthreads); in k1k_flow the worker warps, without the
// control warp.
template <int RT> __device__ __forceinline__ void bar_rt() { asm volatile("bar.sync 1, %0;" ::"n"(RT * 32) : "memory"); }

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

// The per-pass kernels' shared-memory tables: the compact image (FFT twiddles + Makhoul bases) where
// the factors are computed (fp32, COFEM_1K_CTAB), else the [0, n) prefix of the full layout.
template <typename T, int PASS> __device__ __forceinline__ Tw<T> load_tab_pass(const DctArgs& a, cplx<T>* sm) {
  if constexpr (ctp<T, PASS>()) return load_tables_ct<T>(tab1k<T>(a), sm);
  else return load_tables<T>(tab1k<T>(a), sm, ntab<T, PASS>());
}

// ---------------------------------------------------------------- pass A
// Shared memory: [RT warps][WREG] (FFT exchange / output tile row) then the twiddle tables.
// Persistent kernels: work item w = (column j0 + w / NTILE, tile w % NTILE), grid-strided.
template <typename T> struct Work { static constexpr int NTILE = L / Geo<T>::RT; };

template <typename T, bool CG = false>
__device__ __forceinline__ void rows_inv_item(const DctArgs& a, int j, int tile, int dir, double bcoef, T* sm,
                                              const Tw<T>& tb);

template <typename T>
#ifndef COFEM_1K_INV_TMA
#define COFEM_1K_INV_TMA 0    // pass A (fp32 probes) with TMA bulk staging of each warp's next row (A/B switch)
#endif
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
  // pass A needs the FFT twiddles and the DCT-III pre tables only: the [0, TPRE) prefix (12.8 KB in fp32)
  const Tw<T> tb = load_tab_pass<T, 0>(a, reinterpret_cast<cplx<T>*>(sm + RT * WREG));   // + barrier
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

template <typename T, bool CG>
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
      for (int i = 0; i < 4; ++i) pv[i] = ldx<CG>(pr + lane + 32 * (4 * h + i));
      if (dir) {
        float4 rv[4], dd[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) { rv[i] = ldx<CG>(rr + lane + 32 * (4 * h + i)); dd[i] = dv[lane + 32 * (4 * h + i)]; }
#ifdef COFEM_EXP_FUSE_EMU   // timing experiment only: the extra traffic of a fused update (q read, r write)
        {
          const float4* __restrict__ qq4 = reinterpret_cast<const float4*>(c.q + rb);
          float4* rw = const_cast<float4*>(rr);
          const float z0 = (float)(a.beta * 0.0);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 qv = qq4[lane + 32 * (4 * h + i)];
            rv[i].x -= z0 * qv.x; rv[i].y -= z0 * qv.y; rv[i].z -= z0 * qv.z; rv[i].w -= z0 * qv.w;
            rw[lane + 32 * (4 * h + i)] = rv[i];
          }
        }
#endif
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
  pre_all<T, ctp<T, 0>() && !CG>(lane, A, B, C, E, va, vb, tb);
  T* reg = sm + warp * WREG;
  fft512<T, +1>(va, vb, lane, reinterpret_cast<cplx<T>*>(reg), tb);
  const int ja = lane, jb = lane ? 64 - lane : 32;
#pragma unroll
  for (int r = 0; r < 8; ++r) {     // packed v-order output w[n] = v[2n] + i v[2n+1]
    *reinterpret_cast<cplx<T>*>(reg + 2 * (ja + 64 * r)) = va[r];
    *reinterpret_cast<cplx<T>*>(reg + 2 * (jb + 64 * r)) = vb[r];
  }
  bar_rt<RT>();
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

// ---------------------------------------------------------------- pass A, bulk-staged (fp32 probes)
// each warp's NEXT image row of p and r is copied into shared memory by the TMA
// bulk engine (cp.async.bulk, one 4 KB copy per array, completion on a per-warp mbarrier) while the
// warp runs the current row's FFT, so the row loads leave the critical path whatever the number of
// warps.  16 warps (rows) per CTA, one CTA per SM (212 KB of shared memory: 16 x 8 KB staging, the
// exchange regions, the tables), i.e. the same 16 warps per SM as k1k_rows_inv.  Arithmetic identical
// to rows_inv_item<float>.  Build switch COFEM_1K_INV_TMA (A/B).
namespace rtma {
#ifndef COFEM_1K_TMA_RT
#define COFEM_1K_TMA_RT 16
#endif
#ifndef COFEM_1K_TMA_R
#define COFEM_1K_TMA_R 1      // 1: stage r as well as p
#endif
#ifndef COFEM_1K_TMA_CPS
#define COFEM_1K_TMA_CPS 1    // CTAs per SM of the persistent grid
#endif
constexpr int RT = COFEM_1K_TMA_RT, NT = L / RT, STG = (COFEM_1K_TMA_R ? 2 : 1) * L;
__host__ __device__ constexpr size_t smem_bytes() {
  return (size_t)RT * STG * 4 + (size_t)RT * WREG * 4 + (size_t)TPRE * sizeof(cplx<float>) + (size_t)RT * 8;
}
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(b)));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(b))
               : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done)
                 : "r"(su32(b)), "r"(parity)
                 : "memory");
}
}  // namespace rtma

__global__ void __launch_bounds__(rtma::RT * 32, COFEM_1K_TMA_CPS) k1k_rows_inv_tma(DctArgs a, int j0, int ncols, int dir) {
  using namespace rtma;
  extern __shared__ __align__(16) unsigned char smraw[];   // bulk copies need 16-byte alignment
  float* stg = reinterpret_cast<float*>(smraw);                                  // [RT][STG]: p row, r row
  float* sm = stg + RT * STG;                                                    // [RT][WREG] exchange
  cplx<float>* tabs = reinterpret_cast<cplx<float>*>(sm + RT * WREG);
  uint64_t* bar = reinterpret_cast<uint64_t*>(tabs + TPRE);
  __shared__ ColFlags ci;
  load_colinfo(ci, a.cs, j0, ncols);
  if (!any_active(ci, ncols)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int items = ncols * NT;
  auto next_item = [&](int w) {   // CTA-uniform: the next item of this CTA whose column is active
    for (; w < items; w += gridDim.x)
      if (!ci.frozen[w / NT]) return w;
    return items;
  };
  auto issue = [&](int w) {       // lane 0: this warp's row of item w -> its staging buffer
    const DctCol<float> cn = col_of<float>(a, j0 + w / NT);
    const int64_t rb = (int64_t)((w % NT) * RT + warp) * L;
    const bool rr = COFEM_1K_TMA_R && dir;
    expect_tx(&bar[warp], rr ? 2 * L * 4 : L * 4);
    bulk(stg + warp * STG, cn.p + rb, L * 4, &bar[warp]);
    if (rr) bulk(stg + warp * STG + L, cn.r + rb, L * 4, &bar[warp]);
  };
  int w = next_item(blockIdx.x);
  if (lane == 0) {
    bar_init(&bar[warp]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (w < items) issue(w);
  }
  const Tw<float> tb = load_tables<float>(tab1k<float>(a), tabs, TPRE);   // + barrier
  uint32_t phase = 0;
  const float4* st4p = reinterpret_cast<const float4*>(stg + warp * STG);
  const float4* st4r = reinterpret_cast<const float4*>(stg + warp * STG + (COFEM_1K_TMA_R ? L : 0));
  while (w < items) {
    const int wn = next_item(w + gridDim.x);
    const int jj = w / NT, tile = w % NT, row0 = tile * RT;
    const DctCol<float> c = col_of<float>(a, j0 + jj);
    const int64_t rb = (int64_t)(row0 + warp) * L;
    wait(&bar[warp], phase);
    phase ^= 1u;
    float4 pv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) pv[i] = st4p[lane + 32 * i];
    if (dir) {
      const float bb = (float)ci.b[jj];
      const float4* __restrict__ dv = reinterpret_cast<const float4*>(c.dinv + rb);
      float4* __restrict__ pr = reinterpret_cast<float4*>(c.p + rb);
#pragma unroll
      for (int i = 0; i < 8; ++i) {    // a6: p = M^-1 r + b p
        const float4 rv = COFEM_1K_TMA_R ? st4r[lane + 32 * i] : reinterpret_cast<const float4*>(c.r + rb)[lane + 32 * i];
        const float4 dd = dv[lane + 32 * i];
        pv[i].x = dd.x * rv.x + bb * pv[i].x; pv[i].y = dd.y * rv.y + bb * pv[i].y;
        pv[i].z = dd.z * rv.z + bb * pv[i].z; pv[i].w = dd.w * rv.w + bb * pv[i].w;
        pr[lane + 32 * i] = pv[i];
      }
    }
    float4* r4 = reinterpret_cast<float4*>(sm + warp * WREG);
#pragma unroll
    for (int i = 0; i < 8; ++i) r4[lane + 32 * i] = pv[i];
    __syncwarp();                    // the staging buffer is consumed (pv depends on every read of it)
    if (!COFEM_1K_TMA_R && dir && wn < items) {   // r of the next row: L2 prefetch instead
      const int64_t rbn = (int64_t)((wn % NT) * RT + warp) * L;
      pf_line(col_of<float>(a, j0 + wn / NT).r + rbn);
    }
    if (wn < items && lane == 0) issue(wn);
    const float* reg = sm + warp * WREG;
    float A[8], B[8], C[8], E[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      int o[4];
      canon(lane, r, o);
      A[r] = reg[o[0]]; B[r] = reg[o[1]]; C[r] = reg[o[2]]; E[r] = reg[o[3]];
    }
    __syncwarp();                    // fft512 reuses the region
    cplx<float> va[8], vb[8];
    pre_all<float>(lane, A, B, C, E, va, vb, tb);
    float* regw = sm + warp * WREG;
    fft512<float, +1>(va, vb, lane, reinterpret_cast<cplx<float>*>(regw), tb);
    const int ja = lane, jb = lane ? 64 - lane : 32;
#pragma unroll
    for (int r = 0; r < 8; ++r) {     // packed v-order output w[n] = v[2n] + i v[2n+1]
      *reinterpret_cast<cplx<float>*>(regw + 2 * (ja + 64 * r)) = va[r];
      *reinterpret_cast<cplx<float>*>(regw + 2 * (jb + 64 * r)) = vb[r];
    }
    bar_rt<RT>();
    float* __restrict__ out = c.t1;   // T^T[cv][row], line length L: 32-byte segments of 8 rows
#pragma unroll
    for (int it = 0; it < L / (RT * 32); ++it) {
      const int cv = it * RT * 32 + threadIdx.x;
#pragma unroll
      for (int h = 0; h < RT / 8; ++h) {
        float v0[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v0[i] = sm[(8 * h + i) * WREG + cv];
        st32B<float, 8>(out + (int64_t)cv * L + row0 + 8 * h, v0);
      }
    }
    bar_rt<RT>();                    // the exchange regions are reused by the next item
    w = wn;
  }
}

// ---------------------------------------------------------------- pass B
template <typename T, bool CG = false>
__device__ __forceinline__ void cols_item(const DctArgs& a, int j, int tile, T* sm, const Tw<T>& tb);

#ifndef COFEM_1K_COLS_MINB
#define COFEM_1K_COLS_MINB 3   // fp32: 3 CTAs (24 warps) per SM
#endif
template <typename T>
__global__ void __launch_bounds__(Geo<T>::RT * 32, sizeof(T) == 4 ? COFEM_1K_COLS_MINB : 1) k1k_cols(DctArgs a, int j0, int ncols) {
  constexpr int RT = Geo<T>::RT, NT = Work<T>::NTILE;
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sm = reinterpret_cast<T*>(smraw);
  __shared__ ColFlags ci;
  load_colinfo(ci, a.cs, j0, ncols);
  if (!any_active(ci, ncols)) return;
  if (blockIdx.x < ncols * NT && !ci.frozen[blockIdx.x / NT])     // the first item's line, before the tables
    pf_line(col_of<T>(a, j0 + blockIdx.x / NT).t1 + (int64_t)((blockIdx.x % NT) * RT + (threadIdx.x >> 5)) * L);
  const Tw<T> tb = load_tab_pass<T, 1>(a, reinterpret_cast<cplx<T>*>(sm + RT * WREG));   // + barrier
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

template <typename T, bool CG>
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
    A[r] = ldx<CG>(ln + o[0]); B[r] = ldx<CG>(ln + o[1]); C[r] = ldx<CG>(ln + o[2]); E[r] = ldx<CG>(ln + o[3]);
  }
  cplx<T> va[8], vb[8];
  pre_all<T, ctp<T, 1>() && !CG>(lane, A, B, C, E, va, vb, tb);
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
  post_all<T, ctp<T, 1>() && !CG>(lane, va, vb, A, B, C, E, tb);
#pragma unroll
  for (int r = 0; r < 8; ++r) {     // natural-order column values -> tile row (the exchange region is free)
    int o[4];
    canon(lane, r, o);
    reg[o[0]] = A[r]; reg[o[1]] = B[r]; reg[o[2]] = C[r]; reg[o[3]] = E[r];
  }
  bar_rt<RT>();
  T* __restrict__ out = c.t2;       // T2[row][cv] row-major: 32-byte segments of RT v-order columns
#pragma unroll
  for (int it = 0; it < L / (RT * 32); ++it) {
    const int row = it * RT * 32 + threadIdx.x;
    T v[RT];
#pragma unroll
    for (int i = 0; i < RT; ++i) v[i] = sm[i * WREG + row];
    st32B<T, RT>(out + (int64_t)row * L + tile * RT, v);
  }
  bar_rt<RT>();
}


// ---------------------------------------------------------------- pass B, half-warp FFTs (fp32 probes)
// EXPERIMENT (build switch COFEM_1K_COLS_HALF, not the default): correct, but 128 registers (16 warps
// per SM instead of 24) outweigh its 18 % fewer shared-memory wavefronts: C4 fixed-alpha E-step
// 42.6 -> 44.9 ms.
// The column pass with the radix-16 x 32 half-warp FFT pair (fft512h.cuh): 16 lanes per T^T line,
// two lines per warp, 16 lines per CTA item; one exchange per transform (two per line instead of
// four), and the two lines of a warp read the same DCT table and twiddle entries (broadcast).
// Lane (h, t) of warp w owns line 2 w + h of the item and the positions {ka, kb, M + ka, M + kb} +
// 32 k2 (k2 < 16), ka = t, kb = 32 - t (16 for t = 0): the k <-> M - k and k <-> L - k partners of its
// spectral points are its own.
namespace colsh {
constexpr int NL = 16;                             // lines per CTA item
constexpr int NTH = L / NL;                        // items per column
constexpr int TROW = L + 16;                       // tile row stride (floats): the two half-warps of a warp write disjoint banks
constexpr size_t SMEM_X = (size_t)8 * 2 * d1kh::XREG * sizeof(cplx<float>);   // exchange (aliases the tile)
constexpr size_t SMEM_TILE = (size_t)NL * TROW * sizeof(float);
constexpr size_t SMEM_XT = SMEM_X > SMEM_TILE ? SMEM_X : SMEM_TILE;
constexpr size_t SMEM = SMEM_XT + (size_t)2 * M * sizeof(cplx<float>) + (size_t)d1kh::TWTOT * sizeof(cplx<float>);
}

// maskH[line][t] bit 2 m + e = mask at v-order row 2 (t + 16 m) + e (the n-layout of fft512h.cuh)
__global__ void k1k_mask_half(const uint8_t* __restrict__ maskT, unsigned long long* __restrict__ maskH) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= L * 16) return;
  const int line = idx >> 4, t = idx & 15;
  const uint8_t* m = maskT + (int64_t)line * L;
  unsigned long long w = 0;
  for (int mm = 0; mm < 32; ++mm)
    for (int e = 0; e < 2; ++e) w |= (unsigned long long)(m[2 * (t + 16 * mm) + e] != 0) << (2 * mm + e);
  maskH[idx] = w;
}

#ifndef COFEM_1K_COLSH_MINB
#define COFEM_1K_COLSH_MINB 2
#endif
__global__ void __launch_bounds__(256, COFEM_1K_COLSH_MINB) k1k_cols_h(DctArgs a, int j0, int ncols,
                                                                      const unsigned long long* __restrict__ maskH,
                                                                      const cplx<float>* __restrict__ twh) {
  using namespace colsh;
  using T = float;
  extern __shared__ __align__(16) unsigned char smraw[];
  float* tile = reinterpret_cast<float*>(smraw);
  cplx<T>* xall = reinterpret_cast<cplx<T>*>(smraw);
  cplx<T>* ab = reinterpret_cast<cplx<T>*>(smraw + SMEM_XT);                 // Ahat | Bhat (2 M)
  cplx<T>* tw = ab + 2 * M;                                                    // wk | wt
  __shared__ ColFlags ci;
  load_colinfo(ci, a.cs, j0, ncols);
  if (!any_active(ci, ncols)) return;
  {
    const cplx<T>* g = (const cplx<T>*)a.tab1k32 + TAB2;
    for (int i = threadIdx.x; i < 2 * M; i += blockDim.x) ab[i] = g[i];
    for (int i = threadIdx.x; i < d1kh::TWTOT; i += blockDim.x) tw[i] = twh[i];
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, h = lane >> 4, t = lane & 15;
  const int ka = t, kb = d1kh::kb_of(t);
  const bool l0 = t == 0;
  const int lrow = warp * 2 + h;                       // this half-warp's line within the item
  cplx<T>* x = xall + (warp * 2 + h) * d1kh::XREG;
  auto A_ = [&](int k) { return ab[ia(k)]; };
  auto B_ = [&](int k) { return ab[ib(k)]; };
  for (int w = blockIdx.x; w < ncols * NTH; w += gridDim.x) {
    const int jj = w / NTH;
    if (ci.frozen[jj]) continue;
    const int tileidx = w % NTH, line = tileidx * NL + lrow;     // v-order image column cv
    const DctCol<T> c = col_of<T>(a, j0 + jj);
    const T* __restrict__ ln = c.t1 + (int64_t)line * L;
    T A[16], B[16], C[16], E[16];
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) {
      A[k2] = ln[ka + 32 * k2]; B[k2] = ln[kb + 32 * k2]; C[k2] = ln[M + ka + 32 * k2]; E[k2] = ln[M + kb + 32 * k2];
    }
    cplx<T> va[16], vb[16];
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) {                  // DCT-III pre (dct3_pre's arithmetic, Ahat / Bhat tables)
      const int r = 15 - k2;
      T xLa = E[r], xMa = B[r], xLb = C[r], xMb = A[r];
      if (l0) {
        xLa = k2 ? C[16 - k2] : (T)0; xMa = k2 ? A[16 - k2] : C[0];
        xLb = E[r]; xMb = B[r];
      }
      const T xa = (l0 && k2 == 0) ? A[0] * (T)1.41421356237309504880 : A[k2];
      {
        const cplx<T> Aa = A_(ka + 32 * k2), Ba = B_(ka + 32 * k2);
        va[k2] = {xa * Aa.x - xLa * Aa.y + C[k2] * Ba.x - xMa * Ba.y, -xa * Aa.y - xLa * Aa.x - C[k2] * Ba.y - xMa * Ba.x};
      }
      {
        const cplx<T> Ab = A_(kb + 32 * k2), Bb = B_(kb + 32 * k2);
        vb[k2] = {B[k2] * Ab.x - xLb * Ab.y + E[k2] * Bb.x - xMb * Bb.y, -B[k2] * Ab.y - xLb * Ab.x - E[k2] * Bb.y - xMb * Bb.x};
      }
    }
    cplx<T> v[32];
    d1kh::ifft_k2n(va, vb, v, t, x, tw);
    {                                                   // mask (v-order pixel rows of this column)
      const unsigned long long mb = maskH[line * 16 + t];
#pragma unroll
      for (int m = 0; m < 32; ++m) {
        if (!((mb >> (2 * m)) & 1ull)) v[m].x = (T)0;
        if (!((mb >> (2 * m + 1)) & 1ull)) v[m].y = (T)0;
      }
    }
    d1kh::fft_n2k(v, va, vb, t, x, tw);
    // DCT-II post into this line's tile row (natural order); the exchange region aliases the tile,
    // so every half-warp has finished its FFTs first
    bar_rt<8>();
    float* trow = tile + lrow * TROW;
    const T hh = (T)0.70710678118654752440;
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2) {
      const int r = 15 - k2;
      {   // slot a: k = ka + 32 k2
        const cplx<T> Wk = va[k2], Wm = l0 ? va[k2 ? 16 - k2 : 0] : vb[r];
        const cplx<T> Aa = A_(ka + 32 * k2), Ba = B_(ka + 32 * k2);
        const T u = hh * (Wm.x + Wm.y), vv = hh * (Wm.x - Wm.y);
        T lo = Wk.x * Aa.x - Wk.y * Aa.y + u * Ba.x - vv * Ba.y;
        const T hi = Wk.x * Ba.x - Wk.y * Ba.y + vv * Aa.x + u * Aa.y;
        if (l0 && k2 == 0) lo *= (T)0.70710678118654752440;
        trow[ka + 32 * k2] = lo; trow[M + ka + 32 * k2] = hi;
      }
      {   // slot b: k = kb + 32 k2
        const cplx<T> Wk = vb[k2], Wm = l0 ? vb[r] : va[r];
        const cplx<T> Ab = A_(kb + 32 * k2), Bb = B_(kb + 32 * k2);
        const T u = hh * (Wm.x + Wm.y), vv = hh * (Wm.x - Wm.y);
        const T lo = Wk.x * Ab.x - Wk.y * Ab.y + u * Bb.x - vv * Bb.y;
        const T hi = Wk.x * Bb.x - Wk.y * Bb.y + vv * Ab.x + u * Ab.y;
        trow[kb + 32 * k2] = lo; trow[M + kb + 32 * k2] = hi;
      }
    }
    bar_rt<8>();
    T* __restrict__ out = c.t2;                        // T2[row][cv]: 64-byte segments of 16 v-order columns
#pragma unroll
    for (int it = 0; it < L / 256; ++it) {
      const int row = it * 256 + threadIdx.x;
      float v16[16];
#pragma unroll
      for (int i = 0; i < NL; ++i) v16[i] = tile[i * TROW + row];
      float4* o4 = reinterpret_cast<float4*>(out + (int64_t)row * L + tileidx * NL);
#pragma unroll
      for (int q = 0; q < 4; ++q) o4[q] = make_float4(v16[4 * q], v16[4 * q + 1], v16[4 * q + 2], v16[4 * q + 3]);
    }
    bar_rt<8>();
  }
}

// ---------------------------------------------------------------- pass C
template <typename T, bool CG = false>
__device__ __forceinline__ double rows_fwd_item(const DctArgs& a, int j, int tile, T* sm, const Tw<T>& tb);

template <typename T>
#ifndef COFEM_1K_FWD_MINB
#define COFEM_1K_FWD_MINB 0   // 0: no min-blocks bound (nvcc then takes 80 registers, 3 CTAs per SM)
#endif
#if COFEM_1K_FWD_MINB > 0
__global__ void __launch_bounds__(Geo<T>::RT * 32, sizeof(T) == 4 ? COFEM_1K_FWD_MINB : 1) k1k_rows_fwd(DctArgs a, int j0, int ncols) {
#else
__global__ void __launch_bounds__(Geo<T>::RT * 32) k1k_rows_fwd(DctArgs a, int j0, int ncols) {
#endif
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
  const Tw<T> tb = load_tab_pass<T, 2>(a, reinterpret_cast<cplx<T>*>(sm + RT * WREG));   // + barrier
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

template <typename T, bool CG>
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
    for (int r = 0; r < 8; ++r) { va[r] = ldc<CG>(rowc + ja + 64 * r); vb[r] = ldc<CG>(rowc + jb + 64 * r); }
  }
  fft512<T, -1>(va, vb, lane, reinterpret_cast<cplx<T>*>(reg), tb);
  T A[8], B[8], C[8], E[8];
  post_all<T, ctp<T, 2>() && !CG>(lane, va, vb, A, B, C, E, tb);
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
#ifdef COFEM_EXP_FUSE_EMU   // timing experiment only: rho, delta1, delta2 of single-reduction CG in pass C
    double e1 = 0.0, e2 = 0.0, e3 = 0.0;
    const float4* __restrict__ rr4 = reinterpret_cast<const float4*>(c.r + rb);
    const float4* __restrict__ dd4 = reinterpret_cast<const float4*>(c.dinv + rb);
#endif
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float4 pv[4], av[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { pv[i] = ldx<CG>(pp + lane + 32 * (4 * h + i)); av[i] = al[lane + 32 * (4 * h + i)]; }
#ifdef COFEM_EXP_FUSE_EMU
      float4 rv[4], dv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { rv[i] = rr4[lane + 32 * (4 * h + i)]; dv[i] = dd4[lane + 32 * (4 * h + i)]; }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 x = r4[lane + 32 * (4 * h + i)];
        const float xs[4] = {x.x, x.y, x.z, x.w}, rs[4] = {rv[i].x, rv[i].y, rv[i].z, rv[i].w};
        const float ds[4] = {dv[i].x, dv[i].y, dv[i].z, dv[i].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float zr = ds[e] * rs[e], zq = ds[e] * xs[e];
          e1 += (double)rs[e] * (double)zr; e2 += (double)zq * (double)rs[e]; e3 += (double)zq * (double)xs[e];
        }
      }
#endif
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
#ifdef COFEM_EXP_FUSE_EMU
    e1 = warp_sum(e1); e2 = warp_sum(e2); e3 = warp_sum(e3);
    g += 1e-300 * (e1 + e2 + e3);
#endif
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


// ---------------------------------------------------------------- dataflow E-step (fp32 probe columns)
// All U CG iterations of the fp32 probe columns in ONE persistent launch.  The columns are
// independent systems (reading R3), so nothing forces them into lockstep: the work is a stream of
// items -- A (pass A, 8 image rows of one column), B (pass B, 8 T^T lines), C (pass C, 8 rows +
// gamma partials), U (the update a5 of one 2048-element D tile for a GROUP of columns, with the
// group's s accumulator) -- that CTAs take from a global counter in a fixed order.  An item waits
// only for the phase before it of its own column (A(i) <- U(i-1) of its group: b_j; B(i) <- all
// A(i) of the column: the transpose; C(i) <- all B(i); U(i) <- gamma of every column of the group),
// and that phase was dispensed earlier, so the earliest unfinished item can always run: no
// deadlock, whatever the number of resident CTAs.  The G groups are dispensed one phase apart
// (step tau: group g at phase tau - g), so A, B, C and U items of different groups run side by side
// on every SM (HBM-heavy row passes next to the shared-memory-heavy column pass) without the
// launch fill/drain of the per-pass kernels.  Reductions: gamma from one partial per image row
// (pass C), rho' from one partial per D tile, each reduced in fixed order by the CTA that completes
// the phase (deterministic).  Data other items rewrote is read through L2 (CG loads).
namespace flow {
constexpr int MAXG = 8;
constexpr int NT = L / 8;                 // fp32: 8 rows / lines per A, B, C item
struct State {                            // zeroed before every launch
  unsigned long long head;                // next item to dispense
  int nfrozen, pad;
  unsigned cntA[MAXM], cntB[MAXM], cntC[MAXM];   // completed items per probe column (all iterations)
  int doneC[MAXM];                        // iterations whose gamma is applied, per probe column
  int frozen[MAXM];                       // polling mirror of ColState::frozen
  unsigned cntU[MAXG];
  int doneU[MAXG];                        // iterations whose rho' is applied, per group
};
struct Args {
  State* st;
  int K, G, U, ntiles;                    // probe columns (global 1..K), groups, CG iterations, D tiles
  int g0[MAXG + 1];                       // group g = probe columns [g0[g], g0[g+1]) (0-based)
  int H, Gh, VS;                          // halves of a step, groups per half, virtual block size
  long long step, total;                  // items per step; items to dispense
  double invK;                            // 1 / K_total (Eq. 6)
  double* s[MAXG];                        // s accumulator of each group
  double* part2;                          // rho' partials, [column j][tile]
  const uint32_t* bits; int64_t wpc;
  const float *R0, *dinvp;                // for the update items (R is DctArgs::R)
};

__device__ __forceinline__ int ld_acq(const int* p) {
  int v; asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v; asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void st_rel(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// thread 0: wait until *cnt >= target, or the column froze (returns false then)
template <typename C>
__device__ __forceinline__ bool wait_ge(const C* cnt, C target, const int* frozen) {
  for (;;) {
    if (ld_acq(cnt) >= target) return true;
    if (frozen && ld_acq(frozen)) return false;
    __nanosleep(100);
  }
}

// ColState read through L2: other CTAs of the launch rewrite it (the gamma / rho' finishers)
__device__ __forceinline__ ColState ld_cs(const ColState* p) {
  static_assert(sizeof(ColState) == 64, "ColState layout");
  const double* d = reinterpret_cast<const double*>(p);
  const int* n = reinterpret_cast<const int*>(d + 5);
  ColState c;
  c.rho = __ldcg(d); c.rho0 = __ldcg(d + 1); c.gamma = __ldcg(d + 2); c.a = __ldcg(d + 3); c.b = __ldcg(d + 4);
  c.frozen = __ldcg(n); c.frozen_at = __ldcg(n + 1); c.nonfinite = __ldcg(n + 2); c.pad = __ldcg(n + 3);
  c.tau = __ldcg(d + 7);
  return c;
}

__device__ __forceinline__ int size_of(const Args& f, int g, int ph) {
  return ph < 3 ? (f.g0[g + 1] - f.g0[g]) * NT : f.ntiles;
}
// Dispense order.  Step tau holds one block per group: group g at phase counter pi = tau - g
// (pi = 4 i + phase).  A step is split into H halves of Gh groups; within a half the items of its
// blocks are dealt round-robin (item r -> block r mod Gh, index r / Gh), every block padded to the
// virtual size VS (padding items are skipped), so the SMs always hold a mix of the phase types of
// Gh consecutive groups.  A block depends on its own group's block of the previous step, which sat
// in the same half one step earlier: (H - 1) / H of a step apart, so the dependency is complete
// before the block starts (no bubble) when H = 2.
__device__ __forceinline__ void decode(const Args& f, long long q, int& g, int& pi, int& k) {
  const long long tau = q / f.step;
  const int r = (int)(q - tau * f.step);
  const int hs = f.Gh * f.VS, h = r / hs, rr = r - h * hs;
  g = h * f.Gh + rr % f.Gh;
  k = rr / f.Gh;
  pi = (int)tau - g;
  if (g >= f.G || k >= size_of(f, g, pi & 3)) pi = -1;    // padding
}

// Worker barrier: the 8 worker warps of k1k_flow (and the RT warps of the per-pass kernels,
// where it equals __syncthreads); barrier 1, so the control warp never takes part.
template <int N> __device__ __forceinline__ void worker_sync() { asm volatile("bar.sync 1, %0;" ::"n"(N) : "memory"); }

constexpr int NW = 8;                     // worker warps (one image row / T^T line each)
constexpr int FLOW_THREADS = (NW + 1) * 32;   // + the control warp

struct Item {                             // one published work item (ring slot)
  int go;                                 // 1 work, 2 skip, 0 stop
  int ph, i, g, k;                        // phase (A, B, C, U), CG iteration, group, index in block
};
#ifndef COFEM_FLOW_SLOTS
#define COFEM_FLOW_SLOTS 2      // ring depth (items published ahead of the workers)
#endif
constexpr int NSLOT = COFEM_FLOW_SLOTS;
struct Smem {
  Item ring[NSLOT];
  uint64_t full[NSLOT], done[NSLOT];      // mbarriers: item published / item finished by the workers
  double red[NW][MAXM];                   // U items: per-warp rho' sums
  double a[NSLOT][MAXM]; int act[NSLOT][MAXM];   // U items: step lengths / activity of the group, per slot
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
  for (;;) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(su32(b)), "r"(parity) : "memory");
    if (ok) return;
  }
}

// U item: a5 for the columns of group g on D tile t (k_update's arithmetic): r -= a q, z = r / diag,
// rho' partial, s += (a/K) p_k o p (x_k never stored)
__device__ __forceinline__ void update_item(const DctArgs& a, const Args& f, Smem& sh, int slot, int g, int t) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = f.g0[g], c1 = f.g0[g + 1];
  const int64_t d0 = (int64_t)t * VEC_TILE + (int64_t)threadIdx.x * VEC_ELEMS;
  float dp[8];
  {
    const float4 x = *reinterpret_cast<const float4*>(f.dinvp + d0), y = *reinterpret_cast<const float4*>(f.dinvp + d0 + 4);
    dp[0] = x.x; dp[1] = x.y; dp[2] = x.z; dp[3] = x.w; dp[4] = y.x; dp[5] = y.y; dp[6] = y.z; dp[7] = y.w;
  }
  double sacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  bool any = false;
  for (int jj = c0; jj < c1; ++jj) {
    const int cl = jj - c0;
    if (!sh.act[slot][cl]) { if (lane == 0) sh.red[warp][cl] = 0.0; continue; }
    any = true;
    const int64_t o = (int64_t)jj * a.Dp + d0;
    float* Rp = (float*)a.R + o;
    const float* Qp = (const float*)a.Q + o;
    const float* Pp = (const float*)a.P + o;
    float4 r4[2] = {__ldcg(reinterpret_cast<const float4*>(Rp)), __ldcg(reinterpret_cast<const float4*>(Rp) + 1)};
    const float4 q4[2] = {__ldcg(reinterpret_cast<const float4*>(Qp)), __ldcg(reinterpret_cast<const float4*>(Qp) + 1)};
    const float4 p4[2] = {__ldcg(reinterpret_cast<const float4*>(Pp)), __ldcg(reinterpret_cast<const float4*>(Pp) + 1)};
    const uint32_t w = (f.bits[(int64_t)jj * f.wpc + (d0 >> 5)] >> (d0 & 31)) & 0xffu;
    const double ak = sh.a[slot][cl];
    const float akt = (float)ak;
    const double aks = ak * f.invK;
    float* r = reinterpret_cast<float*>(r4);
    const float* q = reinterpret_cast<const float*>(q4);
    const float* pv = reinterpret_cast<const float*>(p4);
    double acc = 0.0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      r[e] = r[e] - akt * q[e];
      const float z = dp[e] * r[e];
      acc += (double)r[e] * (double)z;
      const double pe = (double)pv[e];
      sacc[e] += ((w >> e) & 1u) ? -aks * pe : aks * pe;
    }
    reinterpret_cast<float4*>(Rp)[0] = r4[0]; reinterpret_cast<float4*>(Rp)[1] = r4[1];
    acc = warp_sum(acc);
    if (lane == 0) sh.red[warp][cl] = acc;
  }
  if (any) {
    double* sp = f.s[g] + d0;
    double2 v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) { v[e] = __ldcg(reinterpret_cast<const double2*>(sp) + e); v[e].x += sacc[2 * e]; v[e].y += sacc[2 * e + 1]; }
#pragma unroll
    for (int e = 0; e < 4; ++e) reinterpret_cast<double2*>(sp)[e] = v[e];
  }
  worker_sync<NW * 32>();
  for (int cl = threadIdx.x; cl < c1 - c0; cl += NW * 32) {
    double v = 0.0;
#pragma unroll
    for (int ww = 0; ww < NW; ++ww) v += sh.red[ww][cl];
    f.part2[(int64_t)(c0 + cl + 1) * f.ntiles + t] = v;
  }
}

#ifndef COFEM_FLOW_MINB
#define COFEM_FLOW_MINB 2     // CTAs per SM
#endif
// Warp-specialised: warps 0..7 process items; warp 8 (control) dispenses them into a two-slot ring
// (mbarriers), waits for their dependencies, and after the workers finish an item releases it
// (fence + completion count) and runs the gamma / rho' finishers -- so the worker warps never
// wait on the dispenser atomic, the dependency polls or the release fences.
__global__ void __launch_bounds__(FLOW_THREADS, COFEM_FLOW_MINB) k1k_flow(DctArgs a, Args f) {
  using T = float;
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sm = reinterpret_cast<T*>(smraw);
  __shared__ Smem sh;
  State* st = f.st;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s2 = 0; s2 < NSLOT; ++s2) { mb_init(&sh.full[s2], 1); mb_init(&sh.done[s2], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const Tw<T> tb = load_tables<T>((const cplx<T>*)a.tab1k32, reinterpret_cast<cplx<T>*>(sm + NW * WREG));   // + barrier
  if (warp == NW) {
    // ------------------------------------------------------------ control warp
    // A polling state machine, never blocking on another CTA while it holds finished work: it
    // releases finished items in order, keeps one dequeued candidate, and publishes it into a free
    // slot once its dependency holds (deadlock-free: published items have no open dependencies,
    // and the candidate is the latest item the CTA holds).
    const int U4 = 4 * f.U;
    Item pend[NSLOT] = {}, cand = {};
    int n_pub = 0, n_rel = 0;
    bool have = false, stop = false;
    for (;;) {
      bool progress = false;
      // 1) release the oldest published item once the workers are done with it
      if (n_rel < n_pub) {
        const int slot = n_rel % NSLOT;
        uint32_t ok;
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(su32(&sh.done[slot])), "r"((uint32_t)((n_rel / NSLOT) & 1)) : "memory");
        if (ok) {
          const Item it = pend[slot];
          const int i = it.i, g = it.g;
          if (it.ph < 3) {
            const int jj = f.g0[g] + it.k / NT, j = jj + 1;
            unsigned old = 0;
            if (lane == 0) {
              __threadfence();
              unsigned* cnt = it.ph == 0 ? st->cntA + jj : it.ph == 1 ? st->cntB + jj : st->cntC + jj;
              old = atomicAdd(cnt, 1u);
            }
            old = __shfl_sync(0xffffffffu, old, 0);
            if (it.ph == 2 && old + 1 == (unsigned)(NT * (i + 1))) {   // gamma_j complete (fixed-order reduction)
              __threadfence();
              const double tot = reduce_partials(a.part + (int64_t)j * a.stride, L);
              if (lane == 0) {
                ColState c = ld_cs(a.cs + j);
                finish_gamma(c, tot, i);
                a.cs[j] = c;
                if (c.frozen) { st->frozen[jj] = 1; atomicAdd(&st->nfrozen, 1); }
                __threadfence();
                st_rel(st->doneC + jj, i + 1);
              }
            }
          } else {
            unsigned old = 0;
            if (lane == 0) { __threadfence(); old = atomicAdd(st->cntU + g, 1u); }
            old = __shfl_sync(0xffffffffu, old, 0);
            if (old + 1 == (unsigned)(f.ntiles * (i + 1))) {         // rho' of the group's columns
              __threadfence();
              for (int jj = f.g0[g]; jj < f.g0[g + 1]; ++jj) {
                const int j = jj + 1;
                const double v = reduce_partials(f.part2 + (int64_t)j * f.ntiles, f.ntiles);
                if (lane == 0) {
                  ColState c = ld_cs(a.cs + j);
                  if (!c.frozen) { c.b = v / c.rho; c.rho = v; a.cs[j] = c; }
                }
              }
              if (lane == 0) { __threadfence(); st_rel(st->doneU + g, i + 1); }
            }
          }
          ++n_rel;
          progress = true;
        }
      }
      // 2) dequeue a candidate (skipping items outside the schedule and of frozen columns)
      if (!have && !stop) {
        int go = 1, g = 0, pi = 0, k = 0;
        if (lane == 0) {
          const long long q = (long long)atomicAdd(&st->head, 1ull);
          if (q >= f.total || ld_acq(&st->nfrozen) >= f.K) go = 0;   // done / every column frozen (R5)
          else {
            decode(f, q, g, pi, k);
            if (pi < 0 || pi >= U4) go = 2;
            else if ((pi & 3) < 3 && ld_acq(st->frozen + f.g0[g] + k / NT)) go = 2;
          }
        }
        go = __shfl_sync(0xffffffffu, go, 0);
        if (go == 0) stop = true;
        else if (go == 1) {
          cand.go = 1; cand.g = __shfl_sync(0xffffffffu, g, 0); pi = __shfl_sync(0xffffffffu, pi, 0);
          cand.k = __shfl_sync(0xffffffffu, k, 0); cand.ph = pi & 3; cand.i = pi >> 2;
          have = true;
        }
        progress = true;
      }
      // 3) publish the candidate into a free slot once its dependency holds
      if (have && n_pub - n_rel < NSLOT) {
        int ready = 0;                              // 1 ready, 2 drop (column froze meanwhile)
        if (lane == 0) {
          const int i = cand.i, g = cand.g;
          if (cand.ph < 3) {
            const int jj = f.g0[g] + cand.k / NT;
            if (ld_acq(st->frozen + jj)) ready = 2;
            else if (cand.ph == 0) ready = (i == 0 || ld_acq(st->doneU + g) >= i) ? 1 : 0;
            else if (cand.ph == 1) ready = ld_acq(st->cntA + jj) >= (unsigned)(NT * (i + 1)) ? 1 : 0;
            else ready = ld_acq(st->cntB + jj) >= (unsigned)(NT * (i + 1)) ? 1 : 0;
          } else {
            ready = 1;
            for (int jj = f.g0[g]; jj < f.g0[g + 1]; ++jj)
              if (ld_acq(st->doneC + jj) < i + 1 && !ld_acq(st->frozen + jj)) { ready = 0; break; }
          }
          if (ready == 1) __threadfence();          // acquire side
        }
        ready = __shfl_sync(0xffffffffu, ready, 0);
        if (ready == 2) { have = false; progress = true; }
        else if (ready == 1) {
          const int slot = n_pub % NSLOT;
          if (cand.ph == 3) {                       // U: the group's a_j and activity
            for (int cl = lane; cl < f.g0[cand.g + 1] - f.g0[cand.g]; cl += 32) {
              const int j = f.g0[cand.g] + cl + 1;
              sh.act[slot][cl] = !__ldcg(&a.cs[j].frozen);
              sh.a[slot][cl] = __ldcg(&a.cs[j].a);
            }
          } else {                                  // L2 prefetch of its lines, one 128-B line per lane per row
            const int j = f.g0[cand.g] + cand.k / NT + 1, tile = cand.k % NT;
            const DctCol<T> cn = col_of<T>(a, j);
            for (int w = 0; w < NW; ++w) {
              const int64_t rn = (int64_t)(tile * NW + w) * L + 32 * lane;
              if (cand.ph == 0) {
                asm volatile("prefetch.global.L2 [%0];" ::"l"(cn.p + rn));
                if (cand.i > 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(cn.r + rn));
              } else if (cand.ph == 1) {
                asm volatile("prefetch.global.L2 [%0];" ::"l"(cn.t1 + rn));
              } else {
                asm volatile("prefetch.global.L2 [%0];" ::"l"(cn.t2 + rn));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(cn.p + rn));
              }
            }
          }
          __syncwarp();
          if (lane == 0) { sh.ring[slot] = cand; mb_arrive(&sh.full[slot]); }
          pend[slot] = cand;
          ++n_pub;
          have = false;
          progress = true;
        }
      }
      // 4) stop: every published item released -> publish the stop item and leave
      if (stop && !have && n_rel == n_pub) {
        if (lane == 0) { Item z{}; z.go = 0; sh.ring[n_pub % NSLOT] = z; mb_arrive(&sh.full[n_pub % NSLOT]); }
        break;
      }
      if (!progress) __nanosleep(64);
    }
    return;
  }
  // ------------------------------------------------------------ worker warps 0..7
  for (int n = 0;; ++n) {
    const int slot = n % NSLOT;
    mb_wait(&sh.full[slot], (n / NSLOT) & 1);
    const Item it = sh.ring[slot];
    if (it.go == 0) break;
    if (it.go == 1) {
      if (it.ph < 3) {
        const int jj = f.g0[it.g] + it.k / NT, tile = it.k % NT, j = jj + 1;
        if (it.ph == 0) {
          const double b = __ldcg(&a.cs[j].b);
          rows_inv_item<T, true>(a, j, tile, it.i > 0 ? 1 : 0, b, sm, tb);
        } else if (it.ph == 1) {
          cols_item<T, true>(a, j, tile, sm, tb);
        } else {
          const double gw = rows_fwd_item<T, true>(a, j, tile, sm, tb);
          if (lane == 0) a.part[(int64_t)j * a.stride + tile * NW + warp] = gw;
        }
      } else {
        update_item(a, f, sh, slot, it.g, it.k);
      }
    }
    worker_sync<NW * 32>();                           // item done by every worker (smem reuse, writes)
    if (threadIdx.x == 0) mb_arrive(&sh.done[slot]);
  }
}
}  // namespace flow

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

template <typename T> static size_t smem_bytes(int n = (ntab<T, 1>())) {
  return (size_t)Geo<T>::RT * WREG * sizeof(T) + (size_t)n * sizeof(cplx<T>);
}

template <typename T> static void set_attrs() {
  const int s = (int)smem_bytes<T>();
#if COFEM_1K_INV_TMA
  cudaFuncSetAttribute(k1k_rows_inv_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rtma::smem_bytes());
#endif
  cudaFuncSetAttribute(k1k_rows_inv<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<T>(ntab<T, 0>()));
  cudaFuncSetAttribute(k1k_cols<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, s);
  cudaFuncSetAttribute(k1k_rows_fwd<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<T>(ntab<T, 2>()));
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
  std::vector<cplx<T>> h(TTOT + (ctab<T>() ? NBAS : 0));
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
#ifdef COFEM_1K_TAB6
    put(TP + k, sck * std::conj(q1) * (1.0 + I * std::conj(hh)) / 2.0);
    put(TQ + k, sc * std::conj(q2) * (1.0 - I * std::conj(hh)) / 2.0);
    const C r1 = sk * q1 * (1.0 - I * hh) / 2.0, r2 = sk * q1 * (1.0 + I * hh) / 2.0;
    const C r3 = s * q2 * (1.0 + I * hh) / 2.0, r4 = s * q2 * (1.0 - I * hh) / 2.0;
    // lo = Re(Wk r1) + Re(conj(Wm) r2) = Wk.x r1.x - Wk.y r1.y + Wm.x r2.x + Wm.y r2.y
    put(TR1 + k, r1); put(TR2 + k, r2); put(TR3 + k, r3); put(TR4 + k, r4);
#else
    (void)sck; (void)sk; (void)s; (void)s0;
    put(TAB2 + ia(k), sc * q1 * (1.0 - I * hh) / 2.0);       // Ahat_k
    put(TAB2 + ib(k), sc * q2 * (1.0 + I * hh) / 2.0);       // Bhat_k
#endif
  }
#ifndef COFEM_1K_TAB6
  if (ctab<T>())     // per-lane bases u_k0 = (sc/2) e^{-i pi k0/2L}, v_k0 = (sc/2) e^{-5 i pi k0/2L}, k0 = ja | jb
    for (int lane = 0; lane < 32; ++lane) {
      const int ja = lane, jb = lane ? 64 - lane : 32;
      put(TTOT + lane, sc / 2.0 * e(-PI * ja / (2.0 * L)));
      put(TTOT + 32 + lane, sc / 2.0 * e(-5.0 * PI * ja / (2.0 * L)));
      put(TTOT + 64 + lane, sc / 2.0 * e(-PI * jb / (2.0 * L)));
      put(TTOT + 96 + lane, sc / 2.0 * e(-5.0 * PI * jb / (2.0 * L)));
    }
#endif
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
  if (cudaMalloc(&c->maskH, (size_t)L * 16 * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMalloc(&c->twh, (size_t)d1kh::TWTOT * sizeof(cplx<float>)) != cudaSuccess) {
    c->err = "cudaMalloc half-warp FFT tables"; return COFEM_ERR_OOM;
  }
  {   // W_512^{t k1} in both layouts of fft512h.cuh (fp64 -> fp32)
    std::vector<cplx<float>> hw(d1kh::TWTOT);
    const double PI = 3.14159265358979323846;
    for (int k1 = 0; k1 < 32; ++k1)
      for (int t = 0; t < 16; ++t) {
        const double ang = -2.0 * PI * t * k1 / 512.0;
        const cplx<float> w{(float)cos(ang), (float)sin(ang)};
        hw[d1kh::TWK + k1 * 16 + t] = w;
        hw[d1kh::TWT + t * 32 + k1] = w;
      }
    cudaMemcpy(c->twh, hw.data(), hw.size() * sizeof(hw[0]), cudaMemcpyHostToDevice);
  }
  launch_begin(c, KC_SETUP);
  k1k_mask_lanes<<<L * 32 / 256, 256, 0, c->stream>>>(c->mask_vvT, c->maskL);
  k1k_mask_half<<<L * 16 / 256, 256, 0, c->stream>>>(c->mask_vvT, (unsigned long long*)c->maskH);
  launch_end(c, KC_SETUP);
  cudaFuncSetAttribute(k1k_cols_h, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)colsh::SMEM);
  set_attrs<float>();
  set_attrs<double>();
  {   // dataflow probe kernel: dispenser state and rho' partials (allocated here: E-steps are captured)
    if (cudaMalloc(&c->flow_state, sizeof(flow::State)) != cudaSuccess ||
        cudaMalloc(&c->flow_part2, (size_t)c->m_cap * (c->Dp / VEC_TILE) * sizeof(double)) != cudaSuccess) {
      c->err = "cudaMalloc flow state"; return COFEM_ERR_OOM;
    }
    const size_t smb = (size_t)8 * WREG * sizeof(float) + (size_t)TTOT * sizeof(cplx<float>);
    cudaFuncSetAttribute(flow::k1k_flow, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb);
  }
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
#if COFEM_1K_INV_TMA
  if constexpr (sizeof(T) == 4) {
    const int items = ncols * rtma::NT;   // persistent: one CTA per SM (each warp prefetches its next row)
    int g = std::min(items, c->num_sms * COFEM_1K_TMA_CPS);
    if (j0 > 0 && c->probe_groups > 1) g = std::min(g, (c->num_sms * 120) / 148 * COFEM_1K_TMA_CPS);
    k1k_rows_inv_tma<<<std::max(1, g), rtma::RT * 32, rtma::smem_bytes(), st>>>(a, j0, ncols, dir ? 1 : 0);
  } else
#endif
  k1k_rows_inv<T><<<grid_of((const void*)k1k_rows_inv<T>, smem_bytes<T>(ntab<T, 0>())), blk, smem_bytes<T>(ntab<T, 0>()), st>>>(
      a, j0, ncols, dir ? 1 : 0);
  launch_end(c, mean ? KC_MEAN : KC_DCT_ROWS_INV, st);
  launch_begin(c, mean ? KC_MEAN : KC_DCT_COLS, st);
#ifdef COFEM_1K_COLS_HALF   // experiment build: the half-warp FFT column pass (measured slower)
  if constexpr (sizeof(T) == 4) {
    const int items = ncols * colsh::NTH;
    int g = grid_of((const void*)k1k_cols_h, colsh::SMEM);
    g = std::min(g, items);
    k1k_cols_h<<<std::max(1, g), 256, colsh::SMEM, st>>>(a, j0, ncols, (const unsigned long long*)c->maskH,
                                                         (const cplx<float>*)c->twh);
  } else
#endif
  k1k_cols<T><<<grid_of((const void*)k1k_cols<T>, sm), blk, sm, st>>>(a, j0, ncols);
  launch_end(c, mean ? KC_MEAN : KC_DCT_COLS, st);
  launch_begin(c, mean ? KC_MEAN : KC_DCT_ROWS_FWD, st);
  const size_t smf = smem_bytes<T>(ntab<T, 2>());
  k1k_rows_fwd<T><<<grid_of((const void*)k1k_rows_fwd<T>, smf), blk, smf, st>>>(a, j0, ncols);
  launch_end(c, mean ? KC_MEAN : KC_DCT_ROWS_FWD, st);
  return check_launch(c, "dct1k apply") == cudaSuccess ? COFEM_OK : COFEM_ERR_CUDA;
}

// Column groups of the dataflow kernel: 8 (groups of 4 at K = 32: two halves of 4 groups, so
// the four phase types of consecutive groups share the SMs), fewer when K is small
int dct1k_flow_groups(const Ctx* c, int K) {
  const int want = c->opt.probe_groups > 0 ? c->opt.probe_groups : 4;
  return std::max(1, std::min(K, std::min(want, d1k::flow::MAXG)));
}

// The whole CG loop of the fp32 probe columns as one k1k_flow launch on `st` (the state, the
// group s accumulators and the probe bits are ready; the mean column runs elsewhere).
cofem_status dct1k_flow(Ctx* c, int K, int K_total, cudaStream_t st) {
  using namespace d1k;
  using namespace d1k::flow;
  if (!c->flow_state) { c->err = "flow state not allocated"; return COFEM_ERR_CUDA; }   // dct1k_setup
  Args f;
  memset(&f, 0, sizeof f);
  f.st = (State*)c->flow_state; f.K = K; f.U = c->opt.cg_iters; f.ntiles = (int)(c->Dp / VEC_TILE);
  const int G = dct1k_flow_groups(c, K);
  f.G = G;
  for (int g = 0; g <= G; ++g) f.g0[g] = (int)((int64_t)K * g / G);
  f.H = G >= 2 ? 2 : 1;
  f.Gh = (G + f.H - 1) / f.H;
  f.VS = std::max(f.ntiles, ((K + G - 1) / G) * NT);
  f.step = (long long)f.H * f.Gh * f.VS;
  f.total = f.step * (4LL * f.U + G - 1);
  f.invK = 1.0 / (double)K_total;
  for (int g = 0; g < G; ++g) f.s[g] = g ? c->gs[g] : c->s;
  f.part2 = (double*)c->flow_part2;
  f.bits = c->bits; f.wpc = c->Dp / 32;
  f.dinvp = (const float*)c->dinvp;
  DctArgs a = dct_args(c, K + 1, 0);
  const size_t smb = (size_t)8 * WREG * sizeof(float) + (size_t)TTOT * sizeof(cplx<float>);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k1k_flow, FLOW_THREADS, smb);
  // leave room for the concurrent fp64 mean column (an eighth of the SMs, as the per-pass path)
#ifndef COFEM_FLOW_RESERVE
#define COFEM_FLOW_RESERVE (c->num_sms / 8)
#endif
  const int sms = c->skip_mean ? c->num_sms : c->num_sms - std::max(0, (int)(COFEM_FLOW_RESERVE));
  const int grid = std::max(1, sms * std::max(occ, 1));
  if (cudaMemsetAsync(c->flow_state, 0, sizeof(State), st) != cudaSuccess) { c->err = "memset flow state"; return COFEM_ERR_CUDA; }
  launch_begin(c, KC_DCT_FLOW, st);
  k1k_flow<<<grid, FLOW_THREADS, smb, st>>>(a, f);
  launch_end(c, KC_DCT_FLOW, st);
  return check_launch(c, "k1k_flow") == cudaSuccess ? COFEM_OK : COFEM_ERR_CUDA;
}

cofem_status dct1k_apply(Ctx* c, int j0, int j1, int iter, bool dir, cudaStream_t st) {
  if (j0 == 0 || c->probe64) return dct1k_apply_t<double>(c, j0, j1, iter, dir, st);
  return dct1k_apply_t<float>(c, j0, j1, iter, dir, st);
}

}  // namespace cofem
