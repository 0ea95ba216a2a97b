// fft512.cuh — one-warp 512-point complex FFT (a 1024-point real transform after
// even/odd packing) shared by the 1024 x 1024 DCT fast path (op_dct1k.cu) and the
// overlap-save circular convolution (op_conv_fft.cu).  Product code, sm_100a.
//
// Lane l owns radix-8 butterflies {l, 64 - l} (lane 0: {0, 32}) in the first and last
// Stockham stage, so spectral pairs (k, 512 - k) never leave the lane; the two
// warp-synchronous shared-memory exchanges use padded [r][j] layouts that are
// bank-conflict-free for 8-byte accesses.
#pragma once
#include "fft_common.cuh"

namespace cofem {
namespace d1k {

constexpr int L = 1024, M = 512;
constexpr int XS1 = 66, XS2 = 72;      // exchange row strides in complex entries (conflict-free 8-byte accesses)
constexpr int WREG = 2 * 8 * XS2;      // per-warp smem region (elements of T): exchange buffer / one tile row (>= L)
template <typename T> struct Geo { static constexpr int RT = sizeof(T) == 8 ? 4 : 8; };   // rows (warps) per CTA

// Tables, host-built in fp64 and rounded to T, copied to shared memory by every CTA in
// layouts where each warp access is conflict-free (lanes read consecutive entries):
//   w2[r*8 + k]  = W_64^{r k}      (FFT stage 2, k = lane & 7)
//   w3[r*64 + j] = W_512^{r j}     (FFT stage 3, j = butterfly)
//   DCT-III pre  (Makhoul):  W[k] = u1 P_k + u2 Q_k,  u1 = X[k] - i X[L-k], u2 = X[k+M] - i X[M-k]
//   DCT-II  post:            X[k]   = Re(W_k R1_k) + Re(conj(W_{M-k}) R2_k)
//                            X[k+M] = Re(W_k R3_k) + Re(conj(W_{M-k}) R4_k)
// with the orthonormal scales, the 1/M of the inverse FFT and the even/odd split folded in
// (k < M; the entries are derived in build_tables below).
#ifdef COFEM_1K_TAB6   // round-1 layout: six complex tables per k (P, Q pre; R1..R4 post)
constexpr int TW2 = 0, TW3 = 64, TP = TW3 + 512, TQ = TP + M, TR1 = TQ + M, TR2 = TR1 + M, TR3 = TR2 + M,
              TR4 = TR3 + M, TTOT = TR4 + M;   // offsets in complex entries
constexpr int TPRE = TR1;                      // pass A's prefix
#else                   // Ahat_k, Bhat_k (op_dct1k.cu build_tables): pre and post derive from them
constexpr int TW2 = 0, TW3 = 64, TAB2 = TW3 + 512, TTOT = TAB2 + 2 * M;
constexpr int TPRE = TTOT;
#ifdef COFEM_1K_AB_INTERLEAVE   // [A_0 B_0 A_1 B_1 ..]: one 16-byte load per k (measured +0.7 ms on C4)
__host__ __device__ constexpr int ia(int k) { return 2 * k; }
__host__ __device__ constexpr int ib(int k) { return 2 * k + 1; }
#else                           // [A_0 .. A_{M-1} | B_0 .. B_{M-1}]
__host__ __device__ constexpr int ia(int k) { return k; }
__host__ __device__ constexpr int ib(int k) { return M + k; }
#endif
#endif
// Computed Makhoul factors (fp32 per-pass kernels): Ahat_k = u_k - i v_k, Bhat_k = e^{-i pi/4}(u_k + i v_k)
// with u_k = (sc/2) e^{-i theta k}, v_k = (sc/2) e^{-5 i theta k}, theta = pi/2L; a lane's k are
// k0 + 64 r (k0 = ja or jb), so u_k = u_{k0} e^{-i pi r/32} and v_k = v_{k0} e^{-5 i pi r/32}: four
// per-lane bases [u_ja | v_ja | u_jb | v_jb][lane] replace the 2 x 512-entry tables in shared memory.
// The fp32 table holds them after the full layout (at TTOT); the kernels copy w2 | w3 | bases.
#if defined(COFEM_1K_TAB6)
#undef COFEM_1K_CTAB
#define COFEM_1K_CTAB 0
#endif
#ifndef COFEM_1K_CTAB
#define COFEM_1K_CTAB 0
#endif
constexpr int NBAS = 4 * 32;                 // per-lane bases (complex entries)
constexpr int TBAS = TW3 + 512;              // their offset in the compact shared-memory image
constexpr int TCT = TBAS + NBAS;             // entries of the compact image
// COFEM_1K_CTAB: bit PASS set = pass PASS (0 rows_inv, 1 cols, 2 rows_fwd) computes the factors (fp32)
template <typename T> __host__ __device__ constexpr bool ctab() { return COFEM_1K_CTAB != 0 && sizeof(T) == 4; }
template <typename T, int PASS> __host__ __device__ constexpr bool ctp() {
  return ((COFEM_1K_CTAB >> PASS) & 1) != 0 && sizeof(T) == 4;
}
template <typename T, int PASS> __host__ __device__ constexpr int ntab() {
  return ctp<T, PASS>() ? TCT : PASS == 0 ? TPRE : TTOT;
}
template <typename T> struct Tw { const cplx<T>* base; };

// Compact image for the computed-factor kernels: g[0, TBAS) then the bases g[TTOT, TTOT + NBAS).
template <typename T>
__device__ __forceinline__ Tw<T> load_tables_ct(const cplx<T>* __restrict__ g, cplx<T>* sm) {
  for (int i = threadIdx.x; i < TCT; i += blockDim.x) sm[i] = g[i < TBAS ? i : TTOT + (i - TBAS)];
  __syncthreads();
  return {sm};
}

template <typename T>
__device__ __forceinline__ Tw<T> load_tables(const cplx<T>* __restrict__ g, cplx<T>* sm, int n = TTOT) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = g[i];
  __syncthreads();
  return {sm};
}

template <typename T, int SIGN>
__device__ __forceinline__ void twid(cplx<T>& v, cplx<T> w) { v = SIGN < 0 ? cmul(v, w) : cmulc(v, w); }

// 512-point DFT (SIGN -1) / unnormalised inverse (SIGN +1) by one warp.
// In:  va[r] = x[ja + 64 r], vb[r] = x[jb + 64 r].  Out: va[r] = X[ja + 64 r], vb[r] = X[jb + 64 r].
// Stockham radix-8: stage s reads x[j + 64 r], twiddles by W_{8 Ns}^{r (j mod Ns)}, DFT8,
// writes y[(j / Ns) 8 Ns + (j mod Ns) + r Ns]; Ns = 1, 8, 64.  Exchanges store [r][j]
// (complex entries, row strides XS1 / XS2).
template <typename T, int SIGN>
__device__ __forceinline__ void fft512(cplx<T> (&va)[8], cplx<T> (&vb)[8], int lane, cplx<T>* __restrict__ x,
                                       const Tw<T>& tw) {
  const int ja = lane, jb = lane ? 64 - lane : 32;
  dft8<SIGN>(va); dft8<SIGN>(vb);                       // stage 1 (Ns = 1): butterflies ja, jb
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 8; ++r) { x[r * XS1 + ja] = va[r]; x[r * XS1 + jb] = vb[r]; }
  __syncwarp();
  {   // stage 2 (Ns = 8): butterflies lane, lane + 32; y[i] lives at [(i & 7)][i >> 3]
    const int base = (lane & 7) * XS1 + (lane >> 3);
#pragma unroll
    for (int r = 0; r < 8; ++r) { va[r] = x[base + 8 * r]; vb[r] = x[base + 4 + 8 * r]; }
    const cplx<T>* w2 = tw.base + TW2 + (lane & 7);
#pragma unroll
    for (int r = 1; r < 8; ++r) {
      const cplx<T> w = w2[r * 8];
      twid<T, SIGN>(va[r], w); twid<T, SIGN>(vb[r], w);
    }
  }
  dft8<SIGN>(va); dft8<SIGN>(vb);
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 8; ++r) { x[r * XS2 + lane] = va[r]; x[r * XS2 + lane + 32] = vb[r]; }
  __syncwarp();
  {   // stage 3 (Ns = 64): butterflies ja, jb; y'[i] written by j2 = 8 (i >> 6) + (i & 7), r2 = (i >> 3) & 7
    const int ba = (ja >> 3) * XS2 + (ja & 7), bb = (jb >> 3) * XS2 + (jb & 7);
#pragma unroll
    for (int r = 0; r < 8; ++r) { va[r] = x[ba + 8 * r]; vb[r] = x[bb + 8 * r]; }
    const cplx<T>* w3 = tw.base + TW3;
#ifdef COFEM_FFT_W3_TABLE
#pragma unroll
    for (int r = 1; r < 8; ++r) {
      twid<T, SIGN>(va[r], w3[r * 64 + ja]);
      twid<T, SIGN>(vb[r], w3[r * 64 + jb]);
    }
#else
    // W^{r jb} = W^{64 r} conj(W^{r ja}) = W_8^r conj(W^{r ja}) for jb = 64 - ja (lane > 0); lane 0's
    // jb = 32 twiddle W_16^r is a constant: one table load per r instead of two
    const T h = (T)0.70710678118654752440;
    constexpr double c16[8] = {1.0, 0.92387953251128675613, 0.70710678118654752440, 0.38268343236508977173, 0.0,
                               -0.38268343236508977173, -0.70710678118654752440, -0.92387953251128675613};
#pragma unroll
    for (int r = 1; r < 8; ++r) {
      const cplx<T> wa = w3[r * 64 + ja];
      cplx<T> wb;
      if (r == 1) wb = {h * (wa.x - wa.y), -h * (wa.x + wa.y)};          // W_8^r conj(wa), W_8 = e^{-i pi/4}
      else if (r == 2) wb = {-wa.y, -wa.x};
      else if (r == 3) wb = {-h * (wa.x + wa.y), h * (wa.y - wa.x)};
      else if (r == 4) wb = {-wa.x, wa.y};
      else if (r == 5) wb = {h * (wa.y - wa.x), h * (wa.x + wa.y)};
      else if (r == 6) wb = {wa.y, wa.x};
      else wb = {h * (wa.x + wa.y), h * (wa.x - wa.y)};
      if (lane == 0) wb = {(T)c16[r], -(T)c16[r <= 4 ? 4 - r : r - 4]};   // W_16^r = e^{-i pi r / 8}
      twid<T, SIGN>(va[r], wa);
      twid<T, SIGN>(vb[r], wb);
    }
#endif
  }
  dft8<SIGN>(va); dft8<SIGN>(vb);
  __syncwarp();                                         // exchange region free again
}

// Canonical positions of a lane in a 1024-long line: slot A r -> ja + 64r, B -> jb + 64r,
// C -> 512 + ja + 64r, E -> 512 + jb + 64r (r = 0..7): 32 distinct positions per lane,
// together the whole line; each load/store instruction is coalesced.
__device__ __forceinline__ void canon(int lane, int r, int (&o)[4]) {
  const int ja = lane, jb = lane ? 64 - lane : 32;
  o[0] = ja + 64 * r; o[1] = jb + 64 * r; o[2] = M + ja + 64 * r; o[3] = M + jb + 64 * r;
}

// Per-launch column info, read once per CTA: frozen flags and direction coefficients b_j
// (R5; a6); 1.5 KB of static shared memory.
struct ColFlags {
  int frozen[MAXM];
  double b[MAXM];
};
__device__ __forceinline__ void load_colinfo(ColFlags& ci, const ColState* cs, int j0, int ncols) {
  for (int jj = threadIdx.x; jj < ncols; jj += blockDim.x) {
    const ColState c = cs[j0 + jj];
    ci.frozen[jj] = c.frozen; ci.b[jj] = c.b;
  }
}

// True when some column of the launch is still active.  Each thread reads the entries it
// wrote in load_colinfo, so no barrier is needed before the vote.  A launch whose columns have
// all frozen (R5) returns before staging the tables: every CTA takes the same exit, so the
// last-CTA tickets are untouched.
__device__ __forceinline__ bool any_active(const ColFlags& ci, int ncols) {
  int act = 0;
  for (int jj = threadIdx.x; jj < ncols; jj += blockDim.x) act |= !ci.frozen[jj];
  return __syncthreads_or(act) != 0;
}

}  // namespace d1k
}  // namespace cofem
