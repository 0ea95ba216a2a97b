// op_conv_fft.cu — circular-convolution Gram apply by overlap-save FFT (BASELINE config 5;
// P:17; reading R12), fused with the CG direction update (a6):
//   p = M^-1 r + b p   (iterations > 0),   q = beta g * p + alpha o p,   gamma_j = p_j^T q_j
// g = autocorr(h) is the symmetric (2T-1)-tap Gram stencil (Phi^T Phi circulant).
//
// One warp owns one block of V = 896 outputs: it reads the 1024-sample window starting 64
// before the block (circularly), packs it as 512 complex points z[n] = w[2n] + i w[2n+1],
// runs the one-warp 512-point FFT (fft512.cuh), multiplies by the real window spectrum of g
// in packed form -- Z'[k] = A_k Z[k] + i B_k conj(Z[512-k]) with real A_k, B_k (derivation in
// build_conv_tables) -- and transforms back; outputs at window positions [64, 960) are exact
// (|l| <= 63 < 64).  The input window stays in registers, so q = beta y + alpha o p needs no
// reload of p.  Direct stencil (op_conv.cu) for D < 2048 or T > 64.
// The FFT work is ~4x below the direct 127-tap stencil's FP32 FMA count.
#include <math.h>

#include <algorithm>
#include <vector>

#include "fft512.cuh"

namespace cofem {
namespace cfft {

using namespace d1k;
constexpr int V = 896, HALO = 64;          // valid outputs per window, left halo
constexpr int TAB = TW3 + 512;             // conv coefficient table offset (after the FFT twiddles)
constexpr int TTOTC = TAB + M;             // entries: w2 (64) | w3 (512) | (A_k, B_k) (512)
constexpr int NW = 8;                      // warps (blocks) per CTA

struct ConvArgs {
  int64_t D, Dp; int ncols;
  double beta;
  const double* alpha; const float* alphap;
  // mean column (fp64); p is read from p0 and, with the direction update, written to p0n
  // (ping-pong buffers: overlapping windows read neighbouring blocks' old p)
  const double* p0; double* p0n; const double* r0; const double* dinv64; double* q0;
  // probe block
  const void* P; void* Pn; const void* R; const void* dinvp; void* Q;
  const void* tab32; const void* tab64;
  ColState* cs; double* part; int stride; unsigned* counter; int iter;
  // D-sharded mode: D is this rank's slice; samples outside [0, D) come from the received
  // halo records [side][r | p | dinv][64] (side 0: the 64 before, 1: the 64 after), and
  // per-column totals go to colsum (summed over ranks, then finished)
  const void* halo; const double* halo0; double* colsum;
  int64_t halo_side;   // elements between the side-0 and side-1 blocks of `halo` ([side][K][3][64])
};

template <typename T> struct CCol { const T* p; T* pn; const T* r; const T* dinv; const T* al; T* q; };
template <typename T> __device__ __forceinline__ CCol<T> ccol(const ConvArgs& a, int j) {
  if constexpr (sizeof(T) == 8) {
    if (j == 0) return {a.p0, a.p0n, a.r0, a.dinv64, a.alpha, a.q0};
  }
  const int64_t o = (int64_t)(j - 1) * a.Dp;
  const T* al;
  if constexpr (sizeof(T) == 8) al = a.alpha; else al = a.alphap;
  return {(const T*)a.P + o, (T*)a.Pn + o, (const T*)a.R + o, (const T*)a.dinvp, al, (T*)a.Q + o};
}

// two consecutive samples of the window (positions 2n, 2n+1 = packed point n), one 8- / 16-byte access
template <typename T> struct Vec2;
template <> struct Vec2<float> { using type = float2; };
template <> struct Vec2<double> { using type = double2; };

#ifndef COFEM_CONV_VEC
#define COFEM_CONV_VEC 1     // 0: every window through the general per-sample path (A/B switch)
#endif

#ifndef COFEM_CONV_RB
#define COFEM_CONV_RB 4      // vector path: window points per slot whose r and 1/diag loads are batched
                             // (C5 fixed-alpha E-step: 1 139.5 ms, 2 136.4, 4 135.2, 8 135.2; an L2
                             // prefetch of each warp's next window on top: 148 ms, not kept)
#endif

#ifndef COFEM_CONV_STASH
#define COFEM_CONV_STASH 0   // 1: fp32 interior windows keep the updated p of their valid outputs in shared memory (3 CTAs/SM: C5 196 -> 214 ms, not kept)
#endif
constexpr int STASH = 448;                 // complex points n in [32, 480): window positions [64, 960)
template <typename T>
#ifndef COFEM_CONV_MINB
#if COFEM_CONV_STASH
#define COFEM_CONV_MINB (sizeof(T) == 4 ? 3 : 2)   // fp32: 3 CTAs per SM (shared memory: the p stash)
#else
#define COFEM_CONV_MINB (sizeof(T) == 4 ? 4 : 2)   // fp32: 64 registers, 4 CTAs per SM (C5 228 -> 210 -> 196 ms; the gamma partials sized by the launch, not MAXM, make the 4th CTA fit)
#endif
#endif
__global__ void __launch_bounds__(NW * 32, COFEM_CONV_MINB) k_conv_fft(ConvArgs a, int j0, int dir) {
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sm = reinterpret_cast<T*>(smraw);
  // column flags in static shared memory; the per-warp gamma partials g[NW][ncols] after the
  // tables in dynamic shared memory, sized by the launch's columns (not MAXM)
  __shared__ struct { int frozen[MAXM]; double b[MAXM]; } ci;
  double* gsm = reinterpret_cast<double*>(smraw + NW * WREG * sizeof(T) + TTOTC * sizeof(cplx<T>));
  // fp32: per-warp stash of the window's updated p at its valid outputs (after the gamma partials)
  float2* stash = reinterpret_cast<float2*>(gsm + NW * a.ncols) + (threadIdx.x >> 5) * STASH;
  int act = 0;
  for (int jj = threadIdx.x; jj < a.ncols; jj += blockDim.x) {
    const ColState c = a.cs[j0 + jj];
    ci.frozen[jj] = c.frozen; ci.b[jj] = c.b;
    act |= !c.frozen;
    for (int w = 0; w < NW; ++w) gsm[w * a.ncols + jj] = 0.0;
  }
  // every column frozen (R5): all CTAs exit alike; sharded runs feed a cross-rank sum
  if (!__syncthreads_or(act) && !a.colsum) return;
  const cplx<T>* gtab = reinterpret_cast<const cplx<T>*>(sizeof(T) == 8 ? a.tab64 : a.tab32);
  const Tw<T> tb = load_tables<T>(gtab, reinterpret_cast<cplx<T>*>(sm + NW * WREG), TTOTC);   // + barrier
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ja = lane, jb = lane ? 64 - lane : 32;
  const bool l0 = lane == 0;
  const int64_t nblk = (a.D + V - 1) / V;
  const int64_t ngrp = (nblk + NW - 1) / NW;
  T* reg = sm + warp * WREG;
  // work items column-fastest: the CTAs in flight cover a narrow range of block groups over
  // all columns, so the shared 1/diag and alpha windows (64 MB each at D = 2^24) are read
  // from HBM about once per apply instead of once per column (L2 hits for the others)
  for (int64_t w = blockIdx.x; w < (int64_t)a.ncols * ngrp; w += gridDim.x) {
    const int jj = (int)(w % a.ncols);
    if (ci.frozen[jj]) continue;                                        // CTA-uniform
    const int j = j0 + jj;
    const int64_t blk = (w / a.ncols) * NW + warp;
    if (blk >= nblk) continue;                                          // warp-uniform
    const CCol<T> c = ccol<T>(a, j);
    const int64_t o0 = blk * V, w0 = o0 - HALO;                         // outputs [o0, o0+V), window [w0, w0+1024)
    const int nvalid = (int)min((int64_t)V, a.D - o0);
    const bool fast = w0 >= 0 && w0 + L <= a.D;
    // fp32 interior window with V valid outputs: p kept in the stash, 8-byte stores / alpha loads
    const bool st2 = COFEM_CONV_STASH && sizeof(T) == 4 && fast && !a.halo && nvalid == V;
    if (st2 && lane < 28)                                               // alpha of the outputs -> L2 (3.5 KB)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(c.al + o0 + 32 * lane));
    const T* hal = nullptr;                                             // this column's halo records (sharded)
    int64_t hside = 0;
    if (a.halo) {
      if constexpr (sizeof(T) == 8) {
        if (j == 0) { hal = a.halo0; hside = 192; }
        else { hal = (const T*)a.halo + (int64_t)(j - 1) * 192; hside = a.halo_side; }
      } else { hal = (const T*)a.halo + (int64_t)(j - 1) * 192; hside = a.halo_side; }
    }
    const T bb = (T)ci.b[jj];
    // interior window of a full block (no wrap, no halo records, V valid outputs): packed point n
    // is one vector access at w0 + 2n; the valid outputs [64, 960) are the points n in [32, 480):
    // slot a (n = ja + 64 r) for r >= 1, slot b (n = jb + 64 r) for r <= 6, for every lane.  The
    // pointers do not alias (P / Pn ping-pong, R, 1/diag, alpha, Q), so loads of later points are
    // issued ahead of earlier points' stores (the general path below serialises them).
    using V2 = typename Vec2<T>::type;
    const bool vfast = COFEM_CONV_VEC && !COFEM_CONV_STASH && fast && !hal && nvalid == V;
    cplx<T> va[8], vb[8];
    if (vfast) {
      const V2* __restrict__ p2 = reinterpret_cast<const V2*>(c.p + w0);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const V2 xa = p2[ja + 64 * r], xb = p2[jb + 64 * r];
        va[r] = {xa.x, xa.y}; vb[r] = {xb.x, xb.y};
      }
      if (dir) {                                                        // a6: p = M^-1 r + b p
        const V2* __restrict__ r2 = reinterpret_cast<const V2*>(c.r + w0);
        const V2* __restrict__ d2 = reinterpret_cast<const V2*>(c.dinv + w0);
        V2* __restrict__ pn2 = reinterpret_cast<V2*>(c.pn + w0);
        // r and 1/diag in batches of RB points per slot, all of a batch's loads before its stores
        constexpr int RB = COFEM_CONV_RB;
#pragma unroll
        for (int h = 0; h < 8; h += RB) {
          V2 ra[RB], da[RB], rb[RB], db[RB];
#pragma unroll
          for (int i = 0; i < RB; ++i) {
            ra[i] = r2[ja + 64 * (h + i)]; da[i] = d2[ja + 64 * (h + i)];
            rb[i] = r2[jb + 64 * (h + i)]; db[i] = d2[jb + 64 * (h + i)];
          }
#pragma unroll
          for (int i = 0; i < RB; ++i) {
            const int r = h + i;
            va[r].x = da[i].x * ra[i].x + bb * va[r].x; va[r].y = da[i].y * ra[i].y + bb * va[r].y;
            vb[r].x = db[i].x * rb[i].x + bb * vb[r].x; vb[r].y = db[i].y * rb[i].y + bb * vb[r].y;
            if (r >= 1) { V2 o; o.x = va[r].x; o.y = va[r].y; pn2[ja + 64 * r] = o; }   // own positions only
            if (r <= 6) { V2 o; o.x = vb[r].x; o.y = vb[r].y; pn2[jb + 64 * r] = o; }
          }
        }
      }
    } else
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int sl = 0; sl < 2; ++sl) {
        const int n = (sl ? jb : ja) + 64 * r;
        T x0, x1;
        int64_t i0, i1;
        if (fast) { i0 = w0 + 2 * n; i1 = i0 + 1; }
        else {
          i0 = (w0 + 2 * n) % a.D; if (i0 < 0) i0 += a.D;
          i1 = i0 + 1 == a.D ? 0 : i0 + 1;
        }
        if (!fast && hal) {                                             // sharded edge window: halo records
          const int64_t wi = w0 + 2 * n;
          T v2[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int64_t i = wi + e;
            T pv, rv, dv;
            if (i >= 0 && i < a.D) { pv = c.p[i]; rv = c.r[i]; dv = c.dinv[i]; }
            else if (i < 0 && i >= -64) { const T* h = hal + (64 + i); rv = h[0]; pv = h[64]; dv = h[128]; }
            else if (i >= a.D && i < a.D + 64) { const T* h = hal + hside + (i - a.D); rv = h[0]; pv = h[64]; dv = h[128]; }
            else { pv = 0; rv = 0; dv = 0; }                          // beyond the halo: affects invalid outputs only
            v2[e] = dir ? dv * rv + bb * pv : pv;
          }
          x0 = v2[0]; x1 = v2[1];
        } else {
          if (fast && sizeof(T) == 4) {
            const float2 v = *reinterpret_cast<const float2*>(c.p + i0);
            x0 = (T)v.x; x1 = (T)v.y;
          } else { x0 = c.p[i0]; x1 = c.p[i1]; }
          if (dir) {                                                    // a6: p = M^-1 r + b p
            x0 = c.dinv[i0] * c.r[i0] + bb * x0;
            x1 = c.dinv[i1] * c.r[i1] + bb * x1;
          }
        }
        if (sl) vb[r] = {x0, x1}; else va[r] = {x0, x1};
      }
    }
    if (vfast) {
    } else if (st2) {                // valid outputs: stash p (same lane reads it back), p_new as float2
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int sl = 0; sl < 2; ++sl) {
          const int n = (sl ? jb : ja) + 64 * r;
          if (n >= 32 && n < 32 + STASH) {
            const cplx<T> v = sl ? vb[r] : va[r];
            stash[n - 32] = make_float2((float)v.x, (float)v.y);
            if (dir) *reinterpret_cast<float2*>(c.pn + o0 + 2 * n - HALO) = make_float2((float)v.x, (float)v.y);
          }
        }
    } else if (dir) {                // the direction update is stored by the block that owns the position
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int sl = 0; sl < 2; ++sl) {
          const int n = (sl ? jb : ja) + 64 * r;
          const cplx<T> v = sl ? vb[r] : va[r];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int pos = 2 * n + e;
            if (pos >= HALO && pos < HALO + nvalid) c.pn[o0 + pos - HALO] = e ? v.y : v.x;
          }
        }
    }
    fft512<T, -1>(va, vb, lane, reinterpret_cast<cplx<T>*>(reg), tb);
    // ---- spectral product in packed form: Z'[k] = A_k Z[k] + i B_k conj(Z[(512 - k) mod 512])
    {
      cplx<T> na[8], nb[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const cplx<T> zka = va[r], zma = l0 ? va[(8 - r) & 7] : vb[7 - r];     // k = ja + 64 r
        const cplx<T> zkb = vb[r], zmb = l0 ? vb[7 - r] : va[7 - r];           // k = jb + 64 r
        const cplx<T> ca = tb.base[TAB + ja + 64 * r], cb = tb.base[TAB + jb + 64 * r];
        na[r] = {ca.x * zka.x + ca.y * zma.y, ca.x * zka.y + ca.y * zma.x};
        nb[r] = {cb.x * zkb.x + cb.y * zmb.y, cb.x * zkb.y + cb.y * zmb.x};
      }
#pragma unroll
      for (int r = 0; r < 8; ++r) { va[r] = na[r]; vb[r] = nb[r]; }
    }
    fft512<T, +1>(va, vb, lane, reinterpret_cast<cplx<T>*>(reg), tb);  // y[2n] + i y[2n+1] (1/512 folded in)
    // ---- epilogue: q = beta y + alpha o p at the valid positions, gamma partial
    const T beta = (T)a.beta;
    const T* pcur = dir ? c.pn : c.p;                                   // p of this iteration (own block: just written)
    double g = 0.0;
    if (vfast) {                     // vector epilogue over the 14 valid (r, slot) pairs of every lane
      const V2* __restrict__ pc2 = reinterpret_cast<const V2*>(pcur + w0);
      const V2* __restrict__ al2 = reinterpret_cast<const V2*>(c.al + w0);
      V2* __restrict__ q2 = reinterpret_cast<V2*>(c.q + w0);
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int sl = 0; sl < 2; ++sl) {
          if (sl ? r > 6 : r < 1) continue;
          const int n = (sl ? jb : ja) + 64 * r;
          const cplx<T> y = sl ? vb[r] : va[r];
          const V2 pv = pc2[n], av = al2[n];
          V2 qv;
          qv.x = beta * y.x + av.x * pv.x; qv.y = beta * y.y + av.y * pv.y;          // a3
          q2[n] = qv;
          g += (double)pv.x * (double)qv.x + (double)pv.y * (double)qv.y;            // a4
        }
    } else if (st2) {                // p from the stash, alpha / q as float2
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int sl = 0; sl < 2; ++sl) {
          const int n = (sl ? jb : ja) + 64 * r;
          if (n >= 32 && n < 32 + STASH) {
            const cplx<T> y = sl ? vb[r] : va[r];
            const int64_t i = o0 + 2 * n - HALO;
            const float2 pv = stash[n - 32];
            const float2 av = *reinterpret_cast<const float2*>(c.al + i);
            const float q0 = (float)beta * (float)y.x + av.x * pv.x, q1 = (float)beta * (float)y.y + av.y * pv.y;   // a3
            *reinterpret_cast<float2*>(c.q + i) = make_float2(q0, q1);
            g += (double)pv.x * (double)q0 + (double)pv.y * (double)q1;                                           // a4
          }
        }
    } else
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int sl = 0; sl < 2; ++sl) {
        const int n = (sl ? jb : ja) + 64 * r;
        const cplx<T> y = sl ? vb[r] : va[r];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int pos = 2 * n + e;
          if (pos >= HALO && pos < HALO + nvalid) {
            const int64_t i = o0 + pos - HALO;
            const T pv = pcur[i];
            const T qv = beta * (e ? y.y : y.x) + c.al[i] * pv;         // a3
            c.q[i] = qv;
            g += (double)pv * (double)qv;                               // a4
          }
        }
      }
    g = warp_sum(g);
    if (lane == 0) gsm[warp * a.ncols + jj] += g;
  }
  // gamma_j: CTA partials (fixed warp order) -> part[j][cta]; the last CTA reduces (R5)
  __syncthreads();
  for (int jj = threadIdx.x; jj < a.ncols; jj += blockDim.x) {
    double v = 0.0;
#pragma unroll
    for (int ww = 0; ww < NW; ++ww) v += gsm[ww * a.ncols + jj];
    a.part[(int64_t)(j0 + jj) * a.stride + blockIdx.x] = v;
  }
  __threadfence();
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(a.counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int jj = warp; jj < a.ncols; jj += NW) {
    const int j = j0 + jj;
    const double tot = reduce_partials(a.part + (int64_t)j * a.stride, gridDim.x);
    if (lane == 0) {
      if (a.colsum) a.colsum[j] = tot;                                  // sharded: summed over ranks, then finished
      else if (!ci.frozen[jj]) { ColState cc = a.cs[j]; finish_gamma(cc, tot, a.iter); a.cs[j] = cc; }
    }
  }
  if (threadIdx.x == 0) *a.counter = 0u;
}

// Tables: FFT twiddles (fft512.cuh layout) and the packed-domain conv coefficients.
// With X = DFT_1024(window), the circular window convolution is Y = G o X, G_k =
// sum_{|l| < T} g_l e^{-2 pi i k l / 1024} (real: g symmetric).  With E_k, O_k the DFTs of the
// even / odd samples (Z = E + i O, E_k = (Z_k + conj Z_{M-k}) / 2, O_k = (Z_k - conj Z_{M-k}) / 2i),
// X_k = E_k + W^k O_k, X_{k+M} = E_k - W^k O_k (W = e^{-2 pi i/1024}), and the packed inverse
// Z'_k = E'_k + i O'_k with E' = (Y_k + Y_{k+M})/2, O' = (Y_k - Y_{k+M}) W^{-k}/2 gives
//   Z'_k = (S_k - D_k sin th_k) Z_k + i D_k cos th_k conj(Z_{M-k}),
// S_k = (G_k + G_{k+M})/2, D_k = (G_k - G_{k+M})/2, th_k = 2 pi k / 1024; the inverse FFT's 1/512
// is folded into A_k = (S_k - D_k sin th_k)/512 and B_k = D_k cos th_k / 512.
template <typename T> static std::vector<cplx<T>> build_conv_tables(const std::vector<double>& g, int H) {
  using namespace d1k;
  const double PI = 3.14159265358979323846;
  std::vector<cplx<T>> h(TTOTC);
  auto put = [&](int i, double re, double im) { h[i] = cplx<T>{(T)re, (T)im}; };
  for (int r = 0; r < 8; ++r)
    for (int k = 0; k < 8; ++k) put(TW2 + r * 8 + k, cos(-2 * PI * r * k / 64.0), sin(-2 * PI * r * k / 64.0));
  for (int r = 0; r < 8; ++r)
    for (int jj = 0; jj < 64; ++jj) put(TW3 + r * 64 + jj, cos(-2 * PI * r * jj / 512.0), sin(-2 * PI * r * jj / 512.0));
  std::vector<double> G(L);
  for (int k = 0; k < L; ++k) {
    double v = g[H];
    for (int l = 1; l <= H; ++l) v += 2.0 * g[H + l] * cos(2 * PI * (double)k * l / L);
    G[k] = v;
  }
  for (int k = 0; k < M; ++k) {
    const double S = 0.5 * (G[k] + G[k + M]), Dk = 0.5 * (G[k] - G[k + M]), th = 2 * PI * k / L;
    put(TAB + k, (S - Dk * sin(th)) / M, Dk * cos(th) / M);
  }
  return h;
}

template <typename T> static size_t smem_bytes(int ncols) {
  return (size_t)NW * WREG * sizeof(T) + (size_t)TTOTC * sizeof(cplx<T>) + (size_t)NW * ncols * sizeof(double) +
         (COFEM_CONV_STASH && sizeof(T) == 4 ? (size_t)NW * STASH * sizeof(float2) : 0);
}

}  // namespace cfft

// Halo records of every column ([side][column][r | p | dinv][64]): side 0 = this rank's first
// 64 samples (the left neighbour's right halo), side 1 = its last 64 (the right neighbour's
// left halo).  Probe columns in probe precision, the mean column in its own fp64 buffer.
template <typename T>
__global__ void k_conv_pack_halo(int64_t D, int64_t Dp, const T* __restrict__ R, const T* __restrict__ P,
                                 const T* __restrict__ dinv, T* __restrict__ out, int64_t side_stride,
                                 const double* __restrict__ r0, const double* __restrict__ p0,
                                 const double* __restrict__ dinv64, double* __restrict__ out0) {
  const int j = blockIdx.x;                 // 0: mean column, 1..K probes
  for (int t = threadIdx.x; t < 2 * 64; t += blockDim.x) {
    const int side = t >> 6, e = t & 63;
    const int64_t i = side ? D - 64 + e : e;
    if (j == 0) {
      double* o = out0 + side * 192 + e;
      o[0] = r0[i]; o[64] = p0[i]; o[128] = dinv64[i];
    } else {
      T* o = out + side * side_stride + (int64_t)(j - 1) * 192 + e;
      const int64_t b = (int64_t)(j - 1) * Dp + i;
      o[0] = R[b]; o[64] = P[b]; o[128] = dinv[i];
    }
  }
}

// Pack and exchange the halo records of all K + 1 columns with both ring neighbours (one
// NCCL group per precision), on the context stream.
cofem_status conv_halo_exchange(Ctx* c, int K) {
  const int64_t side = (int64_t)c->Kcap * 192;
  if (c->probe64)
    k_conv_pack_halo<double><<<K + 1, 128, 0, c->stream>>>(c->D, c->Dp, (const double*)c->R, (const double*)c->P,
                                                           (const double*)c->dinvp, (double*)c->halo_send, side, c->r0,
                                                           c->p0, c->dinv64, c->halo_send0);
  else
    k_conv_pack_halo<float><<<K + 1, 128, 0, c->stream>>>(c->D, c->Dp, (const float*)c->R, (const float*)c->P,
                                                          (const float*)c->dinvp, (float*)c->halo_send, side, c->r0,
                                                          c->p0, c->dinv64, c->halo_send0);
  if (check_launch(c, "k_conv_pack_halo")) return COFEM_ERR_CUDA;
  const size_t tp = c->probe64 ? 8 : 4;
  char* sp = (char*)c->halo_send;
  char* rp = (char*)c->halo_recv;
  // the probe halos (probe precision) and the mean column's (fp64): one NCCL group, one launch
  cofem_status st = comm_group(c, true);
  if (st != COFEM_OK) return st;
  st = comm_halo(c, sp, sp + side * tp, rp, rp + side * tp, (size_t)K * 192, c->probe64 ? 1 : 0);
  if (st == COFEM_OK) st = comm_halo(c, c->halo_send0, c->halo_send0 + 192, c->halo_recv0, c->halo_recv0 + 192, 192, 1);
  const cofem_status st2 = comm_group(c, false);
  return st != COFEM_OK ? st : st2;
}

bool conv_fft_eligible(const Ctx* c) { return c->D >= 2048 && c->ntaps <= 64 && c->opt.apply_path != 1; }

cofem_status conv_fft_setup(Ctx* c, const std::vector<double>& g) {
  using namespace cfft;
  const int H = c->ntaps - 1;
  auto h32 = build_conv_tables<float>(g, H);
  auto h64 = build_conv_tables<double>(g, H);
  if (cudaMalloc(&c->conv_tab32, h32.size() * sizeof(h32[0])) != cudaSuccess ||
      cudaMalloc(&c->conv_tab64, h64.size() * sizeof(h64[0])) != cudaSuccess) { c->err = "cudaMalloc conv tables"; return COFEM_ERR_OOM; }
  cudaMemcpy(c->conv_tab32, h32.data(), h32.size() * sizeof(h32[0]), cudaMemcpyHostToDevice);
  cudaMemcpy(c->conv_tab64, h64.data(), h64.size() * sizeof(h64[0]), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_conv_fft<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<float>(MAXM));
  cudaFuncSetAttribute(k_conv_fft<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes<double>(MAXM));
  c->part_stride = std::max(c->part_stride, c->num_sms * 8);
  return check_launch(c, "conv fft setup") == cudaSuccess ? COFEM_OK : COFEM_ERR_CUDA;
}

// Columns [j0, j1) of one precision (the fp64 mean column alone, or the probes) on stream st.
cofem_status conv_fft_apply(Ctx* c, int j0, int j1, int iter, bool dir, cudaStream_t st) {
  using namespace cfft;
  ConvArgs a;
  a.D = c->D; a.Dp = c->Dp; a.ncols = j1 - j0; a.beta = c->beta;
  a.alpha = c->alpha; a.alphap = (const float*)c->alphap;
  a.p0 = c->p0; a.p0n = c->p0b; a.r0 = c->r0; a.dinv64 = c->dinv64; a.q0 = c->q0;
  a.P = c->P; a.Pn = c->Pb; a.R = c->R; a.dinvp = c->dinvp; a.Q = c->Q;
  a.tab32 = c->conv_tab32; a.tab64 = c->conv_tab64;
  a.cs = c->cs; a.part = c->part; a.stride = c->part_stride; a.iter = iter;
  a.counter = c->counters + MAXM + 2 + (j0 == 0 ? 1 : 0);
  a.halo = c->sharded ? c->halo_recv : nullptr; a.halo0 = c->sharded ? c->halo_recv0 : nullptr;
  a.halo_side = (int64_t)c->Kcap * 192;
  a.colsum = c->sharded ? c->colsum : nullptr;
  const bool f64 = j0 == 0 || c->probe64;
  const void* fn = f64 ? (const void*)k_conv_fft<double> : (const void*)k_conv_fft<float>;
  const size_t sm = f64 ? smem_bytes<double>(a.ncols) : smem_bytes<float>(a.ncols);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, NW * 32, sm);
  const int64_t items = (int64_t)a.ncols * (((c->D + V - 1) / V + NW - 1) / NW);
  const int grid = (int)std::min<int64_t>(std::min<int64_t>((int64_t)c->num_sms * std::max(occ, 1), items), c->part_stride);
  const int cls = j0 == 0 ? KC_MEAN : KC_CONV_APPLY;
  launch_begin(c, cls, st);
  if (f64) k_conv_fft<double><<<grid, NW * 32, sm, st>>>(a, j0, dir ? 1 : 0);
  else k_conv_fft<float><<<grid, NW * 32, sm, st>>>(a, j0, dir ? 1 : 0);
  launch_end(c, cls, st);
  if (dir) {      // the direction update went to the other buffer: it is the current p from now on
    if (j0 == 0) std::swap(c->p0, c->p0b);
    else std::swap(c->P, c->Pb);
  }
  return check_launch(c, "k_conv_fft") == cudaSuccess ? COFEM_OK : COFEM_ERR_CUDA;
}

}  // namespace cofem
