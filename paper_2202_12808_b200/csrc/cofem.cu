// cofem.cu — C ABI, context, fused CG vector kernels and the E-step / EM driver.
//
// Paper map: Algorithm 1; Eq. 5 b0; Eq. 6 s
// (P:74-78); Eq. 7 batched system; Eq. 8 M-step; CG §3.2
// (P:96-98).  Readings R2-R9 are listed in DESIGN.md §3.
//
// Data layout in HBM: every column is a contiguous D-vector
// padded to Dp (multiple of 2048, zero padding).  Column 0 (mean system) is
// fp64 in its own arrays x0/r0/p0/q0; probe columns 1..K are a [K][Dp] block
// in probe precision TP (fp32 fast / fp64 parity).  The probe x_k are never
// stored: s accumulates (a_k/K) p_k o p_k^(i) every iteration (x_k = sum_i a_k p_k^(i)).
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges for profilers (no cost without a tool)

#include "internal.cuh"

namespace cofem {

static const char* kClassNames[KC_COUNT] = {
    "probe_bits", "pcg_init", "pcg_direction", "pcg_update", "finalize_mstep",
    "dense_phi_p", "dense_phiT_w", "dct_rows_inv", "dct_cols", "dct_rows_fwd",
    "conv_apply", "mean_column", "setup", "dct_flow", "dense_cluster"};

// ------------------------------------------------------------------ bookkeeping
static cudaEvent_t pool_get(Ctx* c) {
  if (!c->ev_pool.empty()) { cudaEvent_t e = c->ev_pool.back(); c->ev_pool.pop_back(); return e; }
  cudaEvent_t e; cudaEventCreate(&e); return e;
}

void launch_begin(Ctx* c, int cls, cudaStream_t st) {
  if (c->prof_mask & (1u << cls)) {
    if (!st) st = c->stream;
    Ctx::Rec r{cls, pool_get(c), pool_get(c), st};
    cudaEventRecord(r.a, st);
    c->prof_recs.push_back(r);
  }
}

void launch_end(Ctx* c, int cls, cudaStream_t st) {
  c->launches++;
  if (c->prof_mask & (1u << cls)) {
    if (!st) st = c->stream;
    // the matching begin is the last record of this stream
    for (auto it = c->prof_recs.rbegin(); it != c->prof_recs.rend(); ++it)
      if (it->st == st) { cudaEventRecord(it->b, st); break; }
  }
}

cudaError_t check_launch(Ctx* c, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) c->err = std::string(what) + ": " + cudaGetErrorString(e);
  return e;
}

static void prof_collect(Ctx* c) {
  if (c->prof_recs.empty()) return;
  if (c->side) cudaStreamSynchronize(c->side);
  for (int g = 1; g < Ctx::MAXG; ++g) if (c->gstream[g]) cudaStreamSynchronize(c->gstream[g]);
  cudaStreamSynchronize(c->stream);
  std::vector<std::vector<std::pair<float, float>>> iv(KC_COUNT);
  const cudaEvent_t ref = c->prof_recs.front().a;
  for (auto& r : c->prof_recs) {
    float ms = 0; cudaEventElapsedTime(&ms, r.a, r.b);
    c->prof_ms[r.cls] += ms; c->prof_cnt[r.cls] += 1;
    float t0 = 0; cudaEventElapsedTime(&t0, ref, r.a);        // may be negative (other streams)
    iv[r.cls].push_back({t0, t0 + ms});
  }
  for (int k = 0; k < KC_COUNT; ++k) {   // busy time = measure of the union of the intervals
    auto& v = iv[k];
    std::sort(v.begin(), v.end());
    double busy = 0; float lo = 0, hi = 0; bool open = false;
    for (auto& x : v) {
      if (!open || x.first > hi) { if (open) busy += hi - lo; lo = x.first; hi = x.second; open = true; }
      else hi = std::max(hi, x.second);
    }
    if (open) busy += hi - lo;
    c->prof_busy[k] += busy;
  }
  for (auto& r : c->prof_recs) { c->ev_pool.push_back(r.a); c->ev_pool.push_back(r.b); }
  c->prof_recs.clear();
}

// ------------------------------------------------------------------ vector kernels
template <typename TP>
struct VecArgs {
  int64_t D, Dp; int K; int m; int64_t wpc;
  double beta; int precond;
  const double* alpha; const double* colsq; const double* b0;
  double* dinv64; TP* dinvp; TP* alphap;
  int jlo, jhi;     // columns [jlo, jhi) processed by k_update (0 = mean system)
  double *x0, *r0, *p0, *q0;
  TP *R, *P, *Q;
  double* s;
  const uint32_t* bits;
  ColState* cs; double* part; int part_stride; unsigned* counter;
  double invK;
  double* colsum;   // sharded mode: per-column totals go here (summed over ranks, then finished)
  double tau;       // freeze threshold on rho / rho0 (ColState::tau)
  int uchunks;      // k_update: probe columns split into uchunks chunks per D tile (1 = all in one item)
  int mean_grid;    // k_update: CTAs [0, mean_grid) update the mean column, tile stride mean_grid
  int warm;         // k_init: the mean column starts from x0 (= mu of the previous E-step; q0 = A x0)
  int nofinish;     // k_update: no rho' reduction (single-reduction CG, R23: rho' came with gamma)
  double* s_part; unsigned* tile_cnt;
  float *Ph, *Pl;   // k_dir (tensor-core dense path): also write the tf32 hi / lo halves of the new P
  int spersist;     // k_update chunks: s_part[chunk] accumulates over the whole E-step (k_sum_chunks adds
                    // them to s at its end) instead of the per-iteration ticketed chunk sum
};

// Probe-stream parameters of the current E-step, read from device memory so that one
// captured CUDA graph serves every E-step (R8: key = seed, counter = (d/128, k, t, tag)).
struct ProbeParams { uint32_t kx, ky; int t, k_offset; long long blk_offset; };   // blk_offset: d_offset / 128
__global__ void k_set_probe_params(ProbeParams* p, ProbeParams v) { *p = v; }

__global__ void k_probe_bits(uint32_t* __restrict__ bits, int64_t wpc, int K, int64_t nblk128,
                             const ProbeParams* __restrict__ pp) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)K * nblk128) return;
  const ProbeParams prm = *pp;
  int k = (int)(idx / nblk128);
  int64_t b = idx - (int64_t)k * nblk128;
  uint4 w = philox4x32_10(make_uint4((uint32_t)(b + prm.blk_offset), (uint32_t)(prm.k_offset + k), (uint32_t)prm.t, PROBE_TAG),
                          make_uint2(prm.kx, prm.ky));
  *reinterpret_cast<uint4*>(bits + (int64_t)k * wpc + b * 4) = w;
}

template <typename T> __device__ __forceinline__ void ld8(const T* p, T (&v)[8]) {
#pragma unroll
  for (int e = 0; e < 8; ++e) v[e] = p[e];
}
template <> __device__ __forceinline__ void ld8<float>(const float* p, float (&v)[8]) {
  float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
template <> __device__ __forceinline__ void ld8<double>(const double* p, double (&v)[8]) {
#pragma unroll
  for (int e = 0; e < 4; ++e) { double2 a = reinterpret_cast<const double2*>(p)[e]; v[2 * e] = a.x; v[2 * e + 1] = a.y; }
}
template <typename T> __device__ __forceinline__ void st8(T* p, const T (&v)[8]);
template <> __device__ __forceinline__ void st8<float>(float* p, const float (&v)[8]) {
  reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}
template <> __device__ __forceinline__ void st8<double>(double* p, const double (&v)[8]) {
#pragma unroll
  for (int e = 0; e < 4; ++e) reinterpret_cast<double2*>(p)[e] = make_double2(v[2 * e], v[2 * e + 1]);
}

// Per-CTA reduction scratch: red[warp][column]; only warp w writes row w (deterministic).
struct VecShared {
  double red[VEC_THREADS / 32][MAXM + 1];   // + k_init's warm-start slot
  double a[MAXM];
  int act[MAXM];
  bool last;
};

// After the tile loop: CTA partials -> part[j][bx]; the last CTA reduces them in fixed
// order and applies `fin(j, sum)` (one warp per column).
template <typename Fin>
__device__ void vec_finish(VecShared& sh, double* part, int stride, unsigned* counter, int jlo, int jhi, Fin fin) {
  __syncthreads();
  for (int j = jlo + threadIdx.x; j < jhi; j += blockDim.x) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < VEC_THREADS / 32; ++w) v += sh.red[w][j];
    part[(int64_t)j * stride + blockIdx.x] = v;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) sh.last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!sh.last) return;
  __threadfence();
  int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = jlo + warp; j < jhi; j += nw) {
    double v = reduce_partials(part + (int64_t)j * stride, gridDim.x);
    if ((threadIdx.x & 31) == 0) fin(j, v);
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// a2: X = 0, R = B, Z = M^-1 R, P = Z, rho = R^T Z; diag(A) = beta colsq + alpha (R6); s = 0.
template <typename TP>
__global__ void __launch_bounds__(VEC_THREADS) k_init(VecArgs<TP> a) {
  __shared__ VecShared sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = threadIdx.x; j <= a.m; j += blockDim.x)
    for (int w = 0; w < VEC_THREADS / 32; ++w) sh.red[w][j] = 0.0;
  __syncthreads();
  const int64_t ntiles = a.Dp / VEC_TILE;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t d0 = tile * VEC_TILE + (int64_t)threadIdx.x * VEC_ELEMS;
    double dv[8], al[8], cq[8], bb[8];
    ld8(a.alpha + d0, al); ld8(a.colsq + d0, cq); ld8(a.b0 + d0, bb);
    TP dp[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      bool valid = d0 + e < a.D;
      double diag = a.beta * cq[e] + al[e];
      dv[e] = valid ? (a.precond ? 1.0 / diag : 1.0) : 0.0;
      dp[e] = (TP)dv[e];
    }
    st8(a.dinv64 + d0, dv); st8(a.dinvp + d0, dp);
    {
      TP ap[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) ap[e] = (TP)al[e];
      st8(a.alphap + d0, ap);
    }
    double z8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    st8(a.s + d0, z8);
    double p8[8], acc = 0.0, acc_b = 0.0;
    if (a.warm) {                  // R20: r0 = b0 - A x0 (q0 holds A x0); rho0 stays b0^T M^-1 b0
      double q8[8];
      ld8(a.q0 + d0, q8);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        acc_b += bb[e] * (dv[e] * bb[e]);
        bb[e] = bb[e] - q8[e];
      }
    } else {
      st8(a.x0 + d0, z8);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) { p8[e] = dv[e] * bb[e]; acc += bb[e] * p8[e]; }
    st8(a.r0 + d0, bb); st8(a.p0 + d0, p8);
    acc = warp_sum(acc);
    if (lane == 0) sh.red[warp][0] += acc;
    if (a.warm) {
      acc_b = warp_sum(acc_b);
      if (lane == 0) sh.red[warp][a.m] += acc_b;          // spare slot m: the cold rho0 of column 0
    }
    for (int k = 0; k < a.K; ++k) {
      uint32_t w = (a.bits[(int64_t)k * a.wpc + (d0 >> 5)] >> (d0 & 31)) & 0xffu;
      TP r[8], p[8];
      double acck = 0.0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        bool valid = d0 + e < a.D;
        r[e] = valid ? (((w >> e) & 1u) ? (TP)-1 : (TP)1) : (TP)0;
        p[e] = dp[e] * r[e];
        acck += (double)r[e] * (double)p[e];
      }
      st8(a.R + (int64_t)k * a.Dp + d0, r); st8(a.P + (int64_t)k * a.Dp + d0, p);
      acck = warp_sum(acck);
      if (lane == 0) sh.red[warp][k + 1] += acck;
    }
  }
  ColState* cs = a.cs;
  double* colsum = a.colsum;
  const double tau = a.tau;
  if (!a.warm) {
    vec_finish(sh, a.part, a.part_stride, a.counter, 0, a.m, [cs, colsum, tau](int j, double v) {
      if (colsum) { colsum[j] = v; return; }
      ColState c; c.rho = v; c.rho0 = v; c.gamma = 0; c.a = 0; c.b = 0;
      c.frozen = 0; c.frozen_at = -1; c.nonfinite = 0; c.pad = 0; c.tau = tau;
      cs[j] = c;
    });
    return;
  }
  // warm start (R20; never sharded): columns [0, m) plus the spare slot m with column 0's cold
  // rho0 = b0^T M^-1 b0, reduced by the warp that finishes column 0 (fixed order)
  __syncthreads();
  for (int j = threadIdx.x; j <= a.m; j += blockDim.x) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < VEC_THREADS / 32; ++w) v += sh.red[w][j];
    a.part[(int64_t)j * a.part_stride + blockIdx.x] = v;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) sh.last = (atomicAdd(a.counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!sh.last) return;
  __threadfence();
  for (int j = warp; j < a.m; j += VEC_THREADS / 32) {
    const double v = reduce_partials(a.part + (int64_t)j * a.part_stride, gridDim.x);
    const double v0 = j == 0 ? reduce_partials(a.part + (int64_t)a.m * a.part_stride, gridDim.x) : v;
    if (lane == 0) {
      ColState c; c.rho = v; c.rho0 = v0; c.gamma = 0; c.a = 0; c.b = 0;
      c.frozen = 0; c.frozen_at = -1; c.nonfinite = 0; c.pad = 0; c.tau = tau;
      cs[j] = c;
    }
  }
  if (threadIdx.x == 0) *a.counter = 0u;
}

// a5: r -= a q; x0 += a0 p0; s += (a_k/K) p_k o P_k; z = M^-1 r; rho' = r^T z; then
// (last CTA) b = rho'/rho, rho = rho'.
#ifndef COFEM_UPD_MINB
#define COFEM_UPD_MINB 3   // two-column kernel: 3 CTAs per SM (85 registers, 64 B spill): C5 217 -> 209.5 ms; 4: 215
#endif
template <typename TP, int UNR>
#ifndef COFEM_UPD1_MINB
#define COFEM_UPD1_MINB 3   // one-column kernel: 80 registers, 3 CTAs per SM (with min-blocks 1 nvcc took 208: C4 53.5 vs 47.7 ms)
#endif
__global__ void __launch_bounds__(VEC_THREADS, UNR == 2 ? COFEM_UPD_MINB : COFEM_UPD1_MINB) k_update(VecArgs<TP> a) {
  __shared__ VecShared sh;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = a.jlo + threadIdx.x; j < a.jhi; j += blockDim.x) {
    ColState c = a.cs[j];
    sh.act[j] = !c.frozen;
    sh.a[j] = c.a;
    for (int w = 0; w < VEC_THREADS / 32; ++w) sh.red[w][j] = 0.0;
  }
  {   // every column of the range frozen (R5): nothing to do (each thread votes on the entries
      // it wrote; all CTAs exit alike, so the tickets stay untouched).  Sharded runs always
      // finish, their column sums feed a cross-rank reduction.
    int act = 0;
    for (int j = a.jlo + threadIdx.x; j < a.jhi; j += blockDim.x) act |= sh.act[j];
    if (!__syncthreads_or(act) && (!a.colsum || a.nofinish)) return;
  }
  const int64_t ntiles = a.Dp / VEC_TILE;
  const int klo = a.jlo > 0 ? a.jlo - 1 : 0, khi = a.jhi - 1;
  // work item = (D tile, chunk of the probe columns); uchunks > 1 only when D is small
  const int ncol = khi - klo, csz = ncol > 0 ? (ncol + a.uchunks - 1) / a.uchunks : 1;
  const int nch = ncol > 0 ? (ncol + csz - 1) / csz : 1;
  // the fp64 mean column over the tiles with the vec_grid stride, whatever the chunking: its
  // rho' partials (and so mu) do not depend on K or max_probes
  if (a.jlo == 0 && sh.act[0] && blockIdx.x < a.mean_grid) {
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += a.mean_grid) {
      const int64_t d0 = tile * VEC_TILE + (int64_t)threadIdx.x * VEC_ELEMS;
      const double a0 = sh.a[0];
      double x[8], r[8], p[8], q[8], dv[8], acc = 0.0;
      ld8(a.x0 + d0, x); ld8(a.r0 + d0, r); ld8(a.p0 + d0, p); ld8(a.q0 + d0, q); ld8(a.dinv64 + d0, dv);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        x[e] = fma(a0, p[e], x[e]);
        r[e] = fma(-a0, q[e], r[e]);
        acc += r[e] * (dv[e] * r[e]);
      }
      st8(a.x0 + d0, x); st8(a.r0 + d0, r);
      acc = warp_sum(acc);
      if (lane == 0) sh.red[warp][0] += acc;
    }
  }
  // probe columns (none in the mean-column launch, jlo = 0, jhi = 1: dinvp is then not read —
  // it holds probe-precision values, Dp floats with fp32 probes)
  for (int64_t item = blockIdx.x; ncol > 0 && item < ntiles * nch; item += gridDim.x) {
    const int64_t tile = item / nch;
    const int chunk = (int)(item % nch);
    const int64_t d0 = tile * VEC_TILE + (int64_t)threadIdx.x * VEC_ELEMS;
    TP dp[8];
    ld8(a.dinvp + d0, dp);
    double sacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    bool any = false;
    const int k1 = min(khi, klo + (chunk + 1) * csz);
    // UNR columns per step: their loads are issued before any of their arithmetic (the
    // per-column operations and the order of the s sums do not depend on UNR)
    for (int k = klo + chunk * csz; k < k1; k += UNR) {
      bool act[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) act[u] = k + u < k1 && sh.act[k + u + 1];   // warp-uniform
      // one-column steps (the concurrent-group DCT path): L2 prefetch of the next column's lines,
      // one 128-byte line per 4 threads (C4 50.2 -> 49.7 ms; the two-column kernel is slower with it)
      if (UNR == 1 && (threadIdx.x & 3) == 0 && k + 1 < k1) {
        const int64_t o = (int64_t)(k + 1) * a.Dp + d0;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.R + o));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.Q + o));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.P + o));
      }
      TP r[UNR][8], q[UNR][8], p[UNR][8];
      uint32_t w[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        w[u] = 0u;
        if (!act[u]) continue;
        const int64_t o = (int64_t)(k + u) * a.Dp + d0;
        ld8(a.R + o, r[u]); ld8(a.Q + o, q[u]); ld8(a.P + o, p[u]);
        w[u] = (a.bits[(int64_t)(k + u) * a.wpc + (d0 >> 5)] >> (d0 & 31)) & 0xffu;
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        if (!act[u]) continue;
        any = true;
        const double ak = sh.a[k + u + 1];
        const TP akt = (TP)ak;
        const double aks = ak * a.invK;
        double acc = 0.0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          r[u][e] = r[u][e] - akt * q[u][e];
          TP z = dp[e] * r[u][e];
          acc += (double)r[u][e] * (double)z;
          double pe = (double)p[u][e];
          sacc[e] += ((w[u] >> e) & 1u) ? -aks * pe : aks * pe;
        }
        st8(a.R + (int64_t)(k + u) * a.Dp + d0, r[u]);
        acc = warp_sum(acc);
        if (lane == 0) sh.red[warp][k + u + 1] += acc;
      }
    }
    if (nch > 1 && a.spersist) {      // this (tile, chunk) item owns s_part[chunk] on the tile: plain RMW
      if (any) {
        double sv[8];
        double* sp = a.s_part + (int64_t)chunk * a.Dp + d0;
        ld8(sp, sv);
#pragma unroll
        for (int e = 0; e < 8; ++e) sv[e] += sacc[e];
        st8(sp, sv);
      }
    } else if (nch == 1) {
      if (any) {
        double sv[8];
        ld8(a.s + d0, sv);
#pragma unroll
        for (int e = 0; e < 8; ++e) sv[e] += sacc[e];
        st8(a.s + d0, sv);
      }
    } else {   // chunk partials; the tile's last chunk adds them to s in chunk order (deterministic)
      st8(a.s_part + (int64_t)chunk * a.Dp + d0, sacc);
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) sh.last = atomicAdd(a.tile_cnt + tile, 1u) == (unsigned)nch - 1;
      __syncthreads();
      if (sh.last) {
        __threadfence();
        double sv[8];
        ld8(a.s + d0, sv);
        for (int ch = 0; ch < nch; ++ch) {
          double pv[8];
          ld8(a.s_part + (int64_t)ch * a.Dp + d0, pv);
#pragma unroll
          for (int e = 0; e < 8; ++e) sv[e] += pv[e];
        }
        st8(a.s + d0, sv);
        if (threadIdx.x == 0) a.tile_cnt[tile] = 0u;
      }
      __syncthreads();
    }
  }
  if (a.nofinish) return;            // single-reduction CG (R23): b and rho' are already in cs
  ColState* cs = a.cs;
  double* colsum = a.colsum;
  vec_finish(sh, a.part, a.part_stride, a.counter, a.jlo, a.jhi, [cs, colsum](int j, double v) {
    if (colsum) { colsum[j] = v; return; }
    ColState c = cs[j];
    if (c.frozen) return;
    c.b = v / c.rho;
    c.rho = v;
    cs[j] = c;
  });
}

// End of an E-step whose k_update accumulated s per column chunk (VecArgs::spersist): s += sum of
// the chunk accumulators in chunk order (deterministic), which are zeroed for the next E-step.
__global__ void k_sum_chunks(int64_t Dp, int nch, double* __restrict__ s, double* __restrict__ s_part) {
  for (int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; d < Dp; d += (int64_t)gridDim.x * blockDim.x) {
    double v = s[d];
    for (int c = 0; c < nch; ++c) { v += s_part[(int64_t)c * Dp + d]; s_part[(int64_t)c * Dp + d] = 0.0; }
    s[d] = v;
  }
}

// a6: P_j = M^-1 R_j + b_j P_j  (separate kernel for dense / conv; fused into DCT pass A).
template <typename TP>
__global__ void __launch_bounds__(VEC_THREADS) k_dir(VecArgs<TP> a) {
  const int j = blockIdx.y;
  const ColState c = a.cs[j];
  if (c.frozen) return;
  const int64_t ntiles = a.Dp / VEC_TILE;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t d0 = tile * VEC_TILE + (int64_t)threadIdx.x * VEC_ELEMS;
    if (j == 0) {
      double r[8], p[8], dv[8];
      ld8(a.r0 + d0, r); ld8(a.p0 + d0, p); ld8(a.dinv64 + d0, dv);
#pragma unroll
      for (int e = 0; e < 8; ++e) p[e] = fma(c.b, p[e], dv[e] * r[e]);
      st8(a.p0 + d0, p);
    } else {
      TP r[8], p[8], dv[8];
      TP* Pk = a.P + (int64_t)(j - 1) * a.Dp + d0;
      ld8(a.R + (int64_t)(j - 1) * a.Dp + d0, r); ld8(Pk, p); ld8(a.dinvp + d0, dv);
      const TP bt = (TP)c.b;
#pragma unroll
      for (int e = 0; e < 8; ++e) p[e] = dv[e] * r[e] + bt * p[e];
      st8(Pk, p);
      if constexpr (sizeof(TP) == 4) {
        if (a.Ph) {   // the next apply's B operand halves (k_tc_split_p's rule: hi = rna tf32, lo = p - hi)
          float h[8], l[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            uint32_t u;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"((float)p[e]));
            h[e] = __uint_as_float(u); l[e] = (float)p[e] - h[e];
          }
          st8(a.Ph + (int64_t)(j - 1) * a.Dp + d0, h); st8(a.Pl + (int64_t)(j - 1) * a.Dp + d0, l);
        }
      }
    }
  }
}

// a8 + a9: mu = x0, s, and (optionally) the M-step alpha = min(1/max(mu^2+s, floor), amax) (Eq. 8).
__global__ void k_finalize(int64_t D, const double* __restrict__ x0, const double* __restrict__ s,
                           double* __restrict__ mu_out, double* __restrict__ s_out, double* __restrict__ alpha_out,
                           double den_floor, double alpha_max) {
  for (int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; d < D; d += (int64_t)gridDim.x * blockDim.x) {
    double mu = x0[d], sv = s[d];
    if (mu_out) mu_out[d] = mu;
    if (s_out) s_out[d] = sv;
    if (alpha_out) alpha_out[d] = fmin(1.0 / fmax(mu * mu + sv, den_floor), alpha_max);
  }
}

__global__ void k_mstep(int64_t D, const double* __restrict__ mu, const double* __restrict__ s,
                        double* __restrict__ alpha_out, double den_floor, double alpha_max) {
  for (int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; d < D; d += (int64_t)gridDim.x * blockDim.x) {
    double m = mu[d];
    alpha_out[d] = fmin(1.0 / fmax(m * m + s[d], den_floor), alpha_max);
  }
}

__global__ void k_check_alpha(int64_t D, const double* __restrict__ alpha, int* __restrict__ bad) {
  for (int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; d < D; d += (int64_t)gridDim.x * blockDim.x) {
    double v = alpha[d];
    if (!(v > 0.0) || !isfinite(v)) atomicExch(bad, 1);
  }
}

// Support certificate (cofem_report.support_*): max|mu| (non-negative doubles order like their bit
// patterns, so an unsigned atomicMax on the bits is exact), then the counts and the smallest
// margin | |mu_d| / max - thr | (again as bit patterns, atomicMin).
struct SupportStats { unsigned long long maxbits, minmargin_bits, count, adjacent; };
__global__ void k_support_max(int64_t D, const double* __restrict__ mu, SupportStats* st) {
  double m = 0.0;
  for (int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; d < D; d += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(mu[d]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(&st->maxbits, (unsigned long long)__double_as_longlong(m));
}
__global__ void k_support_count(int64_t D, const double* __restrict__ mu, double thr, double delta, SupportStats* st) {
  const double mx = __longlong_as_double((long long)st->maxbits);
  unsigned long long cnt = 0, adj = 0;
  double mm = INFINITY;
  for (int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; d < D; d += (int64_t)gridDim.x * blockDim.x) {
    const double a = fabs(mu[d]);
    cnt += a > thr * mx;
    const double margin = mx > 0.0 ? fabs(a / mx - thr) : INFINITY;
    adj += margin < delta;
    mm = fmin(mm, margin);
  }
  for (int o = 16; o > 0; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    adj += __shfl_xor_sync(0xffffffffu, adj, o);
    mm = fmin(mm, __shfl_xor_sync(0xffffffffu, mm, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&st->count, cnt); atomicAdd(&st->adjacent, adj);
    atomicMin(&st->minmargin_bits, (unsigned long long)__double_as_longlong(mm));
  }
}

// Multi-task M-step (reading R22): alpha = 1 / (mean_l mu_l^2 + s), floored / clamped as Eq. 8 (R7).
// MU: L task means, [L][Dp]; the sum runs over l in order (deterministic).
__global__ void k_mstep_multi(int64_t D, int64_t Dp, int L, const double* __restrict__ MU, const double* __restrict__ s,
                              double* __restrict__ alpha_out, double den_floor, double alpha_max) {
  for (int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; d < D; d += (int64_t)gridDim.x * blockDim.x) {
    double den;
    if (L == 1) {                     // exactly k_finalize's expression (L = 1 is Algorithm 1)
      const double m = MU[d];
      den = m * m + s[d];
    } else {
      double acc = 0.0;
      for (int l = 0; l < L; ++l) { const double m = MU[(int64_t)l * Dp + d]; acc += m * m; }
      den = acc / (double)L + s[d];
    }
    alpha_out[d] = fmin(1.0 / fmax(den, den_floor), alpha_max);
  }
}

__global__ void k_add_vec(int64_t n, double* __restrict__ a, const double* __restrict__ b) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] += b[i];
}

// Warm start (R20): p0 = x0 (the previous mu) for one apply of the mean column; the probe columns
// are frozen for that apply (kernels skip them; k_init resets every column afterwards).
__global__ void k_warm_prep(int64_t D, const double* __restrict__ x0, double* __restrict__ p0, ColState* cs, int m) {
  for (int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; d < D; d += (int64_t)gridDim.x * blockDim.x)
    p0[d] = x0[d];
  if (blockIdx.x == 0)
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
      ColState c; c.rho = 1.0; c.rho0 = 1.0; c.gamma = 0; c.a = 0; c.b = 0;
      c.frozen = j > 0; c.frozen_at = j > 0 ? 0 : -1; c.nonfinite = 0; c.pad = 0; c.tau = FREEZE_TAU;
      cs[j] = c;
    }
}

// cofem_estep_probes: the mean system (column 0) is solved by another rank; freeze it at once.
__global__ void k_freeze_col0(ColState* cs) {
  if (threadIdx.x == 0) { cs[0].frozen = 1; cs[0].frozen_at = 0; }
}

// Sharded mode: apply the rank-summed per-column totals (same rules as the in-kernel finishes).
__global__ void k_sharded_finish(ColState* cs, const double* __restrict__ colsum, int m, int mode, int iter, double tau) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const double v = colsum[j];
  ColState c = cs[j];
  if (mode == 0) {
    c.rho = v; c.rho0 = v; c.gamma = 0; c.a = 0; c.b = 0; c.frozen = 0; c.frozen_at = -1; c.nonfinite = 0; c.pad = 0;
    c.tau = tau;
  } else if (mode == 1) {
    finish_gamma(c, v, iter);
  } else if (mode == 3) {            // single-reduction CG (R23): gamma, rho, delta1, delta2 -> a, rho', b
    if (c.frozen) return;
    c.rho = colsum[m + j];             // r^T M^-1 r of the current r (the recurrence below would drift)
    finish_gamma(c, v, iter);
    if (c.frozen) { cs[j] = c; return; }
    const double rn = c.rho - 2.0 * c.a * colsum[2 * m + j] + c.a * c.a * colsum[3 * m + j];
    c.b = rn / c.rho; c.rho = rn;
  } else {
    if (c.frozen) return;
    c.b = v / c.rho; c.rho = v;
  }
  cs[j] = c;
}

cofem_status sharded_finish(Ctx* c, int m, int mode, int iter) {
  cofem_status st = comm_allreduce(c, c->colsum, (size_t)(mode == 3 ? 4 * m : m), 1);
  if (st != COFEM_OK) return st;
  k_sharded_finish<<<1, 160, 0, c->stream>>>(c->cs, c->colsum, m, mode, iter, c->freeze_tau);
  return check_launch(c, "k_sharded_finish") == cudaSuccess ? COFEM_OK : COFEM_ERR_CUDA;
}

// Single-reduction CG (reading R23): rho_j = r_j^T M^-1 r_j and the two dots that give
// rho' = r'^T M^-1 r' of r' = r - a q without r' -- delta1_j = q_j^T M^-1 r_j, delta2_j =
// q_j^T M^-1 q_j -- over this rank's rows, fp64 sums; grid (x, m): CTA partials, the last CTA of
// column j reduces them in fixed order into colsum[m + j], colsum[2m + j], colsum[3m + j].  Frozen
// columns (R5) are skipped (their entries are not read).
template <typename TP>
__global__ void __launch_bounds__(VEC_THREADS) k_sr_dots(VecArgs<TP> a, double* __restrict__ part, unsigned* cnt,
                                                         int stride) {
  const int j = blockIdx.y;
  if (a.cs[j].frozen) return;          // the same for every CTA of the column
  __shared__ double red[VEC_THREADS / 32][3];
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double dr = 0.0, d1 = 0.0, d2 = 0.0;
  const int64_t ntiles = a.Dp / VEC_TILE;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t d0 = tile * VEC_TILE + (int64_t)threadIdx.x * VEC_ELEMS;
    if (j == 0) {
      double r[8], q[8], dv[8];
      ld8(a.r0 + d0, r); ld8(a.q0 + d0, q); ld8(a.dinv64 + d0, dv);
#pragma unroll
      for (int e = 0; e < 8; ++e) { const double z = dv[e] * q[e]; dr += r[e] * (dv[e] * r[e]); d1 += z * r[e]; d2 += z * q[e]; }
    } else {
      TP r[8], q[8], dv[8];
      const int64_t o = (int64_t)(j - 1) * a.Dp + d0;
      ld8(a.R + o, r); ld8(a.Q + o, q); ld8(a.dinvp + d0, dv);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const double z = (double)dv[e] * (double)q[e], re = (double)r[e];
        dr += re * ((double)dv[e] * re); d1 += z * re; d2 += z * (double)q[e];
      }
    }
  }
  dr = warp_sum(dr); d1 = warp_sum(d1); d2 = warp_sum(d2);
  if (lane == 0) { red[warp][0] = dr; red[warp][1] = d1; red[warp][2] = d2; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double v[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int w = 0; w < VEC_THREADS / 32; ++w) { v[0] += red[w][0]; v[1] += red[w][1]; v[2] += red[w][2]; }
#pragma unroll
    for (int i = 0; i < 3; ++i) part[(int64_t)(3 * j + i) * stride + blockIdx.x] = v[i];
    __threadfence();
    last = atomicAdd(cnt + j, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < 32) {
    double t[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) t[i] = reduce_partials(part + (int64_t)(3 * j + i) * stride, gridDim.x);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int i = 0; i < 3; ++i) a.colsum[(i + 1) * a.m + j] = t[i];
      cnt[j] = 0u;
    }
  }
}

template <typename TP>
static VecArgs<TP> vec_args(Ctx* c, int K, double invK) {
  VecArgs<TP> a;
  a.D = c->D; a.Dp = c->Dp; a.K = K; a.m = K + 1; a.wpc = c->Dp / 32;
  a.beta = c->beta; a.precond = c->opt.precond;
  a.alpha = c->alpha; a.colsq = c->colsq; a.b0 = c->b0;
  a.dinv64 = c->dinv64; a.dinvp = (TP*)c->dinvp; a.alphap = (TP*)c->alphap;
  a.jlo = 0; a.jhi = K + 1;
  a.x0 = c->x0; a.r0 = c->r0; a.p0 = c->p0; a.q0 = c->q0;
  a.R = (TP*)c->R; a.P = (TP*)c->P; a.Q = (TP*)c->Q;
  a.s = c->s; a.bits = c->bits;
  a.cs = c->cs; a.part = c->part; a.part_stride = c->part_stride; a.counter = c->counters + MAXM;
  a.invK = invK;
  a.colsum = c->sharded ? c->colsum : nullptr;
  a.tau = c->freeze_tau;
  a.uchunks = c->upd_chunks; a.s_part = c->s_part; a.tile_cnt = c->tile_cnt; a.mean_grid = c->vec_grid;
  a.warm = c->warm_now ? 1 : 0;
  a.nofinish = c->sr ? 1 : 0;
  a.spersist = 0;
  a.Ph = a.Pl = nullptr;
  return a;
}

cofem_status sr_dots(Ctx* c, int m) {
  const int64_t ntiles = c->Dp / VEC_TILE;
  const int gx = (int)std::max<int64_t>(1, std::min<int64_t>({ntiles, (int64_t)c->part_stride,
                                                              ((int64_t)c->num_sms * 4 + m - 1) / m}));
  const dim3 grid((unsigned)gx, (unsigned)m);
  launch_begin(c, KC_UPDATE);
  if (c->probe64) k_sr_dots<double><<<grid, VEC_THREADS, 0, c->stream>>>(vec_args<double>(c, m - 1, 0), c->sr_part, c->sr_cnt, c->part_stride);
  else k_sr_dots<float><<<grid, VEC_THREADS, 0, c->stream>>>(vec_args<float>(c, m - 1, 0), c->sr_part, c->sr_cnt, c->part_stride);
  launch_end(c, KC_UPDATE);
  return check_launch(c, "k_sr_dots") == cudaSuccess ? COFEM_OK : COFEM_ERR_CUDA;
}


cofem_status launch_dir(Ctx* c, int m) {
  int K = m - 1;
  dim3 grid((unsigned)std::min<int64_t>(c->Dp / VEC_TILE, (int64_t)c->num_sms * 4), m);
  launch_begin(c, KC_DIR);
  if (c->probe64) k_dir<double><<<grid, VEC_THREADS, 0, c->stream>>>(vec_args<double>(c, K, 0));
  else {
    VecArgs<float> va = vec_args<float>(c, K, 0);
#ifndef COFEM_DIR_SPLIT
#define COFEM_DIR_SPLIT 1    // A/B build switch: 0 = k_tc_split_p in every apply
#endif
    if (COFEM_DIR_SPLIT && c->kind == COFEM_OP_DENSE && c->dense_tc) {   // the next tensor-core apply skips its split
      dense_tc_p_split(c, &va.Ph, &va.Pl);
      c->p_presplit = va.Ph != nullptr;
    }
    k_dir<float><<<grid, VEC_THREADS, 0, c->stream>>>(va);
  }
  launch_end(c, KC_DIR);
  return check_launch(c, "k_dir") == cudaSuccess ? COFEM_OK : COFEM_ERR_CUDA;
}

// ------------------------------------------------------------------ helpers
static bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

#define CK(call)                                                              \
  do {                                                                        \
    cudaError_t _e = (call);                                                  \
    if (_e != cudaSuccess) {                                                  \
      c->err = std::string(#call) + ": " + cudaGetErrorString(_e);            \
      return _e == cudaErrorMemoryAllocation ? COFEM_ERR_OOM : COFEM_ERR_CUDA; \
    }                                                                         \
  } while (0)

template <typename T>
static cofem_status dalloc(Ctx* c, T** p, size_t n) {
  *p = nullptr;
  if (n == 0) n = 1;
  cudaError_t e = cudaMalloc((void**)p, n * sizeof(T));
  if (e != cudaSuccess) { c->err = std::string("cudaMalloc: ") + cudaGetErrorString(e); return COFEM_ERR_OOM; }
  e = cudaMemsetAsync(*p, 0, n * sizeof(T), c->stream);
  if (e != cudaSuccess) { c->err = cudaGetErrorString(e); return COFEM_ERR_CUDA; }
  return COFEM_OK;
}
#define ALLOC(p, n) do { cofem_status _s = dalloc(c, &(p), (n)); if (_s != COFEM_OK) return _s; } while (0)

// Stage a D-vector input: device pointers are used in place, host ones copied.
static cofem_status stage_in(Ctx* c, const double* src, double* dst_ws, const double** use) {
  if (is_device_ptr(src)) { *use = src; return COFEM_OK; }
  CK(cudaMemcpyAsync(dst_ws, src, c->D * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  *use = dst_ws;
  return COFEM_OK;
}

// alpha > 0 and finite (cofem.h): one check kernel into the flag allocated at setup, read back
// through pinned host memory (no allocation per call).  cofem_em checks only a caller-given
// alpha_init; the alphas of its own M-steps are positive and finite by construction (floor, clamp).
static cofem_status validate_alpha(Ctx* c, const double* alpha_dev) {
  CK(cudaMemsetAsync(c->bad_flag, 0, sizeof(int), c->stream));
  k_check_alpha<<<c->num_sms * 2, 256, 0, c->stream>>>(c->D, alpha_dev, c->bad_flag);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(c->bad_host, c->bad_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (*c->bad_host) { c->err = "alpha must be positive and finite"; return COFEM_ERR_INVALID; }
  return COFEM_OK;
}

// ------------------------------------------------------------------ E-step driver
// U PCG iterations of the 1024 x 1024 DCT fast path: the fp64 mean column (its three
// DCT passes and its update) runs on the side stream concurrently with the probe
// columns on the main stream; the columns are independent (reading R3), so the two
// chains only join at the end of the E-step.
template <typename TP>
static void update_range(Ctx* c, int K, double invK, int jlo, int jhi, unsigned* counter, cudaStream_t st, int cls,
                         double* s_acc = nullptr) {
  VecArgs<TP> a = vec_args<TP>(c, K, invK);
  a.jlo = jlo; a.jhi = jhi; a.counter = counter;
  if (s_acc) a.s = s_acc;
  launch_begin(c, cls, st);
  // two probe columns per step where the update runs alone (conv, dense: C5 242 -> 229 ms per
  // E-step); on the concurrent-group DCT path the lighter one-column kernel (126 vs 80
  // registers) shares the SMs better (C4 52.5 vs 53.6 ms).  Grids: the resident CTAs, 4 / 2 per SM
#ifndef COFEM_UPD_UNR
#define COFEM_UPD_UNR 0   // tuning build switch: force the one- (1) or two-column (2) update
#endif
  constexpr int unr_env = COFEM_UPD_UNR;
  const bool two = jlo >= 1 && jhi - jlo >= 2 && (unr_env ? unr_env == 2 : c->probe_groups <= 1);
  if (jlo == 0 && jhi == 1) k_update<TP, 1><<<c->vec_grid, VEC_THREADS, 0, st>>>(a);
  else if (!two) k_update<TP, 1><<<c->upd_grid, VEC_THREADS, 0, st>>>(a);
  else {
    static int occ2 = 0;            // resident CTAs per SM of the two-column kernel
    if (!occ2) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_update<TP, 2>, VEC_THREADS, 0);
    k_update<TP, 2><<<std::min(c->upd_grid, c->num_sms * std::max(occ2, 1)), VEC_THREADS, 0, st>>>(a);
  }
  launch_end(c, cls, st);
}

// Same for the overlap-save FFT convolution (both paths apply + update per column set).
typedef cofem_status (*SplitApply)(Ctx*, int, int, int, bool, cudaStream_t);
static cofem_status cg_loop_split(Ctx* c, int K, double invK, SplitApply apply) {
  const int m = K + 1;
  // the conv path ping-pongs p between two buffers; every E-step starts from the same
  // assignment (k_init rewrites p), which keeps a captured graph's pointers valid
  void* const P_entry = c->P; double* const p0_entry = c->p0;
  cudaStream_t ms = c->side;
  // fast DCT path: the probe columns run as G independent groups on G streams, so that one
  // group's issue-bound column pass overlaps another's bandwidth-bound passes (C4 fixed-alpha
  // E-step: G = 1 62.7 ms, G = 2 58.3 ms, 57.6 with each probe launch on ~80 % of the SMs;
  // G = 3 59.7, G = 4 61.6)
  const int groups = c->opt.probe_groups > 0 ? c->opt.probe_groups : 2;
  int G = c->fast1k ? std::max(1, std::min(4, groups)) : 1;
  const int gmin = 2;      // measured: groups of >= 2 columns help at every K
  while (G > 1 && ((m - 1) / G < gmin || !c->gs[G - 1])) --G;
  c->probe_groups = G;
  int gj[Ctx::MAXG + 1];
  for (int g = 0; g <= G; ++g) gj[g] = 1 + (int)((int64_t)(m - 1) * g / G);
  CK(cudaEventRecord(c->ev_fork, c->stream));
  CK(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
  for (int g = 1; g < G; ++g) {
    CK(cudaMemsetAsync(c->gs[g], 0, c->Dp * sizeof(double), c->stream));
  }
  if (G > 1) {
    CK(cudaEventRecord(c->ev_fork, c->stream));
    for (int g = 1; g < G; ++g) CK(cudaStreamWaitEvent(c->gstream[g], c->ev_fork, 0));
  }
#ifdef COFEM_EXP_NO_MEAN
  constexpr bool no_mean = true;     // timing experiment build only (results invalid)
#else
  constexpr bool no_mean = false;
#endif
  for (int it = 0; it < c->opt.cg_iters; ++it) {
    cofem_status st;
    if (!no_mean && !c->skip_mean) {
      if ((st = apply(c, 0, 1, it, it > 0, ms)) != COFEM_OK) return st;
      update_range<double>(c, K, invK, 0, 1, c->counters + MAXM + 1, ms, KC_MEAN);
    }
    for (int g = 0; g < G && m > 1; ++g) {          // m = 1: the mean system alone (R22)
      cudaStream_t gst = g ? c->gstream[g] : c->stream;
      unsigned* tk = g ? c->counters + 3 * MAXM + gj[g] : c->counters + MAXM;   // per-group tickets
      if ((st = apply(c, gj[g], gj[g + 1], it, it > 0, gst)) != COFEM_OK) return st;
#ifdef COFEM_EXP_NO_UPD   // timing experiment build only (results invalid): the probe update skipped
      continue;
#endif
      if (c->probe64) update_range<double>(c, K, invK, gj[g], gj[g + 1], tk, gst, KC_UPDATE, g ? c->gs[g] : nullptr);
      else update_range<float>(c, K, invK, gj[g], gj[g + 1], tk, gst, KC_UPDATE, g ? c->gs[g] : nullptr);
    }
    if (check_launch(c, "k_update")) return COFEM_ERR_CUDA;
  }
  CK(cudaEventRecord(c->ev_join, c->side));
  CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  for (int g = 1; g < G; ++g) {
    CK(cudaEventRecord(c->gjoin[g], c->gstream[g]));
    CK(cudaStreamWaitEvent(c->stream, c->gjoin[g], 0));
  }
  for (int g = 1; g < G; ++g) {   // s = s_0 + s_1 + ... in group order (deterministic)
    k_add_vec<<<c->vec_grid, VEC_THREADS, 0, c->stream>>>(c->Dp, c->s, c->gs[g]);
    if (check_launch(c, "k_add_vec")) return COFEM_ERR_CUDA;
  }
  if (c->P != P_entry) { c->Pb = c->P; c->P = P_entry; }
  if (c->p0 != p0_entry) { c->p0b = c->p0; c->p0 = p0_entry; }
  return COFEM_OK;
}

// 1024 x 1024 DCT path, fp32 probes: the probe columns' whole CG loop is one dataflow launch
// (op_dct1k.cu k1k_flow); the fp64 mean column runs its per-pass kernels on the side stream
// concurrently, and the group s accumulators are summed in group order at the end.
[[maybe_unused]] static cofem_status cg_loop_flow(Ctx* c, int K, int K_total, double invK) {
  const int G = dct1k_flow_groups(c, K);
  for (int g = 1; g < G; ++g)
    if (!c->gs[g]) { c->err = "flow: group accumulators missing"; return COFEM_ERR_CUDA; }
  CK(cudaEventRecord(c->ev_fork, c->stream));
  CK(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
  if (!c->skip_mean) {
    for (int it = 0; it < c->opt.cg_iters; ++it) {
      cofem_status st = dct1k_apply(c, 0, 1, it, it > 0, c->side);
      if (st != COFEM_OK) return st;
      update_range<double>(c, K, invK, 0, 1, c->counters + MAXM + 1, c->side, KC_MEAN);
    }
  }
  for (int g = 1; g < G; ++g) CK(cudaMemsetAsync(c->gs[g], 0, c->Dp * sizeof(double), c->stream));
  cofem_status st = dct1k_flow(c, K, K_total, c->stream);
  if (st != COFEM_OK) return st;
  CK(cudaEventRecord(c->ev_join, c->side));
  CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  for (int g = 1; g < G; ++g) {   // s = s_0 + s_1 + ... in group order (deterministic)
    k_add_vec<<<c->vec_grid, VEC_THREADS, 0, c->stream>>>(c->Dp, c->s, c->gs[g]);
    if (check_launch(c, "k_add_vec")) return COFEM_ERR_CUDA;
  }
  return COFEM_OK;
}

// Runs Alg. 1 lines 3-7 with alpha already in c->alpha.  No host sync inside.
static cofem_status cg_loop_conv_sharded(Ctx* c, int K, double invK);

// The device work of one E-step (probes .. end of the CG loop), enqueued on c->stream;
// the probe parameters are already in c->dparams.
static cofem_status estep_body(Ctx* c, int K, int K_total) {
  const int m = K + 1;
  const double invK = 1.0 / (double)K_total;
  const int64_t nblk128 = c->Dp / 128;
  {
    int64_t n = (int64_t)K * nblk128;
    if (n > 0) {       // K = 0: the mean system alone (multi-task EM, R22)
      launch_begin(c, KC_PROBES);
      k_probe_bits<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(c->bits, c->Dp / 32, K, nblk128,
                                                                        (const ProbeParams*)c->dparams);
      launch_end(c, KC_PROBES);
      if (check_launch(c, "k_probe_bits")) return COFEM_ERR_CUDA;
    }
  }
  if (c->warm_now) {   // R20 warm start: q0 = A x0 (x0 = mu of the previous E-step), then k_init uses it
    k_warm_prep<<<c->num_sms * 4, 256, 0, c->stream>>>(c->D, c->x0, c->p0, c->cs, m);
    if (check_launch(c, "k_warm_prep")) return COFEM_ERR_CUDA;
    cofem_status st;
    if (c->fast1k) st = dct1k_apply(c, 0, 1, 0, false, c->stream);
    else if (c->fast_conv) st = conv_fft_apply(c, 0, 1, 0, false, c->stream);
    else if (c->kind == COFEM_OP_DCT2_MASKED) st = dct_apply(c, m, 0, false);
    else if (c->kind == COFEM_OP_DENSE) st = dense_apply(c, m, 0);
    else st = conv_apply(c, m, 0);
    if (st != COFEM_OK) return st;
  }
  launch_begin(c, KC_INIT);
  if (c->probe64) k_init<double><<<c->vec_grid, VEC_THREADS, 0, c->stream>>>(vec_args<double>(c, K, invK));
  else k_init<float><<<c->vec_grid, VEC_THREADS, 0, c->stream>>>(vec_args<float>(c, K, invK));
  launch_end(c, KC_INIT);
  if (check_launch(c, "k_init")) return COFEM_ERR_CUDA;
  if (c->sharded) { cofem_status st = sharded_finish(c, m, 0, 0); if (st != COFEM_OK) return st; }
  if (c->skip_mean) k_freeze_col0<<<1, 32, 0, c->stream>>>(c->cs);   // every kernel skips a frozen column
#ifdef COFEM_1K_FLOW   // experiment build: the dataflow probe kernel (measured slower)
  if (c->fast1k && !c->probe64) return cg_loop_flow(c, K, K_total, invK);
#endif
  if (c->dense_cluster) return dense_cluster_cg(c, K, invK);
  if (c->fast1k) return cg_loop_split(c, K, invK, dct1k_apply);
  if (c->fast_conv && c->sharded) return cg_loop_conv_sharded(c, K, invK);
  if (c->fast_conv) return cg_loop_split(c, K, invK, conv_fft_apply);
  // small D with chunked probe updates: per-chunk s accumulators for the whole E-step
#ifndef COFEM_UPD_SPERSIST
#define COFEM_UPD_SPERSIST 1   // A/B build switch: 0 = the per-iteration ticketed chunk sum
#endif
  const int spersist = COFEM_UPD_SPERSIST && c->upd_chunks > 1 ? 1 : 0;   // s is rank-local in the sharded modes too
  for (int it = 0; it < c->opt.cg_iters; ++it) {
    cofem_status st;
    if (c->kind == COFEM_OP_DCT2_MASKED) {
      st = dct_apply(c, m, it, it > 0);
    } else {
      if (it > 0 && (st = launch_dir(c, m)) != COFEM_OK) return st;
      st = c->kind == COFEM_OP_DENSE ? dense_apply(c, m, it) : conv_apply(c, m, it);
    }
    if (st != COFEM_OK) return st;
    launch_begin(c, KC_UPDATE);
    if (c->probe64) {
      VecArgs<double> va = vec_args<double>(c, K, invK);
      va.spersist = spersist;
      k_update<double, 1><<<c->upd_grid, VEC_THREADS, 0, c->stream>>>(va);
    } else {
      VecArgs<float> va = vec_args<float>(c, K, invK);
      va.spersist = spersist;
      k_update<float, 1><<<c->upd_grid, VEC_THREADS, 0, c->stream>>>(va);
    }
    launch_end(c, KC_UPDATE);
    if (check_launch(c, "k_update")) return COFEM_ERR_CUDA;
    if (c->sharded && !c->sr && (st = sharded_finish(c, m, 2, it)) != COFEM_OK) return st;
  }
  if (spersist) {
    launch_begin(c, KC_UPDATE);
    k_sum_chunks<<<c->num_sms * 4, VEC_THREADS, 0, c->stream>>>(c->Dp, c->upd_chunks, c->s, c->s_part);
    launch_end(c, KC_UPDATE);
    if (check_launch(c, "k_sum_chunks")) return COFEM_ERR_CUDA;
  }
  return COFEM_OK;
}

// D-sharded convolution (BASELINE config 5): one stream (the NCCL calls must
// be ordered); per CG iteration: halo exchange of r, p, 1/diag with both ring neighbours,
// the FFT apply of the mean and the probe columns, the rank-sum of gamma, the update, the
// rank-sum of rho'.
static cofem_status cg_loop_conv_sharded(Ctx* c, int K, double invK) {
  const int m = K + 1;
  void* const P_entry = c->P; double* const p0_entry = c->p0;
  // the fp64 mean column's apply and update run on the side stream, concurrently with the probe
  // columns' (their tickets, partial rows and colsum entries are disjoint); the NCCL calls stay on
  // the context stream, after a join
  auto fork = [c]() -> cofem_status {
    CK(cudaEventRecord(c->ev_fork, c->stream));
    CK(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    return COFEM_OK;
  };
  auto join = [c]() -> cofem_status {
    CK(cudaEventRecord(c->ev_join, c->side));
    CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    return COFEM_OK;
  };
  for (int it = 0; it < c->opt.cg_iters; ++it) {
    cofem_status st;
    if ((st = conv_halo_exchange(c, K)) != COFEM_OK) return st;
    if ((st = fork()) != COFEM_OK) return st;
    if ((st = conv_fft_apply(c, 0, 1, it, it > 0, c->side)) != COFEM_OK) return st;
    if ((st = conv_fft_apply(c, 1, m, it, it > 0, c->stream)) != COFEM_OK) return st;
    if ((st = join()) != COFEM_OK) return st;
    if ((st = sharded_finish(c, m, 1, it)) != COFEM_OK) return st;
    if ((st = fork()) != COFEM_OK) return st;
    update_range<double>(c, K, invK, 0, 1, c->counters + MAXM + 1, c->side, KC_MEAN);
    if (c->probe64) update_range<double>(c, K, invK, 1, m, c->counters + MAXM, c->stream, KC_UPDATE);
    else update_range<float>(c, K, invK, 1, m, c->counters + MAXM, c->stream, KC_UPDATE);
    if (check_launch(c, "k_update")) return COFEM_ERR_CUDA;
    if ((st = join()) != COFEM_OK) return st;
    if ((st = sharded_finish(c, m, 2, it)) != COFEM_OK) return st;
  }
  if (c->P != P_entry) { c->Pb = c->P; c->P = P_entry; }
  if (c->p0 != p0_entry) { c->p0b = c->p0; c->p0 = p0_entry; }
  return COFEM_OK;
}

// Alg. 1 lines 3-7 on the device.  By default the whole E-step (both streams) is captured
// once per (K, K_total) into a CUDA graph and replayed: one launch per E-step instead of
// ~4-8 per CG iteration.  Per-kernel profiling (cofem_profile_enable)
// records events around every launch and therefore runs uncaptured.
static cofem_status estep_device(Ctx* c, int K, uint64_t seed, int t, int k_offset, int K_total) {
  ProbeParams pv{(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32), t, k_offset, (long long)(c->d_offset / 128)};
  k_set_probe_params<<<1, 1, 0, c->stream>>>((ProbeParams*)c->dparams, pv);
  CK(cudaGetLastError());
  if (!c->opt.use_graph || c->prof_mask) return estep_body(c, K, K_total);
  cudaStream_t user = c->stream;
  CK(cudaEventRecord(c->ev_in, user));
  CK(cudaStreamWaitEvent(c->work, c->ev_in, 0));
  c->stream = c->work;
  cofem_status st = COFEM_OK;
  Ctx::GraphSlot* gs = nullptr;
  for (auto& s : c->gslot)
    if (s.exec && s.K == K && s.Kt == K_total && s.skip == (int)c->skip_mean && s.warm == (int)c->warm_now) gs = &s;
  if (!gs) {           // capture into the least recently used slot
    gs = &c->gslot[0];
    for (auto& s : c->gslot) if (s.used < gs->used) gs = &s;
    if (gs->exec) { cudaGraphExecDestroy(gs->exec); gs->exec = nullptr; }
    const int64_t l0 = c->launches, n0 = c->collectives;
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamBeginCapture(c->work, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      st = estep_body(c, K, K_total);
      e = cudaStreamEndCapture(c->work, &g);
    }
    if (e == cudaSuccess && st == COFEM_OK) e = cudaGraphInstantiate(&gs->exec, g, 0);
    if (g) cudaGraphDestroy(g);
    gs->launches = c->launches - l0; gs->colls = c->collectives - n0;
    c->launches = l0; c->collectives = n0;
    if (e != cudaSuccess || st != COFEM_OK) {
      c->stream = user;
      if (st == COFEM_OK) { c->err = std::string("CUDA graph capture: ") + cudaGetErrorString(e); st = COFEM_ERR_CUDA; }
      if (gs->exec) { cudaGraphExecDestroy(gs->exec); gs->exec = nullptr; }
      return st;
    }
    gs->K = K; gs->Kt = K_total; gs->skip = (int)c->skip_mean; gs->warm = (int)c->warm_now;
  }
  gs->used = ++c->gclock;
  cudaError_t e = cudaGraphLaunch(gs->exec, c->work);
  c->launches += gs->launches; c->collectives += gs->colls;
  c->stream = user;
  if (e != cudaSuccess) { c->err = std::string("cudaGraphLaunch: ") + cudaGetErrorString(e); return COFEM_ERR_CUDA; }
  CK(cudaEventRecord(c->ev_out, c->work));
  CK(cudaStreamWaitEvent(user, c->ev_out, 0));
  return COFEM_OK;
}

// Probe-parallel mode (dist_mode 1): the owner split of the GLOBAL K over the ranks
// (paper_2202_12808_b200/dist.py probe_split_owner mirrors it on the host): rank 0 solves the mean
// system and K0 = max(1, min(K - (world - 1), floor((K + mc) / world - mc + 1/2))) probes, mc = the
// mean system's cost in probe columns (it runs concurrently with the probes: 2 on the DCT / FFT
// convolution paths, 0 on the dense tensor-core path where it rides in the same kernels);
// ranks 1.. split the other K - K0 contiguously.
static void split_owner(int K, int W, int r, double mc, int* k_off, int* K_loc, bool* owns) {
  if (W == 1) { *k_off = 0; *K_loc = K; *owns = true; return; }
  const int K0 = std::max(1, std::min(K - (W - 1), (int)floor((K + mc) / W - mc + 0.5)));
  if (r == 0) { *k_off = 0; *K_loc = K0; *owns = true; return; }
  const int rest = K - K0, base = rest / (W - 1), extra = rest % (W - 1), q = r - 1;
  *K_loc = base + (q < extra ? 1 : 0);
  *k_off = K0 + q * base + std::min(q, extra);
  *owns = false;
}
static void pp_split(const Ctx* c, int K, int* k_off, int* K_loc, bool* owns) {
  split_owner(K, c->world, c->rank, c->pp_mean_cost, k_off, K_loc, owns);
}

// One E-step of the probe-parallel mode: this rank's probes (global indices, R8) and, on rank 0,
// the mean system; then s (this rank's partial (1/K) sum, Eq. 6) is summed over the ranks and
// mu = x0 is broadcast from rank 0 -- one all-reduce + one broadcast of D fp64 per E-step, both
// enqueued on the context stream.  Afterwards every rank holds the same x0 and s.
static cofem_status estep_pp(Ctx* c, int K, uint64_t seed, int t, int* K_loc) {
  int off, kl; bool owns;
  pp_split(c, K, &off, &kl, &owns);
  *K_loc = kl;
  c->skip_mean = !owns;
  cofem_status st = estep_device(c, kl, seed, t, off, K);
  c->skip_mean = false;
  if (st != COFEM_OK) return st;
  if ((st = comm_allreduce(c, c->s, (size_t)c->D, 1)) != COFEM_OK) return st;
  return comm_bcast(c, c->x0, (size_t)c->D, 1, 0);
}

static cofem_status check_K(Ctx* c, int K) {
  if (!c->pp) {
    if (K < 1 || K > c->Kcap) { c->err = "K must be in [1, max_probes] (S:148)"; return COFEM_ERR_INVALID; }
    return COFEM_OK;
  }
  if (K < c->world) { c->err = "probe-parallel: K must be >= world (every rank solves >= 1 probe)"; return COFEM_ERR_INVALID; }
  int off, kl; bool owns;
  pp_split(c, K, &off, &kl, &owns);
  if (kl > c->Kcap) { c->err = "probe-parallel: this rank's share of K exceeds max_probes"; return COFEM_ERR_INVALID; }
  return COFEM_OK;
}

static constexpr double SUPPORT_THR = 1e-3, SUPPORT_DELTA = 1e-6;   // reading R16; cofem_report

// Read the column states back (the one end-of-E-step sync) and fill the report; with
// `support`, also the support certificate of mu = x0 (two small kernels, read back with the states).
static cofem_status estep_report(Ctx* c, int m, bool support = true) {
  c->cs_host.resize(m);
  if (support) {
    CK(cudaMemsetAsync(c->sup_stats, 0, sizeof(SupportStats), c->stream));
    CK(cudaMemsetAsync((char*)c->sup_stats + 8, 0x7f, 8, c->stream));     // min margin: a huge double
    k_support_max<<<c->num_sms * 2, 256, 0, c->stream>>>(c->D, c->x0, (SupportStats*)c->sup_stats);
    k_support_count<<<c->num_sms * 2, 256, 0, c->stream>>>(c->D, c->x0, SUPPORT_THR, SUPPORT_DELTA,
                                                            (SupportStats*)c->sup_stats);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(c->sup_host, c->sup_stats, sizeof(SupportStats), cudaMemcpyDeviceToHost, c->stream));
  }
  CK(cudaMemcpyAsync(c->cs_host.data(), c->cs, m * sizeof(ColState), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (support) {
    const SupportStats* h = (const SupportStats*)c->sup_host;
    union { unsigned long long u; double d; } mx{h->maxbits}, mm{h->minmargin_bits};
    c->sup_count = (int64_t)h->count; c->sup_adjacent = (int64_t)h->adjacent;
    c->sup_max = mx.d; c->sup_min_margin = mm.d;
  }
  c->last_cols = m;
  c->frozen_host.resize(m); c->rho_host.resize(m); c->rho0_host.resize(m);
  c->bad_col = -1; c->bad_iter = -1;
  for (int j = 0; j < m; ++j) {
    c->frozen_host[j] = c->cs_host[j].frozen_at;
    c->rho_host[j] = c->cs_host[j].rho;
    c->rho0_host[j] = c->cs_host[j].rho0;
    if (c->cs_host[j].nonfinite && c->bad_col < 0) { c->bad_col = j; c->bad_iter = c->cs_host[j].frozen_at; }
  }
  if (c->bad_col >= 0) {
    char buf[128];
    snprintf(buf, sizeof buf, "numerical breakdown (NaN/Inf) in column %d at CG iteration %d", c->bad_col, c->bad_iter);
    c->err = buf;
    return COFEM_ERR_NUMERIC;
  }
  return COFEM_OK;
}

}  // namespace cofem

using namespace cofem;

// ====================================================================== C ABI
extern "C" {

struct cofem_ctx_s { Ctx c; };

static thread_local std::string g_err;

void cofem_default_options(cofem_options* o) {
  if (!o) return;
  memset(o, 0, sizeof *o);
  o->cg_iters = 100; o->precond = 1; o->den_floor = 1e-12; o->alpha_max = 1e12;
  o->probe_precision = 0; o->max_probes = 32;
  o->rank = 0; o->world = 1; o->nccl_id = nullptr;
  o->cg_rtol = 0.0;
  o->apply_path = 0; o->probe_groups = 0; o->use_graph = 1; o->dist_mode = 0; o->warm_start = 0; o->cg_variant = 0;
}

const char* cofem_version(void) { return "cofem-b200 0.1 (sm_100a)"; }

const char* cofem_kernel_class_name(int32_t cls) {
  return (cls >= 0 && cls < KC_COUNT) ? kClassNames[cls] : nullptr;
}

const char* cofem_last_error(cofem_ctx ctx) { return ctx ? ctx->c.err.c_str() : g_err.c_str(); }

static void free_all(Ctx* c) {
  // the captured graph references NCCL work of the communicator: drain and drop it first
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->work) cudaStreamSynchronize(c->work);
  if (c->side) cudaStreamSynchronize(c->side);
  for (auto& s : c->gslot) if (s.exec) { cudaGraphExecDestroy(s.exec); s.exec = nullptr; }
  comm_destroy(c);
  dense_tc_free(c);
  if (c->phi && !c->phi_owned) c->phi = nullptr;   // borrowed from the caller
  void* ptrs[] = {c->phi, c->mask_vvT, c->dct_tab32, c->dct_tab64, c->taps, c->g64, c->g32, c->b0, c->colsq,
                  c->alpha, c->dinv64, c->dinvp, c->x0, c->r0, c->p0, c->q0, c->R, c->P, c->Q, c->s,
                  c->mu_out, c->s_out, c->alpha_out, c->bits, c->cs, c->part, c->counters,
                  c->ws1, c->ws2, c->ws1d, c->ws2d, c->alphap, c->maskL, c->tab1k32, c->tab1k64,
                  c->Pb, c->p0b, c->conv_tab32, c->conv_tab64, c->colsum,
                  c->halo_send, c->halo_recv, c->halo_send0, c->halo_recv0, c->s_part, c->tile_cnt,
                  c->flow_state, c->flow_part2, c->mt_b0, c->mt_mu, c->b0_saved, c->obs_dev, c->maskH, c->twh,
                  c->sr_part, c->sr_cnt};
  for (void* p : ptrs) if (p) cudaFree(p);
  for (int g = 1; g < Ctx::MAXG; ++g) if (c->gs[g]) cudaFree(c->gs[g]);
  for (auto& r : c->prof_recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->side) cudaStreamDestroy(c->side);
  for (int g = 1; g < Ctx::MAXG; ++g) {
    if (c->gstream[g]) cudaStreamDestroy(c->gstream[g]);
    if (c->gjoin[g]) cudaEventDestroy(c->gjoin[g]);
  }
  if (c->work) cudaStreamDestroy(c->work);
  if (c->ev_in) cudaEventDestroy(c->ev_in);
  if (c->ev_out) cudaEventDestroy(c->ev_out);
  if (c->dparams) cudaFree(c->dparams);
  if (c->bad_flag) cudaFree(c->bad_flag);
  if (c->bad_host) cudaFreeHost(c->bad_host);
  if (c->sup_stats) cudaFree(c->sup_stats);
  if (c->sup_host) cudaFreeHost(c->sup_host);
}

void cofem_destroy(cofem_ctx ctx) {
  if (!ctx) return;
  cudaStreamSynchronize(ctx->c.stream);
  if (ctx->c.work) cudaStreamSynchronize(ctx->c.work);
  free_all(&ctx->c);
  delete ctx;
}

static cofem_status setup_impl(Ctx* c, const cofem_operator* op, const float* y, double beta, const cofem_options* opt) {
  if (!op || !y || !opt) { c->err = "null argument"; return COFEM_ERR_INVALID; }
  if (!(beta > 0.0) || !isfinite(beta)) { c->err = "beta must be > 0"; return COFEM_ERR_INVALID; }
  if (op->D < 1 || op->N < 1) { c->err = "N, D must be >= 1"; return COFEM_ERR_INVALID; }
  if (opt->cg_iters < 1) { c->err = "cg_iters must be >= 1"; return COFEM_ERR_INVALID; }
  if (!(opt->cg_rtol >= 0.0 && opt->cg_rtol < 1.0)) { c->err = "cg_rtol must be in [0, 1)"; return COFEM_ERR_INVALID; }
  if (opt->max_probes < 1 || opt->max_probes + 1 > MAXM) { c->err = "max_probes must be in [1, 128]"; return COFEM_ERR_INVALID; }
  if (opt->den_floor <= 0 || opt->alpha_max <= 0) { c->err = "den_floor and alpha_max must be > 0"; return COFEM_ERR_INVALID; }
  if (opt->apply_path < 0 || opt->apply_path > 2) { c->err = "apply_path must be 0, 1 or 2"; return COFEM_ERR_INVALID; }
  if (opt->probe_groups < 0 || opt->probe_groups > Ctx::MAXG) { c->err = "probe_groups must be in [0, 8]"; return COFEM_ERR_INVALID; }
  if (opt->dist_mode < 0 || opt->dist_mode > 1) { c->err = "dist_mode must be 0 or 1"; return COFEM_ERR_INVALID; }
  if (opt->warm_start < 0 || opt->warm_start > 1) { c->err = "warm_start must be 0 or 1"; return COFEM_ERR_INVALID; }
  if (opt->cg_variant < 0 || opt->cg_variant > 2) { c->err = "cg_variant must be 0, 1 or 2"; return COFEM_ERR_INVALID; }
  c->kind = op->kind; c->N = op->N; c->D = op->D; c->beta = beta; c->opt = *opt;
  c->freeze_tau = std::max(FREEZE_TAU, opt->cg_rtol * opt->cg_rtol);
  if (opt->dist_mode == 1) {                    // probe-parallel (comm.cu: all-reduce of s, broadcast of mu)
    if (!opt->nccl_id || opt->world < 1 || opt->rank < 0 || opt->rank >= opt->world) {
      c->err = "probe-parallel: need nccl_id and 0 <= rank < world"; return COFEM_ERR_INVALID;
    }
    if (op->D_global || op->d_offset) { c->err = "probe-parallel: every rank holds the whole operator (D_global = 0)"; return COFEM_ERR_INVALID; }
    c->pp = true; c->rank = opt->rank; c->world = opt->world;
  } else if (opt->nccl_id || op->D_global) {    // column-sharded dense / D-sharded conv mode (comm.cu)
    if (op->kind == COFEM_OP_DCT2_MASKED) { c->err = "sharded mode: DENSE or CIRCCONV operators only"; return COFEM_ERR_UNSUPPORTED; }
    if (!opt->nccl_id || opt->world < 1 || opt->rank < 0 || opt->rank >= opt->world) {
      c->err = "sharded mode: need nccl_id and 0 <= rank < world"; return COFEM_ERR_INVALID;
    }
    if (op->d_offset < 0 || op->d_offset % 128 || op->D_global < op->d_offset + op->D) {
      c->err = "sharded mode: d_offset must be a multiple of 128 and d_offset + D <= D_global"; return COFEM_ERR_INVALID;
    }
    if (opt->probe_precision) { c->err = "sharded mode: fp32 probes only"; return COFEM_ERR_UNSUPPORTED; }
    if (opt->warm_start) { c->err = "sharded mode: no warm start"; return COFEM_ERR_UNSUPPORTED; }
    c->sharded = true; c->d_offset = op->d_offset; c->D_global = op->D_global;
    c->rank = opt->rank; c->world = opt->world;
  }
  c->probe64 = opt->probe_precision != 0;
  c->Kcap = opt->max_probes; c->m_cap = c->Kcap + 1;
  c->Dp = ((c->D + VEC_TILE - 1) / VEC_TILE) * VEC_TILE;
  CK(cudaGetDevice(&c->device));
  CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
  CK(cudaEventCreate(&c->ev0)); CK(cudaEventCreate(&c->ev1));
  CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  CK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
  for (int g = 1; g < Ctx::MAXG; ++g) {
    CK(cudaStreamCreateWithFlags(&c->gstream[g], cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->gjoin[g], cudaEventDisableTiming));
  }
  CK(cudaStreamCreateWithFlags(&c->work, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming));
  CK(cudaMalloc(&c->dparams, 64));
  CK(cudaMalloc(&c->bad_flag, sizeof(int)));
  CK(cudaMallocHost(&c->bad_host, sizeof(int)));
  CK(cudaMalloc(&c->sup_stats, sizeof(SupportStats)));
  CK(cudaMallocHost(&c->sup_host, sizeof(SupportStats)));

  const size_t tp = c->probe64 ? sizeof(double) : sizeof(float);
  const int64_t Dp = c->Dp;
  ALLOC(c->b0, Dp); ALLOC(c->colsq, Dp); ALLOC(c->alpha, Dp); ALLOC(c->dinv64, Dp);
  { char* p; ALLOC(p, Dp * tp); c->dinvp = p; }
  { char* p; ALLOC(p, Dp * tp); c->alphap = p; }
  ALLOC(c->x0, Dp); ALLOC(c->r0, Dp); ALLOC(c->p0, Dp); ALLOC(c->q0, Dp); ALLOC(c->s, Dp);
  ALLOC(c->mu_out, Dp); ALLOC(c->s_out, Dp); ALLOC(c->alpha_out, Dp);
  { char* p; ALLOC(p, (size_t)c->Kcap * Dp * tp); c->R = p; }
  { char* p; ALLOC(p, (size_t)c->Kcap * Dp * tp); c->P = p; }
  { char* p; ALLOC(p, (size_t)c->Kcap * Dp * tp); c->Q = p; }
  ALLOC(c->bits, (size_t)c->Kcap * (Dp / 32));
  ALLOC(c->cs, c->m_cap);
  ALLOC(c->counters, 4 * MAXM);   // [0, MAXM): per column; [MAXM, MAXM + 4): per-launch tickets; probe groups
                                  // g >= 1 of the fast DCT path: [2 MAXM + j0) DCT, [3 MAXM + j0) update
  c->vec_grid = (int)std::min<int64_t>(Dp / VEC_TILE, (int64_t)c->num_sms * 4);
  {   // k_update: with fewer D tiles than 2 per SM, split the probe columns into chunks as well
    const int64_t ntiles = Dp / VEC_TILE;
    int ch = 1;
    if (ntiles < 2 * c->num_sms && c->Kcap > 1)
      ch = (int)std::min<int64_t>(c->Kcap, (2 * c->num_sms + ntiles - 1) / ntiles);
    c->upd_chunks = ch;
    c->upd_grid = (int)std::min<int64_t>(ntiles * ch, (int64_t)c->num_sms * 4);
    if (ch > 1) { ALLOC(c->s_part, (size_t)ch * Dp); ALLOC(c->tile_cnt, (size_t)ntiles); }   // zeroed
  }
  c->part_stride = std::max(std::max(c->vec_grid, c->upd_grid), 1);

  if (c->sharded || c->pp) {     // the communicator first: the D-sharded conv setup exchanges y halos
    cofem_status cst = comm_init(c, opt->rank, opt->world, opt->nccl_id);
    if (cst != COFEM_OK) return cst;
  }
  if (c->sharded) {
    if (c->kind == COFEM_OP_CIRCCONV) {
      const size_t tp = c->probe64 ? 8 : 4;
      char* p;
      ALLOC(p, 2 * (size_t)c->Kcap * 192 * tp); c->halo_send = p;
      ALLOC(p, 2 * (size_t)c->Kcap * 192 * tp); c->halo_recv = p;
      ALLOC(c->halo_send0, 2 * 192); ALLOC(c->halo_recv0, 2 * 192);
    }
  }
  // y to device
  const float* y_dev = y;
  float* y_tmp = nullptr;
  if (!is_device_ptr(y)) {
    CK(cudaMalloc(&y_tmp, c->N * sizeof(float)));
    CK(cudaMemcpyAsync(y_tmp, y, c->N * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    y_dev = y_tmp;
  }
  cofem_status st = COFEM_ERR_INVALID;
  if (op->kind == COFEM_OP_DENSE) {
    if (op->ld < op->D || !op->phi) { c->err = "DENSE: phi NULL or ld < D"; st = COFEM_ERR_INVALID; }
    else {
      if (is_device_ptr(op->phi)) {     // borrowed: zero-copy, must outlive the context (cofem.h)
        c->phi = const_cast<float*>(op->phi); c->ld = op->ld; c->phi_owned = false;
        st = dense_setup(c, y_dev);
      } else {                          // host Phi: the library's own device copy (row stride D)
        c->ld = op->D; c->phi_owned = true;
        cudaError_t e = cudaMalloc(&c->phi, (size_t)op->N * op->D * sizeof(float));
        if (e != cudaSuccess) { c->err = "cudaMalloc phi"; st = COFEM_ERR_OOM; }
        else {
          e = cudaMemcpy2DAsync(c->phi, op->D * sizeof(float), op->phi, op->ld * sizeof(float),
                                op->D * sizeof(float), op->N, cudaMemcpyDefault, c->stream);
          st = e == cudaSuccess ? dense_setup(c, y_dev) : COFEM_ERR_CUDA;
          if (e != cudaSuccess) c->err = cudaGetErrorString(e);
        }
      }
    }
  } else if (op->kind == COFEM_OP_DCT2_MASKED) {
    c->rows = op->rows; c->cols = op->cols; c->conv = op->convention;
    auto pow2 = [](int v) { return v >= 16 && v <= 1024 && (v & (v - 1)) == 0; };
    if ((int64_t)op->rows * op->cols != op->D || op->N > op->D || !op->obs_idx) {
      c->err = "DCT2: rows*cols must equal D, N <= D, obs_idx non-NULL"; st = COFEM_ERR_INVALID;
    } else if (!pow2(op->rows) || !pow2(op->cols)) {
      c->err = "DCT2: rows and cols must be powers of two in [16, 1024]"; st = COFEM_ERR_UNSUPPORTED;
    } else if (op->convention != 0 && op->convention != 1) {
      c->err = "DCT2: convention must be 0 or 1"; st = COFEM_ERR_INVALID;
    } else {
      // validate the mask on the host (sorted, distinct, in range)
      std::vector<int64_t> h(op->N);
      cudaError_t e = cudaMemcpy(h.data(), op->obs_idx, op->N * sizeof(int64_t), cudaMemcpyDefault);
      if (e != cudaSuccess) { c->err = cudaGetErrorString(e); st = COFEM_ERR_CUDA; }
      else {
        bool ok = h[0] >= 0 && h[op->N - 1] < op->D;
        for (int64_t i = 1; ok && i < op->N; ++i) ok = h[i] > h[i - 1];
        if (!ok) { c->err = "DCT2: obs_idx must be sorted, distinct, in [0, D)"; st = COFEM_ERR_INVALID; }
        else {
          int64_t* od = nullptr;
          e = cudaMalloc(&od, op->N * sizeof(int64_t));
          if (e == cudaSuccess) e = cudaMemcpyAsync(od, h.data(), op->N * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream);
          st = e == cudaSuccess ? dct_setup(c, y_dev, od) : COFEM_ERR_CUDA;
          cudaStreamSynchronize(c->stream);
          if (od) cudaFree(od);
        }
      }
    }
  } else if (op->kind == COFEM_OP_CIRCCONV) {
    if (op->N != op->D || op->ntaps < 1 || op->ntaps > 64 || op->ntaps > op->D || !op->taps) {
      c->err = "CIRCCONV: need N == D, 1 <= ntaps <= min(64, D), taps non-NULL"; st = COFEM_ERR_INVALID;
    } else {
      std::vector<float> h(op->ntaps);
      cudaError_t e = cudaMemcpy(h.data(), op->taps, op->ntaps * sizeof(float), cudaMemcpyDefault);
      c->ntaps = op->ntaps;
      st = e == cudaSuccess ? conv_setup(c, y_dev, h.data()) : COFEM_ERR_CUDA;
    }
  } else {
    c->err = "unknown operator kind";
  }
  cudaStreamSynchronize(c->stream);
  if (y_tmp) cudaFree(y_tmp);
  if (st != COFEM_OK) return st;
  ALLOC(c->part, (size_t)(c->m_cap + 1) * c->part_stride);   // + k_init's warm-start slot
  c->pp_mean_cost = (c->fast1k || c->fast_conv) ? 2.0 : 0.0;
  if (c->sharded) {
    ALLOC(c->colsum, 4 * MAXM);
    if (c->kind == COFEM_OP_DENSE && !c->dense_tc) {
      c->err = "sharded mode needs the tensor-core dense path (D % 4 == 0, K <= 128)"; return COFEM_ERR_UNSUPPORTED;
    }
    if (c->kind == COFEM_OP_CIRCCONV && !c->fast_conv) {
      c->err = "D-sharded convolution needs the FFT path (local D >= 2048, ntaps <= 64)"; return COFEM_ERR_UNSUPPORTED;
    }
  }
  {   // CG variant (R23): single reduction where it merges collectives -- the column-sharded dense mode
    const bool col_dense = c->sharded && c->kind == COFEM_OP_DENSE;
    if (opt->cg_variant == 2 && !col_dense) {
      c->err = "cg_variant 2 (single-reduction CG): column-sharded dense mode only"; return COFEM_ERR_UNSUPPORTED;
    }
    c->sr = opt->cg_variant == 2 || (opt->cg_variant == 0 && col_dense);
    if (c->sr) { ALLOC(c->sr_part, (size_t)3 * MAXM * c->part_stride); ALLOC(c->sr_cnt, MAXM); }
  }
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaGetLastError());
  return COFEM_OK;
}

cofem_status cofem_setup(cofem_ctx* out, const cofem_operator* op, const float* y, double beta,
                         const cofem_options* opt, void* cuda_stream) {
  if (!out) { g_err = "out is NULL"; return COFEM_ERR_INVALID; }
  *out = nullptr;
  cofem_ctx ctx = new cofem_ctx_s();
  ctx->c.stream = (cudaStream_t)cuda_stream;
  nvtxRangePushA("cofem_setup");
  cofem_status st = setup_impl(&ctx->c, op, y, beta, opt);
  nvtxRangePop();
  if (st != COFEM_OK) {
    g_err = ctx->c.err;
    free_all(&ctx->c);
    delete ctx;
    return st;
  }
  *out = ctx;
  return COFEM_OK;
}

static cofem_status estep_impl(Ctx* c, const double* alpha, int32_t K, uint64_t seed, int32_t t,
                               int32_t k_offset, int32_t K_total, double* mu, double* s) {
  if (!alpha) { c->err = "alpha is NULL"; return COFEM_ERR_INVALID; }
  cofem_status st;
  if ((st = check_K(c, K))) return st;
  if (K_total < K || k_offset < 0) { c->err = "need K_total >= K and k_offset >= 0"; return COFEM_ERR_INVALID; }
  if (c->pp && (k_offset != 0 || K_total != K || c->skip_mean)) {
    c->err = "probe-parallel: pass the global K (k_offset 0, K_total K); cofem_estep_probes is not used";
    return COFEM_ERR_INVALID;
  }
  const double* a_dev;
  st = stage_in(c, alpha, c->alpha, &a_dev);
  if (st) return st;
  if (a_dev != c->alpha) CK(cudaMemcpyAsync(c->alpha, a_dev, c->D * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  if ((st = validate_alpha(c, c->alpha))) return st;
  CK(cudaEventRecord(c->ev0, c->stream));
  int m = K + 1;
  if (c->pp) { int kl; if ((st = estep_pp(c, K, seed, t, &kl))) return st; m = kl + 1; }
  else if ((st = estep_device(c, K, seed, t, k_offset, K_total))) return st;
  const bool mu_dev = mu && is_device_ptr(mu), s_dev = s && is_device_ptr(s);
  launch_begin(c, KC_FINAL);
  k_finalize<<<c->num_sms * 4, 256, 0, c->stream>>>(c->D, c->x0, c->s, mu_dev ? mu : c->mu_out,
                                                     s_dev ? s : c->s_out, nullptr, c->opt.den_floor, c->opt.alpha_max);
  launch_end(c, KC_FINAL);
  if (check_launch(c, "k_finalize")) return COFEM_ERR_CUDA;
  CK(cudaEventRecord(c->ev1, c->stream));
  if (mu && !mu_dev) CK(cudaMemcpyAsync(mu, c->mu_out, c->D * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  if (s && !s_dev) CK(cudaMemcpyAsync(s, c->s_out, c->D * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  st = estep_report(c, m);
  float ms = 0; cudaEventElapsedTime(&ms, c->ev0, c->ev1); c->estep_ms = ms;
  prof_collect(c);
  return st;
}

cofem_status cofem_estep(cofem_ctx ctx, const double* alpha, int32_t K, uint64_t seed, int32_t t,
                         int32_t k_offset, int32_t K_total, double* mu, double* s) {
  if (!ctx) { g_err = "ctx is NULL"; return COFEM_ERR_INVALID; }
  ctx->c.err.clear();
  nvtxRangePushA("cofem_estep");
  const cofem_status st = estep_impl(&ctx->c, alpha, K, seed, t, k_offset, K_total, mu, s);
  nvtxRangePop();
  return st;
}

cofem_status cofem_estep_probes(cofem_ctx ctx, const double* alpha, int32_t K, uint64_t seed, int32_t t,
                                int32_t k_offset, int32_t K_total, double* s) {
  if (!ctx) { g_err = "ctx is NULL"; return COFEM_ERR_INVALID; }
  ctx->c.err.clear();
  if (ctx->c.pp) { ctx->c.err = "cofem_estep_probes: not used in the probe-parallel mode (cofem_estep splits the probes)"; return COFEM_ERR_INVALID; }
  ctx->c.skip_mean = true;
  const cofem_status st = estep_impl(&ctx->c, alpha, K, seed, t, k_offset, K_total, nullptr, s);
  ctx->c.skip_mean = false;
  return st;
}

__global__ void k_apply_prep(int64_t D, int64_t Dp, double beta, int precond, const double* __restrict__ alpha,
                             const double* __restrict__ colsq, double* __restrict__ dinv64, void* dinvp,
                             void* alphap, int probe64) {
  for (int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; d < Dp; d += (int64_t)gridDim.x * blockDim.x) {
    const bool v = d < D;
    const double al = v ? alpha[d] : 0.0, dv = v ? (precond ? 1.0 / (beta * colsq[d] + al) : 1.0) : 0.0;
    dinv64[d] = dv;
    if (probe64) { ((double*)dinvp)[d] = dv; ((double*)alphap)[d] = al; }
    else { ((float*)dinvp)[d] = (float)dv; ((float*)alphap)[d] = (float)al; }
  }
}
__global__ void k_reset_cols(ColState* cs, int m) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  ColState c; c.rho = 1.0; c.rho0 = 1.0; c.gamma = 0; c.a = 0; c.b = 0;
  c.frozen = 0; c.frozen_at = -1; c.nonfinite = 0; c.pad = 0; c.tau = FREEZE_TAU;
  cs[j] = c;
}

static cofem_status apply_impl(Ctx* c, const double* alpha, int32_t K, const double* x0, const void* X, double* q0,
                               void* Q, double* gamma) {
  if (!alpha || !x0 || !X || !q0 || !Q) { c->err = "null argument"; return COFEM_ERR_INVALID; }
  if (K < 1 || K > c->Kcap) { c->err = "K must be in [1, max_probes]"; return COFEM_ERR_INVALID; }
  const size_t tp = c->probe64 ? 8 : 4;
  const int m = K + 1;
  cofem_status st;
  const double* a_dev;
  if ((st = stage_in(c, alpha, c->alpha, &a_dev))) return st;
  if (a_dev != c->alpha) CK(cudaMemcpyAsync(c->alpha, a_dev, c->D * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  if ((st = validate_alpha(c, c->alpha))) return st;
  k_apply_prep<<<c->num_sms * 4, 256, 0, c->stream>>>(c->D, c->Dp, c->beta, c->opt.precond, c->alpha, c->colsq,
                                                       c->dinv64, c->dinvp, c->alphap, c->probe64 ? 1 : 0);
  k_reset_cols<<<1, 256, 0, c->stream>>>(c->cs, m);
  CK(cudaMemcpyAsync(c->p0, x0, c->D * 8, cudaMemcpyDefault, c->stream));
  CK(cudaMemcpy2DAsync(c->P, c->Dp * tp, X, c->D * tp, c->D * tp, K, cudaMemcpyDefault, c->stream));
  CK(cudaGetLastError());
  if (c->fast1k || c->fast_conv) {
    SplitApply apply = c->fast1k ? dct1k_apply : conv_fft_apply;
    if ((st = apply(c, 0, 1, 0, false, c->stream)) != COFEM_OK) return st;
    if ((st = apply(c, 1, m, 0, false, c->stream)) != COFEM_OK) return st;
  } else if (c->kind == COFEM_OP_DCT2_MASKED) {
    if ((st = dct_apply(c, m, 0, false)) != COFEM_OK) return st;
  } else if (c->kind == COFEM_OP_DENSE) {
    if ((st = dense_apply(c, m, 0)) != COFEM_OK) return st;
  } else {
    if ((st = conv_apply(c, m, 0)) != COFEM_OK) return st;
  }
  CK(cudaMemcpyAsync(q0, c->q0, c->D * 8, cudaMemcpyDefault, c->stream));
  CK(cudaMemcpy2DAsync(Q, c->D * tp, c->Q, c->Dp * tp, c->D * tp, K, cudaMemcpyDefault, c->stream));
  c->cs_host.resize(m);
  CK(cudaMemcpyAsync(c->cs_host.data(), c->cs, m * sizeof(ColState), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (gamma)
    for (int j = 0; j < m; ++j) gamma[j] = c->cs_host[j].gamma;
  return COFEM_OK;
}

cofem_status cofem_apply(cofem_ctx ctx, const double* alpha, int32_t K, const double* x0, const void* X, double* q0,
                         void* Q, double* gamma) {
  if (!ctx) { g_err = "ctx is NULL"; return COFEM_ERR_INVALID; }
  ctx->c.err.clear();
  return apply_impl(&ctx->c, alpha, K, x0, X, q0, Q, gamma);
}

cofem_status cofem_mstep(cofem_ctx ctx, const double* mu, const double* s, double* alpha_out) {
  if (!ctx) { g_err = "ctx is NULL"; return COFEM_ERR_INVALID; }
  Ctx* c = &ctx->c;
  c->err.clear();
  if (!mu || !s || !alpha_out) { c->err = "null argument"; return COFEM_ERR_INVALID; }
  const double *mu_d, *s_d;
  cofem_status st;
  if ((st = stage_in(c, mu, c->mu_out, &mu_d))) return st;
  if ((st = stage_in(c, s, c->s_out, &s_d))) return st;
  const bool out_dev = is_device_ptr(alpha_out);
  launch_begin(c, KC_FINAL);
  k_mstep<<<c->num_sms * 4, 256, 0, c->stream>>>(c->D, mu_d, s_d, out_dev ? alpha_out : c->alpha_out,
                                                  c->opt.den_floor, c->opt.alpha_max);
  launch_end(c, KC_FINAL);
  if (check_launch(c, "k_mstep")) return COFEM_ERR_CUDA;
  if (!out_dev) CK(cudaMemcpyAsync(alpha_out, c->alpha_out, c->D * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return COFEM_OK;
}

cofem_status cofem_em(cofem_ctx ctx, int32_t iters, int32_t K, uint64_t seed, int32_t t0,
                      const double* alpha_init, double* alpha_out, double* mu_out, double* s_out) {
  if (!ctx) { g_err = "ctx is NULL"; return COFEM_ERR_INVALID; }
  Ctx* c = &ctx->c;
  c->err.clear();
  if (iters < 1) { c->err = "iters must be >= 1"; return COFEM_ERR_INVALID; }
  cofem_status st;
  if ((st = check_K(c, K))) return st;
  if (alpha_init) {
    const double* a_dev;
    if ((st = stage_in(c, alpha_init, c->alpha, &a_dev))) return st;
    if (a_dev != c->alpha) CK(cudaMemcpyAsync(c->alpha, a_dev, c->D * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    if ((st = validate_alpha(c, c->alpha))) return st;
  } else {
    std::vector<double> ones(c->D, 1.0);   // Alg. 1 line 1
    CK(cudaMemcpyAsync(c->alpha, ones.data(), c->D * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  const bool a_dev = alpha_out && is_device_ptr(alpha_out);
  const bool m_dev = mu_out && is_device_ptr(mu_out);
  const bool s_dev = s_out && is_device_ptr(s_out);
  for (int i = 0; i < iters; ++i) {
    nvtxRangePushA("cofem EM iteration");
    struct PopAtExit { ~PopAtExit() { nvtxRangePop(); } } pop_at_exit;
    CK(cudaEventRecord(c->ev0, c->stream));
    int m = K + 1;
    c->warm_now = c->opt.warm_start && i > 0;          // R20: from the previous E-step's mu (x0)
    if (c->pp) { int kl; st = estep_pp(c, K, seed, t0 + i, &kl); m = kl + 1; }
    else st = estep_device(c, K, seed, t0 + i, 0, K);
    c->warm_now = false;
    if (st) return st;
    const bool lastit = i == iters - 1;
    launch_begin(c, KC_FINAL);
    // the M-step writes the next alpha in place (the E-step state no longer needs it)
    k_finalize<<<c->num_sms * 4, 256, 0, c->stream>>>(
        c->D, c->x0, c->s, lastit ? (m_dev ? mu_out : c->mu_out) : nullptr,
        lastit ? (s_dev ? s_out : c->s_out) : nullptr, c->alpha, c->opt.den_floor, c->opt.alpha_max);
    launch_end(c, KC_FINAL);
    if (check_launch(c, "k_finalize")) return COFEM_ERR_CUDA;
    CK(cudaEventRecord(c->ev1, c->stream));
    st = estep_report(c, m, lastit);
    float ms = 0; cudaEventElapsedTime(&ms, c->ev0, c->ev1); c->estep_ms = ms;
    if (st != COFEM_OK) return st;
  }
  if (alpha_out) CK(cudaMemcpyAsync(alpha_out, c->alpha, c->D * sizeof(double), a_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->stream));
  if (mu_out && !m_dev) CK(cudaMemcpyAsync(mu_out, c->mu_out, c->D * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  if (s_out && !s_dev) CK(cudaMemcpyAsync(s_out, c->s_out, c->D * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  prof_collect(c);
  return COFEM_OK;
}

// NEXT-4 multi-task SBL (reading R22): L tasks share Phi, beta and alpha.  Per EM iteration the
// task means are solved one after another through the E-step machinery (tasks 1..L-1 as
// mean-only E-steps, K = 0; task 0 with the K probes, which give s), then alpha = 1 / (mean_l mu_l^2
// + s).  Each task's b0 = beta Phi^T y_l comes from the operator's own setup arithmetic.
static cofem_status em_multi_impl(Ctx* c, int L, const float* Y, int iters, int K, uint64_t seed, int t0,
                                  const double* alpha_init, double* alpha_out, double* MU_out, double* s_out) {
  if (L < 1 || !Y) { c->err = "multi-task: need L >= 1 and Y"; return COFEM_ERR_INVALID; }
  if (iters < 1) { c->err = "iters must be >= 1"; return COFEM_ERR_INVALID; }
  if (c->sharded || c->pp) { c->err = "multi-task: single-GPU contexts only"; return COFEM_ERR_UNSUPPORTED; }
  if (c->opt.warm_start) { c->err = "multi-task: no warm start"; return COFEM_ERR_UNSUPPORTED; }
  cofem_status st;
  if ((st = check_K(c, K))) return st;
  const int64_t Dp = c->Dp;
  if (L > c->mt_cap) {
    if (c->mt_b0) cudaFree(c->mt_b0);
    if (c->mt_mu) cudaFree(c->mt_mu);
    c->mt_b0 = c->mt_mu = nullptr; c->mt_cap = 0;
    ALLOC(c->mt_b0, (size_t)L * Dp); ALLOC(c->mt_mu, (size_t)L * Dp);
    c->mt_cap = L;
  }
  if (!c->b0_saved) ALLOC(c->b0_saved, Dp);
  CK(cudaMemcpyAsync(c->b0_saved, c->b0, Dp * 8, cudaMemcpyDeviceToDevice, c->stream));
  {   // b0 of every task
    float* ydev = nullptr;
    const bool ydv = is_device_ptr(Y);
    if (!ydv) {
      CK(cudaMalloc(&ydev, (size_t)c->N * sizeof(float)));
    }
    for (int l = 0; l < L && st == COFEM_OK; ++l) {
      const float* yl = Y + (size_t)l * c->N;
      if (!ydv) { CK(cudaMemcpyAsync(ydev, yl, c->N * sizeof(float), cudaMemcpyHostToDevice, c->stream)); yl = ydev; }
      double* out = c->mt_b0 + (size_t)l * Dp;
      st = c->kind == COFEM_OP_DENSE ? dense_b0(c, yl, out) : c->kind == COFEM_OP_DCT2_MASKED ? dct_b0(c, yl, out)
                                                                                          : conv_b0(c, yl, out);
    }
    CK(cudaStreamSynchronize(c->stream));
    if (ydev) cudaFree(ydev);
    if (st != COFEM_OK) return st;
  }
  if (alpha_init) {
    const double* a_dev;
    if ((st = stage_in(c, alpha_init, c->alpha, &a_dev))) return st;
    if (a_dev != c->alpha) CK(cudaMemcpyAsync(c->alpha, a_dev, c->D * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    if ((st = validate_alpha(c, c->alpha))) return st;
  } else {
    std::vector<double> ones(c->D, 1.0);
    CK(cudaMemcpyAsync(c->alpha, ones.data(), c->D * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  for (int i = 0; i < iters; ++i) {
    CK(cudaEventRecord(c->ev0, c->stream));
    for (int l = L - 1; l >= 0; --l) {      // task 0 last: its E-step (with the probes) leaves s
      CK(cudaMemcpyAsync(c->b0, c->mt_b0 + (size_t)l * Dp, Dp * 8, cudaMemcpyDeviceToDevice, c->stream));
      if ((st = estep_device(c, l ? 0 : K, seed, t0 + i, 0, l ? 1 : K))) return st;
      CK(cudaMemcpyAsync(c->mt_mu + (size_t)l * Dp, c->x0, Dp * 8, cudaMemcpyDeviceToDevice, c->stream));
      if (l && (st = estep_report(c, 1, false))) return st;
    }
    launch_begin(c, KC_FINAL);
    k_mstep_multi<<<c->num_sms * 4, 256, 0, c->stream>>>(c->D, Dp, L, c->mt_mu, c->s, c->alpha, c->opt.den_floor,
                                                          c->opt.alpha_max);
    launch_end(c, KC_FINAL);
    if (check_launch(c, "k_mstep_multi")) return COFEM_ERR_CUDA;
    CK(cudaEventRecord(c->ev1, c->stream));
    st = estep_report(c, K + 1, i == iters - 1);
    float ms = 0; cudaEventElapsedTime(&ms, c->ev0, c->ev1); c->estep_ms = ms;
    if (st != COFEM_OK) return st;
  }
  CK(cudaMemcpyAsync(c->b0, c->b0_saved, Dp * 8, cudaMemcpyDeviceToDevice, c->stream));   // the context's own y again
  if (alpha_out) CK(cudaMemcpyAsync(alpha_out, c->alpha, c->D * 8, cudaMemcpyDefault, c->stream));
  if (s_out) CK(cudaMemcpyAsync(s_out, c->s, c->D * 8, cudaMemcpyDefault, c->stream));
  if (MU_out) CK(cudaMemcpy2DAsync(MU_out, c->D * 8, c->mt_mu, Dp * 8, c->D * 8, L, cudaMemcpyDefault, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  prof_collect(c);
  return COFEM_OK;
}

cofem_status cofem_em_multi(cofem_ctx ctx, int32_t L, const float* Y, int32_t iters, int32_t K, uint64_t seed,
                            int32_t t0, const double* alpha_init, double* alpha_out, double* MU_out, double* s_out) {
  if (!ctx) { g_err = "ctx is NULL"; return COFEM_ERR_INVALID; }
  ctx->c.err.clear();
  return em_multi_impl(&ctx->c, L, Y, iters, K, seed, t0, alpha_init, alpha_out, MU_out, s_out);
}

cofem_status cofem_last_report(cofem_ctx ctx, cofem_report* out) {
  if (!ctx || !out) { g_err = "null argument"; return COFEM_ERR_INVALID; }
  Ctx* c = &ctx->c;
  out->cols = c->last_cols; out->cg_iters = c->opt.cg_iters;
  out->frozen_at = c->frozen_host.data(); out->rho = c->rho_host.data(); out->rho0 = c->rho0_host.data();
  out->bad_col = c->bad_col; out->bad_iter = c->bad_iter;
  out->estep_ms_last = c->estep_ms; out->launches = c->launches; out->collectives = c->collectives;
  out->support_count = c->sup_count; out->support_adjacent = c->sup_adjacent;
  out->support_max_abs_mu = c->sup_max; out->support_min_margin = c->sup_min_margin;
  out->support_delta = SUPPORT_DELTA;
  return COFEM_OK;
}

cofem_status cofem_probe_split(int32_t K, int32_t world, int32_t rank, double mean_cost, int32_t* k_offset,
                               int32_t* K_local, int32_t* owns_mean) {
  if (world < 1 || rank < 0 || rank >= world || K < world || !k_offset || !K_local || !owns_mean || !(mean_cost >= 0)) {
    g_err = "cofem_probe_split: need K >= world >= 1, 0 <= rank < world, mean_cost >= 0";
    return COFEM_ERR_INVALID;
  }
  int off, kl; bool owns;
  split_owner(K, world, rank, mean_cost, &off, &kl, &owns);
  *k_offset = off; *K_local = kl; *owns_mean = owns ? 1 : 0;
  return COFEM_OK;
}

cofem_status cofem_profile_enable(cofem_ctx ctx, uint32_t mask) {
  if (!ctx) { g_err = "ctx is NULL"; return COFEM_ERR_INVALID; }
  ctx->c.prof_mask = mask;
  return COFEM_OK;
}

cofem_status cofem_profile_read(cofem_ctx ctx, int32_t cls, double* total_ms, int64_t* count, int32_t reset) {
  if (!ctx || cls < 0 || cls >= KC_COUNT) { g_err = "bad argument"; return COFEM_ERR_INVALID; }
  Ctx* c = &ctx->c;
  prof_collect(c);
  if (total_ms) *total_ms = c->prof_ms[cls];
  if (count) *count = c->prof_cnt[cls];
  if (reset) { c->prof_ms[cls] = 0; c->prof_cnt[cls] = 0; c->prof_busy[cls] = 0; }
  return COFEM_OK;
}

cofem_status cofem_profile_busy(cofem_ctx ctx, int32_t cls, double* busy_ms) {
  if (!ctx || cls < 0 || cls >= KC_COUNT || !busy_ms) { g_err = "bad argument"; return COFEM_ERR_INVALID; }
  prof_collect(&ctx->c);
  *busy_ms = ctx->c.prof_busy[cls];
  return COFEM_OK;
}

}  // extern "C"
