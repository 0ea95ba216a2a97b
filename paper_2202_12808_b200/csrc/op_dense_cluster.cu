// op_dense_cluster.cu — the whole CG loop of a SMALL dense problem (Alg. 1 lines 3-7 after the
// probes and k_init; BASELINE config 1, N x D = 100 x 400) in ONE thread-block cluster.
//
// At this size every kernel of the per-iteration path (W = Phi P, Q = beta Phi^T W + alpha o P,
// the update, the direction) is a few microseconds of latency around almost no work, so the graph
// of ~6 launches per CG iteration costs ~46 us per iteration (C1).  Here the NC CTAs of one cluster
// each hold a column slice of Phi (and the matching rows of every vector) in shared memory for the
// whole E-step, and the three reductions of a CG iteration run through distributed shared memory
// (DSMEM) between cluster barriers instead of through HBM and kernel boundaries:
//   W = sum_c Phi_c P_c     : each CTA writes its partial [N][K], then CTA c sums rows [c N/NC, ..)
//                             over the NC partials in fixed order and stores them into EVERY CTA's W
//   gamma_j, rho'_j         : per-CTA partials, every CTA sums the NC partials in fixed order and
//                             takes the same step lengths / freeze decisions (R5) on its own copy
// Four cluster barriers per CG iteration, no global memory traffic inside the loop.  The probe
// columns may be split over several clusters of one launch (dcl_groups; cluster 0 also solves the
// mean system), each writing its own s partial; the partials are summed in cluster order.
//
// Arithmetic mirrors the SIMT kernels (op_dense.cu) and k_update / k_dir (cofem.cu): probe columns
// in probe precision TP with fp32 Phi, the mean column in fp64 (fp32 Phi promoted exactly), gamma,
// rho', s in fp64; the same freeze rule (finish_gamma).  Used when the problem fits one cluster's
// shared memory (dense_cluster_eligible), cofem_options.apply_path = 0, single GPU / probe-parallel.
#include <cooperative_groups.h>

#include <algorithm>

#include "internal.cuh"

namespace cofem {
namespace dcl {

namespace cg = cooperative_groups;

#ifndef COFEM_DCL_EXP
#define COFEM_DCL_EXP 0   // timing experiments only (results invalid): 1 no GEMM loops, 2 also no DSMEM W
#endif
#ifndef COFEM_DCL_NC
#define COFEM_DCL_NC 8
#endif
// C1 E-step (fixed alpha): KG 8 / 256 threads 1.61 ms, KG 4 / 256 1.51, KG 4 / 512 1.43, KG 4 / 384 1.38;
// 16-CTA clusters measured slower
#ifndef COFEM_DCL_THREADS
#define COFEM_DCL_THREADS 384
#endif
#ifndef COFEM_DCL_KG
#define COFEM_DCL_KG 4
#endif
constexpr int NC = COFEM_DCL_NC;            // CTAs per cluster (8: the portable maximum)
constexpr int THREADS = COFEM_DCL_THREADS;
constexpr int KG = COFEM_DCL_KG;            // probe columns per thread work unit (register accumulators)

constexpr int MAXCL = 8;                    // clusters per launch (probe-column groups)

struct Args {
  const float* phi; int64_t ld;
  int N, D, Dc, DcP, K, U;
  int ncl, Kmax;                    // clusters: cluster g solves probes [K g / ncl, K (g+1) / ncl) (+ the mean if g = 0)
  double* sg[MAXCL];                // cluster g's s partial (sg[0] = s); summed in cluster order afterwards
  double beta, invK;
  const double* alpha; const double* dinv64; const void* dinvp;
  double* x0; const double* r0; const double* p0;
  const void* R; const void* P;
  double* s; const uint32_t* bits; int64_t Dp, wpc;
  ColState* cs;
};

// Shared-memory layout (bytes, 16-aligned pieces), sized for K probe columns.  The probe arrays are
// stored [d][KP] and W [n][KP] (KP = K rounded up to KG, zero columns): the KG columns of a work unit
// are one 32- / 64-byte vector per d (or n) in the two products.
struct Layout {
  size_t phi, Pp, Rp, Qp, dvp, x, r, p, q, dv, al, sacc, wpart, wfull, w0part, w0full, gpart, rpart, cs, coef, sgn,
      total;
};
__host__ __device__ inline size_t al16(size_t v) { return (v + 15) & ~size_t(15); }
__host__ __device__ inline int kpad(int K) { return ((K + KG - 1) / KG) * KG; }
__host__ __device__ inline Layout layout(int N, int Dc, int DcP, int K, size_t tp) {
  Layout L;
  const int KP = kpad(K);
  size_t o = 0;
  L.phi = o; o = al16(o + (size_t)N * DcP * 4);
  L.Pp = o; o = al16(o + (size_t)Dc * KP * tp);
  L.Rp = o; o = al16(o + (size_t)Dc * KP * tp);
  L.Qp = o; o = al16(o + (size_t)Dc * KP * tp);
  L.dvp = o; o = al16(o + (size_t)Dc * tp);
  L.x = o; o = al16(o + (size_t)Dc * 8);
  L.r = o; o = al16(o + (size_t)Dc * 8);
  L.p = o; o = al16(o + (size_t)Dc * 8);
  L.q = o; o = al16(o + (size_t)Dc * 8);
  L.dv = o; o = al16(o + (size_t)Dc * 8);
  L.al = o; o = al16(o + (size_t)Dc * 8);
  L.sacc = o; o = al16(o + (size_t)Dc * 8);
  L.wpart = o; o = al16(o + (size_t)N * KP * tp);
  L.wfull = o; o = al16(o + (size_t)N * KP * tp);
  L.w0part = o; o = al16(o + (size_t)N * 8);
  L.w0full = o; o = al16(o + (size_t)N * 8);
  L.gpart = o; o = al16(o + (size_t)(K + 1) * 8);
  L.rpart = o; o = al16(o + (size_t)(K + 1) * 8);
  L.cs = o; o = al16(o + (size_t)(K + 1) * sizeof(ColState));
  L.coef = o; o = al16(o + (size_t)KP * 8);
  L.sgn = o; o = al16(o + (size_t)Dc * KP);
  L.total = o;
  return L;
}

// KG consecutive values of probe precision from 16-byte-aligned shared memory
template <typename TP> __device__ __forceinline__ void ldkg(const TP* p, TP (&v)[KG]) {
  static_assert(KG % 4 == 0, "KG");
  if constexpr (sizeof(TP) == 4) {
#pragma unroll
    for (int i = 0; i < KG / 4; ++i) {
      const float4 x = reinterpret_cast<const float4*>(p)[i];
      v[4 * i] = x.x; v[4 * i + 1] = x.y; v[4 * i + 2] = x.z; v[4 * i + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < KG / 2; ++i) {
      const double2 x = reinterpret_cast<const double2*>(p)[i];
      v[2 * i] = x.x; v[2 * i + 1] = x.y;
    }
  }
}

template <typename TP>
__global__ void __cluster_dims__(NC, 1, 1) __launch_bounds__(THREADS) k_dense_cluster_cg(Args a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // probe-column group of this cluster: local column j (0 = mean, on cluster 0 only) is global
  // column jg(j); with one cluster this is the whole E-step
  const int cid = blockIdx.x / NC, klo = (int)((int64_t)a.K * cid / a.ncl), khi = (int)((int64_t)a.K * (cid + 1) / a.ncl);
  const bool has_mean = cid == 0;
  auto jg = [&](int j) { return j == 0 ? 0 : klo + j; };
  const int N = a.N, K = khi - klo, m = K + 1, Dc = a.Dc, DcP = a.DcP, KP = kpad(K), G = KP / KG;
  const Layout L = layout(N, Dc, DcP, a.Kmax, sizeof(TP));
  float* phs = reinterpret_cast<float*>(smraw + L.phi);     // [N][DcP]
  TP* Ps = reinterpret_cast<TP*>(smraw + L.Pp);             // [Dc][KP]
  TP* Rs = reinterpret_cast<TP*>(smraw + L.Rp);
  TP* Qs = reinterpret_cast<TP*>(smraw + L.Qp);
  TP* dvp = reinterpret_cast<TP*>(smraw + L.dvp);           // [Dc] 1/diag in probe precision
  double* xs = reinterpret_cast<double*>(smraw + L.x);      // mean column [Dc]
  double* rs = reinterpret_cast<double*>(smraw + L.r);
  double* ps = reinterpret_cast<double*>(smraw + L.p);
  double* qs = reinterpret_cast<double*>(smraw + L.q);
  double* dv = reinterpret_cast<double*>(smraw + L.dv);
  double* als = reinterpret_cast<double*>(smraw + L.al);
  double* sacc = reinterpret_cast<double*>(smraw + L.sacc);
  TP* wpart = reinterpret_cast<TP*>(smraw + L.wpart);       // [N][KP]
  TP* wfull = reinterpret_cast<TP*>(smraw + L.wfull);
  double* w0part = reinterpret_cast<double*>(smraw + L.w0part);
  double* w0full = reinterpret_cast<double*>(smraw + L.w0full);
  double* gpart = reinterpret_cast<double*>(smraw + L.gpart);
  double* rpart = reinterpret_cast<double*>(smraw + L.rpart);
  ColState* cs = reinterpret_cast<ColState*>(smraw + L.cs);
  double* coef = reinterpret_cast<double*>(smraw + L.coef);   // [KP] a_k / K of the active columns, else 0
  uint8_t* sgn = smraw + L.sgn;                             // [Dc][KP] probe bit (1: -1)

  // ---- this CTA's slice d in [d0, d0 + Dl) of Phi and of every vector (state after k_init)
  const int d0 = rank * Dc;
  const int Dl = max(0, min(Dc, a.D - d0));
  for (int i = tid; i < N * DcP; i += THREADS) {
    const int n = i / DcP, dl = i % DcP;
    phs[i] = dl < Dl ? a.phi[(int64_t)n * a.ld + d0 + dl] : 0.0f;
  }
  const TP* Pg = reinterpret_cast<const TP*>(a.P);
  const TP* Rg = reinterpret_cast<const TP*>(a.R);
  const TP* dvg = reinterpret_cast<const TP*>(a.dinvp);
  for (int i = tid; i < Dc * KP; i += THREADS) {
    const int dl = i / KP, k = i % KP;
    const bool v = dl < Dl && k < K;
    const int d = d0 + dl;
    Ps[i] = v ? Pg[(int64_t)(klo + k) * a.Dp + d] : (TP)0;
    Rs[i] = v ? Rg[(int64_t)(klo + k) * a.Dp + d] : (TP)0;
    Qs[i] = (TP)0;
    sgn[i] = v ? (uint8_t)((a.bits[(int64_t)(klo + k) * a.wpc + (d >> 5)] >> (d & 31)) & 1u) : (uint8_t)0;
  }
  for (int i = tid; i < N * KP; i += THREADS) { wpart[i] = (TP)0; wfull[i] = (TP)0; }
  for (int dl = tid; dl < Dc; dl += THREADS) {
    const bool v = dl < Dl;
    const int d = d0 + dl;
    dvp[dl] = v ? dvg[d] : (TP)0;
    xs[dl] = v ? a.x0[d] : 0.0; rs[dl] = v ? a.r0[d] : 0.0; ps[dl] = v ? a.p0[d] : 0.0; qs[dl] = 0.0;
    dv[dl] = v ? a.dinv64[d] : 0.0; als[dl] = v ? a.alpha[d] : 0.0; sacc[dl] = v && has_mean ? a.s[d] : 0.0;
  }
  for (int j = tid; j < m; j += THREADS) {
    cs[j] = a.cs[jg(j)];
    if (j == 0 && !has_mean) cs[0].frozen = 1;     // the mean system is cluster 0's
  }
  const int Nr = (N + NC - 1) / NC, n_lo = min(N, rank * Nr), n_hi = min(N, n_lo + Nr);
  cl.sync();

#pragma unroll 1
  for (int it = 0; it < a.U; ++it) {
    // every column frozen (R5): nothing left to do (the state is the same in every CTA)
    int act = 0;
    for (int j = tid; j < m; j += THREADS) act |= !cs[j].frozen;
    if (!__syncthreads_or(act)) break;
    // ---- 1. W partial = Phi_c P_c (probe precision) and Phi_c p0 (fp64)
    for (int u = tid; u < (COFEM_DCL_EXP >= 1 ? 0 : N * (G + (has_mean ? 1 : 0))); u += THREADS) {
      const int n = u % N, g = u / N;
      const float* ph = phs + n * DcP;
      if (g < G) {
        TP acc[KG];
#pragma unroll
        for (int i = 0; i < KG; ++i) acc[i] = (TP)0;
        for (int dl = 0; dl < Dl; ++dl) {
          const TP f = (TP)ph[dl];
          TP pv[KG];
          ldkg(Ps + dl * KP + g * KG, pv);
#pragma unroll
          for (int i = 0; i < KG; ++i) acc[i] += f * pv[i];
        }
#pragma unroll
        for (int i = 0; i < KG; ++i) wpart[n * KP + g * KG + i] = acc[i];
      } else {
        double acc0 = 0.0;
        for (int dl = 0; dl < Dl; ++dl) acc0 += (double)ph[dl] * ps[dl];
        w0part[n] = acc0;
      }
    }
    cl.sync();
    // ---- 2. rows [n_lo, n_hi): sum the NC partials in rank order, store into every CTA's W
    const int kw = K + (has_mean ? 1 : 0);          // W columns: the probes (+ the mean)
    for (int i = tid; i < (COFEM_DCL_EXP >= 2 ? 0 : (n_hi - n_lo) * kw); i += THREADS) {
      const int n = n_lo + i / kw, k = i % kw;
      if (k < K) {
        TP x[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) x[c] = cl.map_shared_rank(wpart, c)[n * KP + k];
        TP v = (TP)0;
#pragma unroll
        for (int c = 0; c < NC; ++c) v += x[c];
#pragma unroll
        for (int c = 0; c < NC; ++c) cl.map_shared_rank(wfull, c)[n * KP + k] = v;
      } else {
        double x[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) x[c] = cl.map_shared_rank(w0part, c)[n];
        double v = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) v += x[c];
#pragma unroll
        for (int c = 0; c < NC; ++c) cl.map_shared_rank(w0full, c)[n] = v;
      }
    }
    cl.sync();
    // ---- 3. Q = beta Phi_c^T W + alpha o P (a3), q0 likewise in fp64; gamma partials (a4)
    const TP betat = (TP)a.beta;
    for (int u = tid; u < (COFEM_DCL_EXP >= 1 ? 0 : Dl * (G + (has_mean ? 1 : 0))); u += THREADS) {
      const int dl = u % Dl, g = u / Dl;
      if (g < G) {
        TP acc[KG];
#pragma unroll
        for (int i = 0; i < KG; ++i) acc[i] = (TP)0;
        for (int n = 0; n < N; ++n) {
          const TP f = (TP)phs[n * DcP + dl];
          TP wv[KG];
          ldkg(wfull + n * KP + g * KG, wv);
#pragma unroll
          for (int i = 0; i < KG; ++i) acc[i] += f * wv[i];
        }
        const TP alt = (TP)als[dl];
        TP pv[KG];
        ldkg(Ps + dl * KP + g * KG, pv);
#pragma unroll
        for (int i = 0; i < KG; ++i) Qs[dl * KP + g * KG + i] = betat * acc[i] + alt * pv[i];
      } else {
        double acc0 = 0.0;
        for (int n = 0; n < N; ++n) acc0 += (double)phs[n * DcP + dl] * w0full[n];
        qs[dl] = a.beta * acc0 + als[dl] * ps[dl];
      }
    }
    __syncthreads();
    for (int j = warp; j < m; j += THREADS / 32) {   // one warp per column: lane-strided, then the tree
      double g = 0.0;
      if (j == 0) { if (has_mean) for (int dl = lane; dl < Dl; dl += 32) g += ps[dl] * qs[dl]; }
      else for (int dl = lane; dl < Dl; dl += 32) g += (double)Ps[dl * KP + j - 1] * (double)Qs[dl * KP + j - 1];
      g = warp_sum(g);
      if (lane == 0) gpart[j] = g;
    }
    cl.sync();
    // ---- 4. gamma_j over the cluster (rank order); freeze rule and a_j on every CTA's copy
    for (int j = tid; j < m; j += THREADS) {
      double x[NC], v = 0.0;
#pragma unroll
      for (int c = 0; c < NC; ++c) x[c] = cl.map_shared_rank(gpart, c)[j];
#pragma unroll
      for (int c = 0; c < NC; ++c) v += x[c];
      if (COFEM_DCL_EXP == 0) finish_gamma(cs[j], v, it);
      if (j > 0) coef[j - 1] = cs[j].frozen ? 0.0 : cs[j].a * a.invK;
    }
    __syncthreads();
    // ---- 5. a5: x0 += a0 p0, r -= a q, s += (a_k / K) p_k o z_k; rho' partials
    for (int u = tid; u < Dl * K; u += THREADS) {
      const int dl = u / K, k = u % K;
      if (cs[k + 1].frozen) continue;
      const TP akt = (TP)cs[k + 1].a;
      Rs[dl * KP + k] = Rs[dl * KP + k] - akt * Qs[dl * KP + k];
    }
    if (!cs[0].frozen) {
      const double a0 = cs[0].a;
      for (int dl = tid; dl < Dl; dl += THREADS) {
        xs[dl] = fma(a0, ps[dl], xs[dl]);
        rs[dl] = fma(-a0, qs[dl], rs[dl]);
      }
    }
    for (int dl = tid; dl < Dl; dl += THREADS) {    // the probe estimator, columns in order (k_update)
      double sv = 0.0;
      for (int k = 0; k < K; ++k) {
        const double aks = coef[k], pe = (double)Ps[dl * KP + k];
        sv += sgn[dl * KP + k] ? -aks * pe : aks * pe;
      }
      sacc[dl] += sv;
    }
    __syncthreads();
    for (int j = warp; j < m; j += THREADS / 32) {
      double v = 0.0;
      if (!cs[j].frozen) {
        if (j == 0) {
          for (int dl = lane; dl < Dl; dl += 32) v += rs[dl] * (dv[dl] * rs[dl]);
        } else {
          for (int dl = lane; dl < Dl; dl += 32) {
            const TP r = Rs[dl * KP + j - 1], z = dvp[dl] * r;
            v += (double)r * (double)z;
          }
        }
      }
      v = warp_sum(v);
      if (lane == 0) rpart[j] = v;
    }
    cl.sync();
    // ---- 6. rho'_j over the cluster; b_j; direction p = M^-1 r + b p (a6) for the next iteration
    for (int j = tid; j < m; j += THREADS) {
      if (cs[j].frozen) continue;
      double x[NC], v = 0.0;
#pragma unroll
      for (int c = 0; c < NC; ++c) x[c] = cl.map_shared_rank(rpart, c)[j];
#pragma unroll
      for (int c = 0; c < NC; ++c) v += x[c];
      cs[j].b = v / cs[j].rho;
      cs[j].rho = v;
    }
    __syncthreads();
    for (int u = tid; u < Dl * K; u += THREADS) {
      const int dl = u / K, k = u % K;
      if (cs[k + 1].frozen) continue;
      const TP bt = (TP)cs[k + 1].b;
      Ps[dl * KP + k] = dvp[dl] * Rs[dl * KP + k] + bt * Ps[dl * KP + k];
    }
    if (!cs[0].frozen) {
      const double b0 = cs[0].b;
      for (int dl = tid; dl < Dl; dl += THREADS) ps[dl] = fma(b0, ps[dl], dv[dl] * rs[dl]);
    }
    __syncthreads();
  }
  // ---- results: mu slice, s slice; the column states (identical in every CTA) from rank 0
  for (int dl = tid; dl < Dl; dl += THREADS) {
    if (has_mean) a.x0[d0 + dl] = xs[dl];
    a.sg[cid][d0 + dl] = sacc[dl];
  }
  if (rank == 0)
    for (int j = tid; j < m; j += THREADS)
      if (j > 0 || has_mean) a.cs[jg(j)] = cs[j];
  cl.sync();                         // no CTA leaves while others may still read its shared memory
}

struct Parts { double* p[MAXCL]; };
__global__ void k_sum_parts(int64_t D, int ncl, Parts sp) {
  for (int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; d < D; d += (int64_t)gridDim.x * blockDim.x) {
    double v = sp.p[0][d];
    for (int g = 1; g < ncl; ++g) v += sp.p[g][d];
    sp.p[0][d] = v;
  }
}

}  // namespace dcl

static size_t dcl_smem(const Ctx* c, int K) {
  const int Dc = (int)((c->D + dcl::NC - 1) / dcl::NC);
  return dcl::layout((int)c->N, Dc, Dc | 1, K, c->probe64 ? 8 : 4).total;
}

// Clusters per E-step: the probe columns split over ncl concurrent clusters (each on its own NC
// SMs, each with its own copy of Phi's slices; the columns are independent systems, R3), so each
// cluster's per-iteration loops (products, update, per-column dots) cover a quarter of the columns
// while the barrier and reduction latency stays the same; options.probe_groups, else COFEM_DCL_GROUPS.
#ifndef COFEM_DCL_GROUPS
#define COFEM_DCL_GROUPS 0   // 0 = auto: max(min(4, K), ceil(K / KG)) -- whole KG-column units per cluster
#endif                       // (C1 E-step, fixed alpha: 1 cluster 1.36 ms, 2 1.13, 3 1.00, 4 0.99, 5 0.96, 7 0.96)
static int dcl_groups(const Ctx* c, int K) {
  int g = c->opt.probe_groups > 0 ? c->opt.probe_groups
                                  : COFEM_DCL_GROUPS > 0 ? COFEM_DCL_GROUPS
                                                         : std::max(std::min(4, K), (K + dcl::KG - 1) / dcl::KG);
  g = std::max(1, std::min(g, std::min(dcl::MAXCL, K)));
  while (g > 1 && !c->gs[g - 1]) --g;
  return g;
}

bool dense_cluster_eligible(const Ctx* c) {
  if (c->kind != COFEM_OP_DENSE || c->sharded || c->opt.apply_path != 0) return false;
  if (c->D < dcl::NC || c->N > (1 << 16)) return false;
  return dcl_smem(c, c->Kcap) <= (size_t)200 * 1024;
}

cofem_status dense_cluster_setup(Ctx* c) {
  const int sm = (int)dcl_smem(c, c->Kcap);
  if (dcl::NC > 8) {
    cudaFuncSetAttribute(dcl::k_dense_cluster_cg<double>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(dcl::k_dense_cluster_cg<float>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  cudaError_t e = c->probe64 ? raise_smem_attr((const void*)dcl::k_dense_cluster_cg<double>, sm)
                              : raise_smem_attr((const void*)dcl::k_dense_cluster_cg<float>, sm);
  if (e != cudaSuccess) { c->err = std::string("dense cluster setup: ") + cudaGetErrorString(e); return COFEM_ERR_CUDA; }
  c->dense_cluster = true;
  for (int g = 1; g < dcl::MAXCL && g < Ctx::MAXG; ++g)      // the clusters' s partials (dcl_groups)
    if (!c->gs[g]) {
      if (cudaMalloc(&c->gs[g], c->Dp * sizeof(double)) != cudaSuccess) { c->gs[g] = nullptr; cudaGetLastError(); break; }
      cudaMemset(c->gs[g], 0, c->Dp * sizeof(double));          // the padding [D, Dp) stays 0
    }
  return COFEM_OK;
}

// All U CG iterations of the E-step (state initialised by k_init) in one cluster launch.
cofem_status dense_cluster_cg(Ctx* c, int K, double invK) {
  dcl::Args a;
  a.phi = c->phi; a.ld = c->ld; a.N = (int)c->N; a.D = (int)c->D;
  a.Dc = (int)((c->D + dcl::NC - 1) / dcl::NC); a.DcP = a.Dc | 1; a.K = K; a.U = c->opt.cg_iters;
  a.beta = c->beta; a.invK = invK;
  a.alpha = c->alpha; a.dinv64 = c->dinv64; a.dinvp = c->dinvp;
  a.x0 = c->x0; a.r0 = c->r0; a.p0 = c->p0; a.R = c->R; a.P = c->P;
  a.s = c->s; a.bits = c->bits; a.Dp = c->Dp; a.wpc = c->Dp / 32; a.cs = c->cs;
  a.ncl = dcl_groups(c, K);
  a.Kmax = (K + a.ncl - 1) / a.ncl;
  for (int g = 0; g < dcl::MAXCL; ++g) a.sg[g] = g == 0 ? c->s : (g < a.ncl ? c->gs[g] : nullptr);
  const size_t sm = dcl::layout(a.N, a.Dc, a.DcP, a.Kmax, c->probe64 ? 8 : 4).total;
  launch_begin(c, KC_DENSE_CLUSTER);
  if (c->probe64) dcl::k_dense_cluster_cg<double><<<dcl::NC * a.ncl, dcl::THREADS, sm, c->stream>>>(a);
  else dcl::k_dense_cluster_cg<float><<<dcl::NC * a.ncl, dcl::THREADS, sm, c->stream>>>(a);
  if (a.ncl > 1)                      // s = ((s_0 + s_1) + s_2) + s_3 in cluster order (deterministic)
  {
    dcl::Parts sp;
    for (int g = 0; g < dcl::MAXCL; ++g) sp.p[g] = a.sg[g];
    dcl::k_sum_parts<<<c->num_sms * 2, 256, 0, c->stream>>>(c->D, a.ncl, sp);
  }
  launch_end(c, KC_DENSE_CLUSTER);
  return check_launch(c, "k_dense_cluster_cg") == cudaSuccess ? COFEM_OK : COFEM_ERR_CUDA;
}

}  // namespace cofem
