// op_dense_tc.cu — dense Gram apply on the 5th-generation tensor cores (sm_100a):
//   W = Phi P            (N x K probes; split-K over D)          k_tc_phiP
//   Q = beta Phi^T W + alpha o P,  gamma_j = p_j^T q_j           k_tc_phiTW
// (Eq. 7; batched "matrix-matrix" CG apply, §3.2; BASELINE north_star:
// "tcgen05/TMA tiles with a 3xTF32 split").
//
// 3xTF32: C = A_hi B_hi + A_hi B_lo + A_lo B_hi on kind::tf32 MMAs with fp32 accumulation in
// TMEM.  B (the probe block, small) is split once per apply with hi = round-to-nearest tf32; A
// (Phi) is written to TMEM as is — the tensor core reads only the tf32 bits of an fp32 operand
// (truncation, tools/tf32_semantics.cu) — with lo = x - trunc(x) (exact, |lo| < 2^-10 |x|); the
// dropped A_lo B_lo term is <= 2^-21 |A||B| per product.
//
// Per CTA (one 128-row output tile; 18 warps):
//   warp 0      TMA producer: Phi tile (16 KB) + B_hi, B_lo tiles (K-major, SWIZZLE_128B) + 32
//               fp64 mean-column operands per 32-wide K step into a 6-stage smem ring
//   warp 1      TMEM allocator + tcgen05.mma issuer (whole warp, elect.sync per instruction;
//               A from TMEM, B from smem), one wait and one commit per PAIR of K steps
//   warps 2-17  "splitters", 4 groups x one warp per TMEM lane quarter: each thread owns one
//               output row m; group g splits the K steps kt = g (mod 4): reads its row of the
//               Phi tile from smem (Phi^T's transposition happens here for k_tc_phiTW: the
//               tile is MN-major in smem), writes x and lo = x - trunc(x) into TMEM, then
//               accumulates the fp64 mean column (column 0 of B = [b0 | p_1..p_K], R2, R10)
//               with DFMA; they promote the round-toward-zero TMEM accumulator into RN fp32
//               register sums every pair and run the epilogue (q, gamma partials / W partials).
// The probe B operand's hi/lo split is done once per apply in global memory (B is
// O((N + D) K), Phi is O(N D)).  Only the probe columns use the tensor cores; parity mode
// (fp64 probes) keeps the SIMT path (op_dense.cu).  Measured design notes: DESIGN.md §7.2.
#include <cuda.h>
#include <stdio.h>

#include <algorithm>

#include "internal.cuh"

namespace cofem {
namespace tc {

constexpr int BM = 128, BK = 32;
constexpr int NGROUP = 4;                  // splitter groups: group g handles K steps kt = g (mod NGROUP)
constexpr int NSPLIT = 4 * NGROUP;         // splitter warps (one per TMEM lane quarter per group)
constexpr int THREADS = 64 + 32 * NSPLIT;  // warps 0-1 + splitters
constexpr int NAB = 4;                     // TMEM A buffers (hi 32 | lo 32 columns each) over all M-tiles
constexpr int TMEM_COLS = 512;             // [0, 256) two accumulator buffers; [256, 512) A buffers (1 CTA / SM)
constexpr int TM_A = 256;
// The tensor core's fp32 accumulation rounds toward zero, so its error grows linearly with the
// number of accumulated MMAs (measured: 3xTF32 apply error 6e-5 at N = 8192 with one TMEM
// accumulator, tools/tc_error_probe.py).  The accumulator is therefore promoted every pair of
// K steps (K = 64) into round-to-nearest fp32 register sums held by the splitter warps, with
// NACC TMEM accumulator buffers so the MMAs of the next pairs overlap the promotion.
//
// Pair protocol.  The single MMA-issuing thread is the serial bottleneck of this kernel (each
// tcgen05.mma costs ~45 issue cycles, a commit ~44, an mbarrier wait ~90; tools/mma_rate.cu,
// tools/tc_trace.py), so it works on PAIRS of K steps: one split_done wait, 16 MMAs (fused)
// and ONE commit (pair_done) per pair; pair_done frees the pair's smem stages (producer), its
// TMEM A buffers (splitters, two pairs later) and is the chunk-complete signal (promotion).
#ifdef COFEM_TC_EXP_SLEEP
constexpr int SPLIT_SLEEP = 40;            // ns between the splitters' barrier polls
#else
constexpr int SPLIT_SLEEP = 0;             // spinning on try_wait measured 2 % faster on C3 than a 40 ns back-off
#endif
constexpr int PLAG = 2;                    // splitters promote pair c at the top of pair c + PLAG (right when its
                                           // A buffers free up); deadlock-free for 2 <= PLAG < NACC + 3

// ---------------------------------------------------------------- PTX wrappers
#ifdef COFEM_TC_EXP_TRACE   // timing experiment: clock64 of pipeline events in CTA (0, 0) of k_tc_phiTW
__device__ long long g_tc_trace[1024][10];
#define TC_TRACE(kt, ev) \
  { if (MN && blockIdx.x == 0 && blockIdx.y == 0 && (kt) < 1024) g_tc_trace[kt][ev] = clock64(); }
#else
#define TC_TRACE(kt, ev) {}
#endif
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
// Bounded wait: a protocol error records (block, warp, barrier offset, parity) in
// g_tc_stuck and ends the thread instead of hanging the GPU (the host reports it as
// COFEM_ERR_CUDA with the record).
__device__ unsigned long long g_tc_stuck[4];
// sleep_ns > 0: back off between polls (the splitter warps share issue slots with the
// single-thread MMA issuer, whose instruction chain must not be starved by spinning).
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity, int sleep_ns = 0) {
  for (long long spin = 0;; ++spin) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(su32(b)), "r"(parity)
        : "memory");
    if (done) return;
    if (sleep_ns) __nanosleep(sleep_ns);
    if (spin > (1ll << 24)) {
      if (atomicCAS(&g_tc_stuck[0], 0ull, 1ull) == 0ull) {
        g_tc_stuck[1] = ((unsigned long long)blockIdx.x << 32) | (blockIdx.y << 16) | (threadIdx.x >> 5);
        g_tc_stuck[2] = ((unsigned long long)(su32(b) & 0xFFFF) << 32) | parity;
      }
      asm volatile("exit;");
    }
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          su32(dst)),
      "l"(map), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem], kind::tf32, M = 128, cta_group::1
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
// Warp-converged forms: all 32 lanes execute them with warp-uniform operands and elect.sync
// picks the issuing lane inside the asm block, so ptxas emits a predicated UTCHMMA instead of
// an ELECT loop per instruction (measured 34 vs 70 cycles per N = 64 MMA, tools/mma_rate.cu).
__device__ __forceinline__ void mma_ts_e(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit_e(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)) : "memory");
}

// 32 consecutive 32-bit TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
      "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
      "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr), "f"(v[0]),
               "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "r"(taddr)
               : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, "
      "[%16];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]), "=f"(v[8]),
        "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor: K-major, 128-byte swizzle (the layout TMA writes for a
// box whose inner dimension is 128 B): rows of 128 B, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t desc_k_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address >> 4
  d |= (uint64_t)1 << 16;                          // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;                // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                          // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                          // SWIZZLE_128B
  return d;
}
// Instruction descriptor: kind::tf32, fp32 accumulate, A and B K-major, M = 128, N = bn.
__host__ __device__ constexpr uint32_t idesc_tf32(int bn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(bn >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

// hi = x rounded to the nearest tf32 (cvt.rna), so lo = x - hi is exact and |lo| <= 2^-11 |x|.
// The same rounding (to nearest, ties away) on the integer pipe: add half a tf32 ulp to the
// magnitude bits and clear the 13 low bits (finite x; the splitters' hot loop avoids the
// conversion unit, which the fp64 mean-column F2F already keeps busy).
__device__ __forceinline__ float tf32_hi_alu(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Kernel modes.  0: bn <= 64, fused N = 2 bn MMAs, 2 accumulator buffers of 128 columns;
// 1: bn <= 64, three N = bn MMAs per K = 8, 4 buffers of 64 columns (the MMA of pair p waits for
// the promotion of pair p - 4: never on the critical path); 2: bn <= 128, unfused, 2 x 128.
// Pipeline depth: 6 stages of <= 33 KB (bn <= 64) or 4 of <= 49 KB (bn <= 128).
// 3: bn <= 32 (C2), three N = bn MMAs, 4 accumulator buffers of only 32 columns, so TMEM holds
// SIX A buffers (three pairs): the splitters run two pairs ahead of the MMAs instead of one
// (the split chain MMA(p) -> split(p + NP) -> MMA(p + NP) is what bounds these kernels).
#ifndef COFEM_TC_M3_STAGES
#define COFEM_TC_M3_STAGES 8 // 6: 17.97 ms at PLAG 3
#endif
#ifndef COFEM_TC_M3_PLAG
#define COFEM_TC_M3_PLAG 2   // C2 E-step: 2 17.90 ms, 3 18.07, 4 18.04 (mode 1: 19.10)
#endif
// 4: bn <= 32, FUSED: one N = 2 bn = 64 MMA forms A_hi [B_hi | B_lo] and one N = bn MMA adds A_lo B_hi
// (2 MMAs per K = 8 instead of 3, against the issuing thread's ~42 cycles per tcgen05.mma --
// tools/tc_trace.py C2: 1009 of mode 3's 1579-cycle pair period), 4 accumulators of 64, four A
// buffers.  Measured slower than mode 3 (C2 E-step 16.2 vs 15.5 ms): build switch only.
__host__ __device__ constexpr int stages_of(int mode) { return mode == 2 ? 4 : (mode == 3 || mode == 4) ? COFEM_TC_M3_STAGES : 6; }
__host__ __device__ constexpr int nacc_of(int mode) { return mode == 1 || mode == 3 || mode == 4 ? 4 : 2; }
__host__ __device__ constexpr int accw_of(int mode) { return mode == 3 ? 32 : (mode == 1 || mode == 4) ? 64 : 128; }
__host__ __device__ constexpr int nabuf_of(int mode) { return mode == 3 ? 6 : 4; }        // TMEM A buffers
__host__ __device__ constexpr int tma_of(int mode) { return mode == 3 ? 128 : TM_A; }     // their base column
__host__ __device__ constexpr int plag_of(int mode) { return mode == 3 ? COFEM_TC_M3_PLAG : PLAG; }
__host__ __device__ constexpr bool fused_of(int mode) { return mode == 0 || mode == 4; }

// Accumulator columns promoted (and written by the epilogue) per splitter group: the bn <= 64
// logical columns split evenly over the 4 groups (128 / 4 in mode 2).
__host__ __device__ constexpr int cpg_of(int mode) { return mode == 2 ? 32 : (mode == 3 || mode == 4) ? 8 : 16; }

// Shared-memory plan (dynamic, 1024-aligned):
// STAGES x [A: MT tiles x 16 KB | Bhi bn x 128 B | Blo bn x 128 B | mean-column operand 32 x fp64 (1 KB)]
struct Plan {
  int bn, mt, stages, stage_bytes;
  __host__ __device__ int a_off(int s, int t) const { return s * stage_bytes + t * BM * BK * 4; }
  __host__ __device__ int bhi_off(int s) const { return s * stage_bytes + mt * BM * BK * 4; }
  __host__ __device__ int blo_off(int s) const { return s * stage_bytes + mt * BM * BK * 4 + bn * 128; }
  __host__ __device__ int w_off(int s) const { return s * stage_bytes + mt * BM * BK * 4 + 2 * bn * 128; }
};

struct Bars {
  uint64_t full[8], split_done[4], pair_done[4], chunk_free[4];   // 4 phases apart: no parity aliasing
  uint32_t tmem_base;
  double red[NSPLIT][MAXM];        // epilogue per-warp column partials
  uint64_t mean_free[8];           // stage s's mean-column reads done (producer waits before reuse)
  double mean[NSPLIT][32];         // mean-column partials of the groups
  int last;
};

// TMEM columns: NACC accumulator buffers (one per in-flight promotion chunk), buffer ab of
// M-tile t at (ab MT + t) ACCW; A buffer b of M-tile t at TM_A + (b MT + t) 64 (hi 32 | lo 32),
// NAB / MT buffers cycled.  NACC = 4 (bn <= 64, MT = 1): the MMAs of chunk c + 4 wait for the
// promotion of chunk c, so the promotion latency never stalls the tensor core.  NACC = 2:
// 128-column buffers (bn up to 128, or the fused N = 2 bn MMA; COFEM_TC_FUSE).
template <int MT, int NACC> struct TmemPlan {
  static_assert(NACC * MT * (MT == 2 || NACC == 4 ? 64 : 128) <= TM_A, "TMEM accumulator budget");
  static constexpr int ACCW = (MT == 2 || NACC == 4) ? 64 : 128;
  static constexpr int NABU = NAB / MT;
  static constexpr int CPG = ACCW / NGROUP;        // accumulator columns promoted by each splitter group
  static __device__ __forceinline__ uint32_t acc(int ab, int t) { return (ab * MT + t) * ACCW; }
  static __device__ __forceinline__ uint32_t abuf(int b, int t) { return TM_A + (b * MT + t) * 64; }
};

// ---------------------------------------------------------------- the shared mainloop
// MN = true: A tile t is Phi[n0 : n0+32][d0 + 128 t : +128] as one dense [32][128] box
// (k_tc_phiTW, A = Phi^T, row m = d); false: Phi[n0 + 128 t : +128][d0 : d0+32], K-major
// with the 128-B swizzle (k_tc_phiP, A = Phi, row m = n).  mean_w: the fp64 mean-column
// operand along K (w0 for phiTW, p0 for phiP).  Returns, for a splitter thread, its fp64
// mean-column accumulators of row m of each tile (acc0[t]).
// Row m's 8 K-values [8h, 8h + 8) of a stage's A tile.  MN: [32 n][128 d] dense, a warp reads
// 128 contiguous bytes per n (conflict-free); else row m of 128 B with logical 16-B chunk c at
// physical chunk c ^ (m & 7) (SWIZZLE_128B).
template <bool MN>
__device__ __forceinline__ void load_row8(const unsigned char* a, int m, int h, float (&x)[8]) {
  if (MN) {
    const float* col = reinterpret_cast<const float*>(a) + m;
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = col[(8 * h + i) * BM];
  } else {
    const unsigned char* rowp = a + m * 128;
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      const int c = 2 * h + cc;
      const float4 v = *reinterpret_cast<const float4*>(rowp + ((c ^ (m & 7)) << 4));
      x[4 * cc] = v.x; x[4 * cc + 1] = v.y; x[4 * cc + 2] = v.z; x[4 * cc + 3] = v.w;
    }
  }
}

template <bool MN, int MODE>
__device__ void mainloop(const Plan& pl, unsigned char* sm, Bars& bs, const CUtensorMap* mA, const CUtensorMap* mBh,
                         const CUtensorMap* mBl, int row0, int k0, int nk, const double* __restrict__ mean_w,
                         double (&acc0)[1], float (&sum)[1][cpg_of(MODE)]) {
  constexpr int NACC = nacc_of(MODE), S = stages_of(MODE);      // compile-time: no integer division on the MMA thread's path
  constexpr int CPG = cpg_of(MODE), ACCW = accw_of(MODE), NABUF = nabuf_of(MODE), NP = NABUF / 2, PL = plag_of(MODE);
  struct TP {      // TMEM plan of this mode: NACC accumulators of ACCW columns, NABUF A buffers (hi 32 | lo 32)
    static __device__ __forceinline__ uint32_t acc(int ab, int) { return ab * ACCW; }
    static __device__ __forceinline__ uint32_t abuf(int b, int) { return tma_of(MODE) + b * 64; }
  };
  static_assert(NACC * ACCW <= tma_of(MODE) && tma_of(MODE) + NABUF * 64 <= TMEM_COLS, "TMEM budget");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t tmem = bs.tmem_base;
  const int np = (nk + 1) >> 1;                     // K-step pairs (= promotion chunks)
  constexpr bool fuse = fused_of(MODE);
  acc0[0] = 0.0;
#pragma unroll
  for (int i = 0; i < CPG; ++i) sum[0][i] = 0.f;
  if (warp == 0) {
    if (lane == 0) {                                  // ---- TMA producer
#ifdef COFEM_TC_EXP_NOTMA
      const uint32_t bytes = 0;
#else
      const uint32_t bytes = BM * BK * 4 + 2 * pl.bn * 128 + BK * 8;
#endif
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % S;
        if (kt >= S && !(kt & 1)) {                   // stages of pair (kt - S) / 2 free once its MMAs retired
          const int q = (kt - S) >> 1;
          mbar_wait(&bs.pair_done[q & 3], (q >> 2) & 1);
        }
        if (kt >= S) mbar_wait(&bs.mean_free[s], ((kt / S) - 1) & 1);
        TC_TRACE(kt, 8)
        mbar_expect_tx(&bs.full[s], bytes);
        const int kc = k0 + kt * BK;
#ifdef COFEM_TC_EXP_NOTMA
        if (kc >= 0) continue;
#endif
        if (MN) tma_load_2d(sm + pl.a_off(s, 0), mA, &bs.full[s], row0, kc);
        else tma_load_2d(sm + pl.a_off(s, 0), mA, &bs.full[s], kc, row0);
        tma_load_2d(sm + pl.bhi_off(s), mBh, &bs.full[s], kc, 0);
        tma_load_2d(sm + pl.blo_off(s), mBl, &bs.full[s], kc, 0);
        bulk_load(sm + pl.w_off(s), mean_w + kc, BK * 8, &bs.full[s]);
      }
    }
  } else if (warp == 1) {
    {                                                 // ---- MMA issuer (whole warp, one lane elected per instruction)
      const uint32_t idesc = idesc_tf32(pl.bn);
      // B_hi and B_lo are adjacent K-major row blocks of the stage, so when the accumulator has
      // room for 2 bn columns one N = 2 bn MMA forms A_hi [B_hi | B_lo] (hi.hi in columns
      // [0, bn), hi.lo in [bn, 2 bn), summed at promotion) and one N = bn MMA adds A_lo B_hi:
      // 2 instructions and 2 A-operand reads per K = 8 instead of 3.
      const uint32_t idesc2 = idesc_tf32(2 * pl.bn);
      for (int p = 0; p < np; ++p) {
        const int ab = p % NACC;
        if (p >= NACC) mbar_wait(&bs.chunk_free[ab], ((p / NACC) - 1) & 1);   // chunk p - NACC promoted
        if (lane == 0) TC_TRACE(p, 0)
        mbar_wait(&bs.split_done[p & 3], (p >> 2) & 1);   // both steps split (hence both stages loaded)
        if (lane == 0) TC_TRACE(p, 2)
        fence_after();
        const uint32_t d = tmem + TP::acc(ab, 0);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int kt = 2 * p + h;
          if (kt >= nk) break;
          const int s = kt % S;
          const uint32_t bh = su32(sm + pl.bhi_off(s)), bl = su32(sm + pl.blo_off(s));
          const uint32_t ahi = tmem + TP::abuf(kt % NABUF, 0), alo = ahi + 32;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {        // K = 8 per tf32 MMA; B advances 32 B in the swizzle atom
            const uint64_t dbh = desc_k_sw128(bh + kk * 32);
#ifdef COFEM_TC_EXP_1XTF32   // accuracy experiment (SURVEY §8(d) note 3): one tf32 MMA, no hi/lo corrections
            mma_ts_e(d, ahi + kk * 8, dbh, idesc, (h | kk) != 0);
            (void)alo; (void)bl; (void)fuse; (void)idesc2;
#else
            if (fuse) {
              mma_ts_e(d, ahi + kk * 8, dbh, idesc2, (h | kk) != 0);
            } else {
              mma_ts_e(d, ahi + kk * 8, dbh, idesc, (h | kk) != 0);
              mma_ts_e(d, ahi + kk * 8, desc_k_sw128(bl + kk * 32), idesc, 1);
            }
            mma_ts_e(d, alo + kk * 8, dbh, idesc, 1);
#endif
          }
        }
        mma_commit_e(&bs.pair_done[p & 3]);             // stages, A buffers and chunk p: all released here
        if (lane == 0) TC_TRACE(p, 3)
      }
    }
  } else {                                            // ---- splitters / promoters (warps 2 .. 2 + NSPLIT)
    // warp -> TMEM lane quarter q = warp % 4 (hardware rule) and group g: it owns row m for
    // the K steps kt = g (mod NGROUP) -- step h = g & 1 of the pairs p = g >> 1 (mod 2), into
    // TMEM A buffer kt % 4 -- and promotes accumulator columns [g CPG, (g+1) CPG) of row m.
    const int wi = warp - 2, q = warp & 3, g = wi >> 2, m = 32 * q + lane;
    const uint32_t lane_addr = tmem + ((uint32_t)(32 * q) << 16);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};             // independent DFMA chains (fixed-order sums below)
    int cdone = 0;
    auto promote = [&](int c) {                       // chunk (pair) c: TMEM accumulator -> register sums (RN)
      const int ab = c % NACC;
      mbar_wait(&bs.pair_done[c & 3], (c >> 2) & 1, SPLIT_SLEEP);
      if (q == 0 && lane == 0) TC_TRACE(4 * c + g, 7)
      fence_after();
#pragma unroll
      if constexpr (CPG == 8) {                         // modes 3 / 4: 8 columns per group
        if (g * CPG < pl.bn) {
          float v[8];
          tmem_ld8(lane_addr + TP::acc(ab, 0) + g * CPG, v);
          if constexpr (fuse) {                         // + the hi.lo half of the N = 2 bn product
            float u[8];
            tmem_ld8(lane_addr + TP::acc(ab, 0) + pl.bn + g * CPG, u);
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] += u[i];
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) sum[0][i] += v[i];
        }
      } else
      for (int cc = 0; cc < CPG; cc += 16) {
        if (g * CPG + cc >= pl.bn) continue;           // columns past bn carry nothing
#ifdef COFEM_TC_EXP_NOPROMO
        if (cc >= 0) continue;
#endif
        float v[16];
        tmem_ld16(lane_addr + TP::acc(ab, 0) + g * CPG + cc, v);
        if (fuse) {                                   // + the hi.lo half of the N = 2 bn product
          float u[16];
          tmem_ld16(lane_addr + TP::acc(ab, 0) + pl.bn + g * CPG + cc, u);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] += u[i];
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) sum[0][cc + i] += v[i];
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bs.chunk_free[ab]);
    };
    const int nk2 = 2 * np;                           // an odd nk leaves the second half of the last pair empty
    for (int kt = g; kt < nk2; kt += NGROUP) {
      // promote the chunks PLAG pairs behind this step (their MMAs need no split work of ours anymore)
      while (cdone < np && 2 * (cdone + PL) <= kt) promote(cdone++);
      const int p = kt >> 1;
      if (kt < nk) {
        const int s = kt % S;
        if (p >= NP) mbar_wait(&bs.pair_done[(p - NP) & 3], ((p - NP) >> 2) & 1, SPLIT_SLEEP);   // A buffer free
        if (q == 0 && lane == 0) TC_TRACE(kt, 5)
        mbar_wait(&bs.full[s], (kt / S) & 1, SPLIT_SLEEP);
        if (q == 0 && lane == 0) TC_TRACE(kt, 4)
        const unsigned char* a = sm + pl.a_off(s, 0);
        const uint32_t buf = TP::abuf(kt % NABUF, 0);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          float x[8];
          load_row8<MN>(a, m, h, x);
          float lo[8];
#ifdef COFEM_TC_EXP_RNHI
          float hi[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            hi[i] = tf32_hi_alu(x[i]);
            lo[i] = x[i] - hi[i];
          }
          tmem_st8(lane_addr + buf + 8 * h, hi);
#else
          // A_hi = x itself: the tensor core reads only its tf32 bits (truncation, measured by
          // tools/tf32_semantics.cu), so lo = x - trunc(x) is exact and no rounding is needed
#pragma unroll
          for (int i = 0; i < 8; ++i) lo[i] = x[i] - __uint_as_float(__float_as_uint(x[i]) & 0xFFFFE000u);
          tmem_st8(lane_addr + buf + 8 * h, x);
#endif
          tmem_st8(lane_addr + buf + 32 + 8 * h, lo);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bs.split_done[p & 3]);
      if (q == 0 && lane == 0) TC_TRACE(kt, 6)
      if (kt < nk) {   // fp64 mean column (R10) after the MMA's operands are out: off the critical path
        const int s = kt % S;
        const double* w = reinterpret_cast<const double*>(sm + pl.w_off(s));
        const unsigned char* a = sm + pl.a_off(s, 0);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          float x[8];
          load_row8<MN>(a, m, h, x);
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i & 3] = fma((double)x[i], w[8 * h + i], acc[i & 3]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bs.mean_free[s]);
      }
    }
    while (cdone < np) promote(cdone++);
    // combine the groups' partial sums of row m in fixed order (g = 0 .. NGROUP-1)
    bs.mean[wi][lane] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    asm volatile("bar.sync 1, %0;" ::"n"(32 * NSPLIT));
    double v = 0.0;
#pragma unroll
    for (int gg = 0; gg < NGROUP; ++gg) v += bs.mean[4 * gg + (wi & 3)][lane];
    acc0[0] = v;
  }
}

__device__ void setup_cta(Bars& bs, int stages) {
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&bs.full[s], 1); mbar_init(&bs.mean_free[s], 4); }
    for (int b = 0; b < 4; ++b) mbar_init(&bs.split_done[b], 8);      // 2 groups x 4 warps per pair
    for (int b = 0; b < 4; ++b) { mbar_init(&bs.pair_done[b], 1); mbar_init(&bs.chunk_free[b], NSPLIT); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&bs.tmem_base)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
}

__device__ void teardown_cta(Bars& bs) {
  fence_before();
  __syncthreads();
  if ((threadIdx.x >> 5) == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(bs.tmem_base), "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------- K1: W partials = Phi P (split-K over D)
struct PhiPArgs {
  Plan pl;
  int N, D, K, kchunk;             // kchunk: multiple of BK
  const double* p0;                // mean column p (fp64, D)
  float* Wpart;                    // [split][K][Npad]
  double* W0part;                  // [split][Npad]
  int Npad;
  const ColState* cs; int m;       // cs != nullptr: the launch exits when all m columns have frozen
};

// A launch whose columns have all frozen (R5) does nothing: every CTA votes on the same flags
// and returns before any barrier, TMEM or TMA setup (so the phiTW tickets stay untouched).
// Sharded runs pass cs = nullptr (their partial sums feed cross-rank reductions).
__device__ __forceinline__ bool all_frozen(const ColState* cs, int m) {
  if (!cs) return false;
  int act = 0;
  for (int j = threadIdx.x; j < m; j += blockDim.x) act |= !cs[j].frozen;
  return !__syncthreads_or(act);
}

template <int MODE>
__global__ void __launch_bounds__(THREADS, 1) k_tc_phiP(const __grid_constant__ CUtensorMap mA,
                                                        const __grid_constant__ CUtensorMap mBh,
                                                        const __grid_constant__ CUtensorMap mBl, PhiPArgs a) {
  constexpr int MT = 1;
  extern __shared__ __align__(1024) unsigned char sm[];      // no static smem: the dynamic base is 1024-aligned
  if (all_frozen(a.cs, a.m)) return;
  Bars& bs = *reinterpret_cast<Bars*>(sm + a.pl.stages * a.pl.stage_bytes);
  setup_cta(bs, a.pl.stages);
  const int row0 = blockIdx.x * BM * MT, split = blockIdx.y;
  const int k0 = split * a.kchunk, k1 = min(a.D, k0 + a.kchunk);
  const int nk = (k1 - k0 + BK - 1) / BK;
  double acc0[MT];
  float sum[MT][cpg_of(MODE)];
  mainloop<false, MODE>(a.pl, sm, bs, &mA, &mBh, &mBl, row0, k0, nk, a.p0, acc0, sum);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= 2) {
    constexpr int CPG = cpg_of(MODE);
    const int q = warp & 3, g = (warp - 2) >> 2;
    float* wp = a.Wpart + (size_t)split * a.K * a.Npad;
#pragma unroll
    for (int t = 0; t < MT; ++t) {
      const int n = row0 + BM * t + 32 * q + lane;
      if (n < a.N) {
#pragma unroll
        for (int i = 0; i < CPG; ++i) {
          const int col = g * CPG + i;
          if (col < a.K) wp[(size_t)col * a.Npad + n] = sum[t][i];
        }
        if (g == 0) a.W0part[(size_t)split * a.Npad + n] = acc0[t];
      }
    }
  }
  teardown_cta(bs);
}

// Split-K reduction in fixed order -> W_hi, W_lo (3xTF32 halves of W, the B operand of K2) and w0.
__global__ void k_tc_reduce_w(int N, int Npad, int K, int splits, const float* __restrict__ Wpart,
                              const double* __restrict__ W0part, float* __restrict__ Whi, float* __restrict__ Wlo,
                              double* __restrict__ w0) {
  const int64_t tot = (int64_t)K * Npad;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot + Npad; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < tot) {
      const int n = (int)(i % Npad);
      float v = 0.f;
      if (n < N)
        for (int s = 0; s < splits; ++s) v += Wpart[(int64_t)s * tot + i];
      if (Wlo) { const float h = tf32_hi(v); Whi[i] = h; Wlo[i] = v - h; }
      else Whi[i] = v;                                // sharded: raw partial W, split after the all-reduce
    } else {
      const int n = (int)(i - tot);
      double v = 0.0;
      if (n < N)
        for (int s = 0; s < splits; ++s) v += W0part[(int64_t)s * Npad + n];
      w0[n] = v;
    }
  }
}

// Sharded mode: W_hi / W_lo from the rank-summed W (in W_hi), in place.
__global__ void k_tc_split_w(int64_t n, float* __restrict__ Wh, float* __restrict__ Wl) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = Wh[i], h = tf32_hi(v);
    Wh[i] = h; Wl[i] = v - h;
  }
}

// P_hi / P_lo of the probe block (B operand of K1), [K][Dp]
__global__ void k_tc_split_p(int64_t n, const float* __restrict__ P, float* __restrict__ Ph, float* __restrict__ Pl) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = reinterpret_cast<const float4*>(P)[i];
    const float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
    reinterpret_cast<float4*>(Ph)[i] = h;
    reinterpret_cast<float4*>(Pl)[i] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
  }
}

// ---------------------------------------------------------------- K2: Q = beta Phi^T W + alpha o P, gamma
struct PhiTWArgs {
  Plan pl;
  int N, D, K;
  int64_t Dp;
  double beta;
  const double* alpha; const double* w0; const double* p0; double* q0;
  const float* P; float* Q;
  ColState* cs; double* part; int stride; unsigned* counter; int iter;
  double* colsum;
  // split-K over N (gridDim.y splits; build switch COFEM_TC_KSPLIT2): split partials [split][K][Dp] /
  // [split][Dp]; the tile's last split (ticket) sums them in split order
  float* Qpart; double* Q0part; unsigned* tile_cnt;
};

template <int MODE>
__global__ void __launch_bounds__(THREADS, 1) k_tc_phiTW(const __grid_constant__ CUtensorMap mA,
                                                         const __grid_constant__ CUtensorMap mBh,
                                                         const __grid_constant__ CUtensorMap mBl, PhiTWArgs a) {
  constexpr int MT = 1;
  extern __shared__ __align__(1024) unsigned char sm[];      // no static smem: the dynamic base is 1024-aligned
  if (all_frozen(a.colsum ? nullptr : a.cs, a.K + 1)) return;
  Bars& bs = *reinterpret_cast<Bars*>(sm + a.pl.stages * a.pl.stage_bytes);
  for (int i = threadIdx.x; i < NSPLIT * MAXM; i += THREADS) (&bs.red[0][0])[i] = 0.0;
  setup_cta(bs, a.pl.stages);
  const int row0 = blockIdx.x * BM * MT;
  const int nk_all = (a.N + BK - 1) / BK, ks = gridDim.y, split = blockIdx.y;
  const int kchunk = (nk_all + ks - 1) / ks, kt0 = split * kchunk, nk = min(nk_all - kt0, kchunk);
  double acc0[MT];
  float sum[MT][cpg_of(MODE)];
  mainloop<true, MODE>(a.pl, sm, bs, &mA, &mBh, &mBl, row0, kt0 * BK, nk, a.w0, acc0, sum);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = a.K + 1;
  if (ks > 1) {        // split-K: partials out; the tile's last split sums them in split order (deterministic)
    if (warp >= 2) {
      constexpr int CPG = cpg_of(MODE);
      const int q = warp & 3, g = (warp - 2) >> 2, d = row0 + 32 * q + lane;
      if (d < a.D) {
#pragma unroll
        for (int i = 0; i < CPG; ++i) {
          const int k = g * CPG + i;
          if (k < a.K) a.Qpart[((int64_t)split * a.K + k) * a.Dp + d] = sum[0][i];
        }
        if (g == 0) a.Q0part[(int64_t)split * a.Dp + d] = acc0[0];
      }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) bs.last = atomicAdd(a.tile_cnt + blockIdx.x, 1u) == (unsigned)ks - 1;
    __syncthreads();
    if (!bs.last) { teardown_cta(bs); return; }
    __threadfence();
    if (warp >= 2) {
      constexpr int CPG = cpg_of(MODE);
      const int q = warp & 3, g = (warp - 2) >> 2, d = row0 + 32 * q + lane;
      if (d < a.D) {
#pragma unroll
        for (int i = 0; i < CPG; ++i) {
          const int k = g * CPG + i;
          if (k >= a.K) break;
          float v = 0.f;
          for (int sp = 0; sp < ks; ++sp) v += __ldcg(a.Qpart + ((int64_t)sp * a.K + k) * a.Dp + d);
          sum[0][i] = v;
        }
        if (g == 0) {
          double v = 0.0;
          for (int sp = 0; sp < ks; ++sp) v += __ldcg(a.Q0part + (int64_t)sp * a.Dp + d);
          acc0[0] = v;
        }
      }
    }
    if (threadIdx.x == 0) a.tile_cnt[blockIdx.x] = 0u;
  }
  if (warp >= 2) {
    constexpr int CPG = cpg_of(MODE);
    const int wi = warp - 2, q = warp & 3, g = wi >> 2;
    if (g == 0) {     // mean column (fp64): q0 = beta (Phi^T w0)_d + alpha_d p0_d
      double gm = 0.0;
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        const int d = row0 + BM * t + 32 * q + lane;
        if (d < a.D) {
          const double p = a.p0[d], qv = a.beta * acc0[t] + a.alpha[d] * p;
          a.q0[d] = qv;
          gm += p * qv;
        }
      }
      gm = warp_sum(gm);
      if (lane == 0) bs.red[wi][0] = gm;
    }
    const float bt = (float)a.beta;
    float alf[MT];
#pragma unroll
    for (int t = 0; t < MT; ++t) {
      const int d = row0 + BM * t + 32 * q + lane;
      alf[t] = d < a.D ? (float)a.alpha[d] : 0.f;
    }
#pragma unroll
    for (int i = 0; i < CPG; ++i) {
      const int k = g * CPG + i;
      if (k >= a.K) break;                            // warp-uniform
      double gk = 0.0;
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        const int d = row0 + BM * t + 32 * q + lane;
        if (d < a.D) {
          const float p = a.P[(int64_t)k * a.Dp + d];
          const float qv = bt * sum[t][i] + alf[t] * p;   // a3: q = beta Phi^T Phi p + alpha o p
          a.Q[(int64_t)k * a.Dp + d] = qv;
          gk += (double)p * (double)qv;               // a4
        }
      }
      gk = warp_sum(gk);
      if (lane == 0) bs.red[wi][k + 1] = gk;
    }
  }
  __syncthreads();
  // CTA partials (fixed warp order) -> part[j][cta]; last CTA reduces (deterministic), R5
  for (int j = threadIdx.x; j < m; j += THREADS) {
    double v = 0.0;
#pragma unroll
    for (int wi = 0; wi < NSPLIT; ++wi) v += bs.red[wi][j];
    a.part[(int64_t)j * a.stride + blockIdx.x] = v;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) bs.last = atomicAdd(a.counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (bs.last) {
    __threadfence();
    for (int j = warp; j < m; j += THREADS / 32) {
      const double v = reduce_partials(a.part + (int64_t)j * a.stride, gridDim.x);
      if (lane == 0) {
        if (a.colsum) a.colsum[j] = v;              // sharded: summed over ranks, then finished
        else { ColState c = a.cs[j]; finish_gamma(c, v, a.iter); a.cs[j] = c; }
      }
    }
    if (threadIdx.x == 0) *a.counter = 0u;
  }
  teardown_cta(bs);
}

// ---------------------------------------------------------------- host
typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiled encoder() {
  static EncodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiled)p;
  }
  return fn;
}

// 2D fp32 tensor [rows][cols] (cols contiguous, row pitch ld elements), box {bx (cols), by (rows)}, 128-B swizzle
static bool make_map(CUtensorMap* m, const float* base, int64_t cols, int64_t rows, int64_t ld, int bx, int by,
                     bool swizzle = true) {
  EncodeTiled enc = encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)bx, (cuuint32_t)by};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

static Plan plan_for(int bn, int mt, int mode) {
  Plan p;
  p.bn = bn; p.mt = mt;
  p.stage_bytes = mt * BM * BK * 4 + 2 * bn * 128 + 1024;   // + 32 fp64 mean operands, padded to keep 1024-B alignment
  p.stages = stages_of(mode);                                // even: whole pairs
  return p;
}
static size_t smem_of(const Plan& p) { return (size_t)p.stages * p.stage_bytes + sizeof(Bars); }

}  // namespace tc

struct DenseTC {
  CUtensorMap phi_k, phi_mn, phh, pll, whh, wll;
  float *Ph, *Pl, *Wh, *Wl, *Wpart, *Qpart;
  double *W0part, *w0, *Q0part;
  unsigned* tile_cnt;
  int bn, mt, splits, kchunk, Npad, ksplit2;
  int mode;
  tc::Plan pl;
};

void dense_tc_free(Ctx* c) {
  DenseTC* t = (DenseTC*)c->dense_tc;
  if (!t) return;
  void* ptrs[] = {t->Ph, t->Pl, t->Wh, t->Wl, t->Wpart, t->W0part, t->w0, t->Qpart, t->Q0part, t->tile_cnt};
  for (void* p : ptrs) if (p) cudaFree(p);
  delete t;
  c->dense_tc = nullptr;
}

// Set up the tensor-core path (fp32 probes only); leaves c->dense_tc NULL (SIMT path) when
// the shape cannot use it.
cofem_status dense_tc_setup(Ctx* c) {
  using namespace tc;
  if (c->probe64 || c->opt.apply_path == 1) return COFEM_OK;        // parity mode / general kernels: FP32 SIMT
  if (c->D % 4 != 0 || c->ld % 4 != 0 || ((uintptr_t)c->phi & 15) || c->Kcap > 128)
    return COFEM_OK;                                                // TMA: 16-B base and row pitch; N <= 128 per MMA
  if (!encoder()) return COFEM_OK;
  DenseTC* t = new DenseTC();
  memset(t, 0, sizeof *t);
  c->dense_tc = t;
  t->bn = std::max(16, (c->Kcap + 15) / 16 * 16);
  t->mt = 1;                                      // one 128-row M-tile per CTA (pair protocol)
#ifdef COFEM_TC_FUSE
  t->mode = t->bn > 64 ? 2 : 0;                   // timing comparison build (tools/build_variant.sh)
#else
#ifndef COFEM_TC_MODE3
#define COFEM_TC_MODE3 1      // bn <= 32: 1 = mode 3 (six A buffers), 2 = mode 4 (fused: C2 16.2 vs 15.5 ms, slower), 0 = mode 1
#endif
  t->mode = t->bn > 64 ? 2 : (COFEM_TC_MODE3 && t->bn <= 32 ? (COFEM_TC_MODE3 == 2 ? 4 : 3) : 1);
#endif
  t->pl = plan_for(t->bn, t->mt, t->mode);
  if (smem_of(t->pl) > 227 * 1024) { c->err = "dense tc: shared-memory plan too large"; return COFEM_ERR_INVALID; }
  t->Npad = (int)((c->N + 31) / 32 * 32);
  const int rows = BM * t->mt;
  const int mtiles = (int)((c->N + rows - 1) / rows);
  // split-K: the K1 grid (one CTA per SM) is sized to just fill whole waves (>= 8 K steps per split)
  const int ksteps = (int)((c->D + BK - 1) / BK);
  int splits = 1;
  // from ONE wave up (C2: 16 M-tiles x 9 splits = 144 CTAs, E-step 15.7 -> 14.7 ms against 18 splits
  // in two waves; fewer partials for k_tc_reduce_w too); C3 (64 M-tiles) still takes 9 splits
  for (int w = 1; w <= 8; ++w) {
    const int sp = std::max(1, std::min(ksteps / 8, (w * c->num_sms) / mtiles));
    if (sp * mtiles >= (w * c->num_sms * 7) / 8) { splits = sp; break; }
    splits = sp;
  }
#ifdef COFEM_TC_SPLITS
  splits = std::max(1, std::min(ksteps, COFEM_TC_SPLITS));   // tuning build switch: force the K1 split count
#endif
  t->kchunk = ((ksteps + splits - 1) / splits) * BK;
  t->splits = (int)((c->D + t->kchunk - 1) / t->kchunk);
  const size_t pk = (size_t)c->Kcap * c->Dp, wk = (size_t)c->Kcap * t->Npad;
  if (cudaMalloc(&t->Ph, pk * 4) || cudaMalloc(&t->Pl, pk * 4) || cudaMalloc(&t->Wh, wk * 4) ||
      cudaMalloc(&t->Wl, wk * 4) || cudaMalloc(&t->Wpart, (size_t)t->splits * wk * 4) ||
      cudaMalloc(&t->W0part, (size_t)t->splits * t->Npad * 8) || cudaMalloc(&t->w0, (size_t)t->Npad * 8)) {
    c->err = "cudaMalloc dense tensor-core workspace"; return COFEM_ERR_OOM;
  }
  {   // K2 split-K over N while the D tiles alone fill under half of the SMs: the splits stay in one
      // wave, >= 8 K steps each (C2: 63 tiles x 2 = 126 CTAs, E-step 14.77 -> 13.65 ms; C3: 256 tiles,
      // unsplit -- split-K measured slower there)
#ifndef COFEM_TC_KSPLIT2
#define COFEM_TC_KSPLIT2 0    // build switch: force the K2 split count (0 = the rule above)
#endif
    const int tiles2 = (int)((c->D + BM - 1) / BM), nk2 = (int)((c->N + BK - 1) / BK);
    t->ksplit2 = COFEM_TC_KSPLIT2 > 0 ? COFEM_TC_KSPLIT2 : std::min(c->num_sms / std::max(tiles2, 1), nk2 / 8);
    t->ksplit2 = std::max(1, std::min(t->ksplit2, nk2));
    if (t->ksplit2 > 1) {
      if (cudaMalloc(&t->Qpart, (size_t)t->ksplit2 * c->Kcap * c->Dp * 4) ||
          cudaMalloc(&t->Q0part, (size_t)t->ksplit2 * c->Dp * 8) || cudaMalloc(&t->tile_cnt, (size_t)tiles2 * 4)) {
        c->err = "cudaMalloc dense tensor-core split workspace"; return COFEM_ERR_OOM;
      }
      cudaMemset(t->tile_cnt, 0, (size_t)tiles2 * 4);
    }
  }
  cudaMemset(t->Ph, 0, pk * 4); cudaMemset(t->Pl, 0, pk * 4);
  cudaMemset(t->Wh, 0, wk * 4); cudaMemset(t->Wl, 0, wk * 4);
  cudaMemset(t->w0, 0, (size_t)t->Npad * 8);
  bool ok = make_map(&t->phi_k, c->phi, c->D, c->N, c->ld, BK, BM) &&            // K1 A: Phi[n][d], box 32 d x 128 n
            make_map(&t->phi_mn, c->phi, c->D, c->N, c->ld, BM, BK, false) &&    // K2 A: box 128 d x 32 n, dense
            make_map(&t->phh, t->Ph, c->Dp, c->Kcap, c->Dp, BK, t->bn) &&        // K1 B: P_hi, P_lo [K][Dp]
            make_map(&t->pll, t->Pl, c->Dp, c->Kcap, c->Dp, BK, t->bn) &&
            make_map(&t->whh, t->Wh, t->Npad, c->Kcap, t->Npad, BK, t->bn) &&    // K2 B: W_hi, W_lo [K][Npad]
            make_map(&t->wll, t->Wl, t->Npad, c->Kcap, t->Npad, BK, t->bn);
  if (!ok) { c->err = "cuTensorMapEncodeTiled failed"; return COFEM_ERR_CUDA; }
  const int sm = (int)smem_of(t->pl);
  raise_smem_attr((const void*)k_tc_phiP<0>, sm);
  raise_smem_attr((const void*)k_tc_phiP<1>, sm);
  raise_smem_attr((const void*)k_tc_phiP<2>, sm);
  raise_smem_attr((const void*)k_tc_phiP<3>, sm);
  raise_smem_attr((const void*)k_tc_phiP<4>, sm);
  raise_smem_attr((const void*)k_tc_phiTW<0>, sm);
  raise_smem_attr((const void*)k_tc_phiTW<1>, sm);
  raise_smem_attr((const void*)k_tc_phiTW<2>, sm);
  raise_smem_attr((const void*)k_tc_phiTW<3>, sm);
  raise_smem_attr((const void*)k_tc_phiTW<4>, sm);
  c->part_stride = std::max(c->part_stride, (int)((c->D + BM - 1) / BM));
  return check_launch(c, "dense tc setup") == cudaSuccess ? COFEM_OK : COFEM_ERR_CUDA;
}

void dense_tc_p_split(Ctx* c, float** ph, float** pl) {
  DenseTC* t = (DenseTC*)c->dense_tc;
  *ph = t ? t->Ph : nullptr;
  *pl = t ? t->Pl : nullptr;
}

cofem_status dense_tc_apply(Ctx* c, int m, int iter) {
  using namespace tc;
  DenseTC* t = (DenseTC*)c->dense_tc;
  const int K = m - 1;
  const size_t sm = smem_of(t->pl);
  const int rows = BM * t->mt;
  launch_begin(c, KC_DENSE_PHI_P);
  // P_hi / P_lo: already written by the direction kernel (k_dir) when it ran just before this apply
  if (!(c->p_presplit && iter > 0))
    k_tc_split_p<<<c->num_sms * 4, 256, 0, c->stream>>>((int64_t)K * c->Dp, (const float*)c->P, t->Ph, t->Pl);
  c->p_presplit = false;
  PhiPArgs a1;
  a1.pl = t->pl; a1.N = (int)c->N; a1.D = (int)c->D; a1.K = K; a1.kchunk = t->kchunk; a1.p0 = c->p0;
  a1.Wpart = t->Wpart; a1.W0part = t->W0part; a1.Npad = t->Npad;
  a1.cs = c->sharded ? nullptr : c->cs; a1.m = m;
  const dim3 g1((unsigned)((c->N + rows - 1) / rows), t->splits);
  if (t->mode == 0) k_tc_phiP<0><<<g1, THREADS, sm, c->stream>>>(t->phi_k, t->phh, t->pll, a1);
  else if (t->mode == 1) k_tc_phiP<1><<<g1, THREADS, sm, c->stream>>>(t->phi_k, t->phh, t->pll, a1);
  else if (t->mode == 3) k_tc_phiP<3><<<g1, THREADS, sm, c->stream>>>(t->phi_k, t->phh, t->pll, a1);
  else if (t->mode == 4) k_tc_phiP<4><<<g1, THREADS, sm, c->stream>>>(t->phi_k, t->phh, t->pll, a1);
  else k_tc_phiP<2><<<g1, THREADS, sm, c->stream>>>(t->phi_k, t->phh, t->pll, a1);
  k_tc_reduce_w<<<c->num_sms * 4, 256, 0, c->stream>>>((int)c->N, t->Npad, K, t->splits, t->Wpart, t->W0part, t->Wh,
                                                       c->sharded ? nullptr : t->Wl, t->w0);
  if (c->sharded) {      // W = sum over ranks of Phi_r P_r (SURVEY §8(e) column-sharded dense), then split
    cofem_status st;         // the fp32 probe block and the fp64 mean column: one grouped NCCL launch
    if ((st = comm_group(c, true)) != COFEM_OK) return st;
    if ((st = comm_allreduce(c, t->Wh, (size_t)K * t->Npad, 0)) != COFEM_OK) { comm_group(c, false); return st; }
    if ((st = comm_allreduce(c, t->w0, (size_t)t->Npad, 1)) != COFEM_OK) { comm_group(c, false); return st; }
    if ((st = comm_group(c, false)) != COFEM_OK) return st;
    k_tc_split_w<<<c->num_sms * 4, 256, 0, c->stream>>>((int64_t)K * t->Npad, t->Wh, t->Wl);
  }
  launch_end(c, KC_DENSE_PHI_P);
  if (check_launch(c, "k_tc_phiP")) return COFEM_ERR_CUDA;
  PhiTWArgs a2;
  a2.pl = t->pl; a2.N = (int)c->N; a2.D = (int)c->D; a2.K = K; a2.Dp = c->Dp; a2.beta = c->beta;
  a2.alpha = c->alpha; a2.w0 = t->w0; a2.p0 = c->p0; a2.q0 = c->q0; a2.P = (const float*)c->P; a2.Q = (float*)c->Q;
  a2.cs = c->cs; a2.part = c->part; a2.stride = c->part_stride; a2.counter = c->counters + MAXM; a2.iter = iter;
  a2.colsum = c->sharded ? c->colsum : nullptr;
  a2.Qpart = t->Qpart; a2.Q0part = t->Q0part; a2.tile_cnt = t->tile_cnt;
  launch_begin(c, KC_DENSE_PHIT_W);
  const dim3 g2((unsigned)((c->D + rows - 1) / rows), (unsigned)t->ksplit2);
  if (t->mode == 0) k_tc_phiTW<0><<<g2, THREADS, sm, c->stream>>>(t->phi_mn, t->whh, t->wll, a2);
  else if (t->mode == 1) k_tc_phiTW<1><<<g2, THREADS, sm, c->stream>>>(t->phi_mn, t->whh, t->wll, a2);
  else if (t->mode == 3) k_tc_phiTW<3><<<g2, THREADS, sm, c->stream>>>(t->phi_mn, t->whh, t->wll, a2);
  else if (t->mode == 4) k_tc_phiTW<4><<<g2, THREADS, sm, c->stream>>>(t->phi_mn, t->whh, t->wll, a2);
  else k_tc_phiTW<2><<<g2, THREADS, sm, c->stream>>>(t->phi_mn, t->whh, t->wll, a2);
  launch_end(c, KC_DENSE_PHIT_W);
  if (check_launch(c, "k_tc_phiTW")) return COFEM_ERR_CUDA;
  if (c->sharded) {   // gamma (+ delta1, delta2 for the single-reduction CG, R23): one all-reduce
    cofem_status st = c->sr ? sr_dots(c, m) : COFEM_OK;
    if (st == COFEM_OK) st = sharded_finish(c, m, c->sr ? 3 : 1, iter);
    if (st != COFEM_OK) return st;
  }
#ifdef COFEM_TC_DEBUG
  {                                   // synchronous protocol check (debug build)
    cudaStreamSynchronize(c->stream);
    unsigned long long h[4];
    cudaMemcpyFromSymbol(h, g_tc_stuck, sizeof h);
    if (h[0]) {
      fprintf(stderr, "cofem tc: stuck wait: block (%llu,%llu) warp %llu smem offset 0x%llx parity %llu\n", h[1] >> 32,
              (h[1] >> 16) & 0xFFFF, h[1] & 0xFFFF, h[2] >> 32, h[2] & 0xFFFFFFFF);
      c->err = "tensor-core pipeline stall"; return COFEM_ERR_CUDA;
    }
  }
#endif
  return COFEM_OK;
}

}  // namespace cofem

#ifdef COFEM_TC_EXP_TRACE
extern "C" int cofem_tc_trace_dump(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, cofem::tc::g_tc_trace, sizeof(cofem::tc::g_tc_trace));
}
#endif
