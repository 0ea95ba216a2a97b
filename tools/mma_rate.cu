// mma_rate.cu — measured tcgen05.mma issue/throughput ceilings for the shapes the dense
// 3xTF32 path uses (kind::tf32, M = 128, K = 8 per instruction, A from TMEM or shared
// memory, B from shared memory), with kind::f16 (bf16) for comparison.  Data is garbage;
// only the rate matters.  One CTA per SM, one elected thread issues back-to-back MMAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_rate tools/mma_rate.cu -lcuda && /tmp/mma_rate
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_k_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int fmt, int n) {   // fmt: 2 = tf32, 1 = bf16
  return (1u << 4) | ((uint32_t)fmt << 7) | ((uint32_t)fmt << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

template <bool TS, int FMT>
__device__ __forceinline__ void mma(uint32_t d, uint32_t a_tmem, uint64_t adesc, uint64_t bdesc, uint32_t id, uint32_t acc) {
  if (TS) {
    if (FMT == 2)
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                   "r"(a_tmem), "l"(bdesc), "r"(id), "r"(acc) : "memory");
    else
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                   "r"(a_tmem), "l"(bdesc), "r"(id), "r"(acc) : "memory");
  } else {
    if (FMT == 2)
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                   "l"(adesc), "l"(bdesc), "r"(id), "r"(acc) : "memory");
    else
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                   "l"(adesc), "l"(bdesc), "r"(id), "r"(acc) : "memory");
  }
}

// Whole warp converged; one lane elected inside the asm block (no per-MMA ELECT loop in SASS?)
__device__ __forceinline__ void mma_ts_elect(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(id), "r"(acc) : "memory");
}

template <bool TS, int FMT, int NACC, int NCOMMIT>
__global__ void __launch_bounds__(128, 1) k_rate(int n, int reps, unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar, dummy[4];
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&dummy[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    const uint32_t id = idesc(FMT, n), a_t = tbase + 256, d = tbase;
    const uint32_t sa = su32(sm), sb = su32(sm + 16384);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma<TS, FMT>(d + (kk % NACC) * n, a_t + kk * (FMT == 2 ? 8 : 8), desc_k_sw128(sa + kk * 32), desc_k_sw128(sb + kk * 32), id,
                     r != 0);
      // ncommit > 0: one commit every ncommit K-steps of 4 MMAs; < 0: -ncommit commits per K step
      if (NCOMMIT > 0 && (r % NCOMMIT) == NCOMMIT - 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&dummy[0])) : "memory");
      #pragma unroll
      for (int i = 0; i < -NCOMMIT; ++i)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&dummy[i])) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    for (;;) {
      uint32_t done;
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(su32(&bar)) : "memory");
      if (done) break;
    }
    long long t1 = clock64();
    if (blockIdx.x == 0) *cyc = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
  }
}


// The dense path's fused pair pattern: per K = 8, N = 2 bn (A_hi) then N = bn (A_lo) into the
// same accumulator, 8 per K step, one commit per pair of steps.  MODE 0: that pattern;
// 1: the N = 2 bn MMAs only; 2: the N = bn MMAs only; 3: pattern with the N = bn MMA into a
// separate accumulator; 4: N = 2 bn MMAs with alternating A addresses.
template <int MODE>
__global__ void __launch_bounds__(576, 1) k_pair(int bn, int pairs, unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar[4];
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) stop = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (MODE >= 20 ? warp == 0 : threadIdx.x == 0) {
    const uint32_t id1 = idesc(2, bn), id2 = idesc(2, 2 * bn);
    long long t0 = clock64();
    for (int p = 0; p < pairs; ++p) {
      const uint32_t d = tbase + (p & 1) * 128;
      for (int h = 0; h < 2; ++h) {
        const int kt = 2 * p + h;
        const uint32_t bh = su32(sm + (kt % 6) * 16384);
        const uint32_t ahi = tbase + 256 + (kt & 3) * 64, alo = ahi + 32;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t db = desc_k_sw128(bh + kk * 32);
          if (MODE >= 20) {
            if (MODE != 22) mma_ts_elect(d, ahi + kk * 8, db, id2, (h | kk) != 0);
            if (MODE != 21) mma_ts_elect(d, alo + kk * 8, db, id1, MODE == 22 ? (h | kk) != 0 : 1);
          } else {
          if (MODE != 2) mma<true, 2>(d, MODE == 4 && (kk & 1) ? alo + kk * 8 : ahi + kk * 8, 0, db, id2, (h | kk) != 0);
          if (MODE != 1 && MODE != 4) mma<true, 2>(MODE == 3 ? d + 64 : d, alo + kk * 8, 0, db, id1, MODE == 2 ? (h | kk) != 0 : 1);
          }
        }
      }
      if (MODE >= 20)
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&bar[p & 3])) : "memory");
      else
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[p & 3])) : "memory");
    }
    if (MODE >= 20)
      asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&bar[0])) : "memory");
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[0])) : "memory");
    for (;;) {   // wait for everything: the final phase of bar[0] flips after the last commit
      uint32_t done;
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(su32(&bar[0])), "r"((uint32_t)(((pairs + 3) / 4) & 1)) : "memory");
      if (done) break;
    }
    long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = (unsigned long long)(t1 - t0);
    stop = 1;
  } else if (threadIdx.x >= 64 && blockDim.x > 128) {   // idle "splitter" warps polling with back-off
    while (!stop) __nanosleep(MODE >= 10 ? 0 : 40);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
  }
}

template <int MODE>
void run_pair(const char* name, int threads = 128) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8);
  const int smem = 6 * 16384 + 1024, pairs = 1024;
  cudaFuncSetAttribute(k_pair<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_pair<MODE><<<sms, threads, smem>>>(64, 16, cyc);
  k_pair<MODE><<<sms, threads, smem>>>(64, pairs, cyc);
  cudaDeviceSynchronize();
  unsigned long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("pair %-28s thr=%d %7.1f cycles/pair  (%s)\n", name, threads, (double)c / pairs, cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}

template <bool TS, int FMT, int NACC = 1, int NCOMMIT = 0>
void run(const char* name, int n) {
  const int nacc = NACC, ncommit = NCOMMIT;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8);
  const int reps = 4096, smem = 64 * 1024;
  cudaFuncSetAttribute(k_rate<TS, FMT, NACC, NCOMMIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_rate<TS, FMT, NACC, NCOMMIT><<<sms, 128, smem>>>(n, 16, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_rate<TS, FMT, NACC, NCOMMIT><<<sms, 128, smem>>>(n, reps, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double kper = FMT == 2 ? 8 : 16;
  const double flop = 2.0 * 128 * n * kper * 4 * reps * sms;
  printf("%-10s N=%3d nacc=%d commits/4=%d  %7.1f cycles/MMA  %8.1f TFLOP/s  (%s)\n", name, n, nacc, ncommit, (double)c / (4.0 * reps), flop / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}

int main() {
  for (int n : {32, 64, 128, 256}) {
    run<true, 2>("tf32 TS", n);
    run<false, 2>("tf32 SS", n);
    run<false, 1>("bf16 SS", n);
  }
  run<true, 2, 2>("tf32 TS", 64);
  run<true, 2, 4>("tf32 TS", 64);
  // commit cost: one per 8 / 4 / 2 / 1 K-steps of 4 MMAs, then 2 and 3 per K step
  for (int n : {64, 128}) {
    run<true, 2, 1, 8>("tf32 TS", n);
    run<true, 2, 1, 4>("tf32 TS", n);
    run<true, 2, 1, 2>("tf32 TS", n);
    run<true, 2, 1, 1>("tf32 TS", n);
    run<true, 2, 1, -2>("tf32 TS", n);
    run<true, 2, 1, -3>("tf32 TS", n);
  }
  run<false, 1, 1, 1>("bf16 SS", 256);
  run_pair<0>("fused pattern");
  run_pair<1>("N=128 only (8/pair)");
  run_pair<2>("N=64 only (8/pair)");
  run_pair<3>("pattern, separate acc");
  run_pair<4>("N=128 only, alternating A");
  run_pair<0>("fused pattern", 576);
  run_pair<20>("fused pattern, warp+elect");
  run_pair<21>("N=128 only, warp+elect");
  run_pair<22>("N=64 only, warp+elect");
  return 0;
}
