// tf32_semantics.cu — two facts the dense tcgen05 path depends on, measured on the device:
//  (1) what kind::tf32 does with the 13 low mantissa bits of an fp32 operand in shared memory
//      (truncate, round to nearest, or use them), and
//  (2) that an MN-major, 128-B-swizzled A operand (the layout a [32 n][32 d] SWIZZLE_128B TMA
//      box of row-major Phi produces, i.e. Phi^T without a transposed copy) is read correctly
//      with LBO = 4096 B (next 32-row MN block) and SBO = 1024 B (next 8 K).
// One CTA, one M=128, N=16, K=8 MMA per test, D read back through tcgen05.ld.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tf32_semantics tools/tf32_semantics.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_bf16.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstring>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 2) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;   // 2 = SWIZZLE_128B, 1 = SWIZZLE_128B_BASE32B
  return d;
}
// kind::tf32, f32 accumulate, M = 128, N = 16; a_major bit 15 (1 = MN-major)
__host__ __device__ constexpr uint32_t idesc(int n, int a_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

// A: float a[128][8] (m, k) in global; B: float b[16][8] (n, k).  mode 0: A K-major SW128;
// mode 1: A MN-major SW128 (4 blocks of 32 m, LBO 4096; 8 k rows of 128 B).
__global__ void k_test_bf16(const float* a, const float* b, float* d, uint32_t lbo, uint32_t sbo, int amn) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  unsigned char* As = sm;
  unsigned char* Bs = sm + 16384;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 16384 / 4; i += blockDim.x) reinterpret_cast<float*>(As)[i] = 0.f;
  for (int i = tid; i < 2048 / 4; i += blockDim.x) reinterpret_cast<float*>(Bs)[i] = 0.f;
  __syncthreads();
  for (int i = tid; i < 128 * 16; i += blockDim.x) {
    const int m = i / 16, k = i % 16;
    __nv_bfloat16 v = __float2bfloat16(a[m * 16 + k]);
    unsigned char* p;
    if (amn) { const int j = m >> 6, mm = m & 63, c = mm >> 3;
      p = As + j * 2048 + (k >> 3) * 1024 + (k & 7) * 128 + ((c ^ (k & 7)) << 4) + (mm & 7) * 2;   // 8 k rows per 1 KB atom
    } else { const int c = k >> 3; p = As + m * 128 + ((c ^ (m & 7)) << 4) + (k & 7) * 2; }
    *reinterpret_cast<__nv_bfloat16*>(p) = v;
  }
  for (int i = tid; i < 16 * 16; i += blockDim.x) {
    const int n = i / 16, k = i % 16, c = k >> 3;
    *reinterpret_cast<__nv_bfloat16*>(Bs + n * 128 + ((c ^ (n & 7)) << 4) + (k & 7) * 2) = __float2bfloat16(b[n * 16 + k]);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    const uint64_t ad = amn ? desc(su32(As), lbo, sbo) : desc(su32(As), 16, 1024);
    const uint64_t bd = desc(su32(Bs), 16, 1024);
    const uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)amn << 15) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase),
                 "l"(ad), "l"(bd), "r"(id) : "memory");
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  for (;;) {
    uint32_t done;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(su32(&bar)) : "memory");
    if (done) break;
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  float v[16];
  const uint32_t taddr = tbase + ((uint32_t)(32 * warp) << 16);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]), "=f"(v[8]),
        "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int j = 0; j < 16; ++j) d[(32 * warp + lane) * 16 + j] = v[j];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tbase));
  }
}

__global__ void k_test(const float* a, const float* b, float* d, int mode, uint32_t lbo, uint32_t sbo) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  unsigned char* As = sm;              // 16 KB
  unsigned char* Bs = sm + 16384;      // 2 KB (16 rows x 128 B)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 16384 / 4; i += blockDim.x) reinterpret_cast<float*>(As)[i] = 0.f;
  for (int i = tid; i < 2048 / 4; i += blockDim.x) reinterpret_cast<float*>(Bs)[i] = 0.f;
  __syncthreads();
  // K-major SW128: row r (128 B), logical 16-B chunk c at physical c ^ (r & 7)
  auto kmaj = [](unsigned char* base, int r, int k) -> float* {
    const int c = k >> 2;
    return reinterpret_cast<float*>(base + r * 128 + ((c ^ (r & 7)) << 4) + (k & 3) * 4);
  };
  // MN-major SW128: block j = m / 32 at j * 4096; k row at k * 128 B; logical chunk (m % 32) / 4
  // MN-major SWIZZLE_128B_BASE32B: block j = m / 32 at j * 4096; 4-k group at (k / 4) * 512;
  // row k % 4 of 128 B; 32-B unit (m % 32) / 8 at physical unit ^ (k % 4)
  auto mn32 = [](unsigned char* base, int m, int k) -> float* {
    const int j = m >> 5, mm = m & 31, u = mm >> 3, kr = k & 3;
    return reinterpret_cast<float*>(base + j * 4096 + (k >> 2) * 512 + kr * 128 + ((u ^ kr) << 5) + (mm & 7) * 4);
  };
  auto mnmaj = [](unsigned char* base, int m, int k) -> float* {
    const int j = m >> 5, mm = m & 31, c = mm >> 2;
    return reinterpret_cast<float*>(base + j * 4096 + k * 128 + ((c ^ (k & 7)) << 4) + (mm & 3) * 4);
  };
  for (int i = tid; i < 128 * 8; i += blockDim.x) {
    const int m = i / 8, k = i % 8;
    *(mode == 2 ? mn32(As, m, k) : mode ? mnmaj(As, m, k) : kmaj(As, m, k)) = a[m * 8 + k];
  }
  for (int i = tid; i < 16 * 8; i += blockDim.x) {
    const int n = i / 8, k = i % 8;
    *kmaj(Bs, n, k) = b[n * 8 + k];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    const uint64_t ad = mode == 2 ? desc(su32(As), lbo, sbo, 1) : mode ? desc(su32(As), lbo, sbo) : desc(su32(As), 16, 1024);
    const uint64_t bd = desc(su32(Bs), 16, 1024);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase),
                 "l"(ad), "l"(bd), "r"(idesc(16, mode ? 1 : 0)) : "memory");
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  for (;;) {
    uint32_t done;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(su32(&bar)) : "memory");
    if (done) break;
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  float v[16];
  const uint32_t taddr = tbase + ((uint32_t)(32 * warp) << 16);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]), "=f"(v[8]),
        "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int j = 0; j < 16; ++j) d[(32 * warp + lane) * 16 + j] = v[j];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tbase));
  }
}


// (3) the TMA side: Phi [32 n][128 d] row-major (d contiguous) loaded as 4 boxes [32 n][32 d]
// with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B into 4 KB blocks, then MMAs on K-steps kk = 0..3
// (start address + kk * 1024) with the MN-major BASE32B descriptor (LBO 4096, SBO 512).
// D[m][n'] = sum_k Phi[8kk + k][m] * B[n'][k]
__global__ void k_tma(const __grid_constant__ CUtensorMap map, const float* b, float* d, int kk) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar, tbar;
  unsigned char* As = sm;
  unsigned char* Bs = sm + 16384;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 2048 / 4; i += blockDim.x) reinterpret_cast<float*>(Bs)[i] = 0.f;
  __syncthreads();
  for (int i = tid; i < 16 * 8; i += blockDim.x) {
    const int n = i / 8, k = i % 8, c = k >> 2;
    *reinterpret_cast<float*>(Bs + n * 128 + ((c ^ (n & 7)) << 4) + (k & 3) * 4) = b[n * 8 + k];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&tbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&tbar)), "r"(16384) : "memory");
    for (int j = 0; j < 4; ++j)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                   ::"r"(su32(As + j * 4096)), "l"(&map), "r"(su32(&tbar)), "r"(32 * j), "r"(0) : "memory");
  }
  for (;;) {
    uint32_t done;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(su32(&tbar)) : "memory");
    if (done) break;
  }
  if (tid == 0) {
    const uint64_t ad = desc(su32(As) + kk * 1024, 4096, 512, 1);
    const uint64_t bd = desc(su32(Bs), 16, 1024);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase),
                 "l"(ad), "l"(bd), "r"(idesc(16, 1)) : "memory");
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  for (;;) {
    uint32_t done;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(su32(&bar)) : "memory");
    if (done) break;
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  float v[16];
  const uint32_t taddr = tbase + ((uint32_t)(32 * warp) << 16);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]), "=f"(v[8]),
        "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int j = 0; j < 16; ++j) d[(32 * warp + lane) * 16 + j] = v[j];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tbase));
  }
}

static float trunc_tf32(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; float r; memcpy(&r, &u, 4); return r; }
static float rn_tf32(float x) { uint32_t u; memcpy(&u, &x, 4); u = (u + 0x1000u) & 0xFFFFE000u; float r; memcpy(&r, &u, 4); return r; }
static float rne_tf32(float x) {
  uint32_t u; memcpy(&u, &x, 4);
  const uint32_t lsb = (u >> 13) & 1u;
  u = (u + 0xFFFu + lsb) & 0xFFFFE000u; float r; memcpy(&r, &u, 4); return r;
}

int main() {
  srand(7);
  std::vector<float> a(128 * 8), b(16 * 8), d(128 * 16);
  auto rnd = [] { return (float)((rand() / (double)RAND_MAX) * 2.0 - 1.0); };
  for (auto& x : a) x = rnd();                                    // full fp32 mantissas
  for (auto& x : b) x = (float)((rand() % 17) - 8) / 8.0f;        // exact in tf32
  float *da, *db, *dd;
  cudaMalloc(&da, a.size() * 4); cudaMalloc(&db, b.size() * 4); cudaMalloc(&dd, d.size() * 4);
  cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 20480);
  const uint32_t cfg[][3] = {{16, 1024, 0}, {4096, 1024, 1}, {4096, 512, 2}, {512, 4096, 2}};
  for (int ci = 0; ci < 4; ++ci) {
    const int mode = (int)cfg[ci][2];
    k_test<<<1, 128, 20480>>>(da, db, dd, mode, cfg[ci][0], cfg[ci][1]);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost);
    double err[4] = {0, 0, 0, 0}, nrm = 0;   // vs exact, trunc, rn-away, rne
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 16; ++n) {
        double ex = 0, tr = 0, ra = 0, re = 0;
        for (int k = 0; k < 8; ++k) {
          const double bb = b[n * 8 + k], aa = a[m * 8 + k];
          ex += aa * bb; tr += trunc_tf32(aa) * bb; ra += rn_tf32(aa) * bb; re += rne_tf32(aa) * bb;
        }
        const double g = d[m * 16 + n];
        err[0] = fmax(err[0], fabs(g - ex)); err[1] = fmax(err[1], fabs(g - tr));
        err[2] = fmax(err[2], fabs(g - ra)); err[3] = fmax(err[3], fabs(g - re));
        nrm = fmax(nrm, fabs(ex));
      }
    printf("%s A lbo %5u sbo %5u D[0..2] %9.5f %9.5f %9.5f: max|D - ref| / max|D|: exact %.3e  trunc %.3e  rn-away %.3e  rne %.3e  (%s)\n",
           mode == 2 ? "MN-b32  " : mode ? "MN-major" : "K-major ", cfg[ci][0], cfg[ci][1], d[0], d[1], d[16], err[0] / nrm, err[1] / nrm, err[2] / nrm, err[3] / nrm, cudaGetErrorString(e));
  }
  {   // (3) TMA SWIZZLE_128B_ATOM_32B boxes + MN-major BASE32B descriptor
    std::vector<float> phi(32 * 128), b3(16 * 8), d3(128 * 16);
    for (auto& x : phi) x = (float)((rand() % 17) - 8) / 8.0f;
    for (auto& x : b3) x = (float)((rand() % 17) - 8) / 8.0f;
    float *dphi, *db3;
    cudaMalloc(&dphi, phi.size() * 4); cudaMalloc(&db3, b3.size() * 4);
    cudaMemcpy(dphi, phi.data(), phi.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db3, b3.data(), b3.size() * 4, cudaMemcpyHostToDevice);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap map;
    cuuint64_t dims[2] = {128, 32};
    cuuint64_t strides[1] = {128 * 4};
    cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dphi, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 20480);
    for (int kk = 0; kk < 4; ++kk) {
      k_tma<<<1, 128, 20480>>>(map, db3, dd, kk);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(d3.data(), dd, d3.size() * 4, cudaMemcpyDeviceToHost);
      double err = 0, nrm = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 16; ++n) {
          double ex = 0;
          for (int k = 0; k < 8; ++k) ex += (double)phi[(8 * kk + k) * 128 + m] * b3[n * 8 + k];
          err = fmax(err, fabs(d3[m * 16 + n] - ex)); nrm = fmax(nrm, fabs(ex));
        }
      printf("TMA ATOM_32B + MN-b32 kk=%d: rel err %.3e (encode %d, %s)\n", kk, err / nrm, (int)r, cudaGetErrorString(e));
    }
  }
  // bf16 (K = 16 per MMA): K-major reference, then MN-major with (LBO, SBO) candidates
  {
    std::vector<float> a2(128 * 16), b2(16 * 16), d2(128 * 16);
    for (auto& x : a2) x = (float)((rand() % 17) - 8) / 8.0f;
    for (auto& x : b2) x = (float)((rand() % 17) - 8) / 8.0f;
    float *da2, *db2;
    cudaMalloc(&da2, a2.size() * 4); cudaMalloc(&db2, b2.size() * 4);
    cudaMemcpy(da2, a2.data(), a2.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db2, b2.data(), b2.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_test_bf16, cudaFuncAttributeMaxDynamicSharedMemorySize, 20480);
    const uint32_t c2[][3] = {{16, 1024, 0}, {2048, 1024, 1}, {1024, 2048, 1}};
    for (auto& c : c2) {
      k_test_bf16<<<1, 128, 20480>>>(da2, db2, dd, c[0], c[1], (int)c[2]);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(d2.data(), dd, d2.size() * 4, cudaMemcpyDeviceToHost);
      double err = 0, nrm = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 16; ++n) {
          double ex = 0;
          for (int k = 0; k < 16; ++k) ex += (double)a2[m * 16 + k] * b2[n * 16 + k];
          err = fmax(err, fabs(d2[m * 16 + n] - ex)); nrm = fmax(nrm, fabs(ex));
        }
      printf("bf16 %s lbo %5u sbo %5u: rel err %.3e (%s)\n", c[2] ? "MN-major" : "K-major ", c[0], c[1], err / nrm, cudaGetErrorString(e));
    }
  }
  return 0;
}
