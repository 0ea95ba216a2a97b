// microbench.cu — measured B200 ceilings that MEASURED_PEAKS.json does not hold:
// L2-resident read and read+write bandwidth vs working-set size, HBM read+write,
// FP32 FFMA and FP64 DFMA issue rates.  Used for the roofline denominators of
// the L2-resident DCT schedule and the ALU-bound stencil.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench tools/microbench.cu && ./microbench
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_read(const float4* __restrict__ x, size_t n, float* out) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = __ldcg(x + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 123.456f) *out = acc;
}

__global__ void k_rw(float4* __restrict__ x, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float4 v = __ldcg(x + i);
    v.x *= 1.0000001f; v.y *= 1.0000001f; v.z *= 1.0000001f; v.w *= 1.0000001f;
    __stcg(x + i, v);
  }
}

__global__ void k_ffma(float* out, int iters) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const float b = 0.999f, c = 0.001f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
      a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
    }
  }
  float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 1.2345f) *out = s;
}

__global__ void k_dfma(double* out, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999, c = 0.001;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 1.2345) *out = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int l2; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"l2_bytes\": %d, \"clock_khz\": %d", sms, l2, clk);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float* dout; cudaMalloc(&dout, 64);
  const size_t big = (size_t)4 << 30;
  float4* buf; cudaMalloc(&buf, big);
  cudaMemset(buf, 0, big);
  const int grid = sms * 8, blk = 256;
  // L2-resident read / read+write bandwidth vs working set
  size_t sizes_mb[] = {8, 16, 32, 48, 64, 80, 96, 112, 128};
  printf(", \"l2_read_gbs\": {");
  for (int si = 0; si < 9; ++si) {
    size_t n = sizes_mb[si] * ((size_t)1 << 20) / 16;
    for (int w = 0; w < 3; ++w) k_read<<<grid, blk>>>(buf, n, dout);
    const int reps = 50;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) k_read<<<grid, blk>>>(buf, n, dout);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%s\"%zu\": %.0f", si ? ", " : "", sizes_mb[si], reps * n * 16.0 / (ms * 1e-3) / 1e9);
  }
  printf("}, \"l2_rw_gbs\": {");
  for (int si = 0; si < 9; ++si) {
    size_t n = sizes_mb[si] * ((size_t)1 << 20) / 16;
    for (int w = 0; w < 3; ++w) k_rw<<<grid, blk>>>(buf, n);
    const int reps = 50;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) k_rw<<<grid, blk>>>(buf, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%s\"%zu\": %.0f", si ? ", " : "", sizes_mb[si], reps * n * 32.0 / (ms * 1e-3) / 1e9);
  }
  {
    size_t n = big / 16;
    k_rw<<<grid, blk>>>(buf, n);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_rw<<<grid, blk>>>(buf, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("}, \"hbm_rw_gbs_4GiB\": %.0f", 5 * n * 32.0 / (ms * 1e-3) / 1e9);
    k_read<<<grid, blk>>>(buf, n, dout);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_read<<<grid, blk>>>(buf, n, dout);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf(", \"hbm_read_gbs_4GiB\": %.0f", 5 * n * 16.0 / (ms * 1e-3) / 1e9);
  }
  {
    const int iters = 4096, g = sms * 16;
    k_ffma<<<g, 256>>>(dout, 16);
    cudaEventRecord(e0);
    k_ffma<<<g, 256>>>(dout, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * 16 * (double)iters * g * 256;
    printf(", \"fp32_ffma_tflops\": %.1f", fl / (ms * 1e-3) / 1e12);
    k_dfma<<<g, 256>>>((double*)dout, 16);
    cudaEventRecord(e0);
    k_dfma<<<g, 256>>>((double*)dout, iters / 4);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 8 * 16 * (double)(iters / 4) * g * 256;
    printf(", \"fp64_dfma_tflops\": %.1f", fl / (ms * 1e-3) / 1e12);
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf(", \"status\": \"%s\"}\n", cudaGetErrorString(err));
  return err != cudaSuccess;
}
