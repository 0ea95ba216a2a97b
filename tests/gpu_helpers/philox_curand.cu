// Test helper (not product code): evaluates cuRAND's own Philox4x32-10 round function
// (curand_philox4x32_x.h) on counters/keys read from stdin, to pin oracle/philox.py
// against an independent implementation on the device.
#include <cstdio>
#include <curand_kernel.h>
#include <vector>

__global__ void k(const uint4* c, const uint2* key, uint4* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = curand_Philox4x32_10(c[i], key[i]);
}

int main() {
  std::vector<uint4> c; std::vector<uint2> kk;
  unsigned a, b, d, e, f, g;
  while (scanf("%x %x %x %x %x %x", &a, &b, &d, &e, &f, &g) == 6) { c.push_back(make_uint4(a, b, d, e)); kk.push_back(make_uint2(f, g)); }
  int n = (int)c.size();
  uint4 *dc, *dout; uint2* dk;
  cudaMalloc(&dc, n * sizeof(uint4)); cudaMalloc(&dk, n * sizeof(uint2)); cudaMalloc(&dout, n * sizeof(uint4));
  cudaMemcpy(dc, c.data(), n * sizeof(uint4), cudaMemcpyHostToDevice);
  cudaMemcpy(dk, kk.data(), n * sizeof(uint2), cudaMemcpyHostToDevice);
  k<<<(n + 127) / 128, 128>>>(dc, dk, dout, n);
  std::vector<uint4> o(n);
  if (cudaMemcpy(o.data(), dout, n * sizeof(uint4), cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
  for (auto& v : o) printf("%08x %08x %08x %08x\n", v.x, v.y, v.z, v.w);
  return 0;
}
