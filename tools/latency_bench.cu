// Dependent-load latency on sm_100a: one thread chases a random cycle through
// an L2-resident (4 MB) and an HBM-resident (1 GB) buffer.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/latency_bench tools/latency_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

__global__ void chase(const uint32_t* next, int steps, uint32_t* out, long long* cyc) {
  uint32_t p = 0;
  const long long t0 = clock64();
  for (int i = 0; i < steps; ++i) p = __ldcg(next + p);
  const long long t1 = clock64();
  out[0] = p;
  *cyc = t1 - t0;
}

int main() {
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 4);
  cudaMallocManaged(&cyc, 8);
  for (size_t mb : {1, 4, 32, 1024}) {
    const size_t n = mb * (1 << 20) / 4;
    std::vector<uint32_t> h(n);
    // random single cycle over 128-byte-spaced slots
    const size_t stride = 32, m = n / stride;
    std::vector<uint32_t> perm(m);
    for (size_t i = 0; i < m; ++i) perm[i] = static_cast<uint32_t>(i);
    srand(1);
    for (size_t i = m - 1; i > 0; --i) std::swap(perm[i], perm[rand() % (i + 1)]);
    for (size_t i = 0; i < m; ++i) h[perm[i] * stride] = perm[(i + 1) % m] * stride;
    uint32_t* d;
    cudaMalloc(&d, n * 4);
    cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
    const int steps = 20000;
    chase<<<1, 1>>>(d, steps, out, cyc);  // warm
    cudaDeviceSynchronize();
    chase<<<1, 1>>>(d, steps, out, cyc);
    cudaDeviceSynchronize();
    printf("%5zu MB: %7.1f cycles/load  (%.0f ns @1.965GHz)\n", mb, double(*cyc) / steps, double(*cyc) / steps / 1.965);
    cudaFree(d);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
