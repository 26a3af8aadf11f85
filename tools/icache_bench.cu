// Instruction-fetch cost of large straight-line kernels, cold (L2 flushed by a
// 512 MB write) vs warm.  One CTA of 32 threads runs N unrolled FFMAs (16 B
// each), so the code size is ~16*N bytes; a rolled loop of the same work is
// the control.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/icache_bench tools/icache_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int N>
__global__ void straight(float* out, float a, float b) {
  float x = threadIdx.x;
#pragma unroll
  for (int i = 0; i < N; ++i) x = fmaf(x, a, b + static_cast<float>(i));
  if (x == 12345.0f) out[threadIdx.x] = x;
}

__global__ void rolled(float* out, float a, float b, int n) {
  float x = threadIdx.x;
#pragma unroll 1
  for (int i = 0; i < n; ++i) x = fmaf(x, a, b + static_cast<float>(i));
  if (x == 12345.0f) out[threadIdx.x] = x;
}

template <typename F>
void run(const char* name, F launch, char* flush, size_t fbytes) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float cold = 0, warm = 0;
  const int reps = 10;
  for (int r = 0; r < reps; ++r) {
    cudaMemsetAsync(flush, r, fbytes);
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cold += ms;
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    warm += ms;
  }
  printf("%-28s cold %8.2f us   warm %8.2f us\n", name, cold / reps * 1e3, warm / reps * 1e3);
}

int main() {
  float* out;
  char* flush;
  const size_t fbytes = 512ull << 20;
  cudaMalloc(&out, 4096);
  cudaMalloc(&flush, fbytes);
  run("empty rolled n=0", [&] { rolled<<<1, 32>>>(out, 1.0001f, 0.5f, 0); }, flush, fbytes);
  run("rolled n=4096", [&] { rolled<<<1, 32>>>(out, 1.0001f, 0.5f, 4096); }, flush, fbytes);
  run("straight N=256 (4KB)", [&] { straight<256><<<1, 32>>>(out, 1.0001f, 0.5f); }, flush, fbytes);
  run("straight N=1024 (16KB)", [&] { straight<1024><<<1, 32>>>(out, 1.0001f, 0.5f); }, flush, fbytes);
  run("straight N=4096 (64KB)", [&] { straight<4096><<<1, 32>>>(out, 1.0001f, 0.5f); }, flush, fbytes);
  run("straight N=4096 x148 CTAs", [&] { straight<4096><<<148, 32>>>(out, 1.0001f, 0.5f); }, flush, fbytes);
  cudaError_t err = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(err));
  return 0;
}
