// Microbenchmark: throughput of fp16->fp32 conversion paths and LOP3 on sm_100a.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/cvt_bench tools/cvt_bench.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

template <int MODE>
__global__ void k(int iters, uint32_t seed, float* out) {
  uint32_t w[8];
  for (int i = 0; i < 8; ++i) w[i] = seed * (threadIdx.x + 7 * i) | 0x3c003c00u;
  float acc[8] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) {  // __half22float2 (HADD2.F32)
        float2 f = __half22float2(*reinterpret_cast<__half2*>(&w[i]));
        acc[i] += f.x * f.y;
      } else if (MODE == 1) {  // bf16 unpack (shift / mask)
        float a = __uint_as_float(w[i] << 16), b = __uint_as_float(w[i] & 0xffff0000u);
        acc[i] += a * b;
      } else if (MODE == 2) {  // lop3 with two register constants
        uint32_t r;
        asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(w[i]), "r"(0x00030003u * (seed & 1) + 0x00030003u), "r"(0x43004300u | seed));
        acc[i] += __uint_as_float(r);
      } else {  // plain FFMA baseline
        acc[i] = fmaf(acc[i], 1.0001f, __uint_as_float(w[i]));
      }
      w[i] = w[i] * 1664525u + 1013904223u;
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 1.2345f) out[0] = s;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2048;
  void (*ks[4])(int, uint32_t, float*) = {k<0>, k<1>, k<2>, k<3>};
  const char* names[4] = {"half2->float2 (HADD2.F32)", "bf16 shift/mask", "lop3 (2 reg consts)", "ffma+imad baseline"};
  for (int m = 0; m < 4; ++m) {
    float ms = 0;
    for (int r = 0; r < 2; ++r) {
      cudaEventRecord(e0);
      ks[m]<<<nsm, 512>>>(iters, 12345u, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    cudaEventElapsedTime(&ms, e0, e1);
    double warp_ops = double(nsm) * 16 * iters * 8;  // per conversion-site per warp
    printf("%-28s %8.3f ms  %6.2f cycles per (warp-op x SMSP)\n", names[m], ms,
           ms * 1e-3 * 1.9e9 / (warp_ops / (nsm * 4.0)));
  }
  return 0;
}
