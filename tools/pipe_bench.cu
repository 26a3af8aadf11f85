// Per-HMMA cost of the decode mix: 4 LOP3 + {nothing | 1 SHF | 1 IMAD.HI | 1 HADD2.F32 |
// 2 FFMA | 1 IMAD.MOV} with inputs that change every iteration (no folding).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/pipe_bench tools/pipe_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

template <int X>
__global__ void k(int iters, float* out, uint32_t seed) {
  float d[2][4] = {};
  float acc = 0.f;
  uint32_t w0 = seed * threadIdx.x, w1 = w0 ^ 0x5a5a5a5au;
  const uint32_t b = 0x3f803f80u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const uint32_t w = c ? w1 : w0;
      uint32_t src = w;
      if (X == 1) asm volatile("shr.b32 %0, %1, 6;" : "=r"(src) : "r"(w));
      if (X == 2) asm volatile("mul.hi.u32 %0, %1, 0x04000000;" : "=r"(src) : "r"(w));
      uint32_t a[4];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(a[j]) : "r"(src), "r"(0x00030003u << (2 * j)), "r"(0x43004300u));
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b), "r"(b));
      if (X == 3) {
        float f;
        asm volatile("{.reg .f16 l, h; mov.b32 {l, h}, %1; cvt.f32.f16 %0, l;}" : "=f"(f) : "r"(w));
        acc += f;
      }
      if (X == 4) {
        asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(acc) : "f"(d[c][0]), "f"(1.0001f));
        asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(acc) : "f"(d[c][1]), "f"(1.0001f));
      }
    }
    w0 = w0 * 1664525u + 1013904223u;  // IMAD: FMA pipe
    w1 = w1 * 1664525u + 1013904223u;
  }
  const float s = d[0][0] + d[1][0] + acc;
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
  const int iters = 4096, warps = 16;
  auto time = [&](auto kern) {
    float ms = 0;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      kern<<<nsm, warps * 32>>>(iters, out, 12345u);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    return ms * 1e-3 * 1.965e9 / (double(iters) * 2 * warps / 4.0);
  };
  printf("cycles per HMMA per SMSP (4 LOP3 + 1 IMAD each):\n");
  printf("  base            %.2f\n", time(k<0>));
  printf("  + SHF           %.2f\n", time(k<1>));
  printf("  + IMAD.HI       %.2f\n", time(k<2>));
  printf("  + HADD2.F32     %.2f\n", time(k<3>));
  printf("  + 2 FFMA        %.2f\n", time(k<4>));
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
