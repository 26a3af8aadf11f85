// Legacy mma.sync m16n8k32 u8 x s8 -> s32 throughput on sm_100a, alone and with
// n LOP3 per IMMA (fresh inputs each op so nothing folds).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/imma_bench tools/imma_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

template <int NOPS, int CH>
__global__ void k(int iters, int* out, uint32_t seed) {
  int d[CH][4] = {};
  uint32_t w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) w[i] = seed * (threadIdx.x + 7 * i + 1);
  const uint32_t b0 = seed ^ threadIdx.x, b1 = b0 * 3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      uint32_t a[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j < NOPS) {
          asm volatile("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(a[j]) : "r"(w[(c + j) & 7]), "r"(0x03030303u << (2 * (it & 3))), "r"(0u));
        } else {
          a[j] = w[(c + j) & 7];
        }
      }
      asm volatile(
          "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+r"(d[c][0]), "+r"(d[c][1]), "+r"(d[c][2]), "+r"(d[c][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = w[i] * 1664525u + 1013904223u;
  }
  int s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][3];
  if (s == 12345) out[0] = s;
}

template <int CH>
__global__ void hk(int iters, float* out, uint32_t seed) {
  float d[CH][4] = {};
  const uint32_t a0 = seed * threadIdx.x | 0x3f803f80u, b0 = 0x3f803f80u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
          : "r"(a0), "r"(a0), "r"(a0), "r"(a0), "r"(b0), "r"(b0));
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0];
  if (s == 1.2345f) out[0] = s;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2048;
  auto time = [&](auto kern, int ch, int warps) {
    float ms = 0;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      kern<<<nsm, warps * 32>>>(iters, (decltype(out))out, 12345u);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    return ms * 1e-3 * 1.965e9 / (double(iters) * ch * warps / 4.0);
  };
  printf("IMMA k32 u8.s8 (cycles/mma/SMSP): ch=1 w=4 %.2f | ch=4 w=8 %.2f | ch=4 w=16 %.2f\n", time(k<0, 1>, 1, 4),
         time(k<0, 4>, 4, 8), time(k<0, 4>, 4, 16));
  printf("IMMA + 2 LOP3: %.2f | + 4 LOP3: %.2f  (ch=4 w=16)\n", time(k<2, 4>, 4, 16), time(k<4, 4>, 4, 16));
  {
    float ms = 0;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      hk<4><<<nsm, 16 * 32>>>(iters, reinterpret_cast<float*>(out), 12345u);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("HMMA k16 bf16 ref: ch=4 w=16 %.2f\n", ms * 1e-3 * 1.965e9 / (double(iters) * 4 * 16 / 4.0));
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
