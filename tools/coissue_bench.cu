// How many ALU / FMA-pipe instructions co-issue with legacy mma.sync on sm_100a:
// cycles per HMMA per SMSP with N independent ops of one kind per HMMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/coissue_bench tools/coissue_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

enum Op { LOP3, FFMA, IMAD, PRMT, HFMA2, IADD3 };

template <int OP>
__device__ __forceinline__ uint32_t op1(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  if (OP == LOP3) asm volatile("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  if (OP == FFMA) asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  if (OP == IMAD) asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  if (OP == PRMT) asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  if (OP == HFMA2) asm volatile("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  if (OP == IADD3) asm volatile("add.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// NOPS ops per mma; 2 independent accumulator chains; op results feed the A
// operand of the next mma so nothing is dead code.
template <int OP, int NOPS>
__global__ void k(int iters, float* out, uint32_t seed) {
  float d[2][4] = {};
  uint32_t a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i) | 0x3f803f80u;
  const uint32_t b0 = 0x3f803f80u, b1 = b0, m = 0x00030003u, c = 0x43004300u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int ch = 0; ch < 2; ++ch) {
#pragma unroll
      for (int j = 0; j < NOPS; ++j) a[(ch * 4 + j) & 7] = op1<OP>(a[(ch * 4 + j + 3) & 7], m, c);
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(d[ch][0]), "+f"(d[ch][1]), "+f"(d[ch][2]), "+f"(d[ch][3])
          : "r"(a[ch * 4]), "r"(a[ch * 4 + 1]), "r"(a[ch * 4 + 2]), "r"(a[ch * 4 + 3]), "r"(b0), "r"(b1));
    }
  }
  float s = d[0][0] + d[1][0];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += __uint_as_float(a[i]);
  if (s == 1.2345f) out[0] = s;
}

// ops only (no mma): pipe throughput reference
template <int OP>
__global__ void konly(int iters, float* out, uint32_t seed) {
  uint32_t a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i) | 0x3f803f80u;
  const uint32_t m = 0x00030003u, c = 0x43004300u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = op1<OP>(a[(j + 3) & 7], m, c);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += __uint_as_float(a[i]);
  if (s == 1.2345f) out[0] = s;
}

int main() {
  int nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096, warps = 16;
  const double hz = 1.965e9;  // boost clock used by the runs (nvidia-smi)
  auto time = [&](auto kern, int per_iter) {
    float ms = 0;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      kern<<<nsm, warps * 32>>>(iters, out, 12345u);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    // cycles per counted instruction per SMSP
    const double per_smsp = double(iters) * per_iter * warps / 4.0;
    return ms * 1e-3 * hz / per_smsp;
  };
  const char* names[] = {"LOP3", "FFMA", "IMAD", "PRMT", "HFMA2", "IADD3"};
#define ROW(OP)                                                                                    \
  printf("%-6s only: %5.2f cyc/op/SMSP | per mma with n ops: n=0 %5.2f  n=2 %5.2f  n=4 %5.2f  " \
         "n=6 %5.2f  n=8 %5.2f\n",                                                                 \
         names[OP], time(konly<OP>, 8), time(k<OP, 0>, 2), time(k<OP, 2>, 2), time(k<OP, 4>, 2),  \
         time(k<OP, 6>, 2), time(k<OP, 8>, 2));
  ROW(LOP3)
  ROW(FFMA)
  ROW(IMAD)
  ROW(PRMT)
  ROW(HFMA2)
  ROW(IADD3)
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
