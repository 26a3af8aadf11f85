// The tiled kernel's consumer MMA core in isolation (random stage data in shared
// memory, no barriers): cycles per 32-group-pair item for several warp counts
// and instruction schedules.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/core_bench tools/core_bench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

constexpr int kBlk = 640, kCodeBytes = 512, GPI = 32;  // group pairs per item

__device__ __forceinline__ void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_bf16_c(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                           uint32_t b0, uint32_t b1, const float4& c) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%10,%11,%12,%13};"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "f"(c.x), "f"(c.y), "f"(c.z), "f"(c.w));
}
__device__ __forceinline__ uint32_t lop_and_or(uint32_t w, uint32_t m) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(w), "r"(m), "r"(0x43004300u));
  return r;
}
__device__ __forceinline__ float2 h2f2(uint32_t w) {
  float2 f;
  asm("{.reg .f16 l, h; mov.b32 {l, h}, %2; cvt.f32.f16 %0, l; cvt.f32.f16 %1, h;}" : "=f"(f.x), "=f"(f.y) : "r"(w));
  return f;
}

// V = 0: the kernel's schedule (h outer, ks inner); V = 1: both h of a group
// pair interleaved per ks (4 independent chains for NI = 2)
template <int NI, int NT, int V, int kSpanGP>
__device__ __forceinline__ void core(const uint8_t* st, const uint16_t* xs, const float2* sums, int xs_stride,
                                     int warp, int nwarps, float (&acc)[NI][NT][4]) {
  constexpr int TPP = 8 * NT;
  const int lane = threadIdx.x & 31, gid = lane >> 2, tid = lane & 3;
  const uint16_t* xrow[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) xrow[nt] = xs + (nt * 8 + gid) * xs_stride + tid * 4;
  const int nspan = GPI / kSpanGP;
  for (int sp = warp; sp < nspan; sp += nwarps) {
    const int q0 = sp * kSpanGP, q1 = q0 + kSpanGP;
#pragma unroll 2
    for (int q = q0; q < q1; ++q) {
      const uint8_t* blk = st + q * NI * kBlk;
      uint4 cw[NI], mw[NI];
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        cw[i] = *reinterpret_cast<const uint4*>(blk + i * kBlk + lane * 16);
        mw[i] = *reinterpret_cast<const uint4*>(blk + i * kBlk + kCodeBytes + gid * 16);
      }
      float4 xx[2][NT];
      float4 cq[2][NT];  // V == 2: (b0, b1, b0, b1) seed quad, xx.x/.y = (X0, X1)
      float d[2][NI][NT][4];
      uint32_t wa[2][NI][3], wb[2][NI][3];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gl = q * 2 + h;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          if (V == 2) {
            cq[h][nt] = *reinterpret_cast<const float4*>(sums + (gl * TPP + nt * 8 + 2 * tid) * 2);
            const float2 xv = *reinterpret_cast<const float2*>(sums + GPI * 2 * TPP * 2 + gl * TPP + nt * 8 + 2 * tid);
            xx[h][nt] = make_float4(xv.x, 0.f, xv.y, 0.f);
            continue;
          }
          xx[h][nt] = *reinterpret_cast<const float4*>(sums + gl * TPP + nt * 8 + 2 * tid);
#pragma unroll
          for (int i = 0; i < NI; ++i) {
            d[h][i][nt][0] = xx[h][nt].y;
            d[h][i][nt][1] = xx[h][nt].w;
            d[h][i][nt][2] = xx[h][nt].y;
            d[h][i][nt][3] = xx[h][nt].w;
          }
        }
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          wa[h][i][0] = h ? cw[i].z : cw[i].x;
          wb[h][i][0] = h ? cw[i].w : cw[i].y;
          wa[h][i][1] = wa[h][i][0] >> 6;
          wb[h][i][1] = wb[h][i][0] >> 6;
          wa[h][i][2] = wa[h][i][0] >> 12;
          wb[h][i][2] = wb[h][i][0] >> 12;
        }
      }
      auto step = [&](int h, int ks) {
        const int gl = q * 2 + h;
        uint32_t b0[NT], b1[NT];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const uint2 bv = *reinterpret_cast<const uint2*>(xrow[nt] + gl * 64 + ks * 16);
          b0[nt] = bv.x;
          b1[nt] = bv.y;
        }
        const int j0 = 2 * ks, j1 = 2 * ks + 1;
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const uint32_t m0 = 0x00030003u << (2 * (j0 % 3)), m1 = 0x00030003u << (2 * (j1 % 3));
          const uint32_t a0 = lop_and_or(wa[h][i][j0 / 3], m0), a1 = lop_and_or(wb[h][i][j0 / 3], m0);
          const uint32_t a2 = lop_and_or(wa[h][i][j1 / 3], m1), a3 = lop_and_or(wb[h][i][j1 / 3], m1);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            if (V == 2 && ks == 0)
              mma_bf16_c(d[h][i][nt], a0, a1, a2, a3, b0[nt], b1[nt], cq[h][nt]);
            else
              mma_bf16(d[h][i][nt], a0, a1, a2, a3, b0[nt], b1[nt]);
          }
        }
      };
      if (V != 1) {
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) step(h, ks);
      } else {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
#pragma unroll
          for (int h = 0; h < 2; ++h) step(h, ks);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const float2 mA = h2f2(h ? mw[i].y : mw[i].x);
          const float2 mB = h2f2(h ? mw[i].w : mw[i].z);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            acc[i][nt][0] = fmaf(mA.x, d[h][i][nt][0], fmaf(mA.y, xx[h][nt].x, acc[i][nt][0]));
            acc[i][nt][1] = fmaf(mA.x, d[h][i][nt][1], fmaf(mA.y, xx[h][nt].z, acc[i][nt][1]));
            acc[i][nt][2] = fmaf(mB.x, d[h][i][nt][2], fmaf(mB.y, xx[h][nt].x, acc[i][nt][2]));
            acc[i][nt][3] = fmaf(mB.x, d[h][i][nt][3], fmaf(mB.y, xx[h][nt].z, acc[i][nt][3]));
          }
        }
    }
  }
}

template <int NI, int NT, int V, int SP>
__global__ void bench(int items, float* out, long long* cyc) {
  extern __shared__ __align__(16) uint8_t sm[];
  constexpr int TPP = 8 * NT;
  const int xs_stride = GPI * 128 + 8;
  uint8_t* st = sm;
  uint16_t* xs = reinterpret_cast<uint16_t*>(sm + GPI * NI * kBlk);
  float2* sums = reinterpret_cast<float2*>(sm + GPI * NI * kBlk + TPP * xs_stride * 2);
  const int total = GPI * NI * kBlk + TPP * xs_stride * 2 + GPI * 2 * TPP * 8 * 3;
  for (int i = threadIdx.x; i < total / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = (i * 2654435761u) & 0x3c003c00u;  // small finite values
  __syncthreads();
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  float acc[NI][NT][4] = {};
  const long long t0 = clock64();
  for (int it = 0; it < items; ++it) core<NI, NT, V, SP>(st, xs, sums, xs_stride, warp, nwarps, acc);
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < NI; ++i)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) s += acc[i][nt][0] + acc[i][nt][1] + acc[i][nt][2] + acc[i][nt][3];
  if (s == 1.2345f) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int NI, int NT, int V, int SP = 4>
void run(int warps) {
  constexpr int TPP = 8 * NT;
  const int xs_stride = GPI * 128 + 8;
  const int smem = GPI * NI * kBlk + TPP * xs_stride * 2 + GPI * 2 * TPP * 8 * 3;
  cudaFuncSetAttribute(bench<NI, NT, V, SP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4);
  cudaMallocManaged(&cyc, 8);
  const int items = 200;
  bench<NI, NT, V, SP><<<148, warps * 32, smem>>>(items, out, cyc);
  cudaDeviceSynchronize();
  bench<NI, NT, V, SP><<<148, warps * 32, smem>>>(items, out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  const double cpi = double(*cyc) / items;
  const double bytes = GPI * NI * kBlk;
  printf("NI=%d NT=%d V=%d span=%d warps=%2d: %7.0f cycles/item  -> %6.1f B/cycle/SM  = %5.2f TB/s @1.965GHz x148  (%s)\n",
         NI, NT, V, SP, warps, cpi, bytes / cpi, bytes / cpi * 1.965e9 * 148 / 1e12, cudaGetErrorString(e));
  cudaFree(out);
  cudaFree(cyc);
}


// Group-in-N core for single-token passes: the accumulator tile's 8 columns are
// 8 consecutive groups (lane gid feeds its x' row only for k-slices of group
// gid of the tile, else the zero row), so scale/zero are applied once per 8
// groups.  Span = 4 group pairs = one tile.
template <int NI>
__device__ __forceinline__ void core_gn(const uint8_t* st, const uint16_t* xs, const float* bq, const float* xq,
                                        int xs_stride, int zero_row, int warp, int nwarps, float (&acc)[NI][4]) {
  const int lane = threadIdx.x & 31, gid = lane >> 2, tid = lane & 3;
  const int nspan = GPI / 4;
  for (int sp = warp; sp < nspan; sp += nwarps) {
    const int g0 = sp * 8;  // first group of the tile
    const float4 seed = *reinterpret_cast<const float4*>(bq + (sp * 4 + tid) * 4);
    float d[NI][4];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      d[i][0] = seed.x;
      d[i][1] = seed.y;
      d[i][2] = seed.z;
      d[i][3] = seed.w;
    }
#pragma unroll 2
    for (int qq = 0; qq < 4; ++qq) {
      const int q = sp * 4 + qq;
      const uint8_t* blk = st + q * NI * kBlk;
      uint4 cw[NI];
#pragma unroll
      for (int i = 0; i < NI; ++i) cw[i] = *reinterpret_cast<const uint4*>(blk + i * kBlk + lane * 16);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gl = q * 2 + h;
        const uint16_t* xr = xs + ((gl - g0) == gid ? 0 : zero_row) * xs_stride + tid * 4 + gl * 64;
        uint32_t wa[NI][3], wb[NI][3];
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          wa[i][0] = h ? cw[i].z : cw[i].x;
          wb[i][0] = h ? cw[i].w : cw[i].y;
          wa[i][1] = wa[i][0] >> 6;
          wb[i][1] = wb[i][0] >> 6;
          wa[i][2] = wa[i][0] >> 12;
          wb[i][2] = wb[i][0] >> 12;
        }
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint2 bv = *reinterpret_cast<const uint2*>(xr + ks * 16);
          const int j0 = 2 * ks, j1 = 2 * ks + 1;
#pragma unroll
          for (int i = 0; i < NI; ++i) {
            const uint32_t m0 = 0x00030003u << (2 * (j0 % 3)), m1 = 0x00030003u << (2 * (j1 % 3));
            mma_bf16(d[i], lop_and_or(wa[i][j0 / 3], m0), lop_and_or(wb[i][j0 / 3], m0),
                     lop_and_or(wa[i][j1 / 3], m1), lop_and_or(wb[i][j1 / 3], m1), bv.x, bv.y);
          }
        }
      }
    }
    // epilogue once per tile: lane holds D for rows gid, gid+8 x groups g0+2tid, g0+2tid+1
    const float2 xv = *reinterpret_cast<const float2*>(xq + (sp * 4 + tid) * 2);
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const uint4 mw = *reinterpret_cast<const uint4*>(st + (sp * 4 + tid) * NI * kBlk + i * kBlk + kCodeBytes + gid * 16);
      const float2 a0 = h2f2(mw.x), a1 = h2f2(mw.y), b0 = h2f2(mw.z), b1 = h2f2(mw.w);
      acc[i][0] = fmaf(a0.x, d[i][0], fmaf(a0.y, xv.x, acc[i][0]));
      acc[i][1] = fmaf(a1.x, d[i][1], fmaf(a1.y, xv.y, acc[i][1]));
      acc[i][2] = fmaf(b0.x, d[i][2], fmaf(b0.y, xv.x, acc[i][2]));
      acc[i][3] = fmaf(b1.x, d[i][3], fmaf(b1.y, xv.y, acc[i][3]));
    }
  }
}

template <int NI>
__global__ void bench_gn(int items, float* out, long long* cyc) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int xs_stride = GPI * 128 + 8;
  uint8_t* st = sm;
  uint16_t* xs = reinterpret_cast<uint16_t*>(sm + GPI * NI * kBlk);
  float* bq = reinterpret_cast<float*>(sm + GPI * NI * kBlk + 2 * xs_stride * 2);
  float* xq = bq + GPI * 2 * 4;
  const int total = GPI * NI * kBlk + 2 * xs_stride * 2 + GPI * 2 * 4 * 4 + GPI * 2 * 2 * 4;
  for (int i = threadIdx.x; i < total / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = (i * 2654435761u) & 0x3c003c00u;
  __syncthreads();
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  float acc[NI][4] = {};
  const long long t0 = clock64();
  for (int it = 0; it < items; ++it) core_gn<NI>(st, xs, bq, xq, xs_stride, 1, warp, nwarps, acc);
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < NI; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 1.2345f) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int NI>
void run_gn(int warps) {
  const int xs_stride = GPI * 128 + 8;
  const int smem = GPI * NI * kBlk + 2 * xs_stride * 2 + GPI * 2 * 4 * 4 + GPI * 2 * 2 * 4;
  cudaFuncSetAttribute(bench_gn<NI>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4);
  cudaMallocManaged(&cyc, 8);
  const int items = 200;
  bench_gn<NI><<<148, warps * 32, smem>>>(items, out, cyc);
  cudaDeviceSynchronize();
  bench_gn<NI><<<148, warps * 32, smem>>>(items, out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  const double cpi = double(*cyc) / items;
  const double bytes = GPI * NI * kBlk;
  printf("GROUP-N NI=%d warps=%2d:            %7.0f cycles/item  -> %6.1f B/cycle/SM  = %5.2f TB/s  (%s)\n", NI, warps,
         cpi, bytes / cpi, bytes / cpi * 1.965e9 * 148 / 1e12, cudaGetErrorString(e));
  cudaFree(out);
  cudaFree(cyc);
}

// IMMA core (mma.sync m16n8k32 u8 x s8): I8 tile words hold code (m, h, b) of
// lane tid at bit 8b + 2(2m+h) (K = 32m + 16h + 4 tid + b); x as two signed
// 7-bit digits in N columns 2t, 2t+1 (token t <= 3); per (group, token) the
// sums hold {2^-S, -1.5*2^23*2^-S, X, 0}.  The d1 accumulator is seeded with
// the float bits of 1.5*2^23 so 128 d0 + d1 is a float (magic) directly.
__device__ __forceinline__ void imma(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                     uint32_t b1) {
  asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void imma0(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                      uint32_t b1) {
  asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%10,%10,%10};"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "r"(0));
}
// V bit 0: zero-seeded chains (magic added after), bit 1: next group pair's
// code/meta words loaded one iteration ahead
template <int NI, int SP, int V>
__device__ __forceinline__ void core_i8v(const uint8_t* st, const uint8_t* xd, const float4* sums, int xd_stride,
                                         int warp, int nwarps, float (&acc)[NI][2]) {
  const int lane = threadIdx.x & 31, gid = lane >> 2, tid = lane & 3;
  const uint8_t* brow = xd + (gid >> 1) * xd_stride + (gid & 1) * 64 + tid * 8;
  const int nspan = GPI / SP;
  constexpr uint32_t M = 0x03030303u;
  for (int sp = warp; sp < nspan; sp += nwarps) {
    const int q0 = sp * SP, q1 = q0 + SP;
    uint4 cw[NI], mw[NI], ncw[NI], nmw[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      ncw[i] = *reinterpret_cast<const uint4*>(st + q0 * NI * kBlk + i * kBlk + lane * 16);
      nmw[i] = *reinterpret_cast<const uint4*>(st + q0 * NI * kBlk + i * kBlk + kCodeBytes + gid * 16);
    }
#pragma unroll 1
    for (int q = q0; q < q1; ++q) {
      const uint8_t* blk = st + q * NI * kBlk;
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        if (V & 2) {
          cw[i] = ncw[i];
          mw[i] = nmw[i];
          const int qn = q + 1 < q1 ? q + 1 : q;
          ncw[i] = *reinterpret_cast<const uint4*>(st + qn * NI * kBlk + i * kBlk + lane * 16);
          nmw[i] = *reinterpret_cast<const uint4*>(st + qn * NI * kBlk + i * kBlk + kCodeBytes + gid * 16);
        } else {
          cw[i] = *reinterpret_cast<const uint4*>(blk + i * kBlk + lane * 16);
          mw[i] = *reinterpret_cast<const uint4*>(blk + i * kBlk + kCodeBytes + gid * 16);
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gl = q * 2 + h;
        const uint2 bv = *reinterpret_cast<const uint2*>(brow + gl * 128);
        const uint2 bw = *reinterpret_cast<const uint2*>(brow + gl * 128 + 32);
        const float4 sx = sums[gl * 4 + tid];
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const uint32_t wa = h ? cw[i].z : cw[i].x, wb = h ? cw[i].w : cw[i].y;
          int d[4];
          float fa, fb;
          if (V & 1) {
            imma0(d, wa & M, wb & M, (wa >> 2) & M, (wb >> 2) & M, bv.x, bv.y);
            imma(d, (wa >> 4) & M, (wb >> 4) & M, (wa >> 6) & M, (wb >> 6) & M, bw.x, bw.y);
            fa = __int_as_float(d[0] * 128 + (d[1] + 0x4B400000));
            fb = __int_as_float(d[2] * 128 + (d[3] + 0x4B400000));
          } else {
            d[0] = 0; d[1] = 0x4B400000; d[2] = 0; d[3] = 0x4B400000;
            imma(d, wa & M, wb & M, (wa >> 2) & M, (wb >> 2) & M, bv.x, bv.y);
            imma(d, (wa >> 4) & M, (wb >> 4) & M, (wa >> 6) & M, (wb >> 6) & M, bw.x, bw.y);
            fa = __int_as_float(d[0] * 128 + d[1]);
            fb = __int_as_float(d[2] * 128 + d[3]);
          }
          const float ta = fmaf(fa, sx.x, sx.y), tb = fmaf(fb, sx.x, sx.y);
          const float2 mA = h2f2(h ? mw[i].y : mw[i].x);
          const float2 mB = h2f2(h ? mw[i].w : mw[i].z);
          acc[i][0] = fmaf(mA.x, ta, fmaf(mA.y, sx.z, acc[i][0]));
          acc[i][1] = fmaf(mB.x, tb, fmaf(mB.y, sx.z, acc[i][1]));
        }
      }
    }
  }
}

template <int NI, int UNR, int SP>
__device__ __forceinline__ void core_i8(const uint8_t* st, const uint8_t* xd, const float4* sums, int xd_stride,
                                        int warp, int nwarps, float (&acc)[NI][2]) {
  const int lane = threadIdx.x & 31, gid = lane >> 2, tid = lane & 3;
  const uint8_t* brow = xd + (gid >> 1) * xd_stride + (gid & 1) * 64 + tid * 8;
  const int nspan = GPI / SP;
  constexpr uint32_t M = 0x03030303u;
  for (int sp = warp; sp < nspan; sp += nwarps) {
    const int q0 = sp * SP, q1 = q0 + SP;
#pragma unroll UNR
    for (int q = q0; q < q1; ++q) {
      const uint8_t* blk = st + q * NI * kBlk;
      uint4 cw[NI], mw[NI];
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        cw[i] = *reinterpret_cast<const uint4*>(blk + i * kBlk + lane * 16);
        mw[i] = *reinterpret_cast<const uint4*>(blk + i * kBlk + kCodeBytes + gid * 16);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gl = q * 2 + h;
        const uint2 bv = *reinterpret_cast<const uint2*>(brow + gl * 128);  // m = 0; m = 1 at +32
        const uint2 bw = *reinterpret_cast<const uint2*>(brow + gl * 128 + 32);
        const float4 sx = sums[gl * 4 + tid];
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const uint32_t wa = h ? cw[i].z : cw[i].x, wb = h ? cw[i].w : cw[i].y;
          int d[4] = {0, 0x4B400000, 0, 0x4B400000};
          imma(d, wa & M, wb & M, (wa >> 2) & M, (wb >> 2) & M, bv.x, bv.y);
          imma(d, (wa >> 4) & M, (wb >> 4) & M, (wa >> 6) & M, (wb >> 6) & M, bw.x, bw.y);
          const float fa = __int_as_float(d[0] * 128 + d[1]), fb = __int_as_float(d[2] * 128 + d[3]);
          const float ta = fmaf(fa, sx.x, sx.y), tb = fmaf(fb, sx.x, sx.y);
          const float2 mA = h2f2(h ? mw[i].y : mw[i].x);
          const float2 mB = h2f2(h ? mw[i].w : mw[i].z);
          acc[i][0] = fmaf(mA.x, ta, fmaf(mA.y, sx.z, acc[i][0]));
          acc[i][1] = fmaf(mB.x, tb, fmaf(mB.y, sx.z, acc[i][1]));
        }
      }
    }
  }
}

template <int NI, int UNR, int SP>
__global__ void bench_i8(int items, float* out, long long* cyc) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int xd_stride = GPI * 2 * 128 + 16;
  uint8_t* st = sm;
  uint8_t* xd = sm + GPI * NI * kBlk;
  float4* sums = reinterpret_cast<float4*>(sm + GPI * NI * kBlk + 4 * xd_stride);
  const int total = GPI * NI * kBlk + 4 * xd_stride + GPI * 2 * 4 * 16;
  for (int i = threadIdx.x; i < total / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = (i * 2654435761u) & 0x3c003c00u;
  __syncthreads();
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  float acc[NI][2] = {};
  const long long t0 = clock64();
  for (int it = 0; it < items; ++it) {
    if constexpr (UNR >= 10) core_i8v<NI, SP, UNR - 10>(st, xd, sums, xd_stride, warp, nwarps, acc);
    else core_i8<NI, UNR, SP>(st, xd, sums, xd_stride, warp, nwarps, acc);
  }
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < NI; ++i) s += acc[i][0] + acc[i][1];
  if (s == 1.2345f) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int NI, int UNR, int SP = 4>
void run_i8(int warps) {
  const int xd_stride = GPI * 2 * 128 + 16;
  const int smem = GPI * NI * kBlk + 4 * xd_stride + GPI * 2 * 4 * 16;
  cudaFuncSetAttribute(bench_i8<NI, UNR, SP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4);
  cudaMallocManaged(&cyc, 8);
  const int items = 200;
  bench_i8<NI, UNR, SP><<<148, warps * 32, smem>>>(items, out, cyc);
  cudaDeviceSynchronize();
  bench_i8<NI, UNR, SP><<<148, warps * 32, smem>>>(items, out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  const double cpi = double(*cyc) / items;
  const double bytes = GPI * NI * kBlk;
  printf("IMMA NI=%d unroll=%d span=%d warps=%2d:   %7.0f cycles/item  -> %6.1f B/cycle/SM  = %5.2f TB/s  (%s)\n", NI,
         UNR, SP, warps, cpi, bytes / cpi, bytes / cpi * 1.965e9 * 148 / 1e12, cudaGetErrorString(e));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run_i8<2, 1>(8);
  run_i8<2, 10>(8);
  run_i8<2, 11>(8);
  run_i8<2, 12>(8);
  run_i8<2, 13>(8);
  run_i8<2, 1, 2>(16);
  run_i8<2, 11, 2>(16);
  run_i8<2, 13, 2>(16);
  return 0;
  run<2, 1, 0>(8);
  run<2, 1, 2>(8);
  run<2, 1, 2, 2>(16);
  run_gn<2>(8);
  run<1, 1, 0>(8);
  run<1, 1, 2, 2>(16);
  run_gn<1>(8);
  return 0;
}
