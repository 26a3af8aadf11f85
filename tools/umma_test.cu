// Standalone validation of the tcgen05 building blocks used by the prefill GEMM:
// SWIZZLE_128B K-major smem descriptors, the kind::f16 instruction descriptor,
// TMEM alloc / tcgen05.mma / commit->mbarrier / tcgen05.ld, against a host GEMM.
// D[128 x N] = A[128 x K] . B[N x K]^T, bf16 in, fp32 accumulate, K = 128.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/umma_test tools/umma_test.cu
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int M = 128, N = 128, K = 128, KS = 64;  // K slab = one 128-byte swizzle row

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// byte offset of element (r, k) of a [rows x 64] bf16 K-major SWIZZLE_128B slab
__device__ __forceinline__ uint32_t sw128(int r, int k) {
  const uint32_t chunk = static_cast<uint32_t>(k >> 3), within = static_cast<uint32_t>(k & 7) * 2;
  return static_cast<uint32_t>(r) * 128 + ((chunk ^ (r & 7)) << 4) + within;
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {  // K-major, SWIZZLE_128B
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);         // start address
  d |= static_cast<uint64_t>(1) << 16;                       // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;               // SBO: 8-row group stride
  d |= static_cast<uint64_t>(1) << 46;                       // version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;                       // SWIZZLE_128B
  return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n) {
  return (1u << 4)                               // D format F32
         | (1u << 7) | (1u << 10)                // A, B = BF16
         | (static_cast<uint32_t>(n >> 3) << 17)  // N >> 3
         | (static_cast<uint32_t>(m >> 4) << 24); // M >> 4
}

__global__ void umma_kernel(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int* status) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sa = sm;                    // 2 slabs x 16 KB
  uint8_t* sb = sm + 2 * M * 128;      // 2 slabs x 16 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sa + (k / KS) * M * 128 + sw128(r, k % KS)) = A[i];
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sb + (k / KS) * N * 128 + sw128(r, k % KS)) = B[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> async proxy
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = idesc_bf16(M, N);
    for (int ks = 0; ks < K / 16; ++ks) {
      const int slab = ks / 4, kk = ks % 4;  // 4 K=16 steps per 128-byte row: +32 B each
      const uint64_t da = sdesc(smem_u32(sa + slab * M * 128) + kk * 32);
      const uint64_t db = sdesc(smem_u32(sb + slab * N * 128) + kk * 32);
      const uint32_t acc = ks > 0 ? 1u : 0u;
      asm volatile(
          "{.reg .pred p; setp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
  }
  // bounded wait on the commit (trap instead of hanging the GPU)
  uint32_t done = 0;
  for (long spin = 0; spin < (1L << 26) && !done; ++spin)
    asm volatile("{.reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0; selp.b32 %0, 1, 0, P;}"
                 : "=r"(done)
                 : "r"(smem_u32(&bar)));
  if (!done) {
    if (tid == 0) atomicExch(status, 2);
    return;
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // warp w reads TMEM lanes 32w..32w+31 (= rows), 32 columns at a time
  const int row = warp * 32 + (tid & 31);
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    const uint32_t addr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 32; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(N));
  if (tid == 0) atomicExch(status, 1);
}

int main() {
  std::vector<__nv_bfloat16> ha(M * K), hb(N * K);
  std::vector<float> fa(M * K), fb(N * K);
  srand(1);
  for (int i = 0; i < M * K; ++i) {
    fa[i] = __bfloat162float(__float2bfloat16((rand() % 17 - 8) / 8.0f));
    ha[i] = __float2bfloat16(fa[i]);
  }
  for (int i = 0; i < N * K; ++i) {
    fb[i] = __bfloat162float(__float2bfloat16((rand() % 13 - 6) / 4.0f));
    hb[i] = __float2bfloat16(fb[i]);
  }
  __nv_bfloat16 *da, *db;
  float* dd;
  int* st;
  cudaMalloc(&da, M * K * 2);
  cudaMalloc(&db, N * K * 2);
  cudaMalloc(&dd, M * N * 4);
  cudaMalloc(&st, 4);
  cudaMemset(st, 0, 4);
  cudaMemcpy(da, ha.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb.data(), N * K * 2, cudaMemcpyHostToDevice);
  const int smem = 2 * M * 128 + 2 * N * 128 + 1024;
  cudaFuncSetAttribute(umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  umma_kernel<<<1, 128, smem>>>(da, db, dd, st);
  cudaError_t e = cudaDeviceSynchronize();
  int hs = 0;
  cudaMemcpy(&hs, st, 4, cudaMemcpyDeviceToHost);
  std::vector<float> hd(M * N);
  cudaMemcpy(hd.data(), dd, M * N * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  int bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += double(fa[m * K + k]) * fb[n * K + k];
      const double err = fabs(ref - hd[m * N + n]);
      if (err > maxerr) maxerr = err;
      if (err > 1e-3 && bad++ < 5) printf("  mismatch D[%d][%d] = %f, ref %f\n", m, n, hd[m * N + n], ref);
    }
  printf("status %d (%s), max |err| %.3g, bad %d\n", hs, cudaGetErrorString(e), maxerr, bad);
  return (hs == 1 && bad == 0) ? 0 : 1;
}
