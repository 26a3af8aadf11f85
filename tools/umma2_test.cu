// Standalone validation of the CTA-pair (cta_group::2) tcgen05 path used by the
// prefill GEMM: cluster of 2, each CTA holds 128 rows of A and 128 rows of B
// (SWIZZLE_128B K-major), the leader issues tcgen05.mma.cta_group::2 with
// M = 256, N = 256; the peer publishes its smem to the leader's mbarrier with a
// remote release-arrive; the commit is multicast to both CTAs; each CTA reads
// its 128 TMEM lanes.  D[256 x 256] = A[256 x K] . B[256 x K]^T, K = 128.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/umma2_test tools/umma2_test.cu
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int M = 256, N = 256, K = 128, KS = 64, MH = 128, NH = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t sw128(int r, int k) {
  return static_cast<uint32_t>(r) * 128 + ((static_cast<uint32_t>(k >> 3) ^ (r & 7)) << 4) + (k & 7) * 2;
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ bool wait_bar(uint64_t* bar, uint32_t parity) {
  for (long spin = 0; spin < (1L << 26); ++spin) {
    uint32_t ok;
    asm volatile(
        "{.reg .pred P; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%1], %2; selp.b32 %0, 1, 0, P;}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (ok) return true;
  }
  return false;
}

__global__ void __cluster_dims__(2, 1, 1) umma2_kernel(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D,
                                                       int* status, long long* timing) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sa = sm;               // 2 slabs x 16 KB (this CTA's 128 rows of A)
  uint8_t* sb = sm + 2 * MH * 128;  // 2 slabs x 16 KB (this CTA's 128 rows of B)
  __shared__ uint64_t ready, done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t rank = cluster_rank();
  for (int i = tid; i < MH * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sa + (k / KS) * MH * 128 + sw128(r, k % KS)) = A[(rank * MH + r) * K + k];
  }
  for (int i = tid; i < NH * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sb + (k / KS) * NH * 128 + sw128(r, k % KS)) = B[(rank * NH + r) * K + k];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(smem_u32(&ready)));  // own + peer
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(2 * N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();  // barriers initialised + TMEM allocated in both CTAs
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  // publish this CTA's operands to the leader's `ready` barrier
  if (tid == 0) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(&ready)));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
  }
  if (rank == 0 && tid == 0) {
    if (!wait_bar(&ready, 0)) {
      atomicExch(status, 3);
    } else {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t idesc = idesc_bf16(M, N);
      for (int ks = 0; ks < K / 16; ++ks) {
        const int slab = ks / 4, kk = ks % 4;
        const uint64_t da = sdesc(smem_u32(sa + slab * MH * 128) + kk * 32);
        const uint64_t db = sdesc(smem_u32(sb + slab * NH * 128) + kk * 32);
        const uint32_t acc = ks > 0 ? 1u : 0u;
        asm volatile(
            "{.reg .pred p; setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
      const uint16_t mask = 3;
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(&done)),
          "h"(mask)
          : "memory");
    }
  }
  bool ok_done = wait_bar(&done, 0);
  if (ok_done && rank == 0 && tid == 0 && timing != nullptr) {
    // throughput: ITERS x 8 back-to-back MMAs (M=256, N=256, K=16 each) on resident operands
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t idesc = idesc_bf16(M, N);
    long long t0 = clock64();
    for (int it = 0; it < 512; ++it) {
      for (int ks = 0; ks < K / 16; ++ks) {
        const int slab = ks / 4, kk = ks % 4;
        const uint64_t da = sdesc(smem_u32(sa + slab * MH * 128) + kk * 32);
        const uint64_t db = sdesc(smem_u32(sb + slab * NH * 128) + kk * 32);
        asm volatile(
            "{.reg .pred p; setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(tmem + 256),
            "l"(da), "l"(db), "r"(idesc), "r"(1u));
      }
    }
    const uint16_t mask = 3;
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&done)),
        "h"(mask)
        : "memory");
    wait_bar(&done, 1);
    long long t1 = clock64();
    timing[0] = t1 - t0;
  }
  if (ok_done && rank == 1 && tid == 0 && timing != nullptr) wait_bar(&done, 1);
  __syncthreads();
  if (!ok_done) {
    if (tid == 0) atomicExch(status, 2);
  } else {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int row = rank * MH + warp * 32 + (tid & 31);
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
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * N));
  if (tid == 0) atomicAdd(status + 1, 1);
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
  cudaMalloc(&st, 8);
  cudaMemset(st, 0, 8);
  cudaMemset(dd, 0, M * N * 4);
  cudaMemcpy(da, ha.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb.data(), N * K * 2, cudaMemcpyHostToDevice);
  const int smem = 2 * MH * 128 + 2 * NH * 128 + 1024;
  cudaFuncSetAttribute(umma2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long* dt;
  cudaMalloc(&dt, 8);
  cudaMemset(dt, 0, 8);
  umma2_kernel<<<2, 128, smem>>>(da, db, dd, st, dt);
  cudaError_t e = cudaDeviceSynchronize();
  long long ht = 0;
  cudaMemcpy(&ht, dt, 8, cudaMemcpyDeviceToHost);
  printf("timing: 512 x 8 MMAs (M256 N256 K16, SS, cta_group::2): %lld cycles = %.1f cycles/MMA (ideal 128)\n", ht,
         ht / 4096.0);
  int hs[2] = {0, 0};
  cudaMemcpy(hs, st, 8, cudaMemcpyDeviceToHost);
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
      if (err > 1e-3 && bad++ < 8) printf("  mismatch D[%d][%d] = %f, ref %f\n", m, n, hd[m * N + n], ref);
    }
  printf("status %d, ctas done %d (%s), max |err| %.3g, bad %d\n", hs[0], hs[1], cudaGetErrorString(e), maxerr,
         bad);
  return (hs[0] == 0 && hs[1] == 2 && bad == 0) ? 0 : 1;
}
