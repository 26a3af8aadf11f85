// Microbenchmark: per-SM streaming bandwidth of cp.async.bulk (1D TMA) vs LDG.128.
// One persistent CTA per SM streams its contiguous share of a large buffer
// in chunks of C bytes through a ring of S shared-memory stages (bulk), or
// with per-thread 16-byte loads (ldg).  Prints GB/s for each configuration.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bw tools/stream_bw.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void bulk_stream(const uint8_t* src, int64_t per_cta, int chunk, int nstage, int nconsumer,
                            unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)chunk * nstage);
  uint64_t* empty = full + nstage;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nstage; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(nconsumer));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint8_t* base = src + per_cta * blockIdx.x;
  const int nitems = static_cast<int>(per_cta / chunk);
  if (warp == nconsumer) {
    if (lane == 0) {
      for (int k = 0; k < nitems; ++k) {
        const int s = k % nstage;
        if (k >= nstage) {
          uint32_t par = ((k / nstage) - 1) & 1;
          asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(su32(&empty[s])), "r"(par) : "memory");
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(chunk) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(sm + (size_t)s * chunk)), "l"(base + (int64_t)k * chunk), "r"(chunk), "r"(su32(&full[s])) : "memory");
      }
    }
    return;
  }
  unsigned long long acc = 0;
  for (int k = 0; k < nitems; ++k) {
    const int s = k % nstage;
    uint32_t par = (k / nstage) & 1;
    asm volatile("{\n.reg .pred P;\nW2: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W2;\n}" ::"r"(su32(&full[s])), "r"(par) : "memory");
    const uint4* p = reinterpret_cast<const uint4*>(sm + (size_t)s * chunk);
    for (int i = threadIdx.x; i < chunk / 16; i += nconsumer * 32) acc += p[i].x;
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
  }
  if (acc == 0x1234567) atomicAdd(sink, acc);
}

__global__ void ldg_stream(const uint4* src, int64_t per_cta16, int unroll, unsigned long long* sink) {
  const uint4* base = src + per_cta16 * blockIdx.x;
  unsigned long long acc = 0;
  const int T = blockDim.x;
  int64_t i = threadIdx.x;
  for (; i + (int64_t)(7) * T < per_cta16; i += 8 * T) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcs(base + i + u * T);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u].x;
  }
  for (; i < per_cta16; i += T) acc += __ldcs(base + i).x;
  if (acc == 0x1234567) atomicAdd(sink, acc);
}

int main() {
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t total = 3LL << 30;  // 3 GiB
  uint8_t* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  const int chunks[] = {4096, 8192, 16384, 20480, 40960};
  for (int ch : chunks) {
    for (int ns = 2; ns <= 8; ns *= 2) {
      if ((int64_t)ch * ns > 200 * 1024) continue;
      for (int nc : {4, 8, 16}) {
        for (int ctas_per_sm : {1, 2}) {
          if ((int64_t)ch * ns * ctas_per_sm > 200 * 1024) continue;
          const int grid = nsm * ctas_per_sm;
          const int64_t per = (total / grid) / ch * ch;
          const int smem = ch * ns + 2 * ns * 8;
          for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            bulk_stream<<<grid, (nc + 1) * 32, smem>>>(buf, per, ch, ns, nc, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
          }
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          cudaError_t err = cudaGetLastError();
          printf("bulk chunk=%6d stages=%d consumers=%2d ctas/sm=%d : %7.1f GB/s %s\n", ch, ns, nc,
                 ctas_per_sm, per * grid / (ms * 1e6), err == cudaSuccess ? "" : cudaGetErrorString(err));
        }
      }
    }
  }
  for (int threads : {256, 512, 1024}) {
    for (int ctas_per_sm : {1, 2, 4}) {
      if (threads * ctas_per_sm > 2048) continue;
      const int grid = nsm * ctas_per_sm;
      const int64_t per16 = (total / 16) / grid;
      float ms;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        ldg_stream<<<grid, threads>>>(reinterpret_cast<uint4*>(buf), per16, 8, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      cudaEventElapsedTime(&ms, e0, e1);
      printf("ldg threads=%4d ctas/sm=%d : %7.1f GB/s\n", threads, ctas_per_sm,
             per16 * 16.0 * grid / (ms * 1e6));
    }
  }
  return 0;
}
