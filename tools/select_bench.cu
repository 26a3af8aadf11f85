// Warm cost of the router's softmax + stable top-k for one token (E = 8, k = 2):
// the same fp64 operations as select_topk_warp, timed with clock64 per call.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/select_bench tools/select_bench.cu
#include <cfloat>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __noinline__ double pw_sum_small(const double* v, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, v[i]);
    return r;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = v[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], v[i + j]);
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, v[i]);
  return res;
}

__global__ void k(double* g, long long* cyc, int iters, int* out) {
  __shared__ double lg[8 + 64];
  const int lane = threadIdx.x & 31;
  const int E = 8, kk = 2;
  long long t_exp = 0, t_sum = 0, t_div = 0, t_topk = 0;
  int acc = 0;
  for (int it = 0; it < iters; ++it) {
    if (lane < E) lg[lane] = g[lane] + 1e-9 * it;
    __syncwarp();
    long long t0 = clock64();
    double mx = -DBL_MAX;
    for (int e = lane; e < E; e += 32) mx = fmax(mx, lg[e]);
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    for (int e = lane; e < E; e += 32) lg[e] = exp(__dsub_rn(lg[e], mx));
    __syncwarp();
    long long t1 = clock64();
    double den = 0.0;
    if (lane == 0) den = pw_sum_small(lg, E);
    den = __shfl_sync(0xffffffffu, den, 0);
    long long t2 = clock64();
    for (int e = lane; e < E; e += 32) lg[e] = __ddiv_rn(lg[e], den);
    __syncwarp();
    long long t3 = clock64();
    unsigned taken = 0;
    for (int j = 0; j < kk; ++j) {
      double bv = -DBL_MAX;
      int be = 0x7fffffff;
      for (int m = 0, e = lane; e < E; ++m, e += 32)
        if (!((taken >> m) & 1u) && (be == 0x7fffffff || lg[e] > bv)) {
          bv = lg[e];
          be = e;
        }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oe = __shfl_xor_sync(0xffffffffu, be, o);
        if (oe != 0x7fffffff && (be == 0x7fffffff || ov > bv || (ov == bv && oe < be))) {
          bv = ov;
          be = oe;
        }
      }
      if ((be & 31) == lane) taken |= 1u << (be >> 5);
      acc += be;
    }
    long long t4 = clock64();
    t_exp += t1 - t0;
    t_sum += t2 - t1;
    t_div += t3 - t2;
    t_topk += t4 - t3;
  }
  if (lane == 0) {
    cyc[0] = t_exp / iters;
    cyc[1] = t_sum / iters;
    cyc[2] = t_div / iters;
    cyc[3] = t_topk / iters;
    out[0] = acc;
  }
}

int main() {
  double h[8] = {0.3, -0.2, 1.1, 0.7, -1.4, 0.05, 0.9, -0.6};
  double* g;
  long long* cyc;
  int* out;
  cudaMalloc(&g, sizeof(h));
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMallocManaged(&cyc, 4 * sizeof(long long));
  cudaMalloc(&out, 4);
  k<<<1, 32>>>(g, cyc, 10, out);
  cudaDeviceSynchronize();
  k<<<1, 32>>>(g, cyc, 1000, out);
  cudaDeviceSynchronize();
  printf("warm cycles per call: max+exp %lld | pairwise sum (lane 0) %lld | div %lld | top-2 %lld  => total %lld (%.2f us)\n",
         cyc[0], cyc[1], cyc[2], cyc[3], cyc[0] + cyc[1] + cyc[2] + cyc[3],
         (cyc[0] + cyc[1] + cyc[2] + cyc[3]) / 1965.0);
  return 0;
}
