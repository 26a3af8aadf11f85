// K1: fused router -- gate GEMV (fp64) + softmax + stable top-k/top-n, and the
// per-expert pair plan consumed by the expert kernels.
// Reference: ref/moe.py:165-193 (route/softmax), ref/moe.py:234-258 (mixing,
// shared experts).
//
// Grid (token tiles, experts): CTA (tile, e) computes the logits of up to
// kTT tokens against gate row e with wide coalesced fp64 loads.  The last CTA
// of a token tile (atomic ticket) runs softmax + stable top-k for the tile;
// the last tile builds the pair plan -- one launch, no host round trip.
#include <float.h>

#include "common.cuh"
#include "layer.cuh"

namespace lrc {

constexpr int kTT = 8;         // tokens per router CTA
constexpr int kRThreads = 256;

template <typename T>
__device__ __forceinline__ double load_x(const T* x, int64_t i);
template <>
__device__ __forceinline__ double load_x<double>(const double* x, int64_t i) { return x[i]; }
template <>
__device__ __forceinline__ double load_x<float>(const float* x, int64_t i) { return x[i]; }
template <>
__device__ __forceinline__ double load_x<uint16_t>(const uint16_t* x, int64_t i) {
  return static_cast<double>(bf2f(x[i]));
}

// numpy pairwise order for a short fp64 vector (softmax denominator, E <= 256).
__device__ double pw_sum_small(const double* v, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, v[i]);
    return r;
  }
  if (n <= 128) {
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
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pw_sum_small(v, n2), pw_sum_small(v + n2, n - n2));
}

// softmax (ref/moe.py:165-168) + stable descending top-k (np.argsort(-w,
// kind="stable"), ref/moe.py:190: strict '>' keeps the lower index on ties).
__device__ void select_topk(double* lg, int E, int k, int renorm, int64_t b, double* probs,
                            int32_t* topk_idx, float* topk_w) {
  double mx = lg[0];
  for (int e = 1; e < E; ++e) mx = fmax(mx, lg[e]);
  for (int e = 0; e < E; ++e) lg[e] = exp(__dsub_rn(lg[e], mx));
  const double den = pw_sum_small(lg, E);
  for (int e = 0; e < E; ++e) lg[e] = __ddiv_rn(lg[e], den);
  if (probs)
    for (int e = 0; e < E; ++e) probs[b * E + e] = lg[e];
  unsigned long long taken[4] = {0, 0, 0, 0};
  double mix[64];
  for (int j = 0; j < k; ++j) {
    int best = -1;
    double bv = -DBL_MAX;
    for (int e = 0; e < E; ++e) {
      if ((taken[e >> 6] >> (e & 63)) & 1ull) continue;
      if (best < 0 || lg[e] > bv) {
        best = e;
        bv = lg[e];
      }
    }
    taken[best >> 6] |= 1ull << (best & 63);
    topk_idx[b * k + j] = best;
    mix[j] = bv;
  }
  if (renorm) {  // ref/moe.py:234-236, mix.sum() in numpy order
    const double s = pw_sum_small(mix, k);
    if (s > 0.0)
      for (int j = 0; j < k; ++j) mix[j] = __ddiv_rn(mix[j], s);
  }
  for (int j = 0; j < k; ++j) topk_w[b * k + j] = static_cast<float>(mix[j]);
}

// Warp-parallel variant (one warp per token): exp and the top-k argmax run
// across lanes; the softmax denominator keeps numpy's pairwise order (lane 0)
// so weights stay bit-identical to select_topk.
__device__ void select_topk_warp(double* lg, int E, int k, int renorm, int64_t b, double* probs,
                                 int32_t* topk_idx, float* topk_w) {
  const int lane = threadIdx.x & 31;
  double mx = -DBL_MAX;
  for (int e = lane; e < E; e += 32) mx = fmax(mx, lg[e]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  for (int e = lane; e < E; e += 32) lg[e] = exp(__dsub_rn(lg[e], mx));
  __syncwarp();
  double den = 0.0;
  if (lane == 0) den = pw_sum_small(lg, E);
  den = __shfl_sync(0xffffffffu, den, 0);
  for (int e = lane; e < E; e += 32) {
    lg[e] = __ddiv_rn(lg[e], den);
    if (probs) probs[b * E + e] = lg[e];
  }
  __syncwarp();
  uint32_t taken = 0;  // bit m: element lane + 32m already selected
  double mix[64];
  for (int j = 0; j < k; ++j) {
    double bv = -DBL_MAX;
    int be = 0x7fffffff;
    for (int m = 0, e = lane; e < E; ++m, e += 32)
      if (!((taken >> m) & 1u) && (lg[e] > bv || be == 0x7fffffff)) {
        bv = lg[e];
        be = e;
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oe = __shfl_xor_sync(0xffffffffu, be, o);
      if (oe != 0x7fffffff && (be == 0x7fffffff || ov > bv || (ov == bv && oe < be))) {
        bv = ov;
        be = oe;
      }
    }
    if ((be & 31) == lane) taken |= 1u << (be >> 5);
    mix[j] = bv;
    if (lane == 0) topk_idx[b * k + j] = be;
  }
  if (lane == 0) {
    if (renorm) {  // ref/moe.py:234-236, mix.sum() in numpy order
      const double s = pw_sum_small(mix, k);
      if (s > 0.0)
        for (int j = 0; j < k; ++j) mix[j] = __ddiv_rn(mix[j], s);
    }
    for (int j = 0; j < k; ++j) topk_w[b * k + j] = static_cast<float>(mix[j]);
  }
}

__device__ __forceinline__ void griddep_launch_dependents_r() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Speculative low-rank down-projection for a small batch (one token tile):
// t[b][e][proj][j] = V_proj(e)[j, :] . x_b for rows j in block `blk` (8 rows,
// one per warp; proj = blk / (r/8)), for every token of the tile, whether or
// not e turns out to be one of b's top-n experts -- it removes a dependent
// launch between the router and the expert kernels (ref/lowrank.py:165 with
// the factored U.(V.x) order).  Costs < 1% extra bytes at decode sizes.
__device__ void spec_lr_rows(const RouteArgs& ra, const uint16_t* x, int64_t b0, int nb, int e,
                             int blk) {
  const lrc_expert& E = ra.experts[e];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rpb = 8;  // rows per block
  const int nblk1 = (ra.maxr + rpb - 1) / rpb;
  const int proj = blk / nblk1;
  const int j = (blk - proj * nblk1) * rpb + warp;
  const lrc_qmat& V = proj == 0 ? E.v1 : E.v3;
  if (!factor_present(V) || j >= V.rows) {
    if (lane < nb && j < ra.maxr) ra.t[(((b0 + lane) * ra.ne + e) * 3 + proj) * ra.maxr + j] = 0.0f;
    return;
  }
  float acc[kTT];
  const bool g64 = V.dense == nullptr && V.group_size == 64 && ((V.cols * V.bits) % 32) == 0;
  if (V.dense != nullptr) {  // raw fp32 factors (the reference's quantize_factors=False hook)
#pragma unroll
    for (int t = 0; t < kTT; ++t) acc[t] = 0.0f;
    for (int c = lane; c < V.cols; c += 32) {
      const float w = V.dense[static_cast<int64_t>(j) * V.cols + c];
#pragma unroll
      for (int t = 0; t < kTT; ++t)
        if (t < nb) acc[t] = fmaf(w, bf2f(x[(b0 + t) * ra.d + c]), acc[t]);
    }
#pragma unroll
    for (int t = 0; t < kTT; ++t) acc[t] = warp_sum(acc[t]);
  } else if (g64 && V.bits == 3) {
    vrow_dot_tokens<3, kTT>(V, j, x + b0 * ra.d, ra.d, nb, acc);
  } else if (g64 && V.bits == 2) {
    vrow_dot_tokens<2, kTT>(V, j, x + b0 * ra.d, ra.d, nb, acc);
  } else if (g64 && V.bits == 4) {
    vrow_dot_tokens<4, kTT>(V, j, x + b0 * ra.d, ra.d, nb, acc);
  } else {
    const int gs = V.group_size, gpr = (V.cols + gs - 1) / gs;
    const int64_t nbytes = (static_cast<int64_t>(V.rows) * V.cols * V.bits + 7) >> 3;
#pragma unroll
    for (int t = 0; t < kTT; ++t) acc[t] = 0.0f;
    for (int c = lane; c < V.cols; c += 32) {
      const int64_t g = static_cast<int64_t>(j) * gpr + c / gs;
      const float w = fmaf(static_cast<float>(read_code(V.packed, static_cast<int64_t>(j) * V.cols + c,
                                                        V.bits, nbytes)),
                           h2f(V.scales[g]), h2f(V.zeros[g]));
#pragma unroll
      for (int t = 0; t < kTT; ++t)
        if (t < nb) acc[t] = fmaf(w, bf2f(x[(b0 + t) * ra.d + c]), acc[t]);
    }
#pragma unroll
    for (int t = 0; t < kTT; ++t) acc[t] = warp_sum(acc[t]);  // (vrow_dot_tokens reduces itself)
  }
#pragma unroll
  for (int t = 0; t < kTT; ++t)
    if (lane == 0 && t < nb) ra.t[(((b0 + t) * ra.ne + e) * 3 + proj) * ra.maxr + j] = acc[t];
}

template <typename T>
__global__ void __launch_bounds__(kRThreads) gate_kernel(RouteArgs ra) {
  extern __shared__ double sm_lg[];  // [kTT][E] (last CTA only)
  __shared__ double s_red[kTT][kRThreads / 32];
  __shared__ int s_last;
  // blockIdx.z == 0: gate logits of expert e (e < E) + zeroing of this tile's
  // y rows / t2 block; blockIdx.z >= 1: speculative low-rank down-projection
  // t = V.x for 8 rows of V1|V3 of expert e (small batches, see spec_lr_rows).
  const int tile = blockIdx.x, e = blockIdx.y, z = blockIdx.z;
  const int64_t b0 = static_cast<int64_t>(tile) * kTT;
  const int64_t rem = ra.B - b0;
  const int nb = rem < kTT ? static_cast<int>(rem) : kTT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T* x = static_cast<const T*>(ra.x);
  griddep_launch_dependents_r();
  if (z == 0) {
    if (e < ra.E) {
      const double* g = ra.gate_t + static_cast<int64_t>(e) * ra.d;
      double acc[kTT];
#pragma unroll
      for (int t = 0; t < kTT; ++t) acc[t] = 0.0;
      // all of this thread's gate loads are independent: unroll for memory-level parallelism
#pragma unroll 8
      for (int i = threadIdx.x; i < ra.d; i += kRThreads) {
        const double gv = __ldg(g + i);
#pragma unroll
        for (int t = 0; t < kTT; ++t)
          if (t < nb) acc[t] = fma(gv, load_x<T>(x, (b0 + t) * ra.d + i), acc[t]);
      }
#pragma unroll
      for (int t = 0; t < kTT; ++t) {
        const double v = warp_sum_d(acc[t]);
        if (lane == 0) s_red[t][warp] = v;
      }
      __syncthreads();
      if (threadIdx.x < nb) {
        double s = 0.0;
        for (int w = 0; w < kRThreads / 32; ++w) s += s_red[threadIdx.x][w];
        ra.logits[(b0 + threadIdx.x) * ra.E + e] = s;
      }
    }
    if (ra.t2_zero != nullptr && ra.maxr > 0)
      for (int i = threadIdx.x; i < nb * ra.maxr; i += kRThreads) {
        const int t = i / ra.maxr, j = i - t * ra.maxr;
        ra.t2_zero[(((b0 + t) * ra.ne + e) * 3 + 2) * ra.maxr + j] = 0.0f;
      }
    if (ra.y_zero != nullptr && e == 0)
      for (int64_t i = threadIdx.x; i < static_cast<int64_t>(nb) * ra.d; i += kRThreads)
        ra.y_zero[b0 * ra.d + i] = 0.0f;
  } else if constexpr (sizeof(T) == 2) {
    spec_lr_rows(ra, reinterpret_cast<const uint16_t*>(x), b0, nb, e, z - 1);
  }
  // ---- last CTA of this token tile: softmax + top-k
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0)
    s_last = (atomicAdd(&ra.tile_ticket[tile], 1) == static_cast<int>(gridDim.y * gridDim.z) - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int i = threadIdx.x; i < nb * ra.E; i += kRThreads)
    sm_lg[i] = __ldcg(ra.logits + b0 * ra.E + i);
  __syncthreads();
  if (warp < nb)
    select_topk_warp(sm_lg + warp * ra.E, ra.E, ra.k, ra.renorm, b0 + warp, ra.probs, ra.topk_idx,
                     ra.topk_w);
  if (threadIdx.x == 0) ra.tile_ticket[tile] = 0;
  if (ra.plan.ticket == nullptr) return;
  // ---- last tile: build the pair plan for the whole batch
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(ra.plan.ticket, 1) == static_cast<int>(gridDim.x) - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  build_plan_block(ra.plan, ra.topk_idx, ra.topk_w, static_cast<int>(ra.B), ra.k);
  if (threadIdx.x == 0) *ra.plan.ticket = 0;
}

// Pair plan: pair p = b*P + j, P = k + S.  j < k: routed expert topk_idx[b][j],
// weight topk_w, compensated iff j < n.  j >= k: shared expert E + (j-k),
// weight 1, compensated iff compensate_shared (ref/moe.py:249-258).
// Pairs are grouped by expert, ascending pair id inside each expert (stable).
__device__ void build_plan_block(const PlanArgs& pa, const int32_t* topk_idx, const float* topk_w,
                                 int B, int k) {
  const int P = k + pa.num_shared;
  const int NP = B * P;
  const int NE = pa.num_experts + pa.num_shared;
  __shared__ int s_cnt[LRC_MAX_EXPERTS];
  __shared__ int s_off[LRC_MAX_EXPERTS + 1];
  for (int e = threadIdx.x; e < NE; e += blockDim.x) s_cnt[e] = 0;
  __syncthreads();
  for (int p = threadIdx.x; p < NP; p += blockDim.x) {
    const int b = p / P, j = p - b * P;
    int e;
    float w;
    if (j < k) {
      e = __ldcg(topk_idx + b * k + j);
      w = __ldcg(topk_w + b * k + j);
    } else {
      e = pa.num_experts + (j - k);
      w = 1.0f;
    }
    pa.pair_expert[p] = e;
    pa.pair_w[p] = w;
    pa.pair_token[p] = b;
    atomicAdd(&s_cnt[e], 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0, na = 0;
    for (int e = 0; e < NE; ++e) {
      s_off[e] = acc;
      acc += s_cnt[e];
      if (s_cnt[e] > 0) {
        pa.active[na] = e;
        pa.active_off[na] = s_off[e];
        pa.active_cnt[na] = s_cnt[e];
        ++na;
      }
    }
    s_off[NE] = acc;
    pa.counts[0] = na;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    // stable scatter: one warp walks the pairs in order; experts present in a
    // 32-pair chunk are serialised and each advances by its ballot prefix
    int count = 0;
    for (int base = 0; base < NP; base += 32) {
      const int p = base + lane;
      const bool valid = p < NP;
      const int e = valid ? pa.pair_expert[p] : -1;
      int pos = -1;
      unsigned pending = __ballot_sync(0xffffffffu, valid);
      while (pending) {
        const int leader = __ffs(pending) - 1;
        const int le = __shfl_sync(0xffffffffu, e, leader);
        const unsigned same = __ballot_sync(0xffffffffu, valid && e == le);
        if (valid && e == le) pos = s_off[le] + __popc(same & ((1u << lane) - 1u));
        __syncwarp();
        if (lane == leader) s_off[le] += __popc(same);
        __syncwarp();
        pending &= ~same;
      }
      if (valid) pa.pair_list[pos] = p;
      // compensated-pair slots (for the t = V.x buffers), in pair order
      int comp = 0;
      if (valid) {
        const int j = p % P;
        comp = (j < k) ? ((j < pa.top_n) && pa.has_comp[e]) : (pa.compensate_shared && pa.has_comp[e]);
      }
      const unsigned m = __ballot_sync(0xffffffffu, comp);
      if (valid) {
        const int slot = comp ? count + __popc(m & ((1u << lane) - 1u)) : -1;
        pa.pair_comp[p] = slot;
        if (comp) pa.comp_list[slot] = p;
      }
      count += __popc(m);
    }
    if (lane == 0) pa.counts[1] = count;
  }
}

int route_tiles(int64_t B) { return static_cast<int>((B + kTT - 1) / kTT); }

lrc_status launch_route(const RouteArgs& ra, cudaStream_t st) {
  const int smem = kTT * ra.E * static_cast<int>(sizeof(double));
  dim3 grid(route_tiles(ra.B), ra.experts ? ra.ne : ra.E, 1 + ra.spec_blocks);
  switch (ra.x_dtype) {
    case LRC_DTYPE_F64:
      gate_kernel<double><<<grid, kRThreads, smem, st>>>(ra);
      break;
    case LRC_DTYPE_F32:
      gate_kernel<float><<<grid, kRThreads, smem, st>>>(ra);
      break;
    case LRC_DTYPE_BF16:
      gate_kernel<uint16_t><<<grid, kRThreads, smem, st>>>(ra);
      break;
    default:
      return fail(LRC_ERR_INVALID, "route: unknown x dtype");
  }
  LRC_CHECK_LAUNCH();
  return LRC_OK;
}

}  // namespace lrc

extern "C" lrc_status lrc_route(const double* gate_t, const void* x, int x_dtype, int64_t B, int d,
                                int E, int top_k, int top_n, int renormalize, double* probs,
                                int32_t* topk_idx, float* topk_w, void* stream) {
  using namespace lrc;
  if (B < 0 || d <= 0 || E <= 0) return fail(LRC_ERR_INVALID, "route: bad shape");
  if (top_k < 0 || top_n < 0 || top_n > top_k)
    return fail(LRC_ERR_INVALID, "top_n must be <= top_k and both >= 0");
  if (top_k > E) return fail(LRC_ERR_INVALID, "top_k exceeds the number of experts");
  if (top_k > 64 || E > LRC_MAX_EXPERTS) return fail(LRC_ERR_UNSUPPORTED, "route: top_k <= 64, E <= 256");
  if (B == 0) return LRC_OK;
  cudaStream_t st = as_stream(stream);
  // standalone call: scratch from the stream-ordered allocator
  RouteArgs ra{};
  ra.gate_t = gate_t;
  ra.x = x;
  ra.x_dtype = x_dtype;
  ra.B = B;
  ra.d = d;
  ra.E = E;
  ra.k = top_k;
  ra.renorm = renormalize;
  ra.probs = probs;
  ra.topk_idx = topk_idx;
  ra.topk_w = topk_w;
  const int nt = route_tiles(B);
  void* scratch = nullptr;
  const size_t bytes = sizeof(double) * B * E + sizeof(int) * (nt + 1);
  LRC_CUDA_TRY(cudaMallocAsync(&scratch, bytes, st));
  LRC_CUDA_TRY(cudaMemsetAsync(scratch, 0, bytes, st));
  ra.logits = static_cast<double*>(scratch);
  ra.tile_ticket = reinterpret_cast<int*>(ra.logits + B * E);
  lrc_status s = launch_route(ra, st);
  cudaFreeAsync(scratch, st);
  return s;
}
