// Expert-parallel dispatch and combine (the exchange the
// reference's single-device forward does not have -- its combine is
// ref/moe.py:237-258, y = sum over the token's selected experts of w * E(x)).
//
// Fixed-capacity layout, no host synchronisation, static shapes (graph
// capturable with the NCCL all-to-alls between the two kernels):
//   pair p = b k + j (token b, j-th selected expert e = idx[b][j]) goes to rank
//   dest(e) = floor(e G / E) at slot dest * C + (rank of p among the pairs with
//   the same dest, in pair order); C = max_tokens * k rows per destination.
//   Unused slots carry a zero row for the receiver's first expert ceil(r E / G)
//   with weight 0 (they add nothing).
// lrc_ep_dispatch: one kernel builds the slot map (every block recomputes it in
//   shared memory: B k <= 4096 pairs, a per-destination counter scan) and
//   writes the send rows (bf16 x) and metadata {expert, weight bits, comp}.
// lrc_ep_combine: y[b] = sum_j back[slot_of[b k + j]] (gather, no atomics,
//   deterministic).
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "layer.cuh"

namespace lrc {
namespace {

constexpr int kMaxPairs = 4096;
constexpr int kMaxRanks = 64;

// stable per-destination rank of every pair (all threads of the block)
__device__ void ep_slots(const int32_t* idx, int np, int E, int W, int C, int* s_slot) {
  __shared__ int s_cnt[kMaxRanks];
  // chunked scan: 32 pairs per warp-step, ballot per destination
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < W) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  if (warp == 0) {
    for (int base = 0; base < np; base += 32) {
      const int p = base + lane;
      const int e = p < np ? idx[p] : 0;
      const int d = p < np ? (e * W) / E : -1;
      const unsigned same = __match_any_sync(0xffffffffu, d);
      const int before = __popc(same & ((1u << lane) - 1u));
      int pos = 0;
      if (p < np) pos = s_cnt[d] + before;
      __syncwarp();
      // the highest lane of each destination group advances its counter
      if (p < np && (same >> lane) == 1u) s_cnt[d] += __popc(same);
      __syncwarp();
      if (p < np) s_slot[p] = d * C + pos;
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) ep_dispatch_kernel(const int32_t* __restrict__ idx,
                                                           const float* __restrict__ w,
                                                           const uint16_t* __restrict__ x, int B, int k,
                                                           int top_n, int E, int W, int C, int d,
                                                           uint16_t* __restrict__ xs, int32_t* __restrict__ meta,
                                                           int32_t* __restrict__ slot_of) {
  __shared__ int s_slot[kMaxPairs];
  __shared__ int s_pair[kMaxPairs];  // slot -> pair (-1: unused) for this block's slots
  const int np = B * k, ns = W * C;
  ep_slots(idx, np, E, W, C, s_slot);
  // inverse map over all slots (every block; ns <= kMaxPairs)
  for (int i = threadIdx.x; i < ns; i += blockDim.x) s_pair[i] = -1;
  __syncthreads();
  for (int p = threadIdx.x; p < np; p += blockDim.x) s_pair[s_slot[p]] = p;
  __syncthreads();
  if (blockIdx.x == 0)
    for (int p = threadIdx.x; p < np; p += blockDim.x) slot_of[p] = s_slot[p];
  // rows: one warp per slot, 16-byte chunks
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const int chunks = d / 8;
  for (int sl = gw; sl < ns; sl += nw) {
    const int p = s_pair[sl];
    uint4* dst = reinterpret_cast<uint4*>(xs + static_cast<int64_t>(sl) * d);
    if (p >= 0) {
      const uint4* src = reinterpret_cast<const uint4*>(x + static_cast<int64_t>(p / k) * d);
      for (int c = lane; c < chunks; c += 32) dst[c] = src[c];
    } else {
      for (int c = lane; c < chunks; c += 32) dst[c] = make_uint4(0, 0, 0, 0);
    }
    if (lane == 0) {
      const int r = sl / C;
      int e = (r * E + W - 1) / W, wb = 0, cp = 0;  // dummy: the receiver's first expert, weight 0
      if (p >= 0) {
        e = idx[p];
        wb = __float_as_int(w[p]);
        cp = (p % k) < top_n ? 1 : 0;
      }
      meta[3 * sl] = e;
      meta[3 * sl + 1] = wb;
      meta[3 * sl + 2] = cp;
    }
  }
}

__global__ void __launch_bounds__(256) ep_combine_kernel(const float* __restrict__ back,
                                                          const int32_t* __restrict__ slot_of, int B, int k,
                                                          int d, float* __restrict__ y) {
  const int64_t n = static_cast<int64_t>(B) * (d / 4);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int b = static_cast<int>(i / (d / 4)), c = static_cast<int>(i % (d / 4));
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j < k; ++j) {
      const float4 v = reinterpret_cast<const float4*>(back + static_cast<int64_t>(slot_of[b * k + j]) * d)[c];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    reinterpret_cast<float4*>(y + static_cast<int64_t>(b) * d)[c] = acc;
  }
}

}  // namespace
}  // namespace lrc

using namespace lrc;

extern "C" lrc_status lrc_ep_dispatch(const int32_t* topk_idx, const float* topk_w, const uint16_t* x, int64_t B,
                                      int top_k, int top_n, int num_experts, int world, int capacity, int d,
                                      uint16_t* x_send, int32_t* meta_send, int32_t* slot_of, void* stream) {
  if (!topk_idx || !topk_w || !x || !x_send || !meta_send || !slot_of)
    return fail(LRC_ERR_INVALID, "ep_dispatch: null pointer");
  if (B < 0 || top_k < 1 || world < 1 || world > kMaxRanks || num_experts < world || d % 8 != 0 ||
      B * top_k > capacity || static_cast<int64_t>(world) * capacity > kMaxPairs)
    return fail(LRC_ERR_INVALID, "ep_dispatch: bad shape (B k <= capacity, world capacity <= 4096, d % 8 == 0)");
  const int ns = world * capacity;
  const int grid = std::max(1, std::min(148, (ns + 7) / 8));
  ep_dispatch_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      topk_idx, topk_w, x, static_cast<int>(B), top_k, top_n, num_experts, world, capacity, d, x_send, meta_send,
      slot_of);
  LRC_CHECK_LAUNCH();
  return LRC_OK;
}

extern "C" lrc_status lrc_ep_combine(const float* back, const int32_t* slot_of, int64_t B, int top_k, int d,
                                     float* y, void* stream) {
  if (!back || !slot_of || !y) return fail(LRC_ERR_INVALID, "ep_combine: null pointer");
  if (B < 0 || top_k < 1 || d % 4 != 0) return fail(LRC_ERR_INVALID, "ep_combine: bad shape");
  if (B == 0) return LRC_OK;
  const int64_t n = B * (d / 4);
  const int grid = static_cast<int>(std::min<int64_t>(4 * 148, (n + 255) / 256));
  ep_combine_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(back, slot_of, static_cast<int>(B), top_k, d,
                                                                         y);
  LRC_CHECK_LAUNCH();
  return LRC_OK;
}
