// MoE layer object: workspace, generic (reference-layout) expert kernels, LR
// kernels, and the forward orchestration.  Reference: ref/moe.py:196-259,
// ref/lowrank.py:153-165.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"
#include "layer.cuh"
#include "tcd.cuh"

namespace lrc {

// ------------------------------------------------------------ LR kernels ---
// t[b][e][proj][j] = V_proj(e)[j, :] . x_b  for compensated pairs, proj in {w1, w3}
__global__ void __launch_bounds__(256) lr_down_kernel(ExpertArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int task = blockIdx.x * 8 + warp;
  const int per_slot = 2 * a.maxr;
  const int slot = task / per_slot;
  if (slot >= a.plan.counts[1]) return;
  const int rem = task - slot * per_slot;
  const int proj = rem / a.maxr, j = rem - proj * a.maxr;
  const int p = a.plan.comp_list[slot];
  const lrc_expert& E = a.experts[a.plan.pair_expert[p]];
  const lrc_qmat& V = proj == 0 ? E.v1 : E.v3;
  float acc = 0.0f;
  if (qmat_present(V) && j < V.rows) {
    const uint16_t* xb = a.x + static_cast<int64_t>(a.plan.pair_token[p]) * a.hidden;
    const bool g64 = V.dense == nullptr && V.group_size == 64 && ((V.cols * V.bits) % 32) == 0;
    float av[1];
    if (g64 && V.bits == 3) {
      vrow_dot_tokens<3, 1>(V, j, xb, a.hidden, 1, av);
      acc = av[0];
    } else if (g64 && V.bits == 2) {
      vrow_dot_tokens<2, 1>(V, j, xb, a.hidden, 1, av);
      acc = av[0];
    } else if (g64 && V.bits == 4) {
      vrow_dot_tokens<4, 1>(V, j, xb, a.hidden, 1, av);
      acc = av[0];
    } else {
      for (int k = lane; k < V.cols; k += 32) acc = fmaf(qmat_elem(V, j, k), bf2f(xb[k]), acc);
      acc = warp_sum(acc);
    }
  }
  if (lane == 0)
    a.t[((static_cast<int64_t>(a.plan.pair_token[p]) * a.ne + a.plan.pair_expert[p]) * 3 + proj) *
            a.maxr + j] = acc;
}

// index of t[b][e][proj][0] for pair p
__device__ __forceinline__ int64_t t_base(const ExpertArgs& a, int p, int proj) {
  return ((static_cast<int64_t>(a.plan.pair_token[p]) * a.ne + a.plan.pair_expert[p]) * 3 + proj) *
         a.maxr;
}

// U(row, :) . t  (warp-cooperative; all lanes return the sum)
__device__ __forceinline__ float lr_up_dot(const lrc_qmat& U, int row, const float* t) {
  float s = 0.0f;
  for (int j = threadIdx.x & 31; j < U.cols; j += 32) s = fmaf(qmat_elem(U, row, j), t[j], s);
  return warp_sum(s);
}

// --------------------------------------------------- generic expert kernels ---
constexpr int kChunk = 8;

// qrow_dot_g64 with the token count rounded up to 1, 2, 4 or 8 (fewer
// registers and no dead token lanes for the common small counts)
template <int BITS, typename XT>
__device__ __forceinline__ void gdot(const lrc_qmat& W, int row, const XT* const (&xp)[kChunk], int nb,
                                     float (&acc)[kChunk]) {
  if (nb == 1) {
    const XT* const x1[1] = {xp[0]};
    float a1[1];
    qrow_dot_g64<BITS, 1>(W, row, x1, 1, a1);
    acc[0] = a1[0];
  } else if (nb == 2) {
    const XT* const x2[2] = {xp[0], xp[1]};
    float a2[2];
    qrow_dot_g64<BITS, 2>(W, row, x2, 2, a2);
    acc[0] = a2[0];
    acc[1] = a2[1];
  } else if (nb <= 4) {
    const XT* const x4[4] = {xp[0], xp[1], xp[2], xp[3]};
    float a4[4];
    qrow_dot_g64<BITS, 4>(W, row, x4, nb, a4);
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = a4[i];
  } else {
    qrow_dot_g64<BITS, kChunk>(W, row, xp, nb, acc);
  }
}

__global__ void __launch_bounds__(256) up_generic_kernel(ExpertArgs a) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int n_active = a.plan.counts[0];
  const int64_t total = static_cast<int64_t>(n_active) * a.ffn;
  for (int64_t task = gw; task < total; task += nwarps) {
    const int ai = static_cast<int>(task / a.ffn);
    const int f = static_cast<int>(task - static_cast<int64_t>(ai) * a.ffn);
    const lrc_expert& E = a.experts[a.plan.active[ai]];
    const int off = a.plan.active_off[ai], cnt = a.plan.active_cnt[ai];
    for (int c0 = 0; c0 < cnt; c0 += kChunk) {
      const int nch = min(kChunk, cnt - c0);
      float acc1[kChunk], acc3[kChunk];
      const uint16_t* xp[kChunk];
#pragma unroll
      for (int i = 0; i < kChunk; ++i) {
        acc1[i] = acc3[i] = 0.0f;
        int p = a.plan.pair_list[off + c0 + min(i, nch - 1)];
        xp[i] = a.x + static_cast<int64_t>(a.plan.pair_token[p]) * a.hidden;
      }
      const bool fast = a.g64 && E.w1.bits == E.w3.bits;
      if (fast && E.w1.bits == 2) {
        gdot<2>(E.w1, f, xp, nch, acc1);
        gdot<2>(E.w3, f, xp, nch, acc3);
      } else if (fast && E.w1.bits == 3) {
        gdot<3>(E.w1, f, xp, nch, acc1);
        gdot<3>(E.w3, f, xp, nch, acc3);
      } else if (fast && E.w1.bits == 4) {
        gdot<4>(E.w1, f, xp, nch, acc1);
        gdot<4>(E.w3, f, xp, nch, acc3);
      } else {
        for (int k = lane; k < a.hidden; k += 32) {
          const float w1v = qmat_elem(E.w1, f, k), w3v = qmat_elem(E.w3, f, k);
#pragma unroll
          for (int i = 0; i < kChunk; ++i) {
            if (i < nch) {
              const float xv = bf2f(xp[i][k]);
              acc1[i] = fmaf(w1v, xv, acc1[i]);
              acc3[i] = fmaf(w3v, xv, acc3[i]);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < kChunk; ++i) {
          acc1[i] = warp_sum(acc1[i]);
          acc3[i] = warp_sum(acc3[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < kChunk; ++i) {
        if (i < nch) {
          float h1 = acc1[i], h3 = acc3[i];
          const int p = a.plan.pair_list[off + c0 + i];
          const int slot = a.plan.pair_comp[p];
          if (slot >= 0) {
            const float* tp = a.t + t_base(a, p, 0);
            if (qmat_present(E.u1)) h1 += lr_up_dot(E.u1, f, tp);
            if (qmat_present(E.u3)) h3 += lr_up_dot(E.u3, f, tp + a.maxr);
          }
          if (lane == 0) a.a32[static_cast<int64_t>(p) * a.ffn + f] = silu_f(h1) * h3;
        }
      }
    }
  }
}

// t[slot][2][j] = V2(e)[j, :] . a_p
__global__ void __launch_bounds__(256) lr_mid_kernel(ExpertArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int task = blockIdx.x * 8 + warp;
  const int slot = task / a.maxr;
  if (slot >= a.plan.counts[1]) return;
  const int j = task - slot * a.maxr;
  const int p = a.plan.comp_list[slot];
  const lrc_expert& E = a.experts[a.plan.pair_expert[p]];
  float acc = 0.0f;
  if (qmat_present(E.v2) && j < E.v2.rows) {
    const float* ap = a.a32 + static_cast<int64_t>(p) * a.ffn;
    const float* const xp[1] = {ap};
    float av[1];
    if (a.g64 && qmat_g64(E.v2) && E.v2.bits == 3) {
      qrow_dot_g64<3, 1>(E.v2, j, xp, 1, av);
      acc = av[0];
    } else if (a.g64 && qmat_g64(E.v2) && E.v2.bits == 2) {
      qrow_dot_g64<2, 1>(E.v2, j, xp, 1, av);
      acc = av[0];
    } else if (a.g64 && qmat_g64(E.v2) && E.v2.bits == 4) {
      qrow_dot_g64<4, 1>(E.v2, j, xp, 1, av);
      acc = av[0];
    } else {
      for (int k = lane; k < E.v2.cols; k += 32) acc = fmaf(qmat_elem(E.v2, j, k), ap[k], acc);
      acc = warp_sum(acc);
    }
  }
  if (lane == 0) a.t[t_base(a, p, 2) + j] = acc;
}

__global__ void __launch_bounds__(256) down_generic_kernel(ExpertArgs a) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int n_active = a.plan.counts[0];
  const int64_t total = static_cast<int64_t>(n_active) * a.hidden;
  for (int64_t task = gw; task < total; task += nwarps) {
    const int ai = static_cast<int>(task / a.hidden);
    const int r = static_cast<int>(task - static_cast<int64_t>(ai) * a.hidden);
    const lrc_expert& E = a.experts[a.plan.active[ai]];
    const int off = a.plan.active_off[ai], cnt = a.plan.active_cnt[ai];
    for (int c0 = 0; c0 < cnt; c0 += kChunk) {
      const int nch = min(kChunk, cnt - c0);
      float acc[kChunk];
      const float* ap[kChunk];
#pragma unroll
      for (int i = 0; i < kChunk; ++i) {
        acc[i] = 0.0f;
        int p = a.plan.pair_list[off + c0 + min(i, nch - 1)];
        ap[i] = a.a32 + static_cast<int64_t>(p) * a.ffn;
      }
      if (a.g64 && E.w2.bits == 2) {
        gdot<2>(E.w2, r, ap, nch, acc);
      } else if (a.g64 && E.w2.bits == 3) {
        gdot<3>(E.w2, r, ap, nch, acc);
      } else if (a.g64 && E.w2.bits == 4) {
        gdot<4>(E.w2, r, ap, nch, acc);
      } else {
        for (int k = lane; k < a.ffn; k += 32) {
          const float wv = qmat_elem(E.w2, r, k);
#pragma unroll
          for (int i = 0; i < kChunk; ++i)
            if (i < nch) acc[i] = fmaf(wv, ap[i][k], acc[i]);
        }
#pragma unroll
        for (int i = 0; i < kChunk; ++i) acc[i] = warp_sum(acc[i]);
      }
#pragma unroll
      for (int i = 0; i < kChunk; ++i) {
        if (i < nch) {
          float v = acc[i];
          const int p = a.plan.pair_list[off + c0 + i];
          const int slot = a.plan.pair_comp[p];
          if (slot >= 0 && qmat_present(E.u2))
            v += lr_up_dot(E.u2, r, a.t + t_base(a, p, 2));
          if (lane == 0)
            atomicAdd(&a.y[static_cast<int64_t>(a.plan.pair_token[p]) * a.hidden + r],
                      a.plan.pair_w[p] * v);
        }
      }
    }
  }
}

// ------------------------------------------------- dense fp64 (reference) ---
__global__ void dense_up_f64_kernel(const double* w1, const double* w3, int hidden, int ffn,
                                    const double* x, int64_t B, double* act) {
  const int lane = threadIdx.x & 31;
  const int64_t task = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  if (task >= B * ffn) return;
  const int64_t b = task / ffn;
  const int f = static_cast<int>(task - b * ffn);
  double h1 = 0.0, h3 = 0.0;
  for (int k = lane; k < hidden; k += 32) {
    const double xv = x[b * hidden + k];
    h1 = fma(w1[static_cast<int64_t>(f) * hidden + k], xv, h1);
    h3 = fma(w3[static_cast<int64_t>(f) * hidden + k], xv, h3);
  }
  h1 = warp_sum_d(h1);
  h3 = warp_sum_d(h3);
  if (lane == 0) act[task] = h1 / (1.0 + exp(-h1)) * h3;
}

__global__ void dense_down_f64_kernel(const double* w2, int hidden, int ffn, const double* act,
                                      const double* mix, int64_t B, double* y) {
  const int lane = threadIdx.x & 31;
  const int64_t task = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  if (task >= B * hidden) return;
  const int64_t b = task / hidden;
  const int r = static_cast<int>(task - b * hidden);
  double acc = 0.0;
  for (int k = lane; k < ffn; k += 32)
    acc = fma(w2[static_cast<int64_t>(r) * ffn + k], act[b * ffn + k], acc);
  acc = warp_sum_d(acc);
  if (lane == 0) y[task] += (mix ? mix[b] : 1.0) * acc;
}

lrc_status launch_lr_down(const ExpertArgs& a, int np_bound, cudaStream_t st) {
  if (a.maxr == 0) return LRC_OK;
  int tasks = np_bound * 2 * a.maxr;
  static bool carve = false;
  if (!carve && getenv("LRC_NO_CARVEOUT") == nullptr) {  // match the tiled kernels' L1/smem split
    LRC_CUDA_TRY(cudaFuncSetAttribute(lr_down_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    carve = true;
  }
  lr_down_kernel<<<(tasks + 7) / 8, 256, 0, st>>>(a);
  LRC_CHECK_LAUNCH();
  return LRC_OK;
}

}  // namespace lrc

namespace lrc {
// ------------------------------------------------- GPU-driven expert paging ---
// Offload mode (north-star 4) without a host round trip: after the router's
// plan, one launch copies every active expert's block from device-mapped
// pinned host memory into slot a (a = its active index) with 16-byte
// streaming loads across all SMs (8 in flight per thread), then repoints the
// expert's descriptor and its ActiveRec at the slot.  Section order of a block
// (offsets in PagerArgs.off, -1 absent):
// up tiles, down tiles, up LR tiles, down LR tiles, V1 packed/scales/zeros,
// V3 packed/scales/zeros.
struct PagerArgs {
  const uint8_t* const* host;  // [E+S] device-visible block pointers
  int64_t off[10];
  int64_t bytes;               // block bytes (multiple of 16)
  uint8_t* slots;
  int64_t slot_bytes;
  lrc_expert* experts;  // device table
  PlanArgs plan;
  // budgeted LRU over slots shared by every layer (lrc_pager_cache); null:
  // slot a = active index a (no cross-step cache)
  int64_t* owner;            // [n_cache] (layer key << 20 | expert) or -1
  unsigned long long* stamp;  // [n_cache] last use: clock << 12 | order within the step
  unsigned long long* clock;  // step counter
  unsigned long long* stats;  // [2] hits, misses
  int n_cache;
  int layer_key;
  int* slot_of;              // [E+S] per active index: its slot
  int* miss;                 // [E+S] per active index: 1 = copy the block
};

// point expert e's descriptor and active record a at slot s
__device__ void pager_repoint(const PagerArgs& g, int a, int e, int s) {
  const uint8_t* base = g.slots + static_cast<int64_t>(s) * g.slot_bytes;
  auto at = [&](int k) -> const uint8_t* { return g.off[k] >= 0 ? base + g.off[k] : nullptr; };
  lrc_expert d = g.experts[e];
  d.up_tiles = at(0);
  d.down_tiles = at(1);
  d.up_lr_tiles = at(2);
  d.down_lr_tiles = at(3);
  if (g.off[4] >= 0) {
    d.v1.packed = at(4);
    d.v1.scales = reinterpret_cast<const uint16_t*>(at(5));
    d.v1.zeros = reinterpret_cast<const uint16_t*>(at(6));
  }
  if (g.off[7] >= 0) {
    d.v3.packed = at(7);
    d.v3.scales = reinterpret_cast<const uint16_t*>(at(8));
    d.v3.zeros = reinterpret_cast<const uint16_t*>(at(9));
  }
  g.experts[e] = d;
  if (g.plan.arec != nullptr) {
    ActiveRec& R = g.plan.arec[a];
    R.up_tiles = d.up_tiles;
    R.down_tiles = d.down_tiles;
    R.up_lr_tiles = d.up_lr_tiles;
    R.down_lr_tiles = d.down_lr_tiles;
  }
}

// LRU slot assignment for one layer step (one warp).  The step's experts are
// looked up in the order of their first (token, rank) pair -- the reference
// cost model's order (ref/simulate.py:219-227): a hit refreshes its slot; a
// miss takes the least recently used slot not already touched in this step.
__global__ void __launch_bounds__(32) pager_assign_kernel(const PagerArgs g) {
  const int lane = threadIdx.x;
  const int na = g.plan.counts[0];
  const unsigned long long clk = *g.clock + 1;
  // order of the active experts by their first pair (selection sort, na <= 64)
  __shared__ int s_first[LRC_MAX_EXPERTS], s_order[LRC_MAX_EXPERTS];
  for (int a = lane; a < na; a += 32) s_first[a] = g.plan.pair_list[g.plan.active_off[a]];
  __syncwarp();
  if (lane == 0) {
    for (int i = 0; i < na; ++i) s_order[i] = i;
    for (int i = 0; i < na; ++i)
      for (int j = i + 1; j < na; ++j)
        if (s_first[s_order[j]] < s_first[s_order[i]]) {
          const int t = s_order[i];
          s_order[i] = s_order[j];
          s_order[j] = t;
        }
  }
  __syncwarp();
  unsigned long long hits = 0, misses = 0;
  for (int i = 0; i < na; ++i) {
    const int a = s_order[i], e = g.plan.active[a];
    const int64_t key = (static_cast<int64_t>(g.layer_key) << 20) | e;
    const unsigned long long now = (clk << 12) | static_cast<unsigned long long>(min(i, 4095));
    int found = -1;
    for (int s = lane; s < g.n_cache; s += 32)
      if (g.owner[s] == key) found = s;
    for (int o = 16; o > 0; o >>= 1) found = max(found, __shfl_xor_sync(0xffffffffu, found, o));
    int slot = found;
    if (slot < 0) {  // victim: min stamp among slots not touched this step (ties -> lower slot)
      unsigned long long best = ~0ull;
      int bs = 0x7fffffff;
      for (int s = lane; s < g.n_cache; s += 32) {
        const unsigned long long st = g.stamp[s];
        if ((st >> 12) != clk && (st < best || (st == best && s < bs))) {
          best = st;
          bs = s;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int os = __shfl_xor_sync(0xffffffffu, bs, o);
        if (ob < best || (ob == best && os < bs)) {
          best = ob;
          bs = os;
        }
      }
      slot = bs;
    }
    if (lane == 0) {
      g.owner[slot] = key;
      g.stamp[slot] = now;
      g.slot_of[a] = slot;
      g.miss[a] = found < 0 ? 1 : 0;
      pager_repoint(g, a, e, slot);
    }
    __syncwarp();
    if (found < 0) ++misses;
    else ++hits;
  }
  if (lane == 0) {
    *g.clock = clk;
    g.stats[0] += hits;
    g.stats[1] += misses;
  }
}

__global__ void __launch_bounds__(256) pager_kernel(const PagerArgs g) {
  const int a = blockIdx.y;
  if (a >= g.plan.counts[0]) return;
  const int e = g.plan.active[a];
  if (g.owner != nullptr && !g.miss[a]) return;  // resident (cache hit): nothing moves
  const int slot = g.owner != nullptr ? g.slot_of[a] : a;
  const uint4* src = reinterpret_cast<const uint4*>(g.host[e]);
  uint4* dst = reinterpret_cast<uint4*>(g.slots + static_cast<int64_t>(slot) * g.slot_bytes);
  const int64_t n = g.bytes / 16, stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n; i += 8 * stride) {  // 8 loads in flight per thread (host-link latency)
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) __stcs(dst + i + u * stride, v[u]);
  }
  for (; i < n; i += stride) dst[i] = src[i];
  if (g.owner == nullptr && blockIdx.x == 0 && threadIdx.x == 0) pager_repoint(g, a, e, a);
}
}  // namespace lrc

// =========================================================== layer object ===
using namespace lrc;

constexpr int kStageRing = 64;
struct StageEntry {
  lrc_expert e;
  uint8_t has_comp;
};

struct lrc_layer {
  int hidden = 0, ffn = 0, E = 0, S = 0, max_tokens = 0, k_max = 0, maxr = 0;
  int num_sms = 148;
  bool tiled = false;
  bool prefill_ok = false;
  int prefill_bits = 2;  // code width of the prefill packs  // tcgen05 prefill GEMM eligible (2-bit gs64 reference-layout weights)
  uint16_t* lrp = nullptr;     // per-expert bf16 LR packs for the prefill path (built lazily)
  uint8_t* ppk = nullptr;      // per-expert prefill packs of the weight codes (built lazily)
  std::vector<uint8_t> lrp_dirty;  // per expert: packs stale (expert replaced)
  uint16_t* tb = nullptr;      // prefill V.x rows [max_pairs][tb_width] bf16
  bool pager = false;          // GPU-driven expert paging (lrc_layer_set_pager)
  PagerArgs pg{};
  const uint8_t** pg_host = nullptr;  // device copy of the block pointers
  int pg_slots = 0;
  int* pg_scratch = nullptr;  // [2][E+S] slot_of, miss (cache mode)
  int* plan_blk = nullptr;     // parallel plan: per-chunk histograms
  uint32_t* plan_cmask = nullptr;
  int* plan_ticket = nullptr;
  int64_t prefill_min = [] {
    const char* v = getenv("LRC_PREFILL_MIN");
    return v ? static_cast<int64_t>(atoll(v)) : static_cast<int64_t>(128);
  }();
  int last_launches = 0;
  const double* gate_t = nullptr;
  std::vector<lrc_expert> host_experts;
  lrc_expert* d_experts = nullptr;
  StageEntry* h_stage = nullptr;  // pinned ring for stream-ordered descriptor updates
  int stage_next = 0;
  cudaEvent_t stage_ev[kStageRing] = {};
  uint8_t stage_used[kStageRing] = {};
  // workspace
  void* ws = nullptr;
  size_t ws_bytes = 0;
  PlanArgs plan{};
  int32_t* topk_idx = nullptr;
  float* topk_w = nullptr;
  float* t = nullptr;
  float* a32 = nullptr;
  uint16_t* a16 = nullptr;
  int max_pairs = 0;
  double* logits = nullptr;  // router scratch [max_tokens][E]
  int* tile_ticket = nullptr;
  int lr_up_max = 0, lr_down_max = 0;  // largest per-tile low-rank slot (bytes)
  bool pdl = getenv("LRC_NO_PDL") == nullptr;  // programmatic dependent launch
  // host-buffer staging + phase timing
  uint16_t* x_stage = nullptr;
  float* y_stage = nullptr;
  bool profiling = false;
  cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  // tensor-core decode engine (tcd.cu): batches of B <= tcd_max tokens
  int tcd_max = [] {
    const char* v = getenv("LRC_TCD_MAX");
    return v ? atoi(v) : -1;  // -1: auto (on where the tiled kernels do not apply, e.g. 3-bit)
  }();
  bool tcd_ok = false;
  bool g64_ok = false;  // generic path: group-vectorised decode (qrow_dot_g64) for every expert
  int tcd_bits = 2, tcd_fbits = 3;
  std::vector<uint8_t> tcd_dirty;  // per expert: pack stale
  bool tcd_table_dirty = true;
  uint8_t* tcd_packs = nullptr;     // [NE][up | down]
  int64_t tcd_up_bytes = 0, tcd_down_bytes = 0, tcd_lru_bytes = 0, tcd_lrd_bytes = 0;
  std::vector<tcd::Expert> tcd_host;
  tcd::Expert* d_tcd = nullptr;
  float* gate32 = nullptr;          // (E, hidden) fp32 copy of gate_t (fused routing)
  void* tcd_ws = nullptr;
  tcd::Args tcd_args{};
};

static bool has_comp(const lrc_expert& e) {
  auto pres = [](const lrc_qmat& m) { return m.packed != nullptr || m.dense != nullptr; };
  return pres(e.u1) || pres(e.u2) || pres(e.u3);
}

static int rank_of(const lrc_qmat& u) {
  return (u.packed != nullptr || u.dense != nullptr) ? u.cols : 0;
}

static lrc_status validate_expert(const lrc_expert& e, int hidden, int ffn) {
  auto chk = [](const lrc_qmat& m, int rows, int cols, const char* nm) -> lrc_status {
    if (m.packed == nullptr && m.dense == nullptr)
      return fail(LRC_ERR_MISSING, std::string("no artifact for projection ") + nm);
    if (m.rows != rows || m.cols != cols)
      return fail(LRC_ERR_INVALID, std::string("shape mismatch for ") + nm);
    if (m.dense == nullptr && (m.bits < 1 || m.bits > 8 || m.group_size < 1 || !m.scales || !m.zeros))
      return fail(LRC_ERR_INVALID, std::string("bad quantization params for ") + nm);
    return LRC_OK;
  };
  lrc_status s;
  if ((s = chk(e.w1, ffn, hidden, "w1")) != LRC_OK) return s;
  if ((s = chk(e.w3, ffn, hidden, "w3")) != LRC_OK) return s;
  if ((s = chk(e.w2, hidden, ffn, "w2")) != LRC_OK) return s;
  const lrc_qmat* us[3] = {&e.u1, &e.u3, &e.u2};
  const lrc_qmat* vs[3] = {&e.v1, &e.v3, &e.v2};
  const int rows[3] = {ffn, ffn, hidden}, cols[3] = {hidden, hidden, ffn};
  for (int i = 0; i < 3; ++i) {
    int r = rank_of(*us[i]);
    if (r == 0) continue;
    if (us[i]->rows != rows[i] || vs[i]->rows != r || vs[i]->cols != cols[i] ||
        (vs[i]->packed == nullptr && vs[i]->dense == nullptr))
      return fail(LRC_ERR_INVALID, "compensator factor shapes incompatible with the projection");
  }
  return LRC_OK;
}

// The tiled path needs T2 weight tiles for every expert and, for experts with
// compensators, quantized factors re-laid out as LR tiles (raw fp32 factors ->
// generic path).  Also records the largest LR slot the kernels must stage.
static void refresh_tiled(lrc_layer* L) {
  bool ok = (L->hidden % 32) == 0;  // W2 streams as two 16-row-tiled halves
  L->lr_up_max = L->lr_down_max = 0;
  for (auto& e : L->host_experts) {
    ok = ok && e.up_tiles != nullptr && e.down_tiles != nullptr;
    if (!has_comp(e)) continue;
    const lrc_qmat* fs[6] = {&e.u1, &e.v1, &e.u3, &e.v3, &e.u2, &e.v2};
    for (auto f : fs) ok = ok && f->dense == nullptr;
    const LrLayout lay = lr_layout(e);
    ok = ok && (lay.up_total == 0 || e.up_lr_tiles != nullptr);
    ok = ok && (lay.down_total == 0 || e.down_lr_tiles != nullptr);
    L->lr_up_max = std::max(L->lr_up_max, lay.up_total);
    L->lr_down_max = std::max(L->lr_down_max, lay.down_total);
  }
  L->tiled = ok;
  const int old_pbits = L->prefill_bits;
  L->prefill_ok = prefill_eligible(L->host_experts.data(), static_cast<int>(L->host_experts.size()),
                                   L->hidden, L->ffn, L->maxr, &L->prefill_bits);
  if (L->prefill_bits != old_pbits && L->ppk != nullptr) {  // pack size follows the code width
    cudaFree(L->ppk);
    L->ppk = nullptr;
    std::fill(L->lrp_dirty.begin(), L->lrp_dirty.end(), 1);
  }
  L->g64_ok = (L->hidden % 64) == 0 && (L->ffn % 64) == 0;
  for (auto& e : L->host_experts) L->g64_ok = L->g64_ok && qmat_g64(e.w1) && qmat_g64(e.w3) && qmat_g64(e.w2);
  L->tcd_ok = L->maxr <= tcd::kRMax && tcd::eligible(L->host_experts.data(), static_cast<int>(L->host_experts.size()),
                                                      L->hidden, L->ffn, &L->tcd_bits, &L->tcd_fbits);
}

static lrc_status alloc_workspace(lrc_layer* L) {
  const int NE = L->E + L->S;
  const int NP = L->max_tokens * (L->k_max + L->S);
  L->max_pairs = NP;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  size_t o_ticket = take(16), o_counts = take(16), o_hc = take(NE);
  size_t o_pe = take(NP * 4), o_pw = take(NP * 4), o_pt = take(NP * 4), o_pc = take(NP * 4);
  size_t o_pl = take(NP * 4), o_cl = take(NP * 4);
  size_t o_act = take(NE * 4), o_aoff = take(NE * 4), o_acnt = take(NE * 4);
  size_t o_arec = take(NE * sizeof(ActiveRec));
  size_t o_tki = take(size_t(L->max_tokens) * L->k_max * 4);
  size_t o_tkw = take(size_t(L->max_tokens) * L->k_max * 4);
  size_t o_t = take(size_t(L->max_tokens) * NE * 3 * std::max(L->maxr, 1) * 4);
  size_t o_a32 = take(size_t(NP) * L->ffn * 4);
  size_t o_a16 = take(size_t(NP) * L->ffn * 2 + 64);
  size_t o_xs = take(size_t(L->max_tokens) * L->hidden * 2);
  size_t o_ys = take(size_t(L->max_tokens) * L->hidden * 4);
  size_t o_lg = take(size_t(L->max_tokens) * L->E * 8);
  size_t o_tt = take(size_t(route_tiles(L->max_tokens)) * 4 + 16);
  size_t o_tb = take(size_t(NP) * prefill_tb_width(L->maxr) * 2 + 16);
  size_t o_pb = take(size_t(plan_parallel_blocks(NP) + 1) * (NE + 1) * 4);
  size_t o_pcm = take(size_t(NE) * 4 + 16);
  size_t o_ptk = take(16);
  LRC_CUDA_TRY(cudaMalloc(&L->ws, off));
  LRC_CUDA_TRY(cudaMemset(L->ws, 0, off));
  L->ws_bytes = off;
  char* base = static_cast<char*>(L->ws);
  PlanArgs& p = L->plan;
  p.ticket = reinterpret_cast<int*>(base + o_ticket);
  p.counts = reinterpret_cast<int*>(base + o_counts);
  p.has_comp = reinterpret_cast<uint8_t*>(base + o_hc);
  p.pair_expert = reinterpret_cast<int*>(base + o_pe);
  p.pair_w = reinterpret_cast<float*>(base + o_pw);
  p.pair_token = reinterpret_cast<int*>(base + o_pt);
  p.pair_comp = reinterpret_cast<int*>(base + o_pc);
  p.pair_list = reinterpret_cast<int*>(base + o_pl);
  p.comp_list = reinterpret_cast<int*>(base + o_cl);
  p.active = reinterpret_cast<int*>(base + o_act);
  p.active_off = reinterpret_cast<int*>(base + o_aoff);
  p.active_cnt = reinterpret_cast<int*>(base + o_acnt);
  p.arec = reinterpret_cast<ActiveRec*>(base + o_arec);
  p.experts = L->d_experts;
  p.num_experts = L->E;
  p.num_shared = L->S;
  L->topk_idx = reinterpret_cast<int32_t*>(base + o_tki);
  L->topk_w = reinterpret_cast<float*>(base + o_tkw);
  L->t = reinterpret_cast<float*>(base + o_t);
  L->a32 = reinterpret_cast<float*>(base + o_a32);
  L->a16 = reinterpret_cast<uint16_t*>(base + o_a16);
  L->x_stage = reinterpret_cast<uint16_t*>(base + o_xs);
  L->y_stage = reinterpret_cast<float*>(base + o_ys);
  L->logits = reinterpret_cast<double*>(base + o_lg);
  L->tile_ticket = reinterpret_cast<int*>(base + o_tt);
  L->tb = reinterpret_cast<uint16_t*>(base + o_tb);
  L->plan_blk = reinterpret_cast<int*>(base + o_pb);
  L->plan_cmask = reinterpret_cast<uint32_t*>(base + o_pcm);
  L->plan_ticket = reinterpret_cast<int*>(base + o_ptk);
  L->lrp_dirty.assign(NE, 1);  // packs: built before the first prefill call (and after expert updates)
  if (L->maxr) {
    const size_t per = static_cast<size_t>(prefill_lr_pack_elems(L->hidden, L->ffn, L->maxr));
    LRC_CUDA_TRY(cudaMalloc(&L->lrp, per * NE * 2));
  }
  for (auto& e : L->ev) LRC_CUDA_TRY(cudaEventCreate(&e));
  std::vector<uint8_t> hc(NE);
  for (int e = 0; e < NE; ++e) hc[e] = has_comp(L->host_experts[e]) ? 1 : 0;
  LRC_CUDA_TRY(cudaMemcpy(const_cast<uint8_t*>(p.has_comp), hc.data(), NE, cudaMemcpyHostToDevice));
  return LRC_OK;
}

extern "C" lrc_status lrc_layer_create(const double* gate_t, int hidden, int ffn, int num_experts,
                                       int num_shared, const lrc_expert* experts, int max_tokens,
                                       int top_k, lrc_layer** out) {
  if (!out || !gate_t || !experts) return fail(LRC_ERR_INVALID, "layer_create: null argument");
  if (hidden <= 0 || ffn <= 0 || num_experts <= 0 || num_shared < 0 || max_tokens <= 0)
    return fail(LRC_ERR_INVALID, "layer_create: bad dimensions");
  if (num_experts + num_shared > LRC_MAX_EXPERTS)
    return fail(LRC_ERR_UNSUPPORTED, "layer_create: at most 256 experts");
  if (top_k < 0 || top_k > num_experts) return fail(LRC_ERR_INVALID, "top_k exceeds experts");
  auto* L = new lrc_layer();
  L->hidden = hidden;
  L->ffn = ffn;
  L->E = num_experts;
  L->S = num_shared;
  L->max_tokens = max_tokens;
  L->k_max = std::max(top_k, 1);
  L->gate_t = gate_t;
  L->host_experts.assign(experts, experts + num_experts + num_shared);
  for (auto& e : L->host_experts) {
    lrc_status s = validate_expert(e, hidden, ffn);
    if (s != LRC_OK) {
      delete L;
      return s;
    }
    L->maxr = std::max({L->maxr, rank_of(e.u1), rank_of(e.u2), rank_of(e.u3)});
  }
  refresh_tiled(L);
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&L->num_sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t bytes = sizeof(lrc_expert) * L->host_experts.size();
  if (cudaMalloc(&L->d_experts, bytes) != cudaSuccess ||
      cudaMemcpy(L->d_experts, L->host_experts.data(), bytes, cudaMemcpyHostToDevice) != cudaSuccess) {
    delete L;
    return fail(LRC_ERR_CUDA, "layer_create: expert table upload failed");
  }
  lrc_status s = alloc_workspace(L);
  if (s != LRC_OK) {
    cudaFree(L->d_experts);
    delete L;
    return s;
  }
  *out = L;
  return LRC_OK;
}

extern "C" void lrc_layer_destroy(lrc_layer* L) {
  if (!L) return;
  cudaFree(L->d_experts);
  if (L->h_stage) cudaFreeHost(L->h_stage);
  for (auto& ev : L->stage_ev)
    if (ev) cudaEventDestroy(ev);
  cudaFree(L->ws);
  cudaFree(L->lrp);
  cudaFree(L->pg_host);
  cudaFree(L->pg_scratch);
  cudaFree(L->ppk);
  cudaFree(L->tcd_packs);
  cudaFree(L->d_tcd);
  cudaFree(L->gate32);
  cudaFree(L->tcd_ws);
  for (auto& e : L->ev)
    if (e) cudaEventDestroy(e);
  delete L;
}

extern "C" lrc_status lrc_layer_set_expert(lrc_layer* L, int expert_id, const lrc_expert* e) {
  if (!L || !e || expert_id < 0 || expert_id >= L->E + L->S)
    return fail(LRC_ERR_INVALID, "set_expert: bad id");
  lrc_status s = validate_expert(*e, L->hidden, L->ffn);
  if (s != LRC_OK) return s;
  if (std::max({rank_of(e->u1), rank_of(e->u2), rank_of(e->u3)}) > L->maxr)
    return fail(LRC_ERR_UNSUPPORTED, "set_expert: rank above the layer's workspace rank");
  L->host_experts[expert_id] = *e;
  LRC_CUDA_TRY(cudaMemcpy(L->d_experts + expert_id, e, sizeof(lrc_expert), cudaMemcpyHostToDevice));
  if (!L->lrp_dirty.empty()) L->lrp_dirty[expert_id] = 1;
  if (!L->tcd_dirty.empty()) L->tcd_dirty[expert_id] = 1;
  L->tcd_table_dirty = true;
  {
    const uint8_t hc = has_comp(*e) ? 1 : 0;  // top-n decisions of the tiled/prefill plan
    LRC_CUDA_TRY(cudaMemcpy(const_cast<uint8_t*>(L->plan.has_comp) + expert_id, &hc, 1, cudaMemcpyHostToDevice));
  }
  refresh_tiled(L);
  return LRC_OK;
}

// Stream-ordered variant: the device descriptor is written by an async copy on
// `stream` from a pinned staging ring (kStageRing entries per expert slot), so
// it does not serialise against other streams (the offload engine's copies).
// The host-side state (validation, tiled-path eligibility) updates immediately.
extern "C" lrc_status lrc_layer_set_expert_async(lrc_layer* L, int expert_id, const lrc_expert* e,
                                                 void* stream) {
  if (!L || !e || expert_id < 0 || expert_id >= L->E + L->S)
    return fail(LRC_ERR_INVALID, "set_expert: bad id");
  lrc_status s = validate_expert(*e, L->hidden, L->ffn);
  if (s != LRC_OK) return s;
  if (std::max({rank_of(e->u1), rank_of(e->u2), rank_of(e->u3)}) > L->maxr)
    return fail(LRC_ERR_UNSUPPORTED, "set_expert: rank above the layer's workspace rank");
  if (L->h_stage == nullptr) {
    // each ring entry: the descriptor followed by the plan's has_comp byte
    LRC_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&L->h_stage), sizeof(StageEntry) * kStageRing,
                               cudaHostAllocDefault));
    for (auto& ev : L->stage_ev) LRC_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  const int k = L->stage_next++ % kStageRing;
  // the entry's previous async copies must have read it before it is rewritten
  if (L->stage_used[k]) LRC_CUDA_TRY(cudaEventSynchronize(L->stage_ev[k]));
  StageEntry* slot = L->h_stage + k;
  slot->e = *e;
  slot->has_comp = has_comp(*e) ? 1 : 0;
  L->host_experts[expert_id] = *e;
  cudaStream_t st = as_stream(stream);
  LRC_CUDA_TRY(cudaMemcpyAsync(L->d_experts + expert_id, &slot->e, sizeof(lrc_expert), cudaMemcpyHostToDevice, st));
  LRC_CUDA_TRY(cudaMemcpyAsync(const_cast<uint8_t*>(L->plan.has_comp) + expert_id, &slot->has_comp, 1,
                               cudaMemcpyHostToDevice, st));
  LRC_CUDA_TRY(cudaEventRecord(L->stage_ev[k], st));
  L->stage_used[k] = 1;
  if (!L->lrp_dirty.empty()) L->lrp_dirty[expert_id] = 1;
  if (!L->tcd_dirty.empty()) L->tcd_dirty[expert_id] = 1;
  L->tcd_table_dirty = true;
  refresh_tiled(L);
  return LRC_OK;
}

extern "C" lrc_status lrc_layer_set_pager(lrc_layer* L, const void* const* host_blocks, const int64_t* offsets,
                                          int64_t block_bytes, uint8_t* slots, int n_slots, int64_t slot_bytes) {
  if (!L || !host_blocks || !offsets || !slots || n_slots <= 0 || block_bytes <= 0 || block_bytes % 16 ||
      slot_bytes < block_bytes || slot_bytes % 16)
    return fail(LRC_ERR_INVALID, "set_pager: bad arguments");
  if (!L->tiled) return fail(LRC_ERR_UNSUPPORTED, "set_pager: needs the tiled decode layout");
  const int NE = L->E + L->S;
  if (L->pg_host == nullptr) LRC_CUDA_TRY(cudaMalloc(&L->pg_host, sizeof(uint8_t*) * NE));
  LRC_CUDA_TRY(cudaMemcpy(L->pg_host, host_blocks, sizeof(uint8_t*) * NE, cudaMemcpyHostToDevice));
  PagerArgs& g = L->pg;
  g.host = L->pg_host;
  for (int k = 0; k < 10; ++k) g.off[k] = offsets[k];
  g.bytes = block_bytes;
  g.slots = slots;
  g.slot_bytes = slot_bytes;
  g.experts = L->d_experts;
  L->pg_slots = n_slots;
  L->pager = true;
  return LRC_OK;
}

struct lrc_pager_cache {
  int n = 0;
  int64_t* owner = nullptr;
  unsigned long long* stamp = nullptr;
  unsigned long long* clock = nullptr;  // [0] clock, [1] hits, [2] misses
};

extern "C" lrc_status lrc_pager_cache_create(int n_slots, lrc_pager_cache** out) {
  if (!out || n_slots <= 0) return fail(LRC_ERR_INVALID, "pager_cache_create: bad arguments");
  auto* c = new lrc_pager_cache();
  c->n = n_slots;
  if (cudaMalloc(&c->owner, sizeof(int64_t) * n_slots) != cudaSuccess ||
      cudaMalloc(&c->stamp, sizeof(unsigned long long) * n_slots) != cudaSuccess ||
      cudaMalloc(&c->clock, sizeof(unsigned long long) * 3) != cudaSuccess) {
    cudaFree(c->owner);
    cudaFree(c->stamp);
    delete c;
    return fail(LRC_ERR_CUDA, "pager_cache_create: cudaMalloc");
  }
  cudaMemset(c->owner, 0xff, sizeof(int64_t) * n_slots);  // -1: empty
  cudaMemset(c->stamp, 0, sizeof(unsigned long long) * n_slots);
  cudaMemset(c->clock, 0, sizeof(unsigned long long) * 3);
  *out = c;
  return LRC_OK;
}

extern "C" void lrc_pager_cache_destroy(lrc_pager_cache* c) {
  if (!c) return;
  cudaFree(c->owner);
  cudaFree(c->stamp);
  cudaFree(c->clock);
  delete c;
}

extern "C" lrc_status lrc_pager_cache_stats(lrc_pager_cache* c, int64_t* hits_misses) {
  if (!c || !hits_misses) return fail(LRC_ERR_INVALID, "pager_cache_stats: null argument");
  unsigned long long h[3];
  LRC_CUDA_TRY(cudaMemcpy(h, c->clock, sizeof(h), cudaMemcpyDeviceToHost));
  hits_misses[0] = static_cast<int64_t>(h[1]);
  hits_misses[1] = static_cast<int64_t>(h[2]);
  return LRC_OK;
}

extern "C" lrc_status lrc_layer_set_pager_cache(lrc_layer* L, lrc_pager_cache* c, int layer_key) {
  if (!L || !c || layer_key < 0) return fail(LRC_ERR_INVALID, "set_pager_cache: bad arguments");
  if (!L->pager) return fail(LRC_ERR_INVALID, "set_pager_cache: call lrc_layer_set_pager first");
  if (c->n != L->pg_slots) return fail(LRC_ERR_INVALID, "set_pager_cache: cache size != the pager's slot count");
  const int NE = L->E + L->S;
  if (L->pg_scratch == nullptr) LRC_CUDA_TRY(cudaMalloc(&L->pg_scratch, sizeof(int) * 2 * NE));
  PagerArgs& g = L->pg;
  g.owner = c->owner;
  g.stamp = c->stamp;
  g.clock = c->clock;
  g.stats = c->clock + 1;
  g.n_cache = c->n;
  g.layer_key = layer_key;
  g.slot_of = L->pg_scratch;
  g.miss = L->pg_scratch + NE;
  return LRC_OK;
}

extern "C" lrc_status lrc_layer_set_prefill_min(lrc_layer* L, int64_t min_tokens) {
  if (!L) return fail(LRC_ERR_INVALID, "set_prefill_min: null layer");
  L->prefill_min = min_tokens;
  return LRC_OK;
}

extern "C" int lrc_layer_prefill_eligible(const lrc_layer* L) { return L && L->prefill_ok ? 1 : 0; }

extern "C" int lrc_layer_last_launches(const lrc_layer* L) { return L ? L->last_launches : 0; }

// ------------------------------------------------ tcd engine plumbing ----
__global__ void gate32_kernel(const double* g, float* o, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    o[i] = static_cast<float>(g[i]);
}

// L2 norm of each gate row (E, d), rounded up: the routing kernel's fp32 error bound
__global__ void gate_norm_kernel(const double* g, int d, float* out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const double v = g[static_cast<int64_t>(blockIdx.x) * d + i];
    s += v * v;
  }
  s = warp_sum_d(s);
  __shared__ double part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += part[w];
    out[blockIdx.x] = static_cast<float>(sqrt(t) * 1.001);
  }
}

static int64_t tcd_stride(const lrc_layer* L) {  // bytes per expert: codes up|down, LR up|down
  return L->tcd_up_bytes + L->tcd_down_bytes + L->tcd_lru_bytes + L->tcd_lrd_bytes;
}

static bool tcd_fused_routing(const lrc_layer* L) {
  return L->E <= tcd::kFuseMaxE && static_cast<int64_t>(L->E) * L->hidden * 4 <= 160 * 1024;
}

// (Re)build the tcd packs of changed experts, the device expert table, the
// fp32 gate and the workspace.  Not graph-capturable (host copies): the first
// forward after a change runs it, later forwards only check flags.
static lrc_status tcd_prepare(lrc_layer* L, cudaStream_t st) {
  const int NE = L->E + L->S;
  const int T0 = L->ffn / 128;
  if (L->tcd_packs == nullptr) {
    L->tcd_up_bytes = tcd::pack_bytes(L->ffn, L->hidden, 2, L->tcd_bits);
    L->tcd_down_bytes = tcd::pack_bytes(L->hidden, L->ffn, 1, L->tcd_bits);
    if (L->maxr > 0) {
      L->tcd_lru_bytes = static_cast<int64_t>(L->ffn / 128) * tcd::lr_up_tile_bytes(L->maxr);
      L->tcd_lrd_bytes = static_cast<int64_t>(L->hidden / 128) * tcd::lr_down_tile_bytes(L->maxr);
    }
    LRC_CUDA_TRY(cudaMalloc(&L->tcd_packs, static_cast<size_t>(tcd_stride(L)) * NE));
    L->tcd_dirty.assign(NE, 1);
    L->tcd_host.assign(NE, tcd::Expert{});
    LRC_CUDA_TRY(cudaMalloc(&L->d_tcd, sizeof(tcd::Expert) * NE));
    const int64_t ng = static_cast<int64_t>(L->E) * L->hidden;
    LRC_CUDA_TRY(cudaMalloc(&L->gate32, sizeof(float) * (ng + L->E)));
    gate32_kernel<<<148, 256, 0, st>>>(L->gate_t, L->gate32, ng);
    LRC_CHECK_LAUNCH();
    gate_norm_kernel<<<L->E, 256, 0, st>>>(L->gate_t, L->hidden, L->gate32 + ng);
    LRC_CHECK_LAUNCH();
    // workspace
    tcd::Args& a = L->tcd_args;
    a.max_act = std::min({NE, tcd::kMaxTok * L->k_max + L->S, tcd::kMaxAct});
    size_t off = 0;
    auto take = [&](size_t b) {
      size_t o = off;
      off += (b + 255) & ~size_t(255);
      return o;
    };
    const size_t o_gb = take(8), o_tc = take(2 * tcd::kMaxP * 4), o_t13 = take(tcd::kMaxP * 2 * tcd::kRMax * 4);
    const size_t o_t2 = take(2 * tcd::kMaxP * tcd::kRMax * 4), o_xc = take(2 * 4);
    const size_t G0 = L->hidden / 64, G1 = L->ffn / 64;
    const size_t o_xd = take(tcd::kMaxTok * G0 * 512), o_xs = take(tcd::kMaxTok * G0 * 16);
    const size_t o_ad = take(tcd::kMaxP * G1 * 512), o_as = take(tcd::kMaxP * G1 * 16);
    const size_t o_ha = take(static_cast<size_t>(a.max_act) * T0 * 2 * tcd::kMaxTok * 128 * 4);
    const size_t o_hc = take(static_cast<size_t>(a.max_act) * T0 * 4);
    LRC_CUDA_TRY(cudaMalloc(&L->tcd_ws, off));
    LRC_CUDA_TRY(cudaMemsetAsync(L->tcd_ws, 0, off, st));
    char* b = static_cast<char*>(L->tcd_ws);
    a.gbar = reinterpret_cast<unsigned long long*>(b + o_gb);
    a.tcnt = reinterpret_cast<unsigned*>(b + o_tc);
    a.t13 = reinterpret_cast<float*>(b + o_t13);
    a.t2 = reinterpret_cast<float*>(b + o_t2);
    a.xcnt = reinterpret_cast<unsigned*>(b + o_xc);
    a.xdig = reinterpret_cast<uint8_t*>(b + o_xd);
    a.xsum = reinterpret_cast<float4*>(b + o_xs);
    a.adig = reinterpret_cast<uint8_t*>(b + o_ad);
    a.asum = reinterpret_cast<float4*>(b + o_as);
    a.hacc = reinterpret_cast<float*>(b + o_ha);
    a.hcnt = reinterpret_cast<unsigned*>(b + o_hc);
  }
  bool any = false;
  for (int e = 0; e < NE; ++e) {
    if (!L->tcd_dirty[e]) continue;
    const lrc_expert& x = L->host_experts[e];
    uint8_t* up = L->tcd_packs + static_cast<size_t>(tcd_stride(L)) * e;
    uint8_t* down = up + L->tcd_up_bytes;
    uint8_t* lru = down + L->tcd_down_bytes;
    uint8_t* lrd = lru + L->tcd_lru_bytes;
    const lrc_qmat upm[2] = {x.w1, x.w3};
    lrc_status s;
    if ((s = tcd::build_pack(upm, 2, L->tcd_bits, up, st)) != LRC_OK) return s;
    if ((s = tcd::build_pack(&x.w2, 1, L->tcd_bits, down, st)) != LRC_OK) return s;
    const bool comp = has_comp(x);
    if (comp && (s = tcd::build_lr_pack(x, L->hidden, L->ffn, lru, lrd, st)) != LRC_OK) return s;
    tcd::Expert& t = L->tcd_host[e];
    t.up = up;
    t.down = down;
    t.lr_up = comp ? lru : nullptr;
    t.lr_down = comp ? lrd : nullptr;
    t.u1 = x.u1; t.v1 = x.v1; t.u3 = x.u3; t.v3 = x.v3; t.u2 = x.u2; t.v2 = x.v2;
    t.rank = has_comp(x) ? rank_of(x.u1) : 0;
    L->tcd_dirty[e] = 0;
    any = true;
  }
  if (any || L->tcd_table_dirty) {
    LRC_CUDA_TRY(cudaMemcpyAsync(L->d_tcd, L->tcd_host.data(), sizeof(tcd::Expert) * NE, cudaMemcpyHostToDevice, st));
    LRC_CUDA_TRY(cudaStreamSynchronize(st));  // the host table may change before the copy would run
    L->tcd_table_dirty = false;
  }
  return LRC_OK;
}

extern "C" lrc_status lrc_layer_set_tcd_max(lrc_layer* L, int max_tokens) {
  if (!L) return fail(LRC_ERR_INVALID, "set_tcd_max: null layer");
  L->tcd_max = max_tokens;
  return LRC_OK;
}

extern "C" int lrc_layer_tcd_eligible(const lrc_layer* L) { return L && L->tcd_ok ? 1 : 0; }

// NVTX ranges: one per layer call, one per engine (visible in
// nsys / ncu --nvtx; free when no tool is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

static lrc_status forward_impl(lrc_layer* L, const uint16_t* x, int64_t B, int top_k, int top_n,
                               int renormalize, int compensate_shared, float* y, int32_t* topk_idx,
                               float* topk_w, void* stream, bool allow_tiled,
                               const int32_t* pairs_expert = nullptr, const float* pairs_w = nullptr,
                               const uint8_t* pairs_comp = nullptr) {
  if (!L || !x || !y) return fail(LRC_ERR_INVALID, "forward: null argument");
  if (top_k < 0 || top_n < 0 || top_n > top_k)
    return fail(LRC_ERR_INVALID, "top_n must be <= top_k and both >= 0");
  if (top_k > L->E) return fail(LRC_ERR_INVALID, "top_k exceeds the number of experts");
  if (top_k > L->k_max) return fail(LRC_ERR_UNSUPPORTED, "top_k above the layer's workspace");
  if (B < 0 || B > L->max_tokens) return fail(LRC_ERR_UNSUPPORTED, "B above max_tokens");
  NvtxRange nv_call(pairs_expert ? "lrc.layer_forward_pairs" : "lrc.layer_forward");
  cudaStream_t st = as_stream(stream);
  int launches = 0;
  const bool prof = L->profiling;
  if (prof) LRC_CUDA_TRY(cudaEventRecord(L->ev[0], st));
  if (B == 0) {
    L->last_launches = 0;
    return LRC_OK;
  }
  if (L->pager) {  // every distinct expert of the step needs its own slot
    const int64_t distinct = std::min<int64_t>(L->E, B * (pairs_expert ? 1 : top_k)) + (pairs_expert ? 0 : L->S);
    if (distinct > L->pg_slots) return fail(LRC_ERR_UNSUPPORTED, "pager: more distinct experts than slots");
  }
  // ---- tensor-core decode engine: one persistent kernel per layer step
  const int P_tcd = pairs_expert ? 1 : top_k + L->S;
  const int tcd_max = L->tcd_max >= 0 ? L->tcd_max : (L->tiled ? 0 : tcd::kMaxTok);
  if (allow_tiled && L->tcd_ok && !L->pager && tcd_max > 0 && B <= std::min(tcd_max, tcd::kMaxTok) &&
      B * P_tcd <= tcd::kMaxP && top_k <= 8) {
    lrc_status s = tcd_prepare(L, st);
    if (s != LRC_OK) return s;
    int32_t* ti = topk_idx ? topk_idx : L->topk_idx;
    float* tw = topk_w ? topk_w : L->topk_w;
    const bool fused = !pairs_expert && tcd_fused_routing(L);
    const bool pdl = !prof && L->pdl;
    if (prof) LRC_CUDA_TRY(cudaEventRecord(L->ev[1], st));
    if (!pairs_expert && !fused) {  // large expert counts: the cluster router writes the top-k
      RouteArgs ra{};
      ra.gate_t = L->gate_t;
      ra.x = x;
      ra.x_dtype = LRC_DTYPE_BF16;
      ra.B = B;
      ra.d = L->hidden;
      ra.E = L->E;
      ra.k = top_k;
      ra.renorm = renormalize;
      ra.topk_idx = ti;
      ra.topk_w = tw;
      ra.logits = L->logits;
      ra.tile_ticket = L->tile_ticket;
      ra.plan = L->plan;
      ra.plan.ticket = nullptr;  // routing only
      ra.pdl = pdl ? 1 : 0;
      if ((s = launch_route(ra, st)) != LRC_OK) return s;
      ++launches;
    }
    if (prof) LRC_CUDA_TRY(cudaEventRecord(L->ev[2], st));
    tcd::Args a = L->tcd_args;
    a.x = x;
    a.B = static_cast<int>(B);
    a.hidden = L->hidden;
    a.ffn = L->ffn;
    a.E = L->E;
    a.S = pairs_expert ? 0 : L->S;
    a.top_k = pairs_expert ? 1 : top_k;
    a.top_n = pairs_expert ? 1 : top_n;
    a.renorm = renormalize;
    a.comp_shared = compensate_shared;
    a.bits = L->tcd_bits;
    a.fb = L->tcd_fbits;
    a.gate32 = fused ? L->gate32 : nullptr;
    a.gate64 = L->gate_t;
    a.gnorm = L->gate32 + static_cast<int64_t>(L->E) * L->hidden;
    a.pairs_mode = pairs_expert ? 1 : 0;
    a.given_idx = pairs_expert ? pairs_expert : ti;
    a.given_w = pairs_expert ? pairs_w : tw;
    a.given_comp = pairs_comp;
    a.ex = L->d_tcd;
    a.y = y;
    a.topk_idx = ti;
    a.topk_w = tw;
    static const bool stamps = getenv("LRC_TCD_STAMPS") != nullptr;
    a.stamp = stamps ? 1 : 0;
    static const int dbg = getenv("LRC_TCD_DEBUG") ? atoi(getenv("LRC_TCD_DEBUG")) : 0;
    a.dbg = dbg;
    NvtxRange nv_tcd("lrc.tcd");
    if ((s = tcd::launch(a, L->num_sms, st, pdl)) != LRC_OK) return s;
    ++launches;
    if (prof) {
      LRC_CUDA_TRY(cudaEventRecord(L->ev[3], st));
      LRC_CUDA_TRY(cudaEventRecord(L->ev[4], st));
    }
    L->last_launches = launches;
    return LRC_OK;
  }
  PlanArgs plan = L->plan;
  plan.top_n = top_n;
  plan.compensate_shared = compensate_shared;
  plan.comp_rows = pairs_comp;  // pairs mode: per-row flags, no implicit shared pairs
  int32_t* ti = topk_idx ? topk_idx : L->topk_idx;
  float* tw = topk_w ? topk_w : L->topk_w;
  RouteArgs ra{};
  ra.gate_t = L->gate_t;
  ra.x = x;
  ra.x_dtype = LRC_DTYPE_BF16;
  ra.B = B;
  ra.d = L->hidden;
  ra.E = L->E;
  ra.k = top_k;
  ra.renorm = renormalize;
  ra.probs = nullptr;
  ra.topk_idx = ti;
  ra.topk_w = tw;
  ra.logits = L->logits;
  ra.tile_ticket = L->tile_ticket;
  ra.plan = plan;
  // one prologue launch: gate GEMV + softmax/top-k + plan, zeroing of y and the
  // t2 accumulators, and (one token tile) the speculative low-rank V.x
  // (pager mode: the experts' V factors arrive after the router, so no speculative V.x)
  const bool spec = !L->pager && L->maxr > 0 && B <= route_tiles(1) * 8 && route_tiles(B) == 1;
  ra.experts = L->d_experts;
  ra.t = L->t;
  ra.ne = L->E + L->S;
  ra.maxr = L->maxr;
  ra.spec_blocks = spec ? 2 * ((L->maxr + 7) / 8) : 0;
  ra.t2_zero = L->maxr ? L->t : nullptr;
  ra.y_zero = y;
  // PDL: the router's constant-data prologue (expert tables, gate rows, code
  // warm-up) overlaps the previous kernel's tail; it waits before touching x,
  // y, t or the plan
  ra.pdl = (!prof && L->pdl) ? 1 : 0;
  ra.pairs_expert = pairs_expert;
  ra.pairs_w = pairs_w;
  const int P = top_k + (pairs_expert ? 0 : L->S);
  const int np_bound = static_cast<int>(B) * P;
  // large batches: routing only, then the parallel plan (the single-CTA serial
  // plan would take ~1 us per 32 pairs)
  const bool big_plan = np_bound > kSerialPlanMaxPairs;
  if (big_plan) ra.plan.ticket = nullptr;
  static const bool no_bulk = getenv("LRC_NO_BULK_ROUTE") != nullptr;
  nvtxRangePushA("lrc.route");
  lrc_status s = (big_plan && !no_bulk) ? launch_route_bulk(ra, st) : launch_route(ra, st);
  nvtxRangePop();
  if (s != LRC_OK) return s;
  ++launches;
  if (big_plan) {
    if ((s = launch_plan_parallel(plan, ti, tw, static_cast<int>(B), top_k, L->plan_blk, L->plan_cmask,
                                  L->plan_ticket, st)) != LRC_OK)
      return s;
    launches += 2;
  }
  if (L->pager) {  // copy the active experts into their slots, repoint descriptors
    PagerArgs g = L->pg;
    g.plan = plan;
    if (g.owner != nullptr) {
      pager_assign_kernel<<<1, 32, 0, st>>>(g);
      LRC_CHECK_LAUNCH();
      ++launches;
    }
    const unsigned ny = static_cast<unsigned>(std::min(L->pg_slots, L->E + L->S));
    pager_kernel<<<dim3(static_cast<unsigned>(2 * L->num_sms), ny), 256, 0, st>>>(g);
    LRC_CHECK_LAUNCH();
    ++launches;
  }
  if (prof) LRC_CUDA_TRY(cudaEventRecord(L->ev[1], st));
  ExpertArgs a{};
  a.ne = L->E + L->S;
  a.experts = L->d_experts;
  a.plan = plan;
  a.hidden = L->hidden;
  a.ffn = L->ffn;
  a.maxr = L->maxr;
  a.x = x;
  a.t = L->t;
  a.a32 = L->a32;
  a.a16 = L->a16;
  a.y = y;
  a.max_pairs = L->max_pairs;
  a.g64 = (L->g64_ok && !L->pager && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
           (reinterpret_cast<uintptr_t>(L->a32) & 15) == 0) ? 1 : 0;
  // (the pager's descriptors point at slot copies of the tiled layout only)
  // without tiled packs (3-bit codes) the prefill engine also takes the batches
  // above the tensor-core decode engine's range: the generic CUDA-core path is
  // 15x slower there (tools/prefill3_check.py)
  const int64_t pmin = L->tiled ? L->prefill_min : std::min<int64_t>(L->prefill_min, tcd::kMaxTok + 1);
  const bool prefill = allow_tiled && L->prefill_ok && !L->pager && L->prefill_min > 0 && B >= pmin;
  if (!spec && L->maxr && !prefill) {  // exact V.x for the compensated pairs only
    if ((s = launch_lr_down(a, np_bound, st)) != LRC_OK) return s;
    ++launches;
  }
  if (prof) LRC_CUDA_TRY(cudaEventRecord(L->ev[2], st));
  if (prefill) {
    // large batches: tcgen05 grouped dequant-GEMMs (V1|V3.x, up, V2.a, down)
    // (re)build the packs of experts changed since the last prefill call: the
    // weight codes as contiguous per-slab blocks, the LR factors as bf16 rows
    const size_t pb = static_cast<size_t>(prefill_pack_bytes(L->hidden, L->ffn, L->prefill_bits));
    if (L->ppk == nullptr) LRC_CUDA_TRY(cudaMalloc(&L->ppk, pb * L->lrp_dirty.size()));
    const size_t per = static_cast<size_t>(prefill_lr_pack_elems(L->hidden, L->ffn, L->maxr));
    for (size_t i = 0; i < L->lrp_dirty.size(); ++i)
      if (L->lrp_dirty[i]) {
        if ((s = build_prefill_pack(L->host_experts[i], L->hidden, L->ffn, L->prefill_bits, L->ppk + pb * i, st)) != LRC_OK)
          return s;
        if (L->maxr &&
            (s = build_prefill_lr(L->host_experts[i], L->hidden, L->ffn, L->maxr, L->lrp + per * i, st)) != LRC_OK)
          return s;
        L->lrp_dirty[i] = 0;
      }
    NvtxRange nv_pf("lrc.prefill");
    if ((s = launch_prefill(a, np_bound, static_cast<int>(B), L->lrp, L->tb, L->ppk, L->prefill_bits, st, &launches)) != LRC_OK) return s;
    if (prof) LRC_CUDA_TRY(cudaEventRecord(L->ev[3], st));  // phases: up+mid+down lumped into [2]
  } else if (allow_tiled && L->tiled) {
    NvtxRange nv_t("lrc.tiled");
    const int tok_bound = static_cast<int>(std::min<int64_t>(B, L->max_tokens));
    // programmatic dependent launch: the next kernel's CTAs are scheduled as SMs
    // free up and block in griddepcontrol.wait (no PDL while timing phases)
    const bool pdl = !prof && L->pdl;
    if ((s = launch_up_tiled(a, L->num_sms, tok_bound, L->lr_up_max, st, pdl)) != LRC_OK)
      return s;
    if (prof) LRC_CUDA_TRY(cudaEventRecord(L->ev[3], st));
    if ((s = launch_down_tiled(a, L->num_sms, tok_bound, L->lr_down_max, st, pdl)) != LRC_OK)
      return s;
    launches += 2;
  } else {
    NvtxRange nv_g("lrc.generic");
    const int grid = L->num_sms * 4;
    up_generic_kernel<<<grid, 256, 0, st>>>(a);
    LRC_CHECK_LAUNCH();
    if (prof) LRC_CUDA_TRY(cudaEventRecord(L->ev[3], st));
    if (L->maxr) {
      lr_mid_kernel<<<(np_bound * L->maxr + 7) / 8, 256, 0, st>>>(a);
      LRC_CHECK_LAUNCH();
      ++launches;
    }
    down_generic_kernel<<<grid, 256, 0, st>>>(a);
    LRC_CHECK_LAUNCH();
    launches += 2;
  }
  if (prof) LRC_CUDA_TRY(cudaEventRecord(L->ev[4], st));
  L->last_launches = launches;
  return LRC_OK;
}

extern "C" lrc_status lrc_layer_forward(lrc_layer* L, const uint16_t* x, int64_t B, int top_k,
                                        int top_n, int renormalize, int compensate_shared, float* y,
                                        int32_t* topk_idx, float* topk_w, void* stream) {
  return forward_impl(L, x, B, top_k, top_n, renormalize, compensate_shared, y, topk_idx, topk_w,
                      stream, true);
}

extern "C" lrc_status lrc_layer_forward_pairs(lrc_layer* L, const uint16_t* x, int64_t B,
                                              const int32_t* expert, const float* weight,
                                              const uint8_t* comp, float* y, void* stream) {
  if (!expert || !weight || !comp) return fail(LRC_ERR_INVALID, "forward_pairs: null routing");
  return forward_impl(L, x, B, 1, 1, 0, 0, y, nullptr, nullptr, stream, true, expert, weight, comp);
}

extern "C" lrc_status lrc_layer_forward_generic(lrc_layer* L, const uint16_t* x, int64_t B,
                                                int top_k, int top_n, int renormalize,
                                                int compensate_shared, float* y, int32_t* topk_idx,
                                                float* topk_w, void* stream) {
  return forward_impl(L, x, B, top_k, top_n, renormalize, compensate_shared, y, topk_idx, topk_w,
                      stream, false);
}

// Host-buffer staging as kernels (word copies through the UVA mapping of pinned
// memory).  stage-in: releases its dependents at once, copies x, then waits for
// its predecessor (the previous call's stage-out) before completing -- so the
// router's own wait also covers the previous y read.  stage-out: waits for the
// down kernel, then copies y.
// (16-byte words when both sides are 16-byte aligned and the size allows: the
// host side is read/written over the host link, where transaction count, not
// bytes, sets the latency of these small copies)
template <typename W>
__global__ void stage_kernel(const W* __restrict__ src, W* __restrict__ dst, int64_t n, int in) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (!in) asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
  if (in) asm volatile("griddepcontrol.wait;" ::: "memory");
}

static cudaError_t launch_stage(bool in, const void* src, void* dst, size_t bytes, cudaStream_t st,
                                bool pdl) {
  const bool v16 = bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  const int64_t n = static_cast<int64_t>(bytes / (v16 ? 16 : 4));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(std::min<int64_t>(32, (n + 255) / 256)));
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  if (v16)
    return cudaLaunchKernelEx(&cfg, stage_kernel<uint4>, static_cast<const uint4*>(src), static_cast<uint4*>(dst), n,
                              in ? 1 : 0);
  return cudaLaunchKernelEx(&cfg, stage_kernel<uint32_t>, static_cast<const uint32_t*>(src),
                            static_cast<uint32_t*>(dst), n, in ? 1 : 0);
}

extern "C" lrc_status lrc_layer_forward_host(lrc_layer* L, const uint16_t* x_host, int64_t B,
                                             int top_k, int top_n, int renormalize,
                                             int compensate_shared, float* y_host, void* stream) {
  if (!L || !x_host || !y_host) return fail(LRC_ERR_INVALID, "forward_host: null argument");
  if (B < 0 || B > L->max_tokens) return fail(LRC_ERR_UNSUPPORTED, "B above max_tokens");
  cudaStream_t st = as_stream(stream);
  const size_t xb = sizeof(uint16_t) * B * L->hidden, yb = sizeof(float) * B * L->hidden;
  if (B == 0) return LRC_OK;
  // Pinned (device-mapped under UVA) host buffers: the copies are kernels, so the
  // whole call stays one programmatic-dependent-launch chain and the next
  // router still overlaps the previous layer's tail.  Pageable: plain copies.
  cudaPointerAttributes ax{}, ay{};
  const bool mapped = cudaPointerGetAttributes(&ax, x_host) == cudaSuccess &&
                      cudaPointerGetAttributes(&ay, y_host) == cudaSuccess &&
                      ax.type == cudaMemoryTypeHost && ay.type == cudaMemoryTypeHost &&
                      ax.devicePointer != nullptr && ay.devicePointer != nullptr && xb % 4 == 0;
  cudaGetLastError();  // clear a sticky error from probing pageable memory
  const bool pdl = !L->profiling && L->pdl;
  if (mapped) {
    LRC_CUDA_TRY(launch_stage(true, ax.devicePointer, L->x_stage, xb, st, pdl));
  } else {
    LRC_CUDA_TRY(cudaMemcpyAsync(L->x_stage, x_host, xb, cudaMemcpyHostToDevice, st));
  }
  lrc_status s = forward_impl(L, L->x_stage, B, top_k, top_n, renormalize, compensate_shared,
                              L->y_stage, nullptr, nullptr, st, true);
  if (s != LRC_OK) return s;
  if (mapped) {
    LRC_CUDA_TRY(launch_stage(false, L->y_stage, ay.devicePointer, yb, st, pdl));
  } else {
    LRC_CUDA_TRY(cudaMemcpyAsync(y_host, L->y_stage, yb, cudaMemcpyDeviceToHost, st));
  }
  return LRC_OK;
}

extern "C" lrc_status lrc_layer_set_profiling(lrc_layer* L, int enabled) {
  if (!L) return fail(LRC_ERR_INVALID, "set_profiling: null layer");
  L->profiling = enabled != 0;
  return LRC_OK;
}

extern "C" lrc_status lrc_layer_phase_ms(lrc_layer* L, float* ms4) {
  if (!L || !ms4) return fail(LRC_ERR_INVALID, "phase_ms: null argument");
  LRC_CUDA_TRY(cudaEventSynchronize(L->ev[4]));
  for (int i = 0; i < 4; ++i) LRC_CUDA_TRY(cudaEventElapsedTime(&ms4[i], L->ev[i], L->ev[i + 1]));
  return LRC_OK;
}

extern "C" lrc_status lrc_dense_expert_f64(const double* w1, const double* w3, const double* w2,
                                           int hidden, int ffn, const double* x, const double* mix,
                                           int64_t B, double* y, void* stream) {
  if (hidden <= 0 || ffn <= 0 || B < 0) return fail(LRC_ERR_INVALID, "dense_expert: bad shape");
  if (B == 0) return LRC_OK;
  cudaStream_t st = as_stream(stream);
  double* act = nullptr;
  LRC_CUDA_TRY(cudaMallocAsync(&act, sizeof(double) * B * ffn, st));
  int64_t w1n = B * ffn * 32, w2n = B * hidden * 32;
  dense_up_f64_kernel<<<static_cast<unsigned>((w1n + 255) / 256), 256, 0, st>>>(w1, w3, hidden, ffn,
                                                                                 x, B, act);
  dense_down_f64_kernel<<<static_cast<unsigned>((w2n + 255) / 256), 256, 0, st>>>(w2, hidden, ffn,
                                                                                   act, mix, B, y);
  cudaError_t e = cudaGetLastError();
  cudaFreeAsync(act, st);
  if (e != cudaSuccess) return fail(LRC_ERR_CUDA, cudaGetErrorString(e));
  return LRC_OK;
}
