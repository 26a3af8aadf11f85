// K1: fused router prologue -- gate GEMV (fp64) + softmax + stable top-k/top-n,
// the per-expert pair plan consumed by the expert kernels, zeroing of the
// accumulated outputs, and (single token tile) the speculative low-rank
// down-projection t = V.x.
// Reference: ref/moe.py:165-193 (route/softmax), ref/moe.py:234-258 (mixing,
// shared experts), ref/lowrank.py:165 (factored U.(V.x) order).
//
// Grid (token tiles, experts, 1 + V.x row blocks).  CTA (tile, e, 0) computes
// the logits of up to kTT tokens against gate row e; CTAs (tile, e, z>0) the
// speculative V.x rows.  The last CTA of a token tile (atomic ticket) runs the
// warp-parallel softmax + top-k for the tile; the last tile builds the pair
// plan -- one launch, no host round trip.  Code is kept compact on purpose:
// cold straight-line paths in a huge kernel stall on instruction fetch.
#include <float.h>
#include <stdlib.h>

#include "common.cuh"
#include "layer.cuh"

namespace lrc {

constexpr int kTT = 8;  // tokens per router CTA
constexpr int kRThreads = 256;
constexpr int kStampCtas = 1024;

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
__device__ __noinline__ double pw_sum_small(const double* v, int n) {
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

// One warp per token: softmax exactly as ref/moe.py:165-168 (z = l - max,
// exp, divide by the numpy-ordered sum), then k rounds of warp argmax with the
// stable tie rule of np.argsort(-w, kind="stable") (ref/moe.py:190): equal
// weights go to the lower expert index.  lg has E weights + 64 scratch.
__device__ __noinline__ void select_topk_warp(double* lg, int E, int k, int renorm, int64_t b,
                                              double* probs, int32_t* topk_idx, float* topk_w) {
  const int lane = threadIdx.x & 31;
  double mx = -DBL_MAX;
  for (int e = lane; e < E; e += 32) mx = fmax(mx, lg[e]);
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
  for (int j = 0; j < k; ++j) {
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
    if (lane == 0) {
      topk_idx[b * k + j] = be;
      lg[E + j] = bv;  // scratch after the E weights
    }
  }
  __syncwarp();
  if (lane == 0) {
    double* mix = lg + E;
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

// Padded shared-memory x row: 64-column groups at a stride of 66 elements.
__host__ __device__ inline int xs_row_elems(int d) { return ((d + 63) / 64) * 66; }
__device__ inline int xs_col(int c) { return (c >> 6) * 66 + (c & 63); }

// Speculative t[b][e][proj][j] =V_proj(e)[j, :] . x_b for the 8 rows of
// block `blk` (one warp per row) and every token of the tile, whether or not
// e becomes one of b's top-n experts: removes a dependent launch between the
// router and the expert kernels (< 1% extra bytes at decode sizes).  x rows
// come from shared memory (xs: nb x d bf16); each lane preloads the code words
// of its whole groups, then loops over tokens.
__device__ __noinline__ void spec_lr_rows(const RouteArgs& ra, const uint16_t* xs, int64_t b0,
                                          int nb, int e, int blk) {
  const lrc_expert& E = ra.experts[e];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nblk1 = (ra.maxr + 7) / 8;
  const int proj = blk / nblk1;
  const int j = (blk - proj * nblk1) * 8 + warp;
  if (j >= ra.maxr) return;
  const lrc_qmat& V = proj == 0 ? E.v1 : E.v3;
  float* tout = ra.t + ((b0 * ra.ne + e) * 3 + proj) * ra.maxr + j;
  const int64_t tstride = static_cast<int64_t>(ra.ne) * 3 * ra.maxr;
  if (!factor_present(V) || j >= V.rows) {
    if (lane < nb) tout[lane * tstride] = 0.0f;
    return;
  }
  const bool fast = V.dense == nullptr && V.group_size == 64 && V.bits == 3 &&
                    ((V.cols * 3) % 32) == 0 && V.cols <= 64 * 64;
  if (fast) {
    // 3-bit codes, group 64 = 6 words; up to 2 groups per lane (cols <= 4096)
    const int gpr = V.cols / 64 + ((V.cols % 64) != 0);
    const uint32_t* words = reinterpret_cast<const uint32_t*>(V.packed);
    const int64_t nwords = ((static_cast<int64_t>(V.rows) * V.cols * 3 + 7) >> 3) >> 2;
    uint32_t w[2][7];
    float s[2], z[2];
    int nv[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int g = lane + 32 * h;
      nv[h] = (g < gpr) ? min(64, V.cols - g * 64) : 0;
      const int64_t w0 = ((static_cast<int64_t>(j) * V.cols + g * 64) * 3) >> 5;
#pragma unroll
      for (int i = 0; i < 7; ++i) w[h][i] = (nv[h] > 0 && w0 + i < nwords) ? __ldg(words + w0 + i) : 0u;
      s[h] = nv[h] > 0 ? h2f(V.scales[static_cast<int64_t>(j) * gpr + g]) : 0.0f;
      z[h] = nv[h] > 0 ? h2f(V.zeros[static_cast<int64_t>(j) * gpr + g]) : 0.0f;
    }
    const int ldx = xs_row_elems(ra.d);
    for (int t = 0; t < nb; ++t) {
      const uint32_t* xr = reinterpret_cast<const uint32_t*>(xs + t * ldx);
      float acc = 0.0f;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float cx = 0.0f, sx = 0.0f;
        const uint32_t* xg = xr + (lane + 32 * h) * 33;
#pragma unroll
        for (int i2 = 0; i2 < 32; ++i2) {
          if (2 * i2 < nv[h]) {
            const uint32_t xw = xg[i2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int bit = (2 * i2 + q) * 3;
              const float c = static_cast<float>(
                  __funnelshift_r(w[h][bit >> 5], w[h][(bit >> 5) + 1], bit & 31) & 7u);
              const float xv = q ? __uint_as_float(xw & 0xffff0000u) : __uint_as_float(xw << 16);
              cx = fmaf(c, xv, cx);
              sx += xv;
            }
          }
        }
        acc = fmaf(s[h], cx, fmaf(z[h], sx, acc));
      }
      acc = warp_sum(acc);
      if (lane == 0) tout[t * tstride] = acc;
    }
    return;
  }
  const int ldx = xs_row_elems(ra.d);
  for (int t = 0; t < nb; ++t) {  // generic: any bits / group size / raw fp32 factors
    const uint16_t* xr = xs + t * ldx;
    float acc = 0.0f;
    for (int c = lane; c < V.cols; c += 32) acc = fmaf(qmat_elem(V, j, c), bf2f(xr[xs_col(c)]), acc);
    acc = warp_sum(acc);
    if (lane == 0) tout[t * tstride] = acc;
  }
}

__device__ unsigned long long g_route_stamps[kStampCtas * 8];
#define RSTAMP(k)                                                                     \
  do {                                                                                \
    if (ra.stamp && threadIdx.x == 0) {                                               \
      const int cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x; \
      unsigned long long t_;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                          \
      if (cta < kStampCtas) g_route_stamps[cta * 8 + (k)] = t_;                       \
    }                                                                                 \
  } while (0)

template <typename T>
__global__ void __launch_bounds__(kRThreads) route_kernel(const __grid_constant__ RouteArgs ra) {
  extern __shared__ __align__(16) uint8_t rsm[];  // [kTT*(E+64)] f64 logits | x tile (bf16)
  __shared__ double s_red[kTT][kRThreads / 32];
  __shared__ int s_last;
  const int tile = blockIdx.x, e = blockIdx.y, z = blockIdx.z;
  const int64_t b0 = static_cast<int64_t>(tile) * kTT;
  const int64_t rem = ra.B - b0;
  const int nb = rem < kTT ? static_cast<int>(rem) : kTT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T* x = static_cast<const T*>(ra.x);
  RSTAMP(0);
  griddep_launch_dependents_r();
  if (z == 0) {
    if (e < ra.E) {
      const double* g = ra.gate_t + static_cast<int64_t>(e) * ra.d;
      double acc[kTT];
#pragma unroll
      for (int t = 0; t < kTT; ++t) acc[t] = 0.0;
#pragma unroll 4
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
    RSTAMP(6);
    if (ra.t2_zero != nullptr && ra.maxr > 0)
      for (int i = threadIdx.x; i < nb * ra.maxr; i += kRThreads) {
        const int t = i / ra.maxr, j = i - t * ra.maxr;
        ra.t2_zero[(((b0 + t) * ra.ne + e) * 3 + 2) * ra.maxr + j] = 0.0f;
      }
    if (ra.y_zero != nullptr && e == 0)
      for (int64_t i = threadIdx.x; i < static_cast<int64_t>(nb) * ra.d; i += kRThreads)
        ra.y_zero[b0 * ra.d + i] = 0.0f;
  } else if constexpr (sizeof(T) == 2) {
    // stage the tile's token rows once (16-byte copies), then the V.x rows
    // padded layout: 64-column groups at a stride of 33 words, so lanes that
    // each walk their own group hit distinct banks
    uint16_t* xs = reinterpret_cast<uint16_t*>(rsm);
    const uint16_t* xg = reinterpret_cast<const uint16_t*>(x) + b0 * ra.d;
    const int ldx = xs_row_elems(ra.d);
    if ((ra.d % 64) == 0 && (reinterpret_cast<uintptr_t>(xg) & 3) == 0) {
      const int wpr = ra.d / 2;  // words per token row
      uint32_t* xs32 = reinterpret_cast<uint32_t*>(xs);
      const uint32_t* xg32 = reinterpret_cast<const uint32_t*>(xg);
      for (int i = threadIdx.x; i < nb * wpr; i += kRThreads) {
        const int t = i / wpr, w = i - t * wpr;
        xs32[t * (ldx / 2) + (w >> 5) * 33 + (w & 31)] = __ldg(xg32 + i);
      }
    } else {
      for (int i = threadIdx.x; i < nb * ra.d; i += kRThreads) {
        const int t = i / ra.d, c = i - t * ra.d;
        xs[t * ldx + xs_col(c)] = xg[i];
      }
    }
    __syncthreads();
    spec_lr_rows(ra, xs, b0, nb, e, z - 1);
  }
  // ---- last CTA of this token tile: softmax + top-k
  RSTAMP(1);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0)
    s_last = (atomicAdd(&ra.tile_ticket[tile], 1) == static_cast<int>(gridDim.y * gridDim.z) - 1);
  __syncthreads();
  RSTAMP(2);
  if (!s_last) return;
  __threadfence();
  double* lg = reinterpret_cast<double*>(rsm);  // per token: E weights + 64 scratch
  const int ldl = ra.E + 64;
  for (int i = threadIdx.x; i < nb * ra.E; i += kRThreads)
    lg[(i / ra.E) * ldl + i % ra.E] = __ldcg(ra.logits + b0 * ra.E + i);
  __syncthreads();
  if (warp < nb)
    select_topk_warp(lg + warp * ldl, ra.E, ra.k, ra.renorm, b0 + warp, ra.probs, ra.topk_idx,
                     ra.topk_w);
  if (threadIdx.x == 0) ra.tile_ticket[tile] = 0;
  RSTAMP(3);
  if (ra.plan.ticket == nullptr) return;
  // ---- last tile: build the pair plan for the whole batch
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(ra.plan.ticket, 1) == static_cast<int>(gridDim.x) - 1);
  __syncthreads();
  RSTAMP(4);
  if (!s_last) return;
  __threadfence();
  build_plan_block(ra.plan, ra.topk_idx, ra.topk_w, static_cast<int>(ra.B), ra.k);
  if (threadIdx.x == 0) *ra.plan.ticket = 0;
  __syncthreads();
  RSTAMP(5);
}

// Pair plan: pair p = b*P + j, P = k + S.  j < k: routed expert topk_idx[b][j],
// weight topk_w, compensated iff j < n.  j >= k: shared expert E + (j-k),
// weight 1, compensated iff compensate_shared (ref/moe.py:249-258).
// Pairs are grouped by expert, ascending pair id inside each expert (stable).
__device__ __noinline__ void build_plan_block(const PlanArgs& pa, const int32_t* topk_idx,
                                              const float* topk_w, int B, int k) {
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
        if (pa.arec != nullptr) {
          const lrc_expert& X = pa.experts[e];
          const LrLayout L = lr_layout(X);
          ActiveRec& R = pa.arec[na];
          R.up_tiles = X.up_tiles;
          R.down_tiles = X.down_tiles;
          R.up_lr_tiles = X.up_lr_tiles;
          R.down_lr_tiles = X.down_lr_tiles;
          R.e = e;
          R.off = s_off[e];
          R.cnt = s_cnt[e];
          R.up_lr_bytes = L.up_total;
          R.down_lr_bytes = L.down_total;
        }
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
      // compensated-pair slots, in pair order
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
  if (pa.arec == nullptr) return;
  // compensated-pair mask per active expert, 8-pair granularity (one warp each)
  __syncthreads();
  const int na = pa.counts[0];
  for (int a = threadIdx.x >> 5; a < na; a += blockDim.x >> 5) {
    const int off = pa.active_off[a], cnt = pa.active_cnt[a];
    uint32_t mask = 0;
    for (int j0 = 0; j0 < cnt; j0 += 32) {
      const int j = j0 + lane;
      const bool c = j < cnt && pa.pair_comp[pa.pair_list[off + j]] >= 0;
      const unsigned bal = __ballot_sync(0xffffffffu, c);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if ((bal >> (8 * q)) & 0xffu) mask |= 1u << min((j0 >> 3) + q, 31);
    }
    if (lane == 0) pa.arec[a].cmask = mask;
  }
}

int route_tiles(int64_t B) { return static_cast<int>((B + kTT - 1) / kTT); }

lrc_status launch_route(const RouteArgs& ra_in, cudaStream_t st) {
  static const int stamps = getenv("LRC_ROUTE_STAMPS") != nullptr;
  RouteArgs ra = ra_in;
  ra.stamp = stamps;
  // logits scratch (kTT tokens x (E + 64) doubles) shares dynamic smem with the
  // bf16 x tile of the speculative V.x CTAs
  int smem = kTT * (ra.E + 64) * static_cast<int>(sizeof(double));
  if (ra.spec_blocks > 0) smem = max(smem, kTT * xs_row_elems(ra.d) * 2);
  static int configured = -1;
  if (configured < smem) {
    const void* fns[3] = {(const void*)route_kernel<double>, (const void*)route_kernel<float>,
                          (const void*)route_kernel<uint16_t>};
    for (auto f : fns) {
      if (smem > 48 * 1024)
        LRC_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      // same L1/shared split as the tiled expert kernels: no carveout switch
      // (SM drain + reconfiguration) between the launches of a layer
      if (getenv("LRC_NO_CARVEOUT") == nullptr)
        LRC_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    }
    configured = smem;
  }
  dim3 grid(route_tiles(ra.B), ra.experts ? ra.ne : ra.E, 1 + ra.spec_blocks);
  switch (ra.x_dtype) {
    case LRC_DTYPE_F64:
      route_kernel<double><<<grid, kRThreads, smem, st>>>(ra);
      break;
    case LRC_DTYPE_F32:
      route_kernel<float><<<grid, kRThreads, smem, st>>>(ra);
      break;
    case LRC_DTYPE_BF16:
      route_kernel<uint16_t><<<grid, kRThreads, smem, st>>>(ra);
      break;
    default:
      return fail(LRC_ERR_INVALID, "route: unknown x dtype");
  }
  LRC_CHECK_LAUNCH();
  return LRC_OK;
}

}  // namespace lrc

extern "C" lrc_status lrc_debug_stamps(int which, uint64_t* host, int n) {
  using namespace lrc;
  if (n < 0 || n > (which == 0 ? kStampCtas * 8 : 2 * 256 * 8 + 2 * 64 * 6)) return fail(LRC_ERR_INVALID, "stamps: bad count");
  LRC_CUDA_TRY(cudaDeviceSynchronize());
  if (which != 0) {
    tiled_stamps_copy(host, n);
    return LRC_OK;
  }
  LRC_CUDA_TRY(cudaMemcpyFromSymbol(host, g_route_stamps, sizeof(uint64_t) * n));
  void* dev = nullptr;  // cleared after each read: CTAs that skip a point leave 0
  LRC_CUDA_TRY(cudaGetSymbolAddress(&dev, g_route_stamps));
  LRC_CUDA_TRY(cudaMemset(dev, 0, sizeof(g_route_stamps)));
  return LRC_OK;
}

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
