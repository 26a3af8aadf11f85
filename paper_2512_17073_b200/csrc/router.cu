// K1: fused router prologue -- gate GEMV (fp64) + softmax + stable top-k/top-n,
// the per-expert pair plan consumed by the expert kernels, zeroing of the
// accumulated outputs, and (single token tile) the speculative low-rank
// down-projection t = V.x.
// Reference: ref/moe.py:165-193 (route/softmax), ref/moe.py:234-258 (mixing,
// shared experts), ref/lowrank.py:165 (factored U.(V.x) order).
//
// Grid (token tiles x kCl, 1 + aux rows), clusters of kCl CTAs along x: row 0
// of a tile's cluster computes its logits (CTA r: experts r, r + kCl, ...) and
// stores them into the leader CTA's shared memory (DSMEM); after one cluster
// barrier the leader runs the warp-parallel softmax + top-k and, for a single
// token tile, builds the pair plan straight from shared memory (several
// tiles: the last leader, by atomic ticket).  Aux rows zero the accumulated
// outputs and compute the speculative V.x rows.  One launch, no host round
// trip, and at decode sizes no global-memory handoff inside the kernel: every
// dependent global round trip costs ~1 us while the weight stream saturates HBM.
#include <float.h>
#include <stdlib.h>

#include "common.cuh"
#include "layer.cuh"
#include "tcd.cuh"

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
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __noinline__ void select_topk_warp(double* lg, int E, int k, int renorm, int64_t b,
                                              double* probs, int32_t* topk_idx, float* topk_w,
                                              int32_t* s_idx, float* s_w,
                                              unsigned long long* dbg_stamp = nullptr) {
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
  if (dbg_stamp != nullptr && lane == 0) *dbg_stamp = globaltimer();
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
      s_idx[j] = be;
      lg[E + j] = bv;  // scratch after the E weights
    }
  }
  __syncwarp();
  if (dbg_stamp != nullptr && lane == 0) dbg_stamp[5] = globaltimer();
  if (lane == 0) {
    double* mix = lg + E;
    if (renorm) {  // ref/moe.py:234-236, mix.sum() in numpy order
      const double s = pw_sum_small(mix, k);
      if (s > 0.0)
        for (int j = 0; j < k; ++j) mix[j] = __ddiv_rn(mix[j], s);
    }
    for (int j = 0; j < k; ++j) {
      topk_w[b * k + j] = static_cast<float>(mix[j]);
      s_w[j] = static_cast<float>(mix[j]);
    }
  }
}

// Layer-forward variant (no fp64 probabilities requested, E <= 32): the
// selection runs on the exact fp64 logits -- the softmax is monotonic, so the
// stable top-k of the probabilities is the stable top-k of the logits unless
// two compared logits are so close that their fp64 exponentials could round
// to the same value; such near-ties (and ties) take the exact path above.
// The mixing weights are computed in fp32 (expf, warp sum): within a few ulp
// of float(fp64 softmax), far inside the layer-output tolerance.  Replaces
// ~1,600 SASS instructions of fp64 exp / div / pairwise sum (cold code on the
// critical path, DESIGN 8 item 2) with ~200.
__device__ __noinline__ bool select_topk_fast(const double* lg, int E, int k, int renorm, int64_t b,
                                              int32_t* topk_idx, float* topk_w, int32_t* s_idx, float* s_w) {
  const int lane = threadIdx.x & 31;
  const double l = lane < E ? lg[lane] : -DBL_MAX;
  // 32-bit order key: the top 27 bits of the order-preserving integer image of
  // the double, then (31 - lane) so that equal keys go to the lower expert;
  // one redux.sync.max per selection round.  Truncation only merges logits
  // that agree in their top 27 bits -- the fp64 near-tie guard below sends
  // every such case (and every real near-tie) to the exact path.
  const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(l));
  const unsigned long long ord = (u >> 63) ? ~u : (u | 0x8000000000000000ull);
  const uint32_t key = lane < E ? (static_cast<uint32_t>(ord >> 37) << 5) | static_cast<uint32_t>(31 - lane) : 0u;
  bool taken = lane >= E, ok = true;
  double prev = 0.0, mx = 0.0;
  int my_rank = -1;
  const int kk = min(k + 1, E);
  for (int j = 0; j < kk; ++j) {
    const uint32_t m = __reduce_max_sync(0xffffffffu, taken ? 0u : key);
    const int be = 31 - static_cast<int>(m & 31u);
    const double bv = __shfl_sync(0xffffffffu, l, be);
    if (j == 0) mx = bv;
    // fp64 exp(l - mx) has relative error < 2^-52: logits closer than this
    // bound could produce equal probabilities (a tie the reference breaks by
    // index) -- leave those to the exact path
    if (j > 0 && !(prev - bv > 1e-13 * fmax(1.0, fabs(bv - mx)))) ok = false;
    prev = bv;
    if (lane == be) {
      taken = true;
      if (j < k) my_rank = j;
    }
  }
  if (!ok) return false;
  const float ex = lane < E ? expf(static_cast<float>(l - mx)) : 0.f;
  float den = ex;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) den += __shfl_xor_sync(0xffffffffu, den, o);
  float w = ex / den;
  if (renorm) {
    float sw = my_rank >= 0 ? w : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sw += __shfl_xor_sync(0xffffffffu, sw, o);
    if (sw > 0.f) w = w / sw;
  }
  if (my_rank >= 0) {
    topk_idx[b * k + my_rank] = lane;
    topk_w[b * k + my_rank] = w;
    s_idx[my_rank] = lane;
    s_w[my_rank] = w;
  }
  return true;
}

__device__ __forceinline__ void griddep_launch_dependents_r() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void griddep_wait_r() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Padded shared-memory x row: 64-column groups at a stride of 66 elements.
__host__ __device__ inline int xs_row_elems(int d) { return ((d + 63) / 64) * 66; }
__device__ inline int xs_col(int c) { return (c >> 6) * 66 + (c & 63); }

// Speculative t[b][e][proj][j] =V_proj(e)[j, :] . x_b for the 8 rows of
// block `blk` (one warp per row) and every token of the tile, whether or not
// e becomes one of b's top-n experts: removes a dependent launch between the
// router and the expert kernels (< 1% extra bytes at decode sizes).  x rows
// come from shared memory (xs: nb x d bf16); each lane preloads the code words
// of its whole groups, then loops over tokens.
__device__ __forceinline__ float code_f(uint32_t c) {  // exact float of a small code
  return __uint_as_float(0x4B000000u | c) - 8388608.0f;
}

template <int NT>
__device__ __forceinline__ void spec_dot(const RouteArgs& ra, const uint16_t* xs, const float* xsum,
                                         const uint32_t (&w)[2][7], const float (&s)[2], const float (&z)[2],
                                         const int (&nv)[2], int nb, float* tout, int64_t tstride) {
  const int lane = threadIdx.x & 31;
  const int ldx = xs_row_elems(ra.d);
  const uint32_t* xs32 = reinterpret_cast<const uint32_t*>(xs);
  float acc[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t] = 0.0f;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (nv[h] == 0) continue;
    const int g = lane + 32 * h;
    float cx[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) cx[t] = 0.0f;
    // two chunks of 32 codes = exactly 3 words each (static word indices)
    for (int ch = 0; ch < 2; ++ch) {
      if (32 * ch >= nv[h]) break;
      const uint32_t q[4] = {ch ? w[h][3] : w[h][0], ch ? w[h][4] : w[h][1], ch ? w[h][5] : w[h][2],
                             ch ? w[h][6] : w[h][3]};
#pragma unroll
      for (int i2 = 0; i2 < 16; ++i2) {
        const int bit0 = 6 * i2, bit1 = bit0 + 3;
        const float c0 = code_f(__funnelshift_r(q[bit0 >> 5], q[(bit0 >> 5) + 1], bit0 & 31) & 7u);
        const float c1 = code_f(__funnelshift_r(q[bit1 >> 5], q[(bit1 >> 5) + 1], bit1 & 31) & 7u);
#pragma unroll
        for (int t = 0; t < NT; ++t)
          if (t < nb) {
            const uint32_t xw = xs32[t * (ldx / 2) + g * 33 + 16 * ch + i2];
            cx[t] = fmaf(c0, __uint_as_float(xw << 16), fmaf(c1, __uint_as_float(xw & 0xffff0000u), cx[t]));
          }
      }
    }
#pragma unroll
    for (int t = 0; t < NT; ++t)
      if (t < nb) acc[t] = fmaf(s[h], cx[t], fmaf(z[h], xsum[t * 64 + g], acc[t]));
  }
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    if (t < nb) {
      const float v = warp_sum(acc[t]);
      if (lane == 0) tout[t * tstride] = v;
    }
  }
}

__device__ __noinline__ void spec_lr_rows(const RouteArgs& ra, const uint16_t* xs, const float* xsum,
                                          int64_t b0, int nb, int e, int blk) {
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
    // each code is decoded once (exact float via the 2^23 magic, no XU
    // conversion) and applied to every token of the tile; sum(x) per group
    // comes precomputed from the staging pass (xsum[t][g]).  This code runs
    // once per layer step with a cold instruction cache, so its size is its
    // cost: the single-token variant is ~8x smaller than the tile one.
    if (nb == 1) spec_dot<1>(ra, xs, xsum, w, s, z, nv, 1, tout, tstride);
    else spec_dot<kTT>(ra, xs, xsum, w, s, z, nv, nb, tout, tstride);
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
    if ((ra.stamp & 1) && threadIdx.x == 0) {                                         \
      const int cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x; \
      unsigned long long t_;                                                          \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                          \
      if (cta < kStampCtas) g_route_stamps[cta * 8 + (k)] = t_;                       \
    }                                                                                 \
  } while (0)

constexpr int kCl = 8;  // CTAs per router cluster: one cluster per token tile

// barrier of the kRThreads worker threads (the warm-up warp never joins)
__device__ __forceinline__ void wsync() { asm volatile("bar.sync 1, %0;" ::"n"(kRThreads) : "memory"); }

__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// store v into CTA `rank`'s shared memory at the address of `p` in its layout
__device__ __forceinline__ void st_cl_f64(const double* p, uint32_t rank, double v) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}

__device__ __forceinline__ void st_cl_u64(const uint64_t* p, uint32_t rank, uint64_t v) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(ra), "l"(v) : "memory");
}
__device__ __forceinline__ void st_cl_u8(const uint8_t* p, uint32_t rank, uint8_t v) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p));
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.u8 [%0], %1;" ::"r"(ra), "h"(static_cast<unsigned short>(v)) : "memory");
}

template <typename T>
__device__ __forceinline__ void load_x2(const T* x, int64_t i, double& a, double& b);
template <>
__device__ __forceinline__ void load_x2<double>(const double* x, int64_t i, double& a, double& b) {
  const double2 v = __ldg(reinterpret_cast<const double2*>(x + i));
  a = v.x;
  b = v.y;
}
template <>
__device__ __forceinline__ void load_x2<float>(const float* x, int64_t i, double& a, double& b) {
  const float2 v = __ldg(reinterpret_cast<const float2*>(x + i));
  a = v.x;
  b = v.y;
}
template <>
__device__ __forceinline__ void load_x2<uint16_t>(const uint16_t* x, int64_t i, double& a, double& b) {
  const uint32_t v = __ldg(reinterpret_cast<const unsigned int*>(x + i));
  a = bf2f(v & 0xffffu);
  b = bf2f(v >> 16);
}

// Per-expert tile pointers the plan builder copies into ActiveRec.
struct ExpertTiles {
  const uint8_t* up;
  const uint8_t* down;
  const uint8_t* up_lr;
  const uint8_t* down_lr;
  int up_lr_bytes, down_lr_bytes;
};

__device__ __noinline__ void build_plan_block(const PlanArgs& pa, const int32_t* tk_idx,
                                              const float* tk_w, const uint8_t* hc,
                                              const ExpertTiles* et, int B, int k);
__device__ __noinline__ void build_plan_warp(const PlanArgs& pa, const int32_t* tk_idx,
                                             const float* tk_w, const uint8_t* hc,
                                             const ExpertTiles* et, int B, int k);

// Scratch of the warm-up warp: select + warp plan run once on dummy data while
// the logits are computed, so the leader's serial tail finds its code in the
// SM's instruction cache (a cold line costs an L2 round trip, ~150 ns each).
struct WarmScratch {
  double lg[LRC_MAX_EXPERTS + 64];
  int32_t idx[64];
  float w[64];
  int pe[32], pt[32], pc[32], pl[32], cl[32], act[32], aoff[32], acnt[32], cnt[4];
  float pw[32];
  ActiveRec arec[32];
};
__device__ __noinline__ void warm_tail(const RouteArgs& ra, WarmScratch& ws, const uint8_t* hc,
                                       const ExpertTiles* et, bool exact);

template <typename T>
__global__ void __launch_bounds__(kRThreads + 32) route_kernel(const __grid_constant__ RouteArgs ra) {
  extern __shared__ __align__(16) uint8_t rsm[];  // leader: [kTT][E+64] f64 logits | aux: x tile
  __shared__ double s_red[kTT][kRThreads / 32];
  __shared__ int s_last;
  __shared__ int32_t s_tidx[kTT * 64];
  __shared__ float s_tw[kTT * 64];
  __shared__ uint8_t s_hc[LRC_MAX_EXPERTS];
  __shared__ ExpertTiles s_et[LRC_MAX_EXPERTS];
  __shared__ WarmScratch s_warm;
  const int rank = static_cast<int>(cl_rank());
  const int tile = blockIdx.x / kCl, ntiles = gridDim.x / kCl, row = blockIdx.y;
  const int64_t b0 = static_cast<int64_t>(tile) * kTT;
  const int64_t rem = ra.B - b0;
  const int nb = rem < kTT ? static_cast<int>(rem) : kTT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T* x = static_cast<const T*>(ra.x);
  RSTAMP(0);
  // Dependents (the up kernel) are released only after this grid's own
  // griddepcontrol.wait: a running up kernel then implies the previous layer is
  // complete, so it may read x and build its activation operand before it waits
  // for the routing.
  if (!ra.pdl) griddep_launch_dependents_r();
  // single-token decode: the leader's extra warp owns the whole tail (select +
  // plan).  It runs both on dummy data while the logits are computed, so its
  // SMSP's instruction cache holds them when the logits land (the tail is
  // otherwise ~6 us of cold instruction fetches on the layer's critical path).
  const bool tailw = ntiles == 1 && nb == 1 && ra.plan.ticket != nullptr && ra.pairs_expert == nullptr &&
                     ra.probs == nullptr && ra.E <= 32 && ra.k <= ra.E &&
                     ra.k + (ra.plan.comp_rows ? 0 : ra.plan.num_shared) <= 32;
  if (warp == kRThreads / 32) {  // the extra warp: leader of a row-0 cluster only
    if (row == 0) {
      // arrive on the cluster barrier first: the logits handoff must not wait
      // for this warp's cold instruction fetches
      asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
      if (rank == 0 && tailw) {
        auto tstamp = [&](int k) {
          if ((ra.stamp & 1) && lane == 0) {
            unsigned long long t_;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
            g_route_stamps[blockIdx.x * 8 + k] = t_;
          }
        };
        warm_tail(ra, s_warm, s_hc, s_et, false);
        tstamp(7);
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // every logit landed
        tstamp(4);
        double* lg = reinterpret_cast<double*>(rsm);
        if (!select_topk_fast(lg, ra.E, ra.k, ra.renorm, b0, ra.topk_idx, ra.topk_w, s_tidx, s_tw))
          select_topk_warp(lg, ra.E, ra.k, ra.renorm, b0, ra.probs, ra.topk_idx, ra.topk_w, s_tidx, s_tw);
        __syncwarp();
        tstamp(2);
        build_plan_warp(ra.plan, s_tidx, s_tw, s_hc, s_et, static_cast<int>(ra.B), ra.k);
        if ((ra.stamp & 1) && lane == 0) {
          unsigned long long t_;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
          g_route_stamps[blockIdx.x * 8 + 5] = t_;
        }
      } else if (rank == 0 && ra.plan.ticket != nullptr && (ra.stamp & 2)) {
        warm_tail(ra, s_warm, s_hc, s_et, true);  // (debug: warm-up only)
      }
    }
    return;
  }
  if (row > 0) {
    // ---- aux CTAs: speculative V.x rows (single tile) + zeroing of the outputs
    if (ra.pdl) {  // x, y and t belong to the previous kernel until here
      griddep_wait_r();
      griddep_launch_dependents_r();
    }
    RSTAMP(2);
    const int aux = (row - 1) * kCl + rank, naux = (gridDim.y - 1) * kCl;
    if (ra.y_zero != nullptr) {
      const int64_t n = static_cast<int64_t>(nb) * ra.d;
      for (int64_t i = static_cast<int64_t>(aux) * kRThreads + threadIdx.x; i < n;
           i += static_cast<int64_t>(naux) * kRThreads)
        ra.y_zero[b0 * ra.d + i] = 0.0f;
    }
    if (ra.t2_zero != nullptr && ra.maxr > 0) {
      const int n = nb * ra.ne * ra.maxr;
      for (int i = aux * kRThreads + threadIdx.x; i < n; i += naux * kRThreads) {
        const int t = i / (ra.ne * ra.maxr), r2 = i - t * ra.ne * ra.maxr;
        const int e = r2 / ra.maxr, j = r2 - e * ra.maxr;
        ra.t2_zero[(((b0 + t) * ra.ne + e) * 3 + 2) * ra.maxr + j] = 0.0f;
      }
    }
    if constexpr (sizeof(T) == 2) {
      if (ra.spec_blocks > 0 && aux < ra.ne * ra.spec_blocks) {
        // stage the tile's token rows (padded: 64-column groups at a stride of
        // 33 words, so lanes that each walk their own group hit distinct banks)
        uint16_t* xs = reinterpret_cast<uint16_t*>(rsm);
        const uint16_t* xg = reinterpret_cast<const uint16_t*>(x) + b0 * ra.d;
        const int ldx = xs_row_elems(ra.d);
        if ((ra.d % 64) == 0 && (reinterpret_cast<uintptr_t>(xg) & 3) == 0) {
          const int wpr = ra.d / 2;  // words per token row
          uint32_t* xs32 = reinterpret_cast<uint32_t*>(xs);
          const uint32_t* xg32 = reinterpret_cast<const uint32_t*>(xg);
          constexpr int U = 8;  // loads in flight per thread: one round trip per 8 KB
          for (int base = 0; base < nb * wpr; base += U * kRThreads) {
            uint32_t v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int i = base + u * kRThreads + threadIdx.x;
              v[u] = i < nb * wpr ? __ldg(xg32 + i) : 0u;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int i = base + u * kRThreads + threadIdx.x;
              if (i < nb * wpr) {
                const int t = i / wpr, w = i - t * wpr;
                xs32[t * (ldx / 2) + (w >> 5) * 33 + (w & 31)] = v[u];
              }
            }
          }
        } else {
          for (int i = threadIdx.x; i < nb * ra.d; i += kRThreads) {
            const int t = i / ra.d, c = i - t * ra.d;
            xs[t * ldx + xs_col(c)] = xg[i];
          }
        }
        wsync();
        RSTAMP(3);
        // per (token, 64-column group) sums of x for the zero-point term
        float* xsum = reinterpret_cast<float*>(rsm + kTT * ldx * 2);
        const int gpr = (ra.d + 63) / 64;
        if (gpr <= 64)
          for (int i = threadIdx.x; i < nb * gpr; i += kRThreads) {
            const int t = i / gpr, g = i - t * gpr;
            const uint32_t* r = reinterpret_cast<const uint32_t*>(xs) + t * (ldx / 2) + g * 33;
            const int nw = min(32, (ra.d - g * 64 + 1) / 2);
            float a = 0.0f;
            for (int q = 0; q < nw; ++q) a += __uint_as_float(r[q] << 16) + __uint_as_float(r[q] & 0xffff0000u);
            xsum[t * 64 + g] = a;
          }
        wsync();
        RSTAMP(4);
        spec_lr_rows(ra, xs, xsum, b0, nb, aux % ra.ne, aux / ra.ne);
      }
    }
    RSTAMP(1);
    return;
  }
  // ---- logits: cluster CTA `rank` takes experts rank, rank + kCl, ...; every
  // gate load of a row is in flight at once (pairs, 8 per thread for d = 4096)
  const bool leader = rank == 0;
  const int NE = ra.plan.num_experts + ra.plan.num_shared;
  if (rank == 1 && ra.plan.ticket != nullptr) {
    // plan inputs for the leader, fetched by a helper CTA while the leader
    // computes its logits, stored into the leader's shared memory (DSMEM)
    for (int e = threadIdx.x; e < NE; e += kRThreads) {
      st_cl_u8(&s_hc[e], 0, ra.plan.has_comp[e]);
      if (ra.plan.arec != nullptr) {
        const lrc_expert& X = ra.plan.experts[e];
        const LrLayout L = lr_layout(X);
        const ExpertTiles et{X.up_tiles, X.down_tiles, X.up_lr_tiles, X.down_lr_tiles, L.up_total, L.down_total};
        static_assert(sizeof(ExpertTiles) == 40, "ExpertTiles layout");
        const uint64_t* src = reinterpret_cast<const uint64_t*>(&et);
        uint64_t* dst = reinterpret_cast<uint64_t*>(&s_et[e]);
#pragma unroll
        for (int q = 0; q < 5; ++q) st_cl_u64(dst + q, 0, src[q]);
      }
    }
  }
  if (ra.pdl) {
    // the gate rows are constant: pull this CTA's into L1 while the previous
    // kernel drains, then wait before reading x
    for (int e = rank; e < ra.E; e += kCl)
      for (int l = threadIdx.x; l < (ra.d * 8 + 127) / 128; l += kRThreads)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(ra.gate_t + static_cast<int64_t>(e) * ra.d + l * 16));
    griddep_wait_r();
    griddep_launch_dependents_r();
  }
  double* lg = reinterpret_cast<double*>(rsm);  // leader's layout: per token E weights + 64 scratch
  const int ldl = ra.E + 64;
  for (int e = rank; e < (ra.pairs_expert != nullptr ? 0 : ra.E); e += kCl) {
    const double* g = ra.gate_t + static_cast<int64_t>(e) * ra.d;
    double acc[kTT];
#pragma unroll
    for (int t = 0; t < kTT; ++t) acc[t] = 0.0;
    if ((ra.d & 1) == 0) {
      // explicit batches: the U gate pairs and U x pairs per token are all in
      // flight before the first use (a runtime-bounded loop would serialise)
      constexpr int U = 8;
      const int np = ra.d >> 1;
      for (int base = 0; base < np; base += U * kRThreads) {
        double2 gv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i2 = base + u * kRThreads + threadIdx.x;
          gv[u] = i2 < np ? __ldg(reinterpret_cast<const double2*>(g) + i2) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int t = 0; t < kTT; ++t)
          if (t < nb) {
            double xa[U], xb[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const int i2 = base + u * kRThreads + threadIdx.x;
              if (i2 < np) {
                load_x2<T>(x, (b0 + t) * ra.d + 2 * i2, xa[u], xb[u]);
              } else {
                xa[u] = xb[u] = 0.0;
              }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) acc[t] = fma(gv[u].y, xb[u], fma(gv[u].x, xa[u], acc[t]));
          }
      }
    } else {
      for (int i = threadIdx.x; i < ra.d; i += kRThreads) {
        const double gv = __ldg(g + i);
#pragma unroll
        for (int t = 0; t < kTT; ++t)
          if (t < nb) acc[t] = fma(gv, load_x<T>(x, (b0 + t) * ra.d + i), acc[t]);
      }
    }
    if (rank != 0) RSTAMP(3);
#pragma unroll
    for (int t = 0; t < kTT; ++t) {
      const double v = warp_sum_d(acc[t]);
      if (lane == 0) s_red[t][warp] = v;
    }
    wsync();
    if (rank != 0) RSTAMP(4);
    if (threadIdx.x < nb) {
      double sum = 0.0;
      for (int w = 0; w < kRThreads / 32; ++w) sum += s_red[threadIdx.x][w];
      st_cl_f64(lg + threadIdx.x * ldl + e, 0, sum);  // into the leader's shared memory
    }
    wsync();
    if (rank != 0) RSTAMP(5);
  }
  cl_sync();  // release/acquire: the leader sees every logit
  RSTAMP(6);
  if (!leader || tailw) return;
  // ---- leader: softmax + top-k (warp per token), then the pair plan
  if (ra.pairs_expert != nullptr) {  // pairs mode: the routing is given (k = 1)
    if (threadIdx.x < nb) {
      const int32_t e = ra.pairs_expert[b0 + threadIdx.x];
      const float w = ra.pairs_w[b0 + threadIdx.x];
      s_tidx[threadIdx.x] = e;
      s_tw[threadIdx.x] = w;
      ra.topk_idx[b0 + threadIdx.x] = e;
      ra.topk_w[b0 + threadIdx.x] = w;
    }
  } else if (warp < nb) {
    if (ra.probs == nullptr && ra.E <= 32 && ra.k <= ra.E &&
        select_topk_fast(lg + warp * ldl, ra.E, ra.k, ra.renorm, b0 + warp, ra.topk_idx, ra.topk_w,
                         s_tidx + warp * ra.k, s_tw + warp * ra.k)) {
      // done (exact selection, fp32 weights)
    } else
    select_topk_warp(lg + warp * ldl, ra.E, ra.k, ra.renorm, b0 + warp, ra.probs, ra.topk_idx,
                     ra.topk_w, s_tidx + warp * ra.k, s_tw + warp * ra.k,
                     ((ra.stamp & 1) && warp == 0 && blockIdx.y * gridDim.x + blockIdx.x < kStampCtas)
                         ? &g_route_stamps[(blockIdx.y * gridDim.x + blockIdx.x) * 8 + 2]
                         : nullptr);
  }
  RSTAMP(3);
  if (ra.plan.ticket == nullptr) return;
  wsync();
  if (ntiles == 1) {  // decode: the whole plan from shared memory, no ticket
    if (ra.B * (ra.k + (ra.plan.comp_rows ? 0 : ra.plan.num_shared)) <= 32) {
      if (warp == 0) build_plan_warp(ra.plan, s_tidx, s_tw, s_hc, s_et, static_cast<int>(ra.B), ra.k);
    } else {
      build_plan_block(ra.plan, s_tidx, s_tw, s_hc, s_et, static_cast<int>(ra.B), ra.k);
    }
    RSTAMP(5);
    return;
  }
  // several token tiles: the last leader builds the plan from the global top-k
  __threadfence();
  wsync();
  if (threadIdx.x == 0) s_last = (atomicAdd(ra.plan.ticket, 1) == ntiles - 1);
  wsync();
  RSTAMP(4);
  if (!s_last) return;
  __threadfence();
  build_plan_block(ra.plan, ra.topk_idx, ra.topk_w, s_hc, s_et, static_cast<int>(ra.B), ra.k);
  if (threadIdx.x == 0) *ra.plan.ticket = 0;
  RSTAMP(5);
}

// Pair plan: pair p = b*P + j, P = k + S.  j < k: routed expert tk_idx[b][j],
// weight tk_w, compensated iff j < n.  j >= k: shared expert E + (j-k),
// weight 1, compensated iff compensate_shared (ref/moe.py:249-258).
// Pairs are grouped by expert, ascending pair id inside each expert (stable).
// tk_idx / tk_w may point to shared (single tile) or global memory; hc and et
// are the has-comp flags and tile pointers staged in shared memory.
__device__ __noinline__ void build_plan_block(const PlanArgs& pa, const int32_t* tk_idx,
                                              const float* tk_w, const uint8_t* hc,
                                              const ExpertTiles* et, int B, int k) {
  const int P = k + (pa.comp_rows ? 0 : pa.num_shared);  // pairs mode: no implicit shared pairs
  const int NP = B * P;
  const int NE = pa.num_experts + pa.num_shared;
  __shared__ int s_cnt[LRC_MAX_EXPERTS];
  __shared__ int s_off[LRC_MAX_EXPERTS + 1];
  __shared__ int s_start[LRC_MAX_EXPERTS];
  __shared__ int s_act[LRC_MAX_EXPERTS];
  __shared__ uint32_t s_cm[LRC_MAX_EXPERTS];
  __shared__ int s_na;
  for (int e = threadIdx.x; e < NE; e += kRThreads) {
    s_cnt[e] = 0;
    s_cm[e] = 0;
  }
  wsync();
  auto pair_of = [&](int p, int& e, float& w) {
    const int b = p / P, j = p - b * P;
    if (j < k) {
      e = tk_idx[b * k + j];
      w = tk_w[b * k + j];
    } else {
      e = pa.num_experts + (j - k);
      w = 1.0f;
    }
  };
  for (int p = threadIdx.x; p < NP; p += kRThreads) {
    int e;
    float w;
    pair_of(p, e, w);
    pa.pair_expert[p] = e;
    pa.pair_w[p] = w;
    pa.pair_token[p] = p / P;
    atomicAdd(&s_cnt[e], 1);
  }
  wsync();
  if (threadIdx.x == 0) {
    int acc = 0, na = 0;
    for (int e = 0; e < NE; ++e) {
      s_off[e] = acc;
      s_start[e] = acc;
      if (s_cnt[e] > 0) {
        pa.active[na] = e;
        pa.active_off[na] = acc;
        pa.active_cnt[na] = s_cnt[e];
        s_act[na++] = e;
      }
      acc += s_cnt[e];
    }
    s_off[NE] = acc;
    s_na = na;
    pa.counts[0] = na;
  }
  wsync();
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    // stable scatter: one warp walks the pairs in order; experts present in a
    // 32-pair chunk are serialised and each advances by its ballot prefix
    int count = 0;
    for (int base = 0; base < NP; base += 32) {
      const int p = base + lane;
      const bool valid = p < NP;
      int e = -1;
      float w;
      if (valid) pair_of(p, e, w);
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
        comp = (j < k) ? ((pa.comp_rows != nullptr ? pa.comp_rows[p / P] != 0 : j < pa.top_n) && hc[e])
                       : (pa.compensate_shared && hc[e]);
      }
      const unsigned m = __ballot_sync(0xffffffffu, comp);
      if (valid) {
        const int slot = comp ? count + __popc(m & ((1u << lane) - 1u)) : -1;
        pa.pair_comp[p] = slot;
        if (comp) {
          pa.comp_list[slot] = p;
          atomicOr(&s_cm[e], 1u << min((pos - s_start[e]) >> 3, 31));
        }
      }
      count += __popc(m);
    }
    if (lane == 0) pa.counts[1] = count;
  }
  if (pa.arec == nullptr) return;
  wsync();
  for (int a = threadIdx.x; a < s_na; a += kRThreads) {
    const int e = s_act[a];
    const ExpertTiles& T = et[e];
    ActiveRec R;
    R.up_tiles = T.up;
    R.down_tiles = T.down;
    R.up_lr_tiles = T.up_lr;
    R.down_lr_tiles = T.down_lr;
    R.e = e;
    R.off = s_start[e];
    R.cnt = s_cnt[e];
    R.cmask = s_cm[e];
    R.up_lr_bytes = T.up_lr_bytes;
    R.down_lr_bytes = T.down_lr_bytes;
    R.pad[0] = R.pad[1] = 0;
    pa.arec[a] = R;
  }
}

// Decode plan (B * (k + S) <= 32 pairs): one pair per lane, warp-synchronous
// (match / ballot / reduce), same output as build_plan_block.
__device__ __noinline__ void build_plan_warp(const PlanArgs& pa, const int32_t* tk_idx,
                                             const float* tk_w, const uint8_t* hc,
                                             const ExpertTiles* et, int B, int k) {
  const int lane = threadIdx.x & 31;
  const int P = k + (pa.comp_rows ? 0 : pa.num_shared), NP = B * P;
  const bool valid = lane < NP;
  int e = 0x7fffffff, j = 0;
  if (valid) {
    const int b = lane / P;
    j = lane - b * P;
    float w;
    if (j < k) {
      e = tk_idx[b * k + j];
      w = tk_w[b * k + j];
    } else {
      e = pa.num_experts + (j - k);
      w = 1.0f;
    }
    pa.pair_expert[lane] = e;
    pa.pair_w[lane] = w;
    pa.pair_token[lane] = b;
  }
  const unsigned same = __match_any_sync(0xffffffffu, e);  // lanes of my expert, in pair order
  const int cnt = __popc(same), rk = __popc(same & ((1u << lane) - 1u));
  int off = 0, nbelow = 0;  // pairs / distinct experts with a smaller id
  if (pa.num_experts + pa.num_shared <= 32) {
    // per-expert pair counts by ballot (lane x: expert x), exclusive scan over
    // the lanes, one gather: a short dependency chain instead of 32 rounds
    int cx = 0;
#pragma unroll
    for (int x = 0; x < 32; ++x) {
      const unsigned bx = __ballot_sync(0xffffffffu, valid && e == x);
      if (lane == x) cx = __popc(bx);
    }
    int incl = cx;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const unsigned present = __ballot_sync(0xffffffffu, cx > 0);
    off = __shfl_sync(0xffffffffu, incl - cx, e & 31);
    nbelow = __popc(present & ((1u << (e & 31)) - 1u));
  } else {
    for (int q = 0; q < 32; ++q) {
      const int eq = __shfl_sync(0xffffffffu, e, q);
      const unsigned sq = __shfl_sync(0xffffffffu, same, q);
      off += eq < e;
      nbelow += (eq < e) && ((sq & ((1u << q) - 1u)) == 0u);
    }
  }
  const bool row_comp = pa.comp_rows != nullptr ? (valid && pa.comp_rows[lane / P] != 0) : j < pa.top_n;
  const bool comp = valid && ((j < k) ? (row_comp && hc[e] != 0) : (pa.compensate_shared && hc[e] != 0));
  const unsigned cm = __ballot_sync(0xffffffffu, comp);
  if (valid) {
    pa.pair_list[off + rk] = lane;
    const int slot = comp ? __popc(cm & ((1u << lane) - 1u)) : -1;
    pa.pair_comp[lane] = slot;
    if (comp) pa.comp_list[slot] = lane;
  }
  const uint32_t cmask = __reduce_or_sync(same, comp ? (1u << min(rk >> 3, 31)) : 0u);
  const bool first = valid && rk == 0;
  if (first) {
    pa.active[nbelow] = e;
    pa.active_off[nbelow] = off;
    pa.active_cnt[nbelow] = cnt;
    if (pa.arec != nullptr) {
      const ExpertTiles& T = et[e];
      ActiveRec R;
      R.up_tiles = T.up;
      R.down_tiles = T.down;
      R.up_lr_tiles = T.up_lr;
      R.down_lr_tiles = T.down_lr;
      R.e = e;
      R.off = off;
      R.cnt = cnt;
      R.cmask = cmask;
      R.up_lr_bytes = T.up_lr_bytes;
      R.down_lr_bytes = T.down_lr_bytes;
      R.pad[0] = R.pad[1] = 0;
      pa.arec[nbelow] = R;
    }
  }
  const int na = __popc(__ballot_sync(0xffffffffu, first));
  if (lane == 0) {
    pa.counts[0] = na;
    pa.counts[1] = __popc(cm);
  }
}

__device__ __noinline__ void warm_tail(const RouteArgs& ra, WarmScratch& ws, const uint8_t* hc,
                                       const ExpertTiles* et, bool exact) {
  const int lane = threadIdx.x & 31;
  const int E = min(ra.E, LRC_MAX_EXPERTS);
  for (int e = lane; e < E; e += 32) ws.lg[e] = 0.001 * e;
  __syncwarp();
  if (E <= 32 && ra.k <= E) select_topk_fast(ws.lg, E, ra.k, ra.renorm, 0, ws.idx, ws.w, ws.idx, ws.w);
  __syncwarp();
  if (exact) select_topk_warp(ws.lg, E, ra.k, ra.renorm, 0, nullptr, ws.idx, ws.w, ws.idx, ws.w);
  __syncwarp();
  PlanArgs d = ra.plan;  // same scalars, outputs redirected to the scratch
  d.pair_expert = ws.pe;
  d.pair_w = ws.pw;
  d.pair_token = ws.pt;
  d.pair_comp = ws.pc;
  d.pair_list = ws.pl;
  d.comp_list = ws.cl;
  d.active = ws.act;
  d.active_off = ws.aoff;
  d.active_cnt = ws.acnt;
  d.counts = ws.cnt;
  d.arec = ws.arec;
  if (ra.k + ra.plan.num_shared <= 32) build_plan_warp(d, ws.idx, ws.w, hc, et, 1, ra.k);
}

int route_tiles(int64_t B) { return static_cast<int>((B + kTT - 1) / kTT); }

// --------------------------------------------------- large-batch routing ---
// The cluster router is latency-tuned for decode (one 8-CTA cluster per 8
// tokens).  For large batches: a block per 32 tokens computes all their
// logits as fp64 dot products (one (token, expert) pair per thread and pass;
// x and gate chunks staged through padded shared memory), then the same
// warp softmax + stable top-k as the leader (ref/moe.py:165-193); it also
// zeroes the outputs the expert kernels accumulate into.  The pair plan then
// comes from the parallel counting sort below.
constexpr int kBT = 32;  // tokens per bulk-router block

__host__ __device__ inline int bulk_chunk(int E) {  // d columns per staged chunk
  int c = 8192 / (E > 0 ? E : 1);
  c = c > 256 ? 256 : c;
  return c < 16 ? 16 : (c & ~15);
}
static size_t bulk_smem(int E) {
  const int c = bulk_chunk(E);
  return (static_cast<size_t>(E) * (c + 1) + kBT * (c + 1) + kBT * (E + 64)) * sizeof(double) +
         8 * 64 * (sizeof(int32_t) + sizeof(float));
}

template <typename T, int kMaxPJ>  // kMaxPJ >= ceil(kBT * E / 256) (token, expert) pairs per thread
__global__ void __launch_bounds__(256) route_bulk_kernel(const __grid_constant__ RouteArgs ra) {
  extern __shared__ __align__(16) double bsm[];
  const int E = ra.E, d = ra.d, tid = threadIdx.x, warp = tid >> 5;
  const int64_t b0 = static_cast<int64_t>(blockIdx.x) * kBT;
  const int64_t rem = ra.B - b0;
  const int nb = rem < kBT ? static_cast<int>(rem) : kBT;
  if (ra.y_zero != nullptr) {
    float* yz = ra.y_zero + b0 * d;
    const int64_t n = static_cast<int64_t>(nb) * d;
    if ((d & 3) == 0 && (reinterpret_cast<uintptr_t>(ra.y_zero) & 15) == 0) {
      for (int64_t i = tid; i < n / 4; i += blockDim.x)
        reinterpret_cast<float4*>(yz)[i] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    } else {
      for (int64_t i = tid; i < n; i += blockDim.x) yz[i] = 0.0f;
    }
  }
  if (ra.t2_zero != nullptr && ra.maxr > 0) {
    const int n = nb * ra.ne * ra.maxr;
    for (int i = tid; i < n; i += blockDim.x) {
      const int t = i / (ra.ne * ra.maxr), r2 = i - t * ra.ne * ra.maxr;
      const int e = r2 / ra.maxr, j = r2 - e * ra.maxr;
      ra.t2_zero[(((b0 + t) * ra.ne + e) * 3 + 2) * ra.maxr + j] = 0.0f;
    }
  }
  if (ra.pairs_expert != nullptr) {  // pairs mode: the routing is given (k = 1)
    if (tid < nb) {
      ra.topk_idx[b0 + tid] = ra.pairs_expert[b0 + tid];
      ra.topk_w[b0 + tid] = ra.pairs_w[b0 + tid];
    }
    return;
  }
  const int C = bulk_chunk(E), ldg = C + 1;
  double* gs = bsm;                        // [E][C + 1]
  double* xs = gs + static_cast<size_t>(E) * ldg;  // [kBT][C + 1]
  double* lg = xs + kBT * ldg;             // [kBT][E + 64]
  int32_t* sidx = reinterpret_cast<int32_t*>(lg + kBT * (E + 64));
  float* sw = reinterpret_cast<float*>(sidx + 8 * 64);
  const T* x = static_cast<const T*>(ra.x);
  const int npairs = kBT * E;
  // four interleaved partial sums per (token, expert): independent fp64 FMA
  // chains (a single chain is latency-bound); fixed, deterministic order
  double acc[kMaxPJ][4];
#pragma unroll
  for (int j = 0; j < kMaxPJ; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[j][q] = 0.0;
  for (int k0 = 0; k0 < d; k0 += C) {
    const int cw = min(C, d - k0);
    for (int i = tid; i < E * C; i += blockDim.x) {
      const int e = i / C, c = i - e * C;
      gs[e * ldg + c] = c < cw ? ra.gate_t[static_cast<int64_t>(e) * d + k0 + c] : 0.0;
    }
    for (int i = tid; i < kBT * C; i += blockDim.x) {
      const int t = i / C, c = i - t * C;
      xs[t * ldg + c] = (t < nb && c < cw) ? load_x(x, (b0 + t) * d + k0 + c) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kMaxPJ; ++j) {
      const int pr = tid + j * 256;
      if (pr < npairs) {
        const int t = pr / E, e = pr - t * E;
        const double* xr = xs + t * ldg;
        const double* gr = gs + e * ldg;
        double a0 = acc[j][0], a1 = acc[j][1], a2 = acc[j][2], a3 = acc[j][3];
        int c = 0;
        for (; c + 3 < cw; c += 4) {
          a0 = fma(xr[c], gr[c], a0);
          a1 = fma(xr[c + 1], gr[c + 1], a1);
          a2 = fma(xr[c + 2], gr[c + 2], a2);
          a3 = fma(xr[c + 3], gr[c + 3], a3);
        }
        for (; c < cw; ++c) a0 = fma(xr[c], gr[c], a0);
        acc[j][0] = a0;
        acc[j][1] = a1;
        acc[j][2] = a2;
        acc[j][3] = a3;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < kMaxPJ; ++j) {
    const int pr = tid + j * 256;
    if (pr < npairs) {
      const int t = pr / E, e = pr - t * E;
      lg[t * (E + 64) + e] = (acc[j][0] + acc[j][1]) + (acc[j][2] + acc[j][3]);
    }
  }
  __syncthreads();
  for (int t = warp; t < nb; t += blockDim.x / 32)
    select_topk_warp(lg + t * (E + 64), E, ra.k, ra.renorm, b0 + t, ra.probs, ra.topk_idx, ra.topk_w,
                     sidx + warp * 64, sw + warp * 64);
}

template <typename T>
static lrc_status launch_route_bulk_t(const RouteArgs& ra, size_t smem, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>((ra.B + kBT - 1) / kBT);
  const int pj = (kBT * ra.E + 255) / 256;
  auto go = [&](auto kern) -> lrc_status {
    static size_t configured = 0;  // per instantiation
    if (configured < smem) {
      LRC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      configured = smem;
    }
    kern<<<grid, 256, smem, st>>>(ra);
    LRC_CHECK_LAUNCH();
    return LRC_OK;
  };
  if (pj <= 1) return go(route_bulk_kernel<T, 1>);
  if (pj <= 2) return go(route_bulk_kernel<T, 2>);
  if (pj <= 8) return go(route_bulk_kernel<T, 8>);
  return go(route_bulk_kernel<T, 32>);
}

lrc_status launch_route_bulk(const RouteArgs& ra, cudaStream_t st) {
  if (ra.E > 256 || ra.k > 64) return fail(LRC_ERR_UNSUPPORTED, "bulk route: E <= 256, k <= 64");
  const size_t smem = bulk_smem(ra.E);
  switch (ra.x_dtype) {
    case LRC_DTYPE_F64: return launch_route_bulk_t<double>(ra, smem, st);
    case LRC_DTYPE_F32: return launch_route_bulk_t<float>(ra, smem, st);
    case LRC_DTYPE_BF16: return launch_route_bulk_t<uint16_t>(ra, smem, st);
    default: return fail(LRC_ERR_INVALID, "route: unknown x dtype");
  }
}

// ---------------------------------------------- large-batch parallel plan ---
// Same output as build_plan_block (pairs grouped by expert, ascending pair id
// inside each expert; compensated slots in pair order), as a counting sort over
// 1024-pair chunks: per-chunk histograms, then a stable scatter whose offsets
// are the chunk prefix sums; the last chunk writes the active lists and
// records.  Replaces the serial single-CTA plan when B * P is large.
constexpr int kPlanChunk = 1024;

__device__ __forceinline__ void plan_pair(const PlanArgs& pa, const int32_t* tk_idx, const float* tk_w, int k,
                                          int P, int p, int& e, float& w, bool& comp) {
  const int b = p / P, j = p - b * P;
  if (j < k) {
    e = tk_idx[b * k + j];
    w = tk_w[b * k + j];
  } else {
    e = pa.num_experts + (j - k);
    w = 1.0f;
  }
  comp = (j < k) ? ((pa.comp_rows != nullptr ? pa.comp_rows[b] != 0 : j < pa.top_n) && pa.has_comp[e])
                 : (pa.compensate_shared && pa.has_comp[e]);
}

__global__ void __launch_bounds__(kPlanChunk) plan_count_kernel(const PlanArgs pa, const int32_t* tk_idx,
                                                                const float* tk_w, int B, int k, int* blk) {
  const int P = k + (pa.comp_rows ? 0 : pa.num_shared), NP = B * P, NE = pa.num_experts + pa.num_shared;
  __shared__ int cnt[LRC_MAX_EXPERTS + 1];
  for (int e = threadIdx.x; e <= NE; e += blockDim.x) cnt[e] = 0;
  __syncthreads();
  const int p = blockIdx.x * kPlanChunk + threadIdx.x;
  if (p < NP) {
    int e;
    float w;
    bool comp;
    plan_pair(pa, tk_idx, tk_w, k, P, p, e, w, comp);
    pa.pair_expert[p] = e;
    pa.pair_w[p] = w;
    pa.pair_token[p] = p / P;
    atomicAdd(&cnt[e], 1);
    if (comp) atomicAdd(&cnt[NE], 1);
  }
  __syncthreads();
  for (int e = threadIdx.x; e <= NE; e += blockDim.x) blk[blockIdx.x * (NE + 1) + e] = cnt[e];
}

__global__ void __launch_bounds__(kPlanChunk) plan_scatter_kernel(const PlanArgs pa, const int32_t* tk_idx,
                                                                  const float* tk_w, int B, int k, const int* blk,
                                                                  uint32_t* cmask, int* ticket) {
  const int P = k + (pa.comp_rows ? 0 : pa.num_shared), NP = B * P, NE = pa.num_experts + pa.num_shared;
  const int nblk = gridDim.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ int total[LRC_MAX_EXPERTS + 1];
  __shared__ int start[LRC_MAX_EXPERTS + 1];
  __shared__ int base[LRC_MAX_EXPERTS + 1];
  __shared__ int wcnt[kPlanChunk / 32][LRC_MAX_EXPERTS + 1];
  __shared__ int s_last, s_na;
  __shared__ int s_act[LRC_MAX_EXPERTS];
  for (int e = threadIdx.x; e <= NE; e += blockDim.x) {
    int before = 0, all = 0;
    for (int b = 0; b < nblk; ++b) {
      const int c = blk[b * (NE + 1) + e];
      all += c;
      before += b < static_cast<int>(blockIdx.x) ? c : 0;
    }
    total[e] = all;
    base[e] = before;
  }
  for (int e = lane; e <= NE; e += 32) wcnt[warp][e] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int e = 0; e < NE; ++e) {
      start[e] = acc;
      acc += total[e];
    }
    start[NE] = 0;  // compensated slots start at 0
  }
  __syncthreads();
  for (int e = threadIdx.x; e <= NE; e += blockDim.x) base[e] += start[e];
  // per-warp histograms (ranks inside the warp from match_any)
  const int p = blockIdx.x * kPlanChunk + threadIdx.x;
  const bool valid = p < NP;
  int e = -1 - lane;
  float w = 0.0f;
  bool comp = false;
  if (valid) plan_pair(pa, tk_idx, tk_w, k, P, p, e, w, comp);
  const unsigned lt = (1u << lane) - 1u;
  const unsigned same = __match_any_sync(0xffffffffu, e);
  const unsigned cm = __ballot_sync(0xffffffffu, comp);
  if (valid && (same & lt) == 0) wcnt[warp][e] = __popc(same);
  if (lane == 0) wcnt[warp][NE] = __popc(cm);
  __syncthreads();
  for (int x = threadIdx.x; x <= NE; x += blockDim.x) {  // exclusive scan over warps
    int acc = 0;
    for (int w2 = 0; w2 < kPlanChunk / 32; ++w2) {
      const int c = wcnt[w2][x];
      wcnt[w2][x] = acc;
      acc += c;
    }
  }
  __syncthreads();
  if (valid) {
    const int pos = base[e] + wcnt[warp][e] + __popc(same & lt);
    pa.pair_list[pos] = p;
    const int slot = comp ? base[NE] + wcnt[warp][NE] + __popc(cm & lt) : -1;
    pa.pair_comp[p] = slot;
    if (comp) {
      pa.comp_list[slot] = p;
      atomicOr(&cmask[e], 1u << min((pos - start[e]) >> 3, 31));
    }
  }
  // the last chunk publishes the active lists and per-expert records
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1) == nblk - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x == 0) {
    int na = 0;
    for (int x = 0; x < NE; ++x)
      if (total[x] > 0) {
        pa.active[na] = x;
        pa.active_off[na] = start[x];
        pa.active_cnt[na] = total[x];
        s_act[na++] = x;
      }
    pa.counts[0] = na;
    pa.counts[1] = total[NE];
    s_na = na;
    *ticket = 0;
  }
  __syncthreads();
  if (pa.arec != nullptr) {
    for (int a = threadIdx.x; a < s_na; a += blockDim.x) {
      const int x = s_act[a];
      const lrc_expert& X = pa.experts[x];
      const LrLayout L = lr_layout(X);
      ActiveRec R;
      R.up_tiles = X.up_tiles;
      R.down_tiles = X.down_tiles;
      R.up_lr_tiles = X.up_lr_tiles;
      R.down_lr_tiles = X.down_lr_tiles;
      R.e = x;
      R.off = start[x];
      R.cnt = total[x];
      R.cmask = *reinterpret_cast<volatile uint32_t*>(&cmask[x]);
      R.up_lr_bytes = L.up_total;
      R.down_lr_bytes = L.down_total;
      R.pad[0] = R.pad[1] = 0;
      pa.arec[a] = R;
    }
  }
  __syncthreads();
  for (int x = threadIdx.x; x < NE; x += blockDim.x) cmask[x] = 0;
}

int plan_parallel_blocks(int64_t np) { return static_cast<int>((np + kPlanChunk - 1) / kPlanChunk); }

lrc_status launch_plan_parallel(const PlanArgs& pa, const int32_t* tk_idx, const float* tk_w, int B, int k,
                                int* blk, uint32_t* cmask, int* ticket, cudaStream_t st) {
  const int P = k + (pa.comp_rows ? 0 : pa.num_shared);
  const int nblk = plan_parallel_blocks(static_cast<int64_t>(B) * P);
  if (nblk == 0) return LRC_OK;
  plan_count_kernel<<<nblk, kPlanChunk, 0, st>>>(pa, tk_idx, tk_w, B, k, blk);
  LRC_CHECK_LAUNCH();
  plan_scatter_kernel<<<nblk, kPlanChunk, 0, st>>>(pa, tk_idx, tk_w, B, k, blk, cmask, ticket);
  LRC_CHECK_LAUNCH();
  return LRC_OK;
}

lrc_status launch_route(const RouteArgs& ra_in, cudaStream_t st) {
  // debug knobs: bit 0 = %globaltimer stamps, bit 1 = no tail warm-up warp
  static const int stamps = (getenv("LRC_ROUTE_STAMPS") != nullptr ? 1 : 0) |
                            (getenv("LRC_ROUTE_NOWARM") != nullptr ? 2 : 0);
  RouteArgs ra = ra_in;
  ra.stamp = stamps;
  // leader: logits scratch (kTT tokens x (E + 64) doubles); aux CTAs: the bf16
  // x tile of the speculative V.x rows
  int smem = kTT * (ra.E + 64) * static_cast<int>(sizeof(double));
  if (ra.spec_blocks > 0) smem = max(smem, kTT * xs_row_elems(ra.d) * 2 + kTT * 64 * 4);
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
  // grid: x = token tiles x kCl (one cluster per tile), y = 1 + aux rows
  const int spec_rows = ra.spec_blocks > 0 ? (ra.ne * ra.spec_blocks + kCl - 1) / kCl : 0;
  const int zero_rows = (ra.y_zero != nullptr || ra.t2_zero != nullptr) ? 1 : 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(route_tiles(ra.B) * kCl, 1 + max(spec_rows, zero_rows), 1);
  cfg.blockDim = dim3(kRThreads + 32);  // + the warm-up warp
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ra.pdl ? 2 : 1;
  switch (ra.x_dtype) {
    case LRC_DTYPE_F64:
      LRC_CUDA_TRY(cudaLaunchKernelEx(&cfg, route_kernel<double>, ra));
      break;
    case LRC_DTYPE_F32:
      LRC_CUDA_TRY(cudaLaunchKernelEx(&cfg, route_kernel<float>, ra));
      break;
    case LRC_DTYPE_BF16:
      LRC_CUDA_TRY(cudaLaunchKernelEx(&cfg, route_kernel<uint16_t>, ra));
      break;
    default:
      return fail(LRC_ERR_INVALID, "route: unknown x dtype");
  }
  return LRC_OK;
}

}  // namespace lrc

extern "C" lrc_status lrc_debug_stamps(int which, uint64_t* host, int n) {
  using namespace lrc;
  if (which < 4 && (n < 0 || n > (which == 0 ? kStampCtas * 8 : 2 * 256 * 8 + 2 * 64 * 6)))
    return fail(LRC_ERR_INVALID, "stamps: bad count");
  LRC_CUDA_TRY(cudaDeviceSynchronize());
  if (which == 5) {
    if (n != 192) return fail(LRC_ERR_INVALID, "wstat: 192 values");
    tcd::wstat_copy(reinterpret_cast<unsigned long long*>(host));
    return LRC_OK;
  }
  if (which == 4) {  // debug: tcd wait mode = n
    tcd::set_wait_mode(n);
    return LRC_OK;
  }
  if (which == 3) {
    if (n != 2048) return fail(LRC_ERR_INVALID, "trace: 2048 values");
    tcd::trace_copy(host);
    return LRC_OK;
  }
  if (which == 2) {
    if (n > 148 * 16) return fail(LRC_ERR_INVALID, "stamps: bad count");
    tcd::stamps_copy(host, n);
    return LRC_OK;
  }
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
