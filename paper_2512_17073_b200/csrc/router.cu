// K1: fused router -- gate GEMV (fp64) + softmax + stable top-k/top-n, and the
// per-expert pair plan consumed by the expert kernels.
// Reference: ref/moe.py:165-193 (route/softmax), ref/moe.py:234-258 (mixing,
// shared experts).
#include <float.h>

#include "common.cuh"
#include "layer.cuh"

namespace lrc {

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

// Route one token per CTA.  Writes probs (optional), topk idx / mixing weight.
// When `plan` is non-null the last CTA to finish (atomic ticket) builds the
// pair plan for the whole batch (no extra launch).
template <typename T>
__global__ void __launch_bounds__(256) route_kernel(const double* __restrict__ gate_t,
                                                    const T* __restrict__ x, int64_t B, int d,
                                                    int E, int k, int renorm,
                                                    double* __restrict__ probs,
                                                    int32_t* __restrict__ topk_idx,
                                                    float* __restrict__ topk_w, PlanArgs plan) {
  extern __shared__ double sm[];
  double* xs = sm;           // d
  double* logit = sm + d;    // E
  const int64_t b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int i = threadIdx.x; i < d; i += blockDim.x) xs[i] = load_x<T>(x, b * d + i);
  __syncthreads();
  for (int e = warp; e < E; e += nw) {
    const double* gr = gate_t + static_cast<int64_t>(e) * d;
    double acc = 0.0;
    for (int i = lane; i < d; i += 32) acc = fma(gr[i], xs[i], acc);
    acc = warp_sum_d(acc);
    if (lane == 0) logit[e] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // softmax exactly as ref/moe.py:165-168: z = l - max; e = exp(z); e / sum(e)
    double mx = logit[0];
    for (int e = 1; e < E; ++e) mx = fmax(mx, logit[e]);
    for (int e = 0; e < E; ++e) logit[e] = exp(__dsub_rn(logit[e], mx));
    double den = pw_sum_small(logit, E);
    for (int e = 0; e < E; ++e) logit[e] = __ddiv_rn(logit[e], den);
    if (probs)
      for (int e = 0; e < E; ++e) probs[b * E + e] = logit[e];
    // stable descending selection: strict '>' keeps the lower index on ties
    // (np.argsort(-w, kind="stable"), ref/moe.py:190)
    unsigned long long taken[4] = {0, 0, 0, 0};
    double mix[64];
    int sel[64];
    double msum = 0.0;
    for (int j = 0; j < k; ++j) {
      int best = -1;
      double bv = -DBL_MAX;
      for (int e = 0; e < E; ++e) {
        if ((taken[e >> 6] >> (e & 63)) & 1ull) continue;
        if (best < 0 || logit[e] > bv) {
          best = e;
          bv = logit[e];
        }
      }
      taken[best >> 6] |= 1ull << (best & 63);
      sel[j] = best;
      mix[j] = bv;
    }
    if (renorm) {
      // mix.sum() in numpy order (pairwise over k values)
      msum = pw_sum_small(mix, k);
      if (msum > 0.0)
        for (int j = 0; j < k; ++j) mix[j] = __ddiv_rn(mix[j], msum);
    }
    for (int j = 0; j < k; ++j) {
      topk_idx[b * k + j] = sel[j];
      topk_w[b * k + j] = static_cast<float>(mix[j]);
    }
  }
  if (plan.ticket == nullptr) return;
  // ---- last CTA builds the plan ----
  __shared__ int is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = atomicAdd(plan.ticket, 1);
    is_last = (t == static_cast<int>(B) - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  build_plan_block(plan, topk_idx, topk_w, static_cast<int>(B), k);
  if (threadIdx.x == 0) *plan.ticket = 0;
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
  __shared__ int s_warp[32];
  __shared__ int s_ncomp;
  for (int e = threadIdx.x; e < NE; e += blockDim.x) s_cnt[e] = 0;
  if (threadIdx.x == 0) s_ncomp = 0;
  __syncthreads();
  // per-pair attributes
  for (int p = threadIdx.x; p < NP; p += blockDim.x) {
    int b = p / P, j = p - b * P;
    int e;
    float w;
    int comp;
    if (j < k) {
      e = topk_idx[b * k + j];
      w = topk_w[b * k + j];
      comp = (j < pa.top_n) && pa.has_comp[e];
    } else {
      e = pa.num_experts + (j - k);
      w = 1.0f;
      comp = pa.compensate_shared && pa.has_comp[e];
    }
    pa.pair_expert[p] = e;
    pa.pair_w[p] = w;
    pa.pair_token[p] = b;
    atomicAdd(&s_cnt[e], 1);
    (void)comp;
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
  // stable scatter: walk pairs in order, one warp-synchronous pass per chunk
  // of 32 pairs; each expert's cursor advances by the ballot prefix.
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    for (int base = 0; base < NP; base += 32) {
      int p = base + lane;
      int e = (p < NP) ? pa.pair_expert[p] : -1;
      int pos = -1;
      // serialise experts present in this chunk
      unsigned pending = __ballot_sync(0xffffffffu, p < NP);
      while (pending) {
        int leader = __ffs(pending) - 1;
        int le = __shfl_sync(0xffffffffu, e, leader);
        unsigned same = __ballot_sync(0xffffffffu, e == le && p < NP);
        if (e == le && p < NP) pos = s_off[le] + __popc(same & ((1u << lane) - 1u));
        __syncwarp();
        if (lane == leader) s_off[le] += __popc(same);
        __syncwarp();
        pending &= ~same;
      }
      if (p < NP) pa.pair_list[pos] = p;
    }
  }
  __syncthreads();
  // compensated-pair slots (for the t = V.x buffers), in pair order
  if (threadIdx.x < 32) {
    int count = 0;
    for (int base = 0; base < NP; base += 32) {
      int p = base + lane;
      int comp = 0;
      if (p < NP) {
        int b = p / P, j = p - b * P;
        int e = pa.pair_expert[p];
        comp = (j < k) ? ((j < pa.top_n) && pa.has_comp[e])
                       : (pa.compensate_shared && pa.has_comp[e]);
      }
      unsigned m = __ballot_sync(0xffffffffu, comp);
      if (p < NP) {
        int slot = comp ? count + __popc(m & ((1u << lane) - 1u)) : -1;
        pa.pair_comp[p] = slot;
        if (comp) pa.comp_list[slot] = p;
      }
      count += __popc(m);
    }
    if (lane == 0) pa.counts[1] = count;
  }
  (void)s_warp;
  (void)s_ncomp;
}

static int route_smem(int d, int E) { return (d + E) * static_cast<int>(sizeof(double)); }

lrc_status launch_route(const double* gate_t, const void* x, int x_dtype, int64_t B, int d, int E,
                        int k, int renorm, double* probs, int32_t* topk_idx, float* topk_w,
                        const PlanArgs& plan, cudaStream_t st) {
  int smem = route_smem(d, E);
  if (smem > 48 * 1024) {
    static const void* fns[3] = {(const void*)route_kernel<double>, (const void*)route_kernel<float>,
                                 (const void*)route_kernel<uint16_t>};
    for (auto f : fns) LRC_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  }
  dim3 grid(static_cast<unsigned>(B));
  switch (x_dtype) {
    case LRC_DTYPE_F64:
      route_kernel<double><<<grid, 256, smem, st>>>(gate_t, (const double*)x, B, d, E, k, renorm,
                                                    probs, topk_idx, topk_w, plan);
      break;
    case LRC_DTYPE_F32:
      route_kernel<float><<<grid, 256, smem, st>>>(gate_t, (const float*)x, B, d, E, k, renorm,
                                                   probs, topk_idx, topk_w, plan);
      break;
    case LRC_DTYPE_BF16:
      route_kernel<uint16_t><<<grid, 256, smem, st>>>(gate_t, (const uint16_t*)x, B, d, E, k,
                                                      renorm, probs, topk_idx, topk_w, plan);
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
  PlanArgs none{};
  return launch_route(gate_t, x, x_dtype, B, d, E, top_k, renormalize, probs, topk_idx, topk_w,
                      none, as_stream(stream));
}
