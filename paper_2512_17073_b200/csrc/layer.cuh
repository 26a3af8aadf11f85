// Device-side structures shared by the router, generic and tiled expert kernels.
#pragma once
#include "common.cuh"

#define LRC_MAX_EXPERTS 256

namespace lrc {

// Pair plan (see build_plan_block in router.cu).
struct PlanArgs {
  int* ticket;
  int num_experts, num_shared, top_n, compensate_shared;
  const uint8_t* has_comp;  // [E+S]
  int* pair_expert;         // [NP]
  float* pair_w;            // [NP]
  int* pair_token;          // [NP]
  int* pair_comp;           // [NP] slot into t buffers or -1
  int* pair_list;           // [NP] pairs grouped by expert
  int* comp_list;           // [NP] compensated pairs by slot
  int* active;              // [E+S] expert ids with >= 1 pair
  int* active_off;          // [E+S] offset into pair_list
  int* active_cnt;          // [E+S]
  int* counts;              // [0] n_active, [1] n_comp
};

__device__ void build_plan_block(const PlanArgs& pa, const int32_t* topk_idx,
                                 const float* topk_w, int B, int k);

lrc_status launch_route(const double* gate_t, const void* x, int x_dtype, int64_t B, int d, int E,
                        int k, int renorm, double* probs, int32_t* topk_idx, float* topk_w,
                        const PlanArgs& plan, cudaStream_t st);

// Arguments of the expert phases.
struct ExpertArgs {
  const lrc_expert* experts;  // device array [E+S]
  PlanArgs plan;
  int hidden, ffn, maxr;
  const uint16_t* x;          // [B][hidden] bf16
  float* t;                   // [NP][3][maxr]  (proj 0 = w1, 1 = w3, 2 = w2)
  float* a32;                 // [NP][ffn] generic path activations
  uint16_t* a16;              // [NP][ffn] bf16 activations (tiled path)
  float* y;                   // [B][hidden] (accumulated)
  int max_pairs;
};

// generic kernels (layer.cu)
lrc_status launch_lr_down(const ExpertArgs& a, int np_bound, cudaStream_t st);

// tiled kernels (fast.cu)
int64_t tiles_bytes(int64_t rows, int64_t cols, int ni);
lrc_status launch_up_tiled(const ExpertArgs& a, int num_sms, int max_tokens_per_expert,
                           cudaStream_t st);
lrc_status launch_down_tiled(const ExpertArgs& a, int num_sms, int max_tokens_per_expert,
                             cudaStream_t st);

}  // namespace lrc
