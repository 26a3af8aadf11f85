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

struct RouteArgs {
  const double* gate_t;
  const void* x;
  int x_dtype;
  int64_t B;
  int d, E, k, renorm;
  double* probs;
  int32_t* topk_idx;
  float* topk_w;
  double* logits;    // [B][E] scratch
  int* tile_ticket;  // [route_tiles(B)] zero-initialised, self-resetting
  PlanArgs plan;     // plan.ticket == nullptr -> routing only
};

__device__ void build_plan_block(const PlanArgs& pa, const int32_t* topk_idx,
                                 const float* topk_w, int B, int k);
int route_tiles(int64_t B);
lrc_status launch_route(const RouteArgs& ra, cudaStream_t st);

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

// Byte layout of the low-rank factor tiles that ride along with a weight tile
// (see fast.cu).  Offsets are per 16-row tile.
struct LrLayout {
  int u1c, u3c, v2c, u1m, u3m, v2m, up_total;  // up: U1, U3 rows + V2^T rows
  int u2c, u2m, down_total;                    // down: U2 rows
};
__host__ __device__ inline int pad16(int x) { return (x + 15) & ~15; }
__host__ __device__ inline bool factor_present(const lrc_qmat& m) {
  return m.packed != nullptr || m.dense != nullptr;
}
__host__ __device__ inline LrLayout lr_layout(const lrc_expert& e) {
  LrLayout L{};
  auto codes = [](const lrc_qmat& m, int r) {
    return factor_present(m) ? pad16((16 * r * m.bits + 7) / 8) : 0;
  };
  auto umeta = [](const lrc_qmat& u) {
    return factor_present(u) ? pad16(16 * ((u.cols + u.group_size - 1) / u.group_size) * 4) : 0;
  };
  const int r1 = factor_present(e.u1) ? e.u1.cols : 0;
  const int r3 = factor_present(e.u3) ? e.u3.cols : 0;
  const int r2 = factor_present(e.u2) ? e.u2.cols : 0;
  int o = 0;
  L.u1c = o; o += codes(e.u1, r1);
  L.u3c = o; o += codes(e.u3, r3);
  L.v2c = o; o += codes(e.v2, r2);
  L.u1m = o; o += umeta(e.u1);
  L.u3m = o; o += umeta(e.u3);
  L.v2m = o; o += factor_present(e.v2) ? pad16(r2 * 4) : 0;
  L.up_total = o;
  o = 0;
  L.u2c = o; o += codes(e.u2, r2);
  L.u2m = o; o += umeta(e.u2);
  L.down_total = o;
  return L;
}

// generic kernels (layer.cu)
lrc_status launch_lr_down(const ExpertArgs& a, int np_bound, cudaStream_t st);

// tiled kernels (fast.cu)
int64_t tiles_bytes(int64_t rows, int64_t cols, int ni);
lrc_status launch_up_tiled(const ExpertArgs& a, int num_sms, int max_tokens_per_expert,
                           int lr_up_max, cudaStream_t st);
lrc_status launch_down_tiled(const ExpertArgs& a, int num_sms, int max_tokens_per_expert,
                             int lr_down_max, cudaStream_t st);

}  // namespace lrc
