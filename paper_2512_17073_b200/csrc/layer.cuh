// Device-side structures shared by the router, generic and tiled expert kernels.
#pragma once
#include "common.cuh"

#define LRC_MAX_EXPERTS 256

namespace lrc {

// Everything the tiled kernels need about one active expert, written by the
// plan builder so their setup is a single dependent round trip.
struct ActiveRec {
  const uint8_t* up_tiles;
  const uint8_t* down_tiles;
  const uint8_t* up_lr_tiles;
  const uint8_t* down_lr_tiles;
  int e, off, cnt;
  uint32_t cmask;  // bit q: pairs [8q, 8q+8) of the expert hold a compensated pair (q >= 31 -> bit 31)
  int up_lr_bytes, down_lr_bytes, pad[2];
};

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
  ActiveRec* arec;          // [E+S] per active expert (layer forward only; null otherwise)
  const lrc_expert* experts;  // device table [E+S] (with arec)
  const uint8_t* comp_rows;   // [B] pairs mode: per-row compensation flag (else top_n rule)
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
  // layer-forward extras (all null/0 for a standalone lrc_route)
  const lrc_expert* experts;  // device table [ne]
  float* t;                   // [B][ne][3][maxr] low-rank vectors
  int ne, maxr;
  int spec_blocks;            // V.x row blocks per expert computed speculatively (0 = none)
  float* t2_zero;             // zero t[b][e][2][:] (tiled path accumulates into it)
  float* y_zero;              // zero y rows
  int stamp;                  // LRC_ROUTE_STAMPS: per-CTA %globaltimer stamps (debug)
  int pdl;                    // launched as a programmatic dependent of the previous kernel
  // pairs mode (expert-parallel receive side): routing is given, one expert per
  // row (k = 1); the gate GEMV and softmax are skipped
  const int32_t* pairs_expert;  // [B] or null
  const float* pairs_w;         // [B]
};

// Row j of a quantized V (group size 64, BITS-bit LSB-first stream) dotted
// with nb bf16 token rows (stride ld): each lane takes whole 64-code groups,
// loads the group's 2*BITS words at once and decodes them with funnel shifts;
// x is read 8 columns (16 B) at a time.  acc[t] is warp-reduced on return.
template <int BITS, int MAXT>
__device__ void vrow_dot_tokens(const lrc_qmat& V, int j, const uint16_t* __restrict__ xt,
                                int64_t ld, int nb, float (&acc)[MAXT]) {
  constexpr int W = 2 * BITS;  // 32-bit words per 64-code group
  const int lane = threadIdx.x & 31;
  const int gpr = (V.cols + 63) / 64;
  const uint32_t* words = reinterpret_cast<const uint32_t*>(V.packed);
  const int64_t nwords = ((static_cast<int64_t>(V.rows) * V.cols * BITS + 7) >> 3) >> 2;
#pragma unroll
  for (int t = 0; t < MAXT; ++t) acc[t] = 0.0f;
  for (int g = lane; g < gpr; g += 32) {
    const int64_t w0 = ((static_cast<int64_t>(j) * V.cols + g * 64) * BITS) >> 5;
    uint32_t w[W + 1];
#pragma unroll
    for (int i = 0; i <= W; ++i) w[i] = (w0 + i < nwords) ? __ldg(words + w0 + i) : 0u;
    const int nv = min(64, V.cols - g * 64);
    const float s = h2f(V.scales[static_cast<int64_t>(j) * gpr + g]);
    const float z = h2f(V.zeros[static_cast<int64_t>(j) * gpr + g]);
    const bool vec = (nv == 64) && (ld % 8) == 0 && ((reinterpret_cast<uintptr_t>(xt) & 15) == 0);
    float cx[MAXT], sx[MAXT];
#pragma unroll
    for (int t = 0; t < MAXT; ++t) cx[t] = sx[t] = 0.0f;
#pragma unroll
    for (int i8 = 0; i8 < 8; ++i8) {
      float c[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int bit = (i8 * 8 + q) * BITS;
        c[q] = static_cast<float>(__funnelshift_r(w[bit >> 5], w[(bit >> 5) + 1], bit & 31) &
                                  ((1u << BITS) - 1u));
      }
#pragma unroll
      for (int t = 0; t < MAXT; ++t) {
        if (t < nb) {
          const uint16_t* xr = xt + t * ld + g * 64 + i8 * 8;
          float xv[8];
          if (vec) {
            const uint4 u = __ldg(reinterpret_cast<const uint4*>(xr));
            const uint32_t u4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              xv[2 * q] = bf2f(u4[q] & 0xffff);
              xv[2 * q + 1] = bf2f(u4[q] >> 16);
            }
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) xv[q] = (i8 * 8 + q < nv) ? bf2f(xr[q]) : 0.0f;
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            cx[t] = fmaf(c[q], xv[q], cx[t]);
            sx[t] += xv[q];
          }
        }
      }
    }
#pragma unroll
    for (int t = 0; t < MAXT; ++t) acc[t] = fmaf(s, cx[t], fmaf(z, sx[t], acc[t]));
  }
#pragma unroll
  for (int t = 0; t < MAXT; ++t) acc[t] = warp_sum(acc[t]);
}

// Row `row` of a quantized weight matrix (group size 64, BITS-bit LSB-first
// stream, rows word-aligned) dotted with NT token vectors xp[t] (bf16 or f32,
// 16-byte aligned, length W.cols): each lane takes whole 64-code groups and
// decodes them with funnel shifts once for all tokens.  acc[t] is
// warp-reduced on return.  The generic expert path for g64 codes of any width
// (ref/quant.py:216-224: W = s * c + z per group).
__device__ __forceinline__ void load8(const uint16_t* p, float (&v)[8]) {
  const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
  const uint32_t u4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    v[2 * q] = bf2f(u4[q] & 0xffff);
    v[2 * q + 1] = bf2f(u4[q] >> 16);
  }
}
__device__ __forceinline__ void load8(const float* p, float (&v)[8]) {
  const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
template <int BITS, int NT, typename XT>
__device__ void qrow_dot_g64(const lrc_qmat& W, int row, const XT* const (&xp)[NT], int nb, float (&acc)[NT]) {
  constexpr int NW = 2 * BITS;  // 32-bit words per 64-code group
  const int lane = threadIdx.x & 31;
  const int gpr = W.cols / 64;
  const uint32_t* words = reinterpret_cast<const uint32_t*>(W.packed) + (static_cast<int64_t>(row) * W.cols * BITS >> 5);
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t] = 0.0f;
  for (int g = lane; g < gpr; g += 32) {
    uint32_t w[NW + 1];
#pragma unroll
    for (int i = 0; i < NW; ++i) w[i] = __ldg(words + g * NW + i);
    w[NW] = 0u;
    const float s = h2f(W.scales[static_cast<int64_t>(row) * gpr + g]);
    const float z = h2f(W.zeros[static_cast<int64_t>(row) * gpr + g]);
    float cx[NT], sx[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) cx[t] = sx[t] = 0.0f;
#pragma unroll
    for (int i8 = 0; i8 < 8; ++i8) {
      float c[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int bit = (i8 * 8 + q) * BITS;
        c[q] = static_cast<float>(__funnelshift_r(w[bit >> 5], w[(bit >> 5) + 1], bit & 31) & ((1u << BITS) - 1u));
      }
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        if (t < nb) {
          float xv[8];
          load8(xp[t] + g * 64 + i8 * 8, xv);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            cx[t] = fmaf(c[q], xv[q], cx[t]);
            sx[t] += xv[q];
          }
        }
      }
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[t] = fmaf(s, cx[t], fmaf(z, sx[t], acc[t]));
  }
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t] = warp_sum(acc[t]);
}
// codes this path takes: packed, group size 64, rows a whole number of words
__host__ __device__ inline bool qmat_g64(const lrc_qmat& W) {
  return W.dense == nullptr && W.packed != nullptr && W.group_size == 64 && (W.cols % 64) == 0 &&
         (W.bits == 2 || W.bits == 3 || W.bits == 4) && ((static_cast<int64_t>(W.cols) * W.bits) % 32) == 0;
}

int route_tiles(int64_t B);
// large-batch plan (router in routing-only mode, then a parallel counting sort)
constexpr int kSerialPlanMaxPairs = 2048;
int plan_parallel_blocks(int64_t np);
lrc_status launch_plan_parallel(const PlanArgs& pa, const int32_t* tk_idx, const float* tk_w, int B, int k,
                                int* blk, uint32_t* cmask, int* ticket, cudaStream_t st);
lrc_status launch_route(const RouteArgs& ra, cudaStream_t st);
lrc_status launch_route_bulk(const RouteArgs& ra, cudaStream_t st);  // large batches, routing only

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
  int ne;                     // experts incl. shared; t is [B][ne][3][maxr]
  int g64;                    // every expert's w1/w3/w2 take qrow_dot_g64 (generic path)
};

// Byte layout of the low-rank factor tiles that ride along with a weight tile
// (see fast.cu).  Offsets are per 16-row tile.
struct LrLayout {
  int u1c, u3c, v2c, u1m, u3m, v2m, up_total;  // up: U1, U3 rows + V2^T rows
  int u2c, u2bc, u2m, u2bm, down_total;        // down: U2 rows of the top / bottom row half
};
__host__ __device__ inline int pad16(int x) { return (x + 15) & ~15; }
__host__ __device__ inline bool factor_present(const lrc_qmat& m) {
  return m.packed != nullptr || m.dense != nullptr;
}
__host__ __device__ inline LrLayout lr_layout(const lrc_expert& e) {
  LrLayout L{};
  // codes are re-laid out as 4-bit nibbles (factor bits <= 4): word-aligned
  // rows, shift-only decode in the epilogue warp
  auto codes = [](const lrc_qmat& m, int r) {
    return factor_present(m) ? pad16((16 * r * 4 + 7) / 8) : 0;
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
  // the down kernel streams W2 as two interleaved row halves (rows [0, H/2) and
  // [H/2, H)), so a down LR tile holds the U2 rows of both halves' tile
  o = 0;
  L.u2c = o; o += codes(e.u2, r2);
  L.u2bc = o; o += codes(e.u2, r2);
  L.u2m = o; o += umeta(e.u2);
  L.u2bm = o; o += umeta(e.u2);
  L.down_total = o;
  return L;
}

void tiled_stamps_copy(uint64_t* host, int n);  // debug (tiled.cu)

// generic kernels (layer.cu)
lrc_status launch_lr_down(const ExpertArgs& a, int np_bound, cudaStream_t st);

// tiled kernels (fast.cu)
int64_t tiles_bytes(int64_t rows, int64_t cols, int ni);
lrc_status launch_up_tiled(const ExpertArgs& a, int num_sms, int max_tokens_per_expert,
                           int lr_up_max, cudaStream_t st, bool pdl);
lrc_status launch_down_tiled(const ExpertArgs& a, int num_sms, int max_tokens_per_expert,
                             int lr_down_max, cudaStream_t st, bool pdl);

// tcgen05 prefill GEMM (prefill.cu)
bool prefill_eligible(const lrc_expert* experts, int n, int hidden, int ffn, int maxr, int* bits);
int64_t prefill_lr_pack_elems(int hidden, int ffn, int maxr);  // bf16 elements per expert
int prefill_tb_width(int maxr);
lrc_status build_prefill_lr(const lrc_expert& e, int hidden, int ffn, int maxr, uint16_t* out, cudaStream_t st);
int64_t prefill_pack_bytes(int hidden, int ffn, int bits);  // per expert
lrc_status build_prefill_pack(const lrc_expert& e, int hidden, int ffn, int bits, uint8_t* out, cudaStream_t st);
lrc_status launch_prefill(const ExpertArgs& a, int np_bound, int max_tok, const uint16_t* lrp, uint16_t* tb,
                          const uint8_t* ppk, int bits, cudaStream_t st, int* launches);

}  // namespace lrc
