// Tensor-core decode engine ("tcd"): one persistent kernel per MoE layer step
// for small batches (B <= 8 tokens).  See tcd.cu for the design.
#pragma once
#include "layer.cuh"

namespace lrc {
namespace tcd {

constexpr int kMaxTok = 8;   // tokens per forward on this path
constexpr int kMaxAct = 64;  // distinct experts per step
constexpr int kMaxP = 64;    // (token, expert) pairs per step
constexpr int kRMax = 64;    // compensator rank
constexpr int kFuseMaxE = 16;  // fused (per-CTA) routing up to this many experts

// Device expert entry: tcd packs (layer-owned) + the reference-layout factors.
struct Expert {
  const uint8_t* up;    // units (tile, group, w1|w3): 128 rows x code bytes + 128 x {s, z} fp16
  const uint8_t* down;  // units (tile, group, w2)
  const uint8_t* lr_up;    // per up tile: U1, U3, V2^T rows as nibbles + fp16 meta (lr_pack)
  const uint8_t* lr_down;  // per down tile: U2 rows
  lrc_qmat u1, v1, u3, v3, u2, v2;
  int rank;             // 0: no compensator
  int pad;
};

// Low-rank tile packs (rank r <= 64, factor bits <= 4): RB = bytes of one
// row's nibbles (16 for r <= 32, 32 for r <= 64).
__host__ __device__ inline int lr_rb(int r) { return r <= 32 ? 16 : 32; }
__host__ __device__ inline int lr_up_tile_bytes(int r) { return 3 * 128 * lr_rb(r) + 2 * 128 * 4 + 2 * kRMax * 4; }
__host__ __device__ inline int lr_down_tile_bytes(int r) { return 128 * lr_rb(r) + 128 * 4; }

struct Args {
  const uint16_t* x;  // [B][hidden] bf16
  int B, hidden, ffn, E, S, top_k, top_n, renorm, comp_shared, bits;
  const float* gate32;   // [E][hidden] fused routing (null: routing given)
  const double* gate64;  // [E][hidden] exact fallback
  const float* gnorm;    // [E] upper bounds of the gate rows' L2 norms (routing error bound)
  const int32_t* given_idx;  // [B][top_k] (external router) or [B] (pairs mode)
  const float* given_w;
  const uint8_t* given_comp;  // pairs mode: per-row compensation flag
  int pairs_mode;
  const Expert* ex;  // [E + S]
  float* y;          // [B][hidden] f32
  int32_t* topk_idx;
  float* topk_w;
  // workspace
  unsigned long long* gbar;  // grid barrier counter (monotonic)
  unsigned* tcnt;            // [2][kMaxP] V.x job counters (parity buffers)
  float* t13;                // [kMaxP][2 * kRMax]
  float* t2;                 // [2][kMaxP][kRMax]
  uint8_t* xdig;             // [max_tok][hidden/64][512] B-operand digit images of x (phase U)
  float4* xsum;              // [max_tok][hidden/64] {2^-S, sum of the scaled integers, 0, 0}
  uint8_t* adig;             // [kMaxP][ffn/64][512] digit images of the activations (phase D)
  float4* asum;              // [kMaxP][ffn/64]
  unsigned* xcnt;            // [2] x-image counters (parity buffers)
  float* hacc;               // [max_act][tiles_up][2][kMaxTok][128] split-tile partial sums
  unsigned* hcnt;            // [max_act][tiles_up]
  int max_act;
  int fb;                    // factor bits (2..4), V group size 64
  int stamp;                 // debug: per-CTA %globaltimer stamps
  int dbg;                   // debug (LRC_TCD_DEBUG): 1 no MMA, 2 no decode/st, 4 no B operand,
                             // 8 no D loads, 16 test_wait spins
};

// host side
bool eligible(const lrc_expert* experts, int n, int hidden, int ffn, int* bits, int* fbits);
int64_t pack_bytes(int rows, int cols, int nmat, int bits);
lrc_status build_pack(const lrc_qmat* mats, int nmat, int bits, uint8_t* out, cudaStream_t st);
lrc_status build_lr_pack(const lrc_expert& e, int hidden, int ffn, uint8_t* up, uint8_t* down, cudaStream_t st);
lrc_status launch(const Args& a, int num_sms, cudaStream_t st, bool pdl);
void stamps_copy(uint64_t* host, int n);
void trace_copy(uint64_t* host);  // [4][256]
void set_wait_mode(int m);
void wstat_copy(unsigned long long* host);  // [24][8]

}  // namespace tcd
}  // namespace lrc
