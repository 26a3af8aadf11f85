/*
 * lrc.h -- C-ABI of the B200-native router-guided low-rank-compensated MoE path.
 *
 * Drop-in boundary for the reference package moe-lrc 0.1.0
 * (/root/reference/pkg/src/moe_lrc, "ref/" below).  The reference is pure
 * Python+numpy and has no FFI; these are the entry points a ctypes binding of
 * that path binds.  Every function:
 *   - takes caller-owned DEVICE pointers (unless stated) and a cudaStream_t
 *     passed as void*; work is stream-ordered and CUDA-graph capturable;
 *   - never allocates on the hot path (lrc_layer_forward uses the layer's
 *     workspace, sized at lrc_layer_create);
 *   - returns an lrc_status; lrc_last_error() holds a message for the calling
 *     thread.  The Python host maps LRC_ERR_INVALID to the reference's
 *     QuantizationError / CompensatorError / MoEError (ValueError family) and
 *     LRC_ERR_MISSING to MissingArtifactError (ref/moe.py:27-32).
 *
 * Numerics contract: integer outputs (codes, packed bytes,
 * routing indices) are bit-exact with the reference; fp64 dequantize is
 * bit-exact; the layer output (bf16 activations, fp16 scale/zero metadata,
 * fp32 accumulation) is within max relative L2 1e-2 of the fp64 reference.
 */
#ifndef LRC_H_
#define LRC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LRC_ABI_VERSION 1

typedef enum {
  LRC_OK = 0,
  LRC_ERR_INVALID = 1,     /* bad shape/config: ValueError family                 */
  LRC_ERR_MISSING = 2,     /* expert record absent: MissingArtifactError          */
  LRC_ERR_CUDA = 3,        /* CUDA runtime error (message has cudaGetErrorString) */
  LRC_ERR_UNSUPPORTED = 4, /* valid but not implemented on this path              */
  LRC_ERR_OOM = 5
} lrc_status;

enum { LRC_DTYPE_F64 = 0, LRC_DTYPE_F32 = 1, LRC_DTYPE_BF16 = 2 };

int lrc_abi_version(void);
const char* lrc_last_error(void);

/* ---------------------------------------------------------------- codes --- */
/* ref/quant.py:243-249 pack_codes: LSB-first continuous bitstream.  out has
 * (count*bits+7)/8 bytes. */
lrc_status lrc_pack_codes(const uint8_t* codes, int64_t count, int bits, uint8_t* packed,
                          void* stream);
/* ref/quant.py:252-262 unpack_codes (K6, bit-exact). */
lrc_status lrc_unpack_codes(const uint8_t* packed, int64_t count, int bits, uint8_t* codes,
                            void* stream);
/* ref/quant.py:216-224 dequantize in fp64, bit-exact (code*scale then +zero,
 * two roundings).  codes uint8 (rows, cols); scales/zeros f64 (rows, ceil(cols/gs)). */
lrc_status lrc_dequantize_f64(const uint8_t* codes, const double* scales, const double* zeros,
                              int64_t rows, int64_t cols, int group_size, double* out,
                              void* stream);
/* ref/quant.py:146-213 quantize: min-max affine fit per group plus
 * hqq_iters rounds of half-quadratic zero refinement (fp64).  Bit-exact with
 * the reference for hqq_iters == 0. */
lrc_status lrc_quantize_f64(const double* w, int64_t rows, int64_t cols, int bits,
                            int group_size, int hqq_iters, double shrink_p, uint8_t* codes,
                            double* scales, double* zeros, void* stream);
/* out += U @ V with U (m, r), V (r, n) dense fp64 (ref/lowrank.py:165). */
lrc_status lrc_add_lowrank_f64(const double* u, const double* v, int64_t m, int64_t n, int r,
                               double* out, void* stream);

/* --------------------------------------------------------------- router --- */
/* ref/moe.py:165-193 route(): probs = softmax(gate.T @ x) in fp64, selected =
 * first top_k of a stable descending sort (ties -> lower index), compensated =
 * first top_n of selected.  gate_t is the TRANSPOSED gate, (E, d) f64.
 * x is (B, d) of x_dtype.  probs (B, E) may be NULL.  topk_w = probs[selected]
 * (renormalised over the top-k when renormalize != 0, ref/moe.py:234-236). */
lrc_status lrc_route(const double* gate_t, const void* x, int x_dtype, int64_t B, int d, int E,
                     int top_k, int top_n, int renormalize, double* probs, int32_t* topk_idx,
                     float* topk_w, void* stream);

/* ------------------------------------------------------------ MoE layer --- */
/* One quantized matrix in the reference storage format: LSB-first packed
 * codes (ref/artifact.py:103-108) + per-group scale/zero as fp16 bit patterns.
 * If `dense` is non-NULL the matrix is instead a raw fp32 row-major matrix
 * (the reference's quantize_factors=False test hook, ref/lowrank.py:144-146). */
typedef struct {
  const uint8_t* packed;
  const uint16_t* scales;
  const uint16_t* zeros;
  const float* dense;
  int32_t rows, cols, bits, group_size;
} lrc_qmat;

/* One expert: SwiGLU projections w1,w3 (ffn, hidden), w2 (hidden, ffn) and an
 * optional rank-r compensator per projection (u (rows, r), v (r, cols)).
 * up_tiles / down_tiles: optional fast tiled layout built by
 * lrc_build_tiles (bits == 2, group_size == 64); NULL -> generic kernels. */
typedef struct {
  lrc_qmat w1, w3, w2;
  int32_t rank;
  lrc_qmat u1, v1, u3, v3, u2, v2;
  const uint8_t* up_tiles;
  const uint8_t* down_tiles;
  const uint8_t* up_lr_tiles;   /* per 16-row tile: U1, U3 rows + V2^T rows (+ fp16 meta) */
  const uint8_t* down_lr_tiles; /* per 16-row tile: U2 rows (+ fp16 meta)                 */
} lrc_expert;

/* Bytes of the fast tiled layout for a (rows, cols) 2-bit gs=64 matrix, with
 * `interleave` matrices of the same shape interleaved (2 for w1|w3, 1 for w2). */
int64_t lrc_tiles_bytes(int64_t rows, int64_t cols, int interleave);
/* Repack `interleave` reference-format matrices into the tiled layout. */
lrc_status lrc_build_tiles(const lrc_qmat* mats, int interleave, uint8_t* tiles, void* stream);
/* Low-rank factor tiles: the rows of U1/U3/V2^T (up) and U2 (down) that belong
 * to each 16-row weight tile, re-laid out contiguously (same 3-bit codes and
 * fp16 metadata) so they stream into shared memory with the weight tile.
 * Sizes are per expert (its factor ranks); requires factor group sizes that
 * are multiples of 16 for V2.  *_bytes may be 0 (no compensator). */
lrc_status lrc_lr_tiles_bytes(const lrc_expert* e, int hidden, int ffn, int64_t* up_bytes,
                              int64_t* down_bytes);
lrc_status lrc_build_lr_tiles(const lrc_expert* e, int hidden, int ffn, uint8_t* up_lr,
                              uint8_t* down_lr, void* stream);
/* Bit-exact inverse (codes of matrix `which`), for the K6 parity test. */
lrc_status lrc_tiles_unpack(const uint8_t* tiles, int64_t rows, int64_t cols, int interleave,
                            int which, uint8_t* codes, void* stream);

typedef struct lrc_layer lrc_layer;

/* gate_t (E, hidden) f64 device; experts: host array of num_experts +
 * num_shared descriptors (shared experts last, ref/moe.py:81-88).  The layer
 * keeps the descriptors (device pointers stay caller-owned) and allocates a
 * workspace for up to max_tokens tokens with top_k routed experts. */
lrc_status lrc_layer_create(const double* gate_t, int hidden, int ffn, int num_experts,
                            int num_shared, const lrc_expert* experts, int max_tokens, int top_k,
                            lrc_layer** out);
void lrc_layer_destroy(lrc_layer* layer);
/* Replace expert descriptors (offload engine: experts move between slots). */
lrc_status lrc_layer_set_expert(lrc_layer* layer, int expert_id, const lrc_expert* e);
/* Stream-ordered lrc_layer_set_expert: the device-side descriptor update is an
 * async copy on `stream` (from a 64-entry pinned staging ring: at most 64
 * updates may be in flight).  Later work on `stream` sees the new expert. */
lrc_status lrc_layer_set_expert_async(lrc_layer* layer, int expert_id, const lrc_expert* e,
                                      void* stream);

/* ref/moe.py:217-259 forward(mode="compensated") for a batch of B tokens:
 * y[b] = sum_{e in top_k(b)} w_be * E_e(x_b) + sum_shared E_s(x_b), with the
 * low-rank term U.(V.x) applied inside the expert kernels for each token's
 * top_n experts only (never materialising Q(W)+UV).  top_n == 0 gives mode
 * "quantized".  x (B, hidden) bf16; y (B, hidden) f32.  topk_idx / topk_w
 * (B, top_k) may be NULL.  compensate_shared as ForwardConfig.
 * Execution: B below the prefill threshold (default 128) runs the decode
 * kernels (router + tiled up/down, 3 PDL-chained launches, graph-capturable);
 * B at or above it runs the tcgen05 grouped dequant-GEMM path (router, parallel
 * plan, V.x / up / V2.a / down GEMMs) when the layer is eligible. */
lrc_status lrc_layer_forward(lrc_layer* layer, const uint16_t* x, int64_t B, int top_k,
                             int top_n, int renormalize, int compensate_shared, float* y,
                             int32_t* topk_idx, float* topk_w, void* stream);
/* Expert-parallel receive side: the routing is GIVEN.  Row b of
 * x goes to expert[b] (0 <= expert < num_experts + num_shared) with mixing
 * weight weight[b]; the low-rank term is applied iff comp[b] != 0 and the
 * expert has a compensator.  y[b] = weight[b] * E_expert[b](x_b) -- the source
 * rank sums its rows back per token (ref/moe.py:237-258 split by expert
 * owner).  No implicit shared experts.  expert/weight/comp are device arrays. */
lrc_status lrc_layer_forward_pairs(lrc_layer* layer, const uint16_t* x, int64_t B,
                                   const int32_t* expert, const float* weight, const uint8_t* comp,
                                   float* y, void* stream);
/* Same computation through the generic (reference-layout) kernels even when
 * tiles exist -- used as an internal cross-check. */
lrc_status lrc_layer_forward_generic(lrc_layer* layer, const uint16_t* x, int64_t B, int top_k,
                                     int top_n, int renormalize, int compensate_shared, float* y,
                                     int32_t* topk_idx, float* topk_w, void* stream);
/* Number of kernel launches the last forward issued on its stream. */
int lrc_layer_last_launches(const lrc_layer* layer);
/* End-to-end variant with HOST buffers: x (B, hidden) bf16 and y (B, hidden)
 * f32 in host memory (pinned for asynchronous copies).  Copies x into the
 * layer's device staging buffer, runs lrc_layer_forward, copies y back; all
 * stream-ordered on `stream` (the caller synchronises). */
lrc_status lrc_layer_forward_host(lrc_layer* layer, const uint16_t* x_host, int64_t B, int top_k,
                                  int top_n, int renormalize, int compensate_shared,
                                  float* y_host, void* stream);
/* Kernel timing: when enabled, forward records CUDA events on its stream
 * around each phase; lrc_layer_phase_ms waits for the last forward and writes
 * {route, lr_down, up, down} durations in milliseconds. */
lrc_status lrc_layer_set_profiling(lrc_layer* layer, int enabled);
/* Batches of B >= min_tokens tokens run the tcgen05 grouped dequant-GEMM
 * (prefill) path when the layer is eligible (2-bit gs=64 weights, hidden and
 * ffn multiples of 64); min_tokens <= 0 disables it.  Default 128 (env
 * LRC_PREFILL_MIN). */
lrc_status lrc_layer_set_prefill_min(lrc_layer* layer, int64_t min_tokens);
/* GPU-driven expert paging (offload without a host round trip): every expert
 * is one block in device-mapped pinned host memory (host_blocks: E+S pointers);
 * offsets[10] = byte offsets in a block of the up tiles, down tiles, up LR
 * tiles, down LR tiles, V1 packed/scales/zeros, V3 packed/scales/zeros (-1 =
 * absent).  Each forward then copies the step's active experts into slots
 * (slot a = the a-th active expert; n_slots must cover the distinct experts a
 * step can select) inside the stream, repoints their descriptors, and runs the
 * tiled decode kernels; no host synchronisation, graph-capturable. */
lrc_status lrc_layer_set_pager(lrc_layer* layer, const void* const* host_blocks, const int64_t* offsets,
                               int64_t block_bytes, uint8_t* slots, int n_slots, int64_t slot_bytes);
/* Budgeted LRU over the pager's slots, shared by every layer that uses the
 * same slot pool (the reference cost model's cache_policy="lru",
 * ref/simulate.py:127-167): a selected expert already resident in a slot moves
 * nothing; a miss takes the least recently used slot not touched in the
 * current step.  n_slots must equal the n_slots given to lrc_layer_set_pager;
 * layer_key distinguishes the layers' experts.  Decisions are made on the
 * device (no host round trip).  Stats = cumulative {hits, misses}. */
typedef struct lrc_pager_cache lrc_pager_cache;
lrc_status lrc_pager_cache_create(int n_slots, lrc_pager_cache** out);
void lrc_pager_cache_destroy(lrc_pager_cache* cache);
lrc_status lrc_pager_cache_stats(lrc_pager_cache* cache, int64_t* hits_misses);
lrc_status lrc_layer_set_pager_cache(lrc_layer* layer, lrc_pager_cache* cache, int layer_key);
int lrc_layer_prefill_eligible(const lrc_layer* layer);
/* Batches of B <= max_tokens (at most 8) tokens run the tensor-core decode
 * engine when the layer is eligible (2- or 3-bit gs=64 weights, hidden and ffn
 * multiples of 128, compensator rank <= 64 with 2..4-bit factors): ONE
 * persistent kernel per layer step -- per-CTA fused routing (E <= 16; larger
 * E uses the cluster router first), tcgen05.mma.kind::i8 with the decoded
 * codes as the TMEM A operand, the low-rank terms, SwiGLU and the weighted
 * combine, split stream-K over all SMs with one grid barrier between the
 * w1|w3 and w2 phases.  0 disables it (the mma.sync tiled kernels run).
 * Default 8 (env LRC_TCD_MAX).  The engine keeps its own copy of the codes in
 * the tcd layout (built lazily on the first eligible forward and after
 * lrc_layer_set_expert*). */
lrc_status lrc_layer_set_tcd_max(lrc_layer* layer, int max_tokens);
int lrc_layer_tcd_eligible(const lrc_layer* layer);
lrc_status lrc_layer_phase_ms(lrc_layer* layer, float* ms4);
/* Debug: %globaltimer (ns) stamps, 8 per CTA, of the last launch of the router
 * (which = 0; enabled by LRC_ROUTE_STAMPS=1 in the environment), of the
 * tiled kernels (which = 1: [down, up][256 CTAs][8]; LRC_TILED_DEBUG bit 3)
 * or of the tensor-core decode kernel (which = 2: [148 CTAs][8]; LRC_TCD_STAMPS=1).
 * Copies n values and clears the device buffer. */
lrc_status lrc_debug_stamps(int which, uint64_t* host, int n);

/* ------------------------------------------------------ expert parallel --- */
/* Dispatch of a rank's routed pairs to the expert owners: pair
 * p = b*top_k + j goes to rank floor(e*world/num_experts), e = topk_idx[p], at
 * slot dest*capacity + (its rank among the pairs with that destination, in
 * pair order).  Writes x_send (world*capacity, d) bf16 rows, meta_send
 * (world*capacity, 3) int32 {expert, float bits of the weight, compensated =
 * j < top_n} and slot_of[p]; unused slots get a zero row for the receiver's
 * first expert ceil(r*num_experts/world) with weight 0.  Requires
 * B*top_k <= capacity and world*capacity <= 4096.  Stream-ordered, no host
 * synchronisation (the NCCL all-to-alls of x_send / meta_send go between
 * this call and the owner's lrc_layer_forward_pairs). */
lrc_status lrc_ep_dispatch(const int32_t* topk_idx, const float* topk_w, const uint16_t* x, int64_t B,
                           int top_k, int top_n, int num_experts, int world, int capacity, int d,
                           uint16_t* x_send, int32_t* meta_send, int32_t* slot_of, void* stream);
/* Combine (ref/moe.py:237-258): y[b] = sum_j back[slot_of[b*top_k + j]] for the
 * rows returned by the reverse all-to-all (already weighted by the owners). */
lrc_status lrc_ep_combine(const float* back, const int32_t* slot_of, int64_t B, int top_k, int d, float* y,
                          void* stream);

/* Dense fp64 expert (mode="reference", ref/moe.py:241-243):
 * y (B, hidden) += w[b] * w2 @ (silu(w1 @ x_b) * (w3 @ x_b)); w may be NULL (=1). */
lrc_status lrc_dense_expert_f64(const double* w1, const double* w3, const double* w2, int hidden,
                                int ffn, const double* x, const double* mix, int64_t B,
                                double* y, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LRC_H_ */
