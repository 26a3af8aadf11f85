// tcgen05 grouped dequant-GEMM for prefill and large batches (SURVEY 8(a) K3,
// config C4).  Semantics: ref/moe.py:217-259 forward(mode="compensated") with
// ref/lowrank.py:153-165 applying U.(V.x) for each token's top-n experts only.
//
// A CTA PAIR (cluster of 2, tcgen05 cta_group::2) computes a [256-row x
// 256-pair] tile of TWO weight matrices that share the B operand, over K in
// 64-column slabs (one 128-byte swizzle row); CTA r holds rows [128r, 128r+128)
// of both A operands and pairs [128r, 128r+128) of B, and its TMEM receives its
// 128 rows x all 256 pairs of both accumulators:
//   up   : W1 and W3 rows [m0, m0+256) x the expert's token rows of x
//          -> SwiGLU in the epilogue -> bf16 activations a16[pair][ffn];
//   down : W2 rows [m0, m0+256) and [m0+256, m0+512) x the pairs' a16 rows
//          -> y[token] += w_pair * (.) with fp32 reductions.
// Roles per CTA (288 threads, one CTA per SM: 223 KB smem, 512 TMEM columns):
//   warps 0-7  producers: thread t dequantizes row t&127 of matrix t>>7 (c*s+z
//              in fp32, rounded once to bf16) from the code ring straight into
//              SWIZZLE_128B smem, gathers its share of the CTA's 128 B rows
//              with cp.async two slabs ahead (zero-filled past the expert's
//              pairs) and arrives on its CTA's stage barrier; after the K loop,
//              the epilogue from its own TMEM.
//   warp 8.1   loader: one cp.async.bulk per A matrix per slab copies the
//              codes + fp16 scale/zero of the CTA's rows (prefill pack) into a
//              6-deep code ring.
//   warp 8.0   leader: issues tcgen05.mma.cta_group::2 (M=256, N=256, K=16)
//              into the two fp32 accumulators and commits each stage back to
//              both CTAs (multicast; 4-stage ring).  Peer: forwards each
//              completed stage to the leader's barrier (one cluster-scope
//              release per stage).
// The pair halves each SM's share of the B operand (gather and smem reads).
// The low-rank term is K augmentation: extra slabs whose A rows hold the U
// factors (up: [U1 | 0] for W1 rows, [0 | U3] for W3 rows; down: U2) and whose
// B rows hold the pair's V.x vector (bf16 [t1 | t3] or t2, zero for
// uncompensated pairs), so U.(V.x) lands in the same accumulator and
// Q(W)+UV^T is never formed.  The V.x vectors come from the same engine run on
// the V factors (modes kVxUp / kVxDown, one accumulator) for the tiles that
// hold a compensated pair.  Factors are repacked once per expert into bf16
// rows (the "LR pack", build_prefill_lr) so every low-rank slab is a plain
// cp.async row copy issued two slabs ahead like B.  The up epilogue stages the
// bf16 activations pair-major in the idle stage memory and writes 16-byte rows.
#include <cuda_bf16.h>

#include <cstdlib>

#include "common.cuh"
#include "layer.cuh"
#include "umma.cuh"

namespace lrc {
namespace {

constexpr int kTM = 128;  // rows per accumulator per CTA (256 per pair)
constexpr int kTN = 256;  // max pairs per tile (MMA N); the kernel takes TN in {64, 128, 256}
constexpr int kBN = 128;  // max B rows per CTA (TN / 2)
constexpr int kKS = 64;   // K slab
constexpr int kStages = 4;
constexpr int kSlabA = kTM * 128;
constexpr int kSlabB = kBN * 128;
constexpr int kStageBytes = 2 * kSlabA + kSlabB;  // 48 KB
constexpr int kProd = 256;
constexpr int kThreads = kProd + 32;
constexpr int kMmaWarp = kProd / 32;
// prefill-pack block: 128 rows x (8 BITS bytes of codes) + 128 x (fp16 scale, fp16 zero)
__host__ __device__ constexpr int cb_bytes(int bits) { return 128 * 8 * bits + 512; }
// code ring depth (slabs, filled by cp.async.bulk): 6 x 2 x 2,560 B (2-bit) or
// 4 x 2 x 3,584 B (3-bit) in the same 30 KB
__host__ __device__ constexpr int cr_depth(int bits) { return bits == 2 ? 6 : 4; }
constexpr int kCR = 6;  // max ring depth
constexpr int kRingBytes = 6 * 2 * cb_bytes(2);
static_assert(4 * 2 * cb_bytes(3) <= kRingBytes, "3-bit code ring");
constexpr int kSmemBytes = kStages * kStageBytes + kRingBytes + 1024;

enum Mode : int {
  kUp = 0,      // A = W1 | W3 rows, B = x rows       -> SwiGLU -> a16
  kDown = 1,    // A = W2 row halves, B = a16 rows    -> y += w * (.)
  kVxUp = 2,    // A = V1 | V3 rows, B = x rows       -> t[.][0|1] (compensated pairs)
  kVxDown = 3,  // A = V2 rows,      B = a16 rows     -> t[.][2]
};

// Per-expert LR pack (bf16, row-major), offsets in elements from the expert's
// base = lrp + e * lrp_stride; R = layer max rank, WU = 64 ceil(2R/64),
// WD = 64 ceil(R/64):
//   u1x [ffn x WU]    [U1 | 0]        u3x [ffn x WU]   [0 | U3]
//   u2x [hidden x WD] [U2 | 0]        vup [2R x hidden] [V1 ; V3]
//   v2  [R x ffn]
struct LrPack {
  int64_t u1x, u3x, u2x, vup, v2, stride;
  int WU, WD;
};
__host__ __device__ inline LrPack lr_pack_layout(int hidden, int ffn, int R) {
  LrPack L{};
  L.WU = 64 * ((2 * R + 63) / 64);
  L.WD = 64 * ((R + 63) / 64);
  int64_t o = 0;
  L.u1x = o; o += static_cast<int64_t>(ffn) * L.WU;
  L.u3x = o; o += static_cast<int64_t>(ffn) * L.WU;
  L.u2x = o; o += static_cast<int64_t>(hidden) * L.WD;
  L.vup = o; o += static_cast<int64_t>(2 * R) * hidden;
  L.v2 = o;  o += static_cast<int64_t>(R) * ffn;
  L.stride = (o + 63) & ~int64_t(63);
  return L;
}

// Prefill pack: the reference codes + metadata of each weight matrix re-laid
// out (same bytes) as blocks of [128 rows][16 B codes] + [128 rows][scale |
// zero << 16], one block per (128-row block, 64-column slab), blocks ordered
// row-block-major, so one slab of one CTA's A rows is ONE contiguous 2,560-byte
// bulk copy.  Rows past the matrix are zero.
struct PPack {
  int64_t w1, w3, w2, stride;  // byte offsets in an expert's pack
};
__host__ __device__ inline PPack ppack_layout(int hidden, int ffn, int bits) {
  const int64_t up = static_cast<int64_t>((ffn + 127) / 128) * (hidden / 64);
  const int64_t dn = static_cast<int64_t>((hidden + 127) / 128) * (ffn / 64);
  const int cb = cb_bytes(bits);
  PPack L;
  L.w1 = 0;
  L.w3 = up * cb;
  L.w2 = 2 * up * cb;
  L.stride = (2 * up + dn) * cb;
  return L;
}

struct PrefillArgs {
  ExpertArgs a;
  int mode;
  int M, K;      // weight rows, main reduction length
  int lr_slabs;  // K-augmentation slabs (0: layer without compensators)
  const uint16_t* lrp;  // LR packs [ne][stride]
  LrPack L;
  uint16_t* tb;  // [max_pairs][WT] bf16 V.x rows ([t1 | t3] after kVxUp, t2 after kVxDown)
  int WT;
  const uint8_t* ppk;  // prefill packs [ne][PL.stride]
  PPack PL;
  int bits, cb, cr;  // code width, pack block bytes, code ring depth
};

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

__device__ __forceinline__ uint64_t f32x2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ uint32_t bf16x2_of(uint64_t v) {  // round both halves to bf16
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  return pack_bf16(lo, hi);
}

// One row of one 64-column slab: 16 B of 2-bit codes (LSB first) and the
// group's fp16 scale / zero bits.
struct RowSlab {
  uint4 c;
  uint32_t s, z;
};

__global__ void build_ppack_kernel(lrc_expert E, int hidden, int ffn, PPack L, int bits, uint8_t* out) {
  const int64_t up = static_cast<int64_t>((ffn + 127) / 128) * (hidden / 64);
  const int cb = cb_bytes(bits), rb = 8 * bits;  // block bytes, code bytes per row slab
  const int64_t nblk = L.stride / cb;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nblk * 128;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t blk = i >> 7;
    const int r = static_cast<int>(i & 127);
    const lrc_qmat& W = blk < up ? E.w1 : (blk < 2 * up ? E.w3 : E.w2);
    const int64_t b = blk < 2 * up ? blk % up : blk - 2 * up;
    const int K = blk < 2 * up ? hidden : ffn, M = blk < 2 * up ? ffn : hidden;
    const int nslab = K / 64;
    const int row = static_cast<int>(b / nslab) * 128 + r, s = static_cast<int>(b % nslab);
    uint2 c[3] = {make_uint2(0, 0), make_uint2(0, 0), make_uint2(0, 0)};
    uint32_t sz = 0;
    if (row < M) {
      // the row slab's codes: 8 BITS bytes of the reference's LSB-first stream
      const uint2* src = reinterpret_cast<const uint2*>(W.packed + ((static_cast<int64_t>(row) * K + s * 64) * bits >> 3));
      for (int i = 0; i < bits; ++i) c[i] = src[i];
      const int64_t g = static_cast<int64_t>(row) * nslab + s;
      sz = static_cast<uint32_t>(W.scales[g]) | (static_cast<uint32_t>(W.zeros[g]) << 16);
    }
    uint8_t* o = out + blk * cb;
    for (int i = 0; i < bits; ++i) *reinterpret_cast<uint2*>(o + rb * r + 8 * i) = c[i];
    *reinterpret_cast<uint32_t*>(o + 128 * rb + 4 * r) = sz;
  }
}

// Dequantize a row slab into its SWIZZLE_128B row.  Code i of a 16-bit field
// is masked in place: (v & 3 << 2i) | 0x4B000000 is the float 2^23 + c*2^2i;
// one FADD2 removes 2^23 and one FFMA2 with s*2^-2i (exact power-of-two
// rescale) and z gives c*s + z with the same single rounding as fmaf(c, s, z).
__device__ __forceinline__ void store_row(uint32_t slab, int r, const RowSlab& v) {
  const float s = h2f(static_cast<uint16_t>(v.s)), z = h2f(static_cast<uint16_t>(v.z));
  uint64_t sp[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) sp[j] = f32x2(s * exp2f(-4.0f * j), s * exp2f(-4.0f * j - 2.0f));
  const uint64_t zz = f32x2(z, z), mm = f32x2(-8388608.0f, -8388608.0f);
  const uint32_t w[4] = {v.c.x, v.c.y, v.c.z, v.c.w};
  uint32_t magic;  // in a register so (b & mask) | magic is ONE lop3 (one immediate per lop3)
  asm("mov.b32 %0, 0x4B000000;" : "=r"(magic));
#pragma unroll
  for (int ch = 0; ch < 8; ++ch) {
    const uint32_t b = (ch & 1) ? (w[ch >> 1] >> 16) : w[ch >> 1];
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t u0, u1;
      asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(u0) : "r"(b), "r"(3u << (4 * j)), "r"(magic));
      asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(u1) : "r"(b), "r"(12u << (4 * j)), "r"(magic));
      const float f0 = __uint_as_float(u0), f1 = __uint_as_float(u1);
      uint64_t t;
      asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(f32x2(f0, f1)), "l"(mm));
      asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(t) : "l"(t), "l"(sp[j]), "l"(zz));
      o[j] = bf16x2_of(t);
    }
    umma::sts128(slab + umma::sw128_chunk(r, ch), o[0], o[1], o[2], o[3]);
  }
}

// 3-bit row slab: 64 codes in 6 words of the LSB-first stream.  Chunk ch (codes
// 8ch..8ch+7) is the 24-bit field at bit 24ch (one funnel shift); code q of
// the field is masked in place into the float 2^23 + c*2^3q (q = 7 is moved
// down 3 bits first: 7*2^21 would carry into the exponent), then as above one
// FADD2 and one FFMA2 with s*2^-3q.
__device__ __forceinline__ void store_row3(uint32_t slab, int r, const uint32_t (&w)[6], uint32_t sb, uint32_t zb) {
  const float s = h2f(static_cast<uint16_t>(sb)), z = h2f(static_cast<uint16_t>(zb));
  uint64_t sp[4];
#pragma unroll
  for (int j = 0; j < 4; ++j)
    sp[j] = f32x2(s * exp2f(-6.0f * j), s * exp2f(j == 3 ? -18.0f : -6.0f * j - 3.0f));
  const uint64_t zz = f32x2(z, z), mm = f32x2(-8388608.0f, -8388608.0f);
  uint32_t magic;
  asm("mov.b32 %0, 0x4B000000;" : "=r"(magic));
#pragma unroll
  for (int ch = 0; ch < 8; ++ch) {
    const int bit = 24 * ch;
    const uint32_t f = __funnelshift_r(w[bit >> 5], w[min((bit >> 5) + 1, 5)], bit & 31);
    const uint32_t f7 = f >> 3;
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t u0, u1;
      asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(u0) : "r"(f), "r"(7u << (6 * j)), "r"(magic));
      if (j == 3)
        asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(u1) : "r"(f7), "r"(7u << 18), "r"(magic));
      else
        asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(u1) : "r"(f), "r"(7u << (6 * j + 3)), "r"(magic));
      uint64_t t;
      asm("add.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(f32x2(__uint_as_float(u0), __uint_as_float(u1))), "l"(mm));
      asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(t) : "l"(t), "l"(sp[j]), "l"(zz));
      o[j] = bf16x2_of(t);
    }
    umma::sts128(slab + umma::sw128_chunk(r, ch), o[0], o[1], o[2], o[3]);
  }
}

// LR pack builder: one thread per element (once per expert upload)
__global__ void build_lr_pack_kernel(lrc_expert E, int hidden, int ffn, int R, LrPack L, uint16_t* out) {
  const int64_t total = L.stride;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float v = 0.0f;
    auto elem = [](const lrc_qmat& m, int64_t r, int64_t c) {
      return (qmat_present(m) && r < m.rows && c < m.cols) ? qmat_elem(m, r, c) : 0.0f;
    };
    if (i < L.u3x) {
      const int64_t r = i / L.WU, c = i % L.WU;
      if (c < R) v = elem(E.u1, r, c);
    } else if (i < L.u2x) {
      const int64_t j = i - L.u3x, r = j / L.WU, c = j % L.WU;
      if (c >= R && c < 2 * R) v = elem(E.u3, r, c - R);
    } else if (i < L.vup) {
      const int64_t j = i - L.u2x, r = j / L.WD, c = j % L.WD;
      if (c < R) v = elem(E.u2, r, c);
    } else if (i < L.v2) {
      const int64_t j = i - L.vup, r = j / hidden, c = j % hidden;
      v = r < R ? elem(E.v1, r, c) : elem(E.v3, r - R, c);
    } else if (i < L.v2 + static_cast<int64_t>(R) * ffn) {
      const int64_t j = i - L.v2, r = j / ffn, c = j % ffn;
      v = elem(E.v2, r, c);
    }
    out[i] = f2bf(v);
  }
}

// TN = pairs per tile (MMA N): small batches take N = 64 / 128 so the tensor
// work follows the expert's token count instead of a fixed 256 columns
template <int TN>
__global__ void __launch_bounds__(kThreads, 1) prefill_kernel(const PrefillArgs P) {
  constexpr int kTN = TN, kBN = TN / 2;
  constexpr uint32_t kIdesc = umma::idesc_bf16(2 * kTM, kTN);
  static_assert(kBN % (kProd / 8) == 0, "B gather: rows bn0 + 32 i");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kStages], empty[kStages], done, rfull[kCR], rempty[kCR];
  __shared__ uint32_t tmem_base;
  __shared__ int s_pair[kTN];
  const ExpertArgs& a = P.a;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = static_cast<int>(umma::cluster_rank());
  const bool b_act = P.mode == kDown || P.mode == kVxDown;  // B rows from a16 (else x)
  const bool vx = P.mode >= kVxUp;

  // blockIdx.y -> (active expert, block of kTN of its pairs), identical in both
  // CTAs of the pair; the grid is an upper bound, surplus pairs leave at once
  // (the per-expert pair counts are loaded in parallel: a scan over global
  // loads would be one dependent L2 round trip per active expert)
  __shared__ int s_cnt[LRC_MAX_EXPERTS];
  const int na = a.plan.counts[0];
  for (int i = tid; i < na; i += kThreads) s_cnt[i] = a.plan.active_cnt[i];
  __syncthreads();
  int yb = blockIdx.y, ai = -1;
  for (int i = 0; i < na; ++i) {
    const int nt = (s_cnt[i] + kTN - 1) / kTN;
    if (yb < nt) {
      ai = i;
      break;
    }
    yb -= nt;
  }
  if (ai < 0) return;
  const int e = a.plan.active[ai];
  const int off = a.plan.active_off[ai] + yb * kTN;
  const int nvalid = min(kTN, s_cnt[ai] - yb * kTN);
  // rows of this CTA's A1 / A3 operands (row of TMEM lane l = base + l)
  const int tile = blockIdx.x >> 1;
  const int a1base = tile * (P.mode == kDown ? 4 * kTM : 2 * kTM) + rank * kTM;
  const int a3base = a1base + (P.mode == kDown ? 2 * kTM : 0);

  int any_comp = 0;
  for (int n = tid; n < kTN; n += kThreads) {
    int p = -1;
    if (n < nvalid) {
      p = a.plan.pair_list[off + n];
      any_comp |= a.plan.pair_comp[p] >= 0;
    }
    s_pair[n] = p;
  }
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      // leader: its producers + the peer's forwarder; peer: its producers
      umma::bar_init(&full[i], rank == 0 ? kProd + 1 : kProd);
      umma::bar_init(&empty[i], 1);
    }
    umma::bar_init(&done, 1);
    for (int i = 0; i < kCR; ++i) {
      umma::bar_init(&rfull[i], 1);
      umma::bar_init(&rempty[i], kProd);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) umma::tmem_alloc2<2 * kTN>(&tmem_base);
  umma::fence_before_sync();
  any_comp = __syncthreads_or(any_comp);  // over all 256 pairs: the same in both CTAs
  umma::cluster_sync();                   // barriers initialised, TMEM allocated in both CTAs
  umma::fence_after_sync();
  const uint32_t tmem = tmem_base;
  if (vx && !any_comp) {  // no compensated pair in this tile: nothing to compute
    umma::fence_before_sync();
    if (warp == kMmaWarp) umma::tmem_dealloc2<2 * kTN>(tmem);
    return;
  }
  const int main_slabs = P.K / kKS;
  const int nslab = main_slabs + ((any_comp && !vx) ? P.lr_slabs : 0);
  const uint16_t* pack = P.lrp ? P.lrp + static_cast<int64_t>(e) * P.L.stride : nullptr;

  if (warp < kMmaWarp) {
    // ------------------------------------------------------------ producers
    const int mat = tid >> 7, rl = tid & (kTM - 1);  // A row rl of A1 (mat 0) / A3 (mat 1)
    const int row = (mat ? a3base : a1base) + rl;
    // copied A rows (bf16 from the LR pack): vx main slabs (V rows) and the
    // K-augmentation slabs (U rows); null = zero row
    const uint16_t* acopy_main = nullptr;  // row start, + 64 s
    const uint16_t* acopy_lr = nullptr;    // row start, + 64 l
    if (pack) {
      if (P.mode == kVxUp && mat == 0 && row < P.M) acopy_main = pack + P.L.vup + static_cast<int64_t>(row) * a.hidden;
      if (P.mode == kVxDown && mat == 0 && row < P.M) acopy_main = pack + P.L.v2 + static_cast<int64_t>(row) * a.ffn;
      if (P.mode == kUp && row < P.M)
        acopy_lr = pack + (mat ? P.L.u3x : P.L.u1x) + static_cast<int64_t>(row) * P.L.WU;
      if (P.mode == kDown && row < P.M) acopy_lr = pack + P.L.u2x + static_cast<int64_t>(row) * P.L.WD;
    }
    // B gather: this CTA's pairs [128 rank, +128): 8 lanes per 128-byte row,
    // rows bn0 + 32 i; per-thread sources fixed for the tile
    const int bc = tid & 7, bn0 = tid >> 3;
    constexpr int kBRows = kBN / (kProd / 8);
    const uint16_t* bsrc[kBRows];
    const uint16_t* tsrc[kBRows];  // the pair's V.x row (K-augmentation slabs)
    uint32_t bmask = 0;
#pragma unroll
    for (int i = 0; i < kBRows; ++i) {
      const int p = s_pair[rank * kBN + bn0 + (kProd / 8) * i];
      bsrc[i] = a.x + bc * 8;
      tsrc[i] = a.x + bc * 8;
      if (p >= 0) {
        bsrc[i] = (b_act ? a.a16 + static_cast<int64_t>(p) * a.ffn
                         : a.x + static_cast<int64_t>(a.plan.pair_token[p]) * a.hidden) + bc * 8;
        if (P.tb) tsrc[i] = P.tb + static_cast<int64_t>(p) * P.WT + bc * 8;
        bmask |= 1u << i;
      }
    }
    const uint32_t sbase = umma::smem_u32(sm);
    const uint32_t bdst0 = sbase + 2 * kSlabA + umma::sw128_chunk(bn0, bc);
    const uint32_t adst0 = sbase + mat * kSlabA + rl * 128;  // + swizzled chunk offset per copy
    // cp.async group of slab s: its B rows and, for copied slabs, this thread's A row
    auto issue = [&](int s) {
      const uint32_t st = (s % kStages) * kStageBytes;
      const bool lr = s >= main_slabs;
      const int k0 = (lr ? s - main_slabs : s) * kKS;
#pragma unroll
      for (int i = 0; i < kBRows; ++i) {
        const bool ok = (bmask >> i) & 1;
        umma::cp_async16(bdst0 + st + i * (kProd / 8) * 128, (lr ? tsrc[i] : bsrc[i]) + (ok ? k0 : 0),
                         ok ? 16u : 0u);
      }
      const uint16_t* ar = lr ? acopy_lr : (vx ? acopy_main : nullptr);
      if (lr || (vx && mat == 0)) {  // (vx: A3 unused)
#pragma unroll
        for (int c = 0; c < 8; ++c)
          umma::cp_async16(adst0 + st + ((static_cast<uint32_t>(c) ^ static_cast<uint32_t>(rl & 7)) << 4),
                           ar ? ar + k0 + 8 * c : a.x, ar ? 16u : 0u);
      }
      umma::cp_async_commit();
    };
    // One slab: dequantize A from the code ring (filled kCR slabs ahead by
    // the bulk-copy loader) unless the slab is copied, wait for the slab's
    // cp.async group, publish the stage; then start the copies two slabs ahead.
    const uint32_t ring = sbase + kStages * kStageBytes + mat * P.cb;
    const int cr = P.cr;
    issue(0);
    if (nslab > 1) issue(1);
    for (int s = 0; s < nslab; ++s) {
      const int stage = s % kStages;
      if (s < main_slabs && !vx) {
        const int slot = s % cr;
        umma::bar_wait(&rfull[slot], (s / cr) & 1);
        const uint32_t blk = ring + slot * 2 * P.cb;
        uint32_t sz;
        if (P.bits == 2) {
          RowSlab v;
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(v.c.x), "=r"(v.c.y), "=r"(v.c.z), "=r"(v.c.w)
                       : "r"(blk + 16 * rl));
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(sz) : "r"(blk + 2048 + 4 * rl));
          umma::bar_arrive(&rempty[slot]);
          v.s = sz & 0xFFFFu;
          v.z = sz >> 16;
          store_row(sbase + stage * kStageBytes + mat * kSlabA, rl, v);
        } else {
          uint32_t w[6];
#pragma unroll
          for (int i = 0; i < 3; ++i)
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(w[2 * i]), "=r"(w[2 * i + 1]) : "r"(blk + 24 * rl + 8 * i));
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(sz) : "r"(blk + 3072 + 4 * rl));
          umma::bar_arrive(&rempty[slot]);
          store_row3(sbase + stage * kStageBytes + mat * kSlabA, rl, w, sz & 0xFFFFu, sz >> 16);
        }
      }
      if (s + 1 < nslab)
        umma::cp_async_wait<1>();  // slab s landed; slab s+1 may be in flight
      else
        umma::cp_async_wait<0>();
      umma::fence_proxy_async();  // generic smem writes (and landed cp.async) -> tensor core
      umma::bar_arrive(&full[stage]);
      const int sb = s + 2;
      if (sb < nslab) {
        if (sb >= kStages) umma::bar_wait_cluster(&empty[sb % kStages], ((sb / kStages) - 1) & 1);
        issue(sb);
      }
    }
  } else if (rank == 0 && lane == 0) {
    // ------------------------------------------------------------ MMA issue (leader)
    for (int s = 0; s < nslab; ++s) {
      const int stage = s % kStages;
      umma::bar_wait_cluster(&full[stage], (s / kStages) & 1);
      umma::fence_after_sync();
      const uint32_t a1 = umma::smem_u32(sm + stage * kStageBytes), a3 = a1 + kSlabA, b = a3 + kSlabA;
#pragma unroll
      for (int kk = 0; kk < kKS / 16; ++kk) {
        const uint32_t acc = (s | kk) != 0 ? 1u : 0u;
        const uint64_t db = umma::sdesc(b + 32 * kk);
        umma::mma2_bf16(tmem, umma::sdesc(a1 + 32 * kk), db, kIdesc, acc);
        if (!vx) umma::mma2_bf16(tmem + kTN, umma::sdesc(a3 + 32 * kk), db, kIdesc, acc);
      }
      umma::commit2(&empty[stage]);
    }
    umma::commit2(&done);
  } else if (lane == 1) {
    // ------------------------------------------------------------ code loader
    // one 2,560-byte bulk copy per A matrix per slab from the prefill pack into
    // the code ring, kCR slabs ahead of the dequantizing producers
    if (!vx && P.ppk) {
      const uint8_t* pk = P.ppk + static_cast<int64_t>(e) * P.PL.stride;
      const int nblkM = (P.M + kTM - 1) / kTM;
      const bool v1 = a1base < P.M, v3 = a3base < P.M;
      const int cb = P.cb, cr = P.cr;
      const uint8_t* s1 = pk + (P.mode == kDown ? P.PL.w2 : P.PL.w1) +
                          static_cast<int64_t>(min(a1base / kTM, nblkM - 1)) * main_slabs * cb;
      const uint8_t* s3 = pk + (P.mode == kDown ? P.PL.w2 : P.PL.w3) +
                          static_cast<int64_t>(min(a3base / kTM, nblkM - 1)) * main_slabs * cb;
      const uint32_t ring0 = umma::smem_u32(sm) + kStages * kStageBytes;
      for (int s = 0; s < main_slabs; ++s) {
        const int slot = s % cr;
        if (s >= cr) umma::bar_wait(&rempty[slot], ((s / cr) - 1) & 1);
        const uint32_t bar = umma::smem_u32(&rfull[slot]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"((v1 ? cb : 0) + (v3 ? cb : 0))
                     : "memory");
        const uint32_t dst = ring0 + slot * 2 * cb;
        if (v1)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
              "l"(s1 + static_cast<int64_t>(s) * cb), "r"(cb), "r"(bar)
              : "memory");
        if (v3)
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  dst + cb),
              "l"(s3 + static_cast<int64_t>(s) * cb), "r"(cb), "r"(bar)
              : "memory");
      }
    }
  } else if (rank == 1 && lane == 0) {
    // ------------------------------------------------------------ forwarder (peer)
    // one cluster-scope release per stage: the peer's stage is complete ->
    // arrive on the leader's barrier (cumulative over the acquired arrivals)
    for (int s = 0; s < nslab; ++s) {
      const int stage = s % kStages;
      umma::bar_wait(&full[stage], (s / kStages) & 1);
      umma::bar_arrive_cta(&full[stage], 0);
    }
  }

  if (warp < kMmaWarp) {
    // ------------------------------------------------------------ epilogue
    // warp w reads TMEM lanes 32(w&3).. (rows) for pair columns [128(w>>2), +128)
    umma::bar_wait_cluster(&done, 0);
    umma::fence_after_sync();
    const int q = warp & 3, half = warp >> 2;
    const uint32_t lbase = tmem + (static_cast<uint32_t>(q * 32) << 16);
    const int ra = a1base + q * 32 + lane, rb = a3base + q * 32 + lane;
    const int cend = min(nvalid, (half + 1) * (kTN / 2));
    // up: activations staged pair-major in the (now idle) stage memory, then
    // written out as 16-byte rows (coalesced) instead of 2-byte scattered stores
    uint16_t* stg = reinterpret_cast<uint16_t*>(sm);  // [kTN pairs][kTM rows] bf16
    for (int c0 = half * (kTN / 2); c0 < cend; c0 += 32) {
      float h1[32], h3[32];
      {
        uint32_t r1[32], r3[32];
        umma::tmem_ld32_nowait(lbase + c0, r1);
        if (!vx) umma::tmem_ld32_nowait(lbase + kTN + c0, r3);
        umma::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          h1[j] = __uint_as_float(r1[j]);
          h3[j] = vx ? 0.0f : __uint_as_float(r3[j]);
        }
      }
      if (P.mode == kUp) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float g = h1[j];
          stg[(c0 + j) * kTM + q * 32 + lane] = f2bf(__fdividef(g, 1.0f + __expf(-g)) * h3[j]);
        }
      } else if (P.mode == kDown) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int n = c0 + j;
          if (n < nvalid) {
            const int p = s_pair[n];
            const float w = a.plan.pair_w[p];
            float* yr = a.y + static_cast<int64_t>(a.plan.pair_token[p]) * a.hidden;
            if (ra < P.M) atomicAdd(yr + ra, w * h1[j]);
            if (rb < P.M) atomicAdd(yr + rb, w * h3[j]);
          }
        }
      } else if (ra < P.WT) {  // V.x rows -> the pair's bf16 t row (zero when uncompensated)
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int n = c0 + j;
          if (n < nvalid) {
            const int p = s_pair[n];
            P.tb[static_cast<int64_t>(p) * P.WT + ra] = a.plan.pair_comp[p] >= 0 ? f2bf(h1[j]) : 0;
          }
        }
      }
    }
    if (P.mode == kUp) {
      asm volatile("bar.sync 1, %0;" ::"n"(kProd) : "memory");  // producers only
      const int r0 = a1base;  // this CTA's rows [r0, r0 + 128)
      for (int i = tid; i < nvalid * (kTM / 8); i += kProd) {
        const int n = i / (kTM / 8), c = i % (kTM / 8);
        const int row = r0 + 8 * c;
        uint16_t* dst = a.a16 + static_cast<int64_t>(s_pair[n]) * a.ffn + row;
        const uint16_t* src = stg + n * kTM + 8 * c;
        if (row + 8 <= P.M) {
          *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
        } else {
          for (int k = 0; k < 8 && row + k < P.M; ++k) dst[k] = src[k];
        }
      }
    }
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::cluster_sync();
  if (warp == kMmaWarp) umma::tmem_dealloc2<2 * kTN>(tmem);
}

}  // namespace

bool prefill_eligible(const lrc_expert* experts, int n, int hidden, int ffn, int maxr, int* bits) {
  if (hidden % kKS != 0 || ffn % kKS != 0 || maxr > kTM || n < 1) return false;
  const int b = experts[0].w1.bits;  // one code width per layer (2 or 3)
  if (b != 2 && b != 3) return false;
  for (int i = 0; i < n; ++i) {
    const lrc_qmat* ws[3] = {&experts[i].w1, &experts[i].w3, &experts[i].w2};
    for (auto w : ws)
      if (w->dense != nullptr || w->packed == nullptr || w->bits != b || w->group_size != kKS ||
          (reinterpret_cast<uintptr_t>(w->packed) & 15) != 0)
        return false;
  }
  *bits = b;
  return true;
}

int64_t prefill_lr_pack_elems(int hidden, int ffn, int maxr) {
  return maxr ? lr_pack_layout(hidden, ffn, maxr).stride : 0;
}
int prefill_tb_width(int maxr) {
  if (!maxr) return 0;
  const LrPack L = lr_pack_layout(64, 64, maxr);
  return L.WU > L.WD ? L.WU : L.WD;
}

lrc_status build_prefill_lr(const lrc_expert& e, int hidden, int ffn, int maxr, uint16_t* out, cudaStream_t st) {
  if (!maxr) return LRC_OK;
  const LrPack L = lr_pack_layout(hidden, ffn, maxr);
  build_lr_pack_kernel<<<592, 256, 0, st>>>(e, hidden, ffn, maxr, L, out);
  LRC_CHECK_LAUNCH();
  return LRC_OK;
}

int64_t prefill_pack_bytes(int hidden, int ffn, int bits) { return ppack_layout(hidden, ffn, bits).stride; }

lrc_status build_prefill_pack(const lrc_expert& e, int hidden, int ffn, int bits, uint8_t* out, cudaStream_t st) {
  build_ppack_kernel<<<592, 256, 0, st>>>(e, hidden, ffn, ppack_layout(hidden, ffn, bits), bits, out);
  LRC_CHECK_LAUNCH();
  return LRC_OK;
}

lrc_status launch_prefill(const ExpertArgs& a, int np_bound, int max_tok, const uint16_t* lrp, uint16_t* tb,
                          const uint8_t* ppk, int bits, cudaStream_t st, int* launches) {
  static bool attr = false;
  if (!attr) {
    LRC_CUDA_TRY(cudaFuncSetAttribute(prefill_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    LRC_CUDA_TRY(cudaFuncSetAttribute(prefill_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    LRC_CUDA_TRY(cudaFuncSetAttribute(prefill_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    attr = true;
  }
  // MMA N per tile: the smallest that holds the largest possible expert batch
  // (an expert sees at most B pairs); LRC_PREFILL_TN overrides
  static const int tn_env = getenv("LRC_PREFILL_TN") ? atoi(getenv("LRC_PREFILL_TN")) : 0;
  const int tn = tn_env == 64 || tn_env == 128 || tn_env == 256 ? tn_env
                 : (max_tok <= 64 ? 64 : (max_tok <= 128 ? 128 : 256));
  PrefillArgs P{};
  P.a = a;
  P.ppk = ppk;
  P.PL = ppack_layout(a.hidden, a.ffn, bits);
  P.bits = bits;
  P.cb = cb_bytes(bits);
  P.cr = cr_depth(bits);
  const int R = lrp ? a.maxr : 0;
  if (R) {
    P.lrp = lrp;
    P.L = lr_pack_layout(a.hidden, a.ffn, R);
    P.tb = tb;
    P.WT = prefill_tb_width(R);
  }
  const int ytiles = (np_bound + tn - 1) / tn + a.ne;  // >= sum over experts of ceil(cnt / tn)
  auto launch = [&](int mode, int M, int K, int lr_slabs, int rows_per_pair) -> lrc_status {
    P.mode = mode;
    P.M = M;
    P.K = K;
    P.lr_slabs = lr_slabs;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * ((M + rows_per_pair - 1) / rows_per_pair), ytiles);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (tn == 64)
      LRC_CUDA_TRY(cudaLaunchKernelEx(&cfg, prefill_kernel<64>, P));
    else if (tn == 128)
      LRC_CUDA_TRY(cudaLaunchKernelEx(&cfg, prefill_kernel<128>, P));
    else
      LRC_CUDA_TRY(cudaLaunchKernelEx(&cfg, prefill_kernel<256>, P));
    ++*launches;
    return LRC_OK;
  };
  lrc_status s;
  if (R && (s = launch(kVxUp, 2 * R, a.hidden, 0, 2 * kTM)) != LRC_OK) return s;
  if ((s = launch(kUp, a.ffn, a.hidden, R ? P.L.WU / kKS : 0, 2 * kTM)) != LRC_OK) return s;
  if (R && (s = launch(kVxDown, R, a.ffn, 0, 2 * kTM)) != LRC_OK) return s;
  return launch(kDown, a.hidden, a.ffn, R ? P.L.WD / kKS : 0, 4 * kTM);
}

}  // namespace lrc
