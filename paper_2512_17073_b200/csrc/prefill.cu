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
// Roles per CTA (288 threads, one CTA per SM: 193 KB smem, 512 TMEM columns):
//   warps 0-7  producers: thread t dequantizes row t&127 of matrix t>>7 (c*s+z
//              in fp32, rounded once to bf16; codes and metadata prefetched four
//              slabs ahead) straight into SWIZZLE_128B smem, gathers its share
//              of the CTA's 128 B rows with cp.async two slabs ahead (zero-filled
//              past the expert's pairs) and release-arrives on the LEADER's
//              stage barrier; after the K loop, the epilogue from its own TMEM.
//   warp 8     (leader CTA) one thread issues tcgen05.mma.cta_group::2
//              (M=256, N=256, K=16) into the two fp32 accumulators and commits
//              each stage back to both CTAs (multicast; 4-stage ring).
// The pair halves each SM's share of the B operand (gather and smem reads).
// The low-rank term is K augmentation: extra slabs whose A rows hold the U
// factors (up: U1 in columns [0, R), U3 in [R, 2R); down: U2) and whose B rows
// hold the pair's V.x vectors t (zero for uncompensated pairs), so U.(V.x)
// lands in the same accumulator and Q(W)+UV^T is never formed.
#include <cuda_bf16.h>

#include "common.cuh"
#include "layer.cuh"
#include "umma.cuh"

namespace lrc {
namespace {

constexpr int kTM = 128;  // rows per accumulator per CTA (256 per pair)
constexpr int kTN = 256;  // pairs per tile (MMA N)
constexpr int kBN = 128;  // B rows per CTA
constexpr int kKS = 64;   // K slab
constexpr int kStages = 4;
constexpr int kSlabA = kTM * 128;
constexpr int kSlabB = kBN * 128;
constexpr int kStageBytes = 2 * kSlabA + kSlabB;  // 48 KB
constexpr int kProd = 256;
constexpr int kThreads = kProd + 32;
constexpr int kMmaWarp = kProd / 32;
constexpr int kSmemBytes = kStages * kStageBytes + 1024;
constexpr int kPD = 4;  // code prefetch distance (slabs)
constexpr uint32_t kIdesc = umma::idesc_bf16(2 * kTM, kTN);

enum Mode : int {
  kUp = 0,      // A = W1 | W3 rows, B = x rows       -> SwiGLU -> a16
  kDown = 1,    // A = W2 row halves, B = a16 rows    -> y += w * (.)
  kVxUp = 2,    // A = V1 | V3 rows, B = x rows       -> t[.][0|1] (compensated pairs)
  kVxDown = 3,  // A = V2 rows,      B = a16 rows     -> t[.][2]
};

struct PrefillArgs {
  ExpertArgs a;
  int mode;
  int M, K;      // weight rows, main reduction length
  int lr_slabs;  // K-augmentation slabs (0: layer without compensators)
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

// Codes and group metadata of one row for one 64-column slab (reference
// layout: row-major LSB-first 2-bit stream, one fp16 scale/zero per group).
// Metadata stays raw until use so a prefetch never waits on its load.
struct RowSlab {
  uint4 c;
  uint32_t s, z;  // fp16 bits
};

// The matrix pointers live in registers (QPtr), not behind the expert-table
// reference, so a prefetch is one dependent-free load.
struct QPtr {
  const uint8_t* packed;
  const uint16_t* scales;
  const uint16_t* zeros;
};

__device__ __forceinline__ RowSlab load_row(const QPtr& W, int row, int M, int K, int k0) {
  RowSlab r{make_uint4(0, 0, 0, 0), 0u, 0u};
  if (row < M) {
    const int64_t e0 = static_cast<int64_t>(row) * K + k0;
    // volatile: issued where written (two slabs ahead), never sunk to the use
    asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.c.x), "=r"(r.c.y), "=r"(r.c.z), "=r"(r.c.w)
                 : "l"(W.packed + (e0 >> 2)));
    const int64_t g = static_cast<int64_t>(row) * (K / kKS) + k0 / kKS;
    asm volatile("ld.global.nc.u16 %0, [%1];" : "=r"(r.s) : "l"(W.scales + g));
    asm volatile("ld.global.nc.u16 %0, [%1];" : "=r"(r.z) : "l"(W.zeros + g));
  }
  return r;
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

__device__ __forceinline__ int64_t t_index(const ExpertArgs& a, int p, int proj) {
  return ((static_cast<int64_t>(a.plan.pair_token[p]) * a.ne + a.plan.pair_expert[p]) * 3 + proj) * a.maxr;
}

template <int BITS>
__device__ __forceinline__ void store_q_row_g64(uint32_t slab, int r, const lrc_qmat& U, int row, int gcol0) {
  const uint32_t* words = reinterpret_cast<const uint32_t*>(U.packed);
  const int64_t bit0 = (static_cast<int64_t>(row) * U.cols + gcol0) * BITS;  // multiple of 64*BITS: word aligned
  const int64_t g = static_cast<int64_t>(row) * (U.cols / kKS) + gcol0 / kKS;
  const float s = h2f(U.scales[g]), z = h2f(U.zeros[g]);
  uint32_t w[2 * BITS + 1];
#pragma unroll
  for (int i = 0; i < 2 * BITS; ++i) w[i] = __ldg(words + (bit0 >> 5) + i);
  w[2 * BITS] = 0u;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int b = (8 * j + q) * BITS;
      v[q] = fmaf(static_cast<float>(__funnelshift_r(w[b >> 5], w[(b >> 5) + 1], b & 31) & ((1u << BITS) - 1u)),
                  s, z);
    }
    umma::sts128(slab + umma::sw128_chunk(r, j), pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
                 pack_bf16(v[6], v[7]));
  }
}

// Columns [gcol0, gcol0 + 64) of row `row` of a quantized (or dense) matrix,
// shifted right by c0 (element col - c0; zero outside [0, cols) and for absent
// rows) -> one SWIZZLE_128B row.  For the low-rank factors: U rows of the
// K-augmentation slabs, V rows of the V.x GEMMs.
__device__ __noinline__ void store_q_row(uint32_t slab, int r, const lrc_qmat& U, int row, int gcol0, int c0) {
  const bool pres = qmat_present(U) && row >= 0 && row < U.rows;
  if (pres && c0 == 0 && U.dense == nullptr && U.group_size == kKS && (U.cols % kKS) == 0 &&
      gcol0 + kKS <= U.cols) {
    if (U.bits == 3) return store_q_row_g64<3>(slab, r, U, row, gcol0);
    if (U.bits == 2) return store_q_row_g64<2>(slab, r, U, row, gcol0);
    if (U.bits == 4) return store_q_row_g64<4>(slab, r, U, row, gcol0);
  }
#pragma unroll 1
  for (int j = 0; j < 8; ++j) {
    float v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int col = gcol0 + 8 * j + q - c0;
      v[q] = (pres && col >= 0 && col < U.cols) ? qmat_elem(U, row, col) : 0.0f;
    }
    umma::sts128(slab + umma::sw128_chunk(r, j), pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
                 pack_bf16(v[6], v[7]));
  }
}

__global__ void __launch_bounds__(kThreads, 1) prefill_kernel(const PrefillArgs P) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[kStages], empty[kStages], done;
  __shared__ uint32_t tmem_base;
  __shared__ int s_pair[kTN];
  const ExpertArgs& a = P.a;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = static_cast<int>(umma::cluster_rank());
  const bool b_act = P.mode == kDown || P.mode == kVxDown;  // B rows from a16 (else x)
  const bool vx = P.mode >= kVxUp;

  // blockIdx.y -> (active expert, block of kTN of its pairs), identical in both
  // CTAs of the pair; the grid is an upper bound, surplus pairs leave at once
  int yb = blockIdx.y, ai = -1;
  const int na = a.plan.counts[0];
  for (int i = 0; i < na; ++i) {
    const int nt = (a.plan.active_cnt[i] + kTN - 1) / kTN;
    if (yb < nt) {
      ai = i;
      break;
    }
    yb -= nt;
  }
  if (ai < 0) return;
  const int e = a.plan.active[ai];
  const lrc_expert& E = a.experts[e];
  const int off = a.plan.active_off[ai] + yb * kTN;
  const int nvalid = min(kTN, a.plan.active_cnt[ai] - yb * kTN);
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

  if (warp < kMmaWarp) {
    // ------------------------------------------------------------ producers
    const int mat = tid >> 7, rl = tid & (kTM - 1);  // A row rl of A1 (mat 0) / A3 (mat 1)
    const lrc_qmat* Wp;
    const int row = (mat ? a3base : a1base) + rl;
    switch (P.mode) {
      case kUp: Wp = mat ? &E.w3 : &E.w1; break;
      case kDown: Wp = &E.w2; break;
      case kVxUp: Wp = mat ? &E.v3 : &E.v1; break;
      default: Wp = mat ? nullptr : &E.v2; break;  // A3 unused (zero)
    }
    const lrc_qmat& W = Wp ? *Wp : E.v2;
    const QPtr Wq{W.packed, W.scales, W.zeros};
    const int qrow = (Wp && row < P.M) ? row : -1;  // quantized-factor row (vx) or -1 = zero
    // B gather: this CTA's pairs [128 rank, +128): 8 lanes per 128-byte row,
    // rows bn0 + 32 i; per-thread sources fixed for the tile
    const int bc = tid & 7, bn0 = tid >> 3;
    constexpr int kBRows = kBN / (kProd / 8);
    const uint16_t* bsrc[kBRows];
    uint32_t bmask = 0;
#pragma unroll
    for (int i = 0; i < kBRows; ++i) {
      const int p = s_pair[rank * kBN + bn0 + (kProd / 8) * i];
      bsrc[i] = a.x + bc * 8;
      if (p >= 0) {
        bsrc[i] = (b_act ? a.a16 + static_cast<int64_t>(p) * a.ffn
                         : a.x + static_cast<int64_t>(a.plan.pair_token[p]) * a.hidden) + bc * 8;
        bmask |= 1u << i;
      }
    }
    const uint32_t bdst0 = umma::smem_u32(sm + 2 * kSlabA) + umma::sw128_chunk(bn0, bc);
    auto issue_b = [&](int s) {
      const uint32_t bb = bdst0 + (s % kStages) * kStageBytes;
      const int k0 = s * kKS;
#pragma unroll
      for (int i = 0; i < kBRows; ++i)
        umma::cp_async16(bb + i * (kProd / 8) * 128, bsrc[i] + ((bmask >> i) & 1 ? k0 : 0),
                         (bmask >> i) & 1 ? 16u : 0u);
      umma::cp_async_commit();
    };
    // One slab: dequantize A (codes prefetched kPD slabs earlier: scattered
    // 16-byte row reads need a long lead under load), wait for this slab's B
    // rows, publish the stage; then start the B gather two slabs ahead and the
    // codes kPD slabs ahead.  Unrolled by kPD + 1 below so the prefetch
    // registers rotate by name (no copies waiting on loads).
    auto step = [&](int s, const RowSlab& cur, RowSlab& dst) {
      const int stage = s % kStages;
      const uint32_t As = umma::smem_u32(sm) + stage * kStageBytes + mat * kSlabA;
      const uint32_t Bs = umma::smem_u32(sm) + stage * kStageBytes + 2 * kSlabA;
      if (s < main_slabs) {
        if (vx)
          store_q_row(As, rl, W, qrow, s * kKS, 0);
        else
          store_row(As, rl, cur);
        if (s + 1 < main_slabs)
          umma::cp_async_wait<1>();  // B(s) landed; B(s+1) may be in flight
        else
          umma::cp_async_wait<0>();
      } else {
        // K augmentation slab: columns [g0, g0 + 64) of [t1 | t3] (up) or t2 (down)
        if (s >= kStages) umma::bar_wait(&empty[stage], ((s / kStages) - 1) & 1);
        const int g0 = (s - main_slabs) * kKS, R = a.maxr;
        if (P.mode == kDown)
          store_q_row(As, rl, E.u2, row, g0, 0);
        else
          store_q_row(As, rl, mat ? E.u3 : E.u1, row, g0, mat ? R : 0);
        if (tid < kBN) {  // one B row per thread
          const int n = tid;
          const int p = s_pair[rank * kBN + n];
          const bool comp = p >= 0 && a.plan.pair_comp[p] >= 0;
#pragma unroll 1
          for (int j = 0; j < 8; ++j) {
            float v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int col = g0 + 8 * j + q;
              float t = 0.0f;
              if (comp) {
                if (P.mode == kDown) {
                  if (col < R) t = a.t[t_index(a, p, 2) + col];
                } else if (col < R) {
                  t = a.t[t_index(a, p, 0) + col];
                } else if (col < 2 * R) {
                  t = a.t[t_index(a, p, 1) + col - R];
                }
              }
              v[q] = t;
            }
            umma::sts128(Bs + umma::sw128_chunk(n, j), pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]),
                         pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7]));
          }
        }
      }
      umma::fence_proxy_async();  // generic smem writes (and landed cp.async) -> tensor core
      umma::bar_arrive(&full[stage]);  // CTA scope: never waits on the prefetches in flight
      const int sb = s + 2;
      if (sb < main_slabs) {
        if (sb >= kStages) umma::bar_wait_cluster(&empty[sb % kStages], ((sb / kStages) - 1) & 1);
        issue_b(sb);
      }
      if (!vx && s + kPD < main_slabs) dst = load_row(Wq, row, P.M, P.K, (s + kPD) * kKS);
    };
    issue_b(0);
    if (main_slabs > 1) issue_b(1);
    RowSlab rs[kPD + 1];
#pragma unroll
    for (int i = 0; i <= kPD; ++i) rs[i] = RowSlab{};
    if (!vx) {
#pragma unroll
      for (int i = 0; i < kPD; ++i)
        if (i < main_slabs) rs[i] = load_row(Wq, row, P.M, P.K, i * kKS);
    }
    for (int s = 0; s < nslab; s += kPD + 1) {
#pragma unroll
      for (int i = 0; i <= kPD; ++i)
        if (s + i < nslab) step(s + i, rs[i], rs[(i + kPD) % (kPD + 1)]);
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
        umma::mma2_bf16(tmem + kTN, umma::sdesc(a3 + 32 * kk), db, kIdesc, acc);
      }
      umma::commit2(&empty[stage]);
    }
    umma::commit2(&done);
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
    for (int c0 = half * (kTN / 2); c0 < cend; c0 += 32) {
      float h1[32], h3[32];
      umma::tmem_ld32(lbase + c0, h1);
      umma::tmem_ld32(lbase + kTN + c0, h3);
      if (P.mode == kUp) {
        if (ra < P.M) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int n = c0 + j;
            if (n < nvalid) {
              const float g = h1[j];
              a.a16[static_cast<int64_t>(s_pair[n]) * a.ffn + ra] =
                  f2bf(__fdividef(g, 1.0f + __expf(-g)) * h3[j]);
            }
          }
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
      } else if (ra < a.maxr) {  // V.x rows -> t of the compensated pairs
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int n = c0 + j;
          if (n < nvalid) {
            const int p = s_pair[n];
            if (a.plan.pair_comp[p] >= 0) {
              if (P.mode == kVxUp) {
                a.t[t_index(a, p, 0) + ra] = h1[j];
                a.t[t_index(a, p, 1) + ra] = h3[j];
              } else {
                a.t[t_index(a, p, 2) + ra] = h1[j];
              }
            }
          }
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

bool prefill_eligible(const lrc_expert* experts, int n, int hidden, int ffn, int maxr) {
  if (hidden % kKS != 0 || ffn % kKS != 0 || maxr > 2 * kTM) return false;
  for (int i = 0; i < n; ++i) {
    const lrc_qmat* ws[3] = {&experts[i].w1, &experts[i].w3, &experts[i].w2};
    for (auto w : ws)
      if (w->dense != nullptr || w->packed == nullptr || w->bits != 2 || w->group_size != kKS ||
          (reinterpret_cast<uintptr_t>(w->packed) & 15) != 0)
        return false;
  }
  return true;
}

lrc_status launch_prefill(const ExpertArgs& a, int np_bound, cudaStream_t st, int* launches) {
  static bool attr = false;
  if (!attr) {
    LRC_CUDA_TRY(cudaFuncSetAttribute(prefill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes));
    attr = true;
  }
  PrefillArgs P{};
  P.a = a;
  const int ytiles = (np_bound + kTN - 1) / kTN + a.ne;  // >= sum over experts of ceil(cnt / kTN)
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
    LRC_CUDA_TRY(cudaLaunchKernelEx(&cfg, prefill_kernel, P));
    ++*launches;
    return LRC_OK;
  };
  lrc_status s;
  const int R = a.maxr;
  if (R && (s = launch(kVxUp, R, a.hidden, 0, 2 * kTM)) != LRC_OK) return s;
  if ((s = launch(kUp, a.ffn, a.hidden, R ? (2 * R + kKS - 1) / kKS : 0, 2 * kTM)) != LRC_OK) return s;
  if (R && (s = launch(kVxDown, R, a.ffn, 0, 2 * kTM)) != LRC_OK) return s;
  return launch(kDown, a.hidden, a.ffn, R ? (R + kKS - 1) / kKS : 0, 4 * kTM);
}

}  // namespace lrc
