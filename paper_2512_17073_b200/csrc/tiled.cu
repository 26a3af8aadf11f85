// Tiled low-bit expert kernels (2-bit codes, group size 64) for sm_100a.
//
// HBM layout ("T2 tiles"): a matrix (M, K) is cut into 16-row tiles and
// 128-column group pairs.  Block (tile t, group-pair q, matrix i) is 640 B:
//   [0,512)   codes: lane l holds 16 B = 4 words W0..W3 (gid = l>>2, tid = l&3);
//             word Wk covers the mma.m16n8k32 K slice k (m = k>>1, half = k&1)
//             of both groups and both rows of the lane: byte b, plane p
//             (bits 8b + 2p) holds the code at column g*64 + 32m + 16half +
//             4tid + b of group g = 2q + (p>>1), row t*16 + gid + 8(p&1).
//             So W & (0x03030303 << 2(p&1)) after W >>= 4 (p >> 1) is one u8
//             A-fragment register: row gid codes x1, row gid+8 codes x4 --
//             a per-row factor, folded into that row's epilogue scale.
//   [512,640) fp16 scale/zero: 16 B per gid {s,z}(A,g0) {s,z}(A,g1) {s,z}(B,g0) {s,z}(B,g1)
//             (A = row t*16+gid, B = row t*16+gid+8)
// Blocks are ordered (t, q, i), so one row tile over a K range is one contiguous
// byte range -> one cp.async.bulk per work item.  The codes are exactly the
// reference's (lrc_tiles_unpack inverts the layout bit-exactly).
//
// Core: mma.sync m16n8k32 u8 x s8 -> s32.  The activation operand is each
// token's 64-column group as a 13-bit integer X = rint(x 2^S) (S per group and
// token: |X| <= 2^12), split into two signed 7-bit digits X = 128 d0 + d1 that
// sit in adjacent N columns (one MMA covers 4 tokens); a lane's accumulator
// pair is then {sum c d0, sum c d1} of one token (x4 for the B row), and
// 128 d0 + d1 + the bits of 1.5 * 2^23 is a float whose mantissa holds the
// exact dot product (|4 sum c X| <= 4 * 192 * 2^12 < 2^22).
// Per group:  y += s * 2^-S (sum c X) + z * sum x   (fp32, ref/quant.py:216-224).
// The x rounding moves each x by at most 2^-12 of the group's largest |x|
// (tests/test_host.py::test_tiled_core_digit_arithmetic; the layer's own
// activations carry bf16 rounding, 2^-9 relative).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "layer.cuh"

namespace lrc {

constexpr int kBlk = 640;
constexpr int kCodeBytes = 512;
constexpr int kNEpi = 2;          // epilogue warps: item k -> warp NW + k % kNEpi
// Consumer warps and their K span per pass width (NQ token quads).  In
// isolation the single-quad core gains from 16 warps on 2-group-pair spans
// (tools/core_bench.cu: 1,854 -> 1,697 cycles per 40 KB item), in the kernel
// it does not (B=1 equal, B=2/4 -4%): 8 warps, 512-column spans everywhere
// (TILED_NW1 / TILED_SPAN1 override the single-quad shape for A/B runs).
#ifndef TILED_NW1
#define TILED_NW1 8
#endif
#ifndef TILED_QUNROLL
#define TILED_QUNROLL 1
#endif
constexpr int kQUnroll = TILED_QUNROLL;  // group pairs per consumer loop body
#ifndef TILED_SPAN1
#define TILED_SPAN1 4
#endif
template <int NQ>
struct KCfg {
  static constexpr int NW = NQ == 1 ? TILED_NW1 : 8;
  static constexpr int SPAN = NQ == 1 ? TILED_SPAN1 : 4;  // group pairs per warp span
  static constexpr int THREADS = (NW + kNEpi + 1) * 32;
};

int64_t tiles_bytes(int64_t rows, int64_t cols, int ni) {
  int64_t rt = (rows + 15) / 16, gp = (cols + 127) / 128;
  return rt * gp * ni * kBlk;
}

// ------------------------------------------------------------------ repack --
__global__ void build_tiles_kernel(lrc_qmat m0, lrc_qmat m1, int ni, int64_t RT, int64_t GP,
                                   uint8_t* __restrict__ tiles) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int lane = static_cast<int>(idx & 31);
  const int64_t blk = idx >> 5;
  if (blk >= RT * GP * ni) return;
  const int i = static_cast<int>(blk % ni);
  const int64_t tq = blk / ni;
  const int64_t q = tq % GP, t = tq / GP;
  const lrc_qmat& m = (i == 0) ? m0 : m1;
  const int gid = lane >> 2, tid = lane & 3;
  const int64_t nbytes = (static_cast<int64_t>(m.rows) * m.cols * m.bits + 7) >> 3;
  uint32_t w[4] = {0u, 0u, 0u, 0u};
  for (int kw = 0; kw < 4; ++kw)
    for (int pl = 0; pl < 4; ++pl) {
      const int64_t r = t * 16 + gid + 8 * (pl & 1);
      for (int b = 0; b < 4; ++b) {
        const int64_t k = (2 * q + (pl >> 1)) * 64 + (kw >> 1) * 32 + (kw & 1) * 16 + tid * 4 + b;
        uint32_t c = 0;
        if (r < m.rows && k < m.cols) c = read_code(m.packed, r * m.cols + k, m.bits, nbytes);
        w[kw] |= c << (8 * b + 2 * pl);
      }
    }
  uint8_t* b = tiles + blk * kBlk;
  *reinterpret_cast<uint4*>(b + lane * 16) = make_uint4(w[0], w[1], w[2], w[3]);
  if (lane < 8) {
    const int gpr = (m.cols + m.group_size - 1) / m.group_size;
    uint16_t v[8];
#pragma unroll
    for (int rs = 0; rs < 2; ++rs)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t r = t * 16 + lane + 8 * rs;
        const int64_t g = 2 * q + h;
        uint16_t s = 0, z = 0;
        if (r < m.rows && g < gpr) {
          s = m.scales[r * gpr + g];
          z = m.zeros[r * gpr + g];
        }
        v[rs * 4 + h * 2] = s;
        v[rs * 4 + h * 2 + 1] = z;
      }
    uint4 mv;
    mv.x = v[0] | (uint32_t(v[1]) << 16);
    mv.y = v[2] | (uint32_t(v[3]) << 16);
    mv.z = v[4] | (uint32_t(v[5]) << 16);
    mv.w = v[6] | (uint32_t(v[7]) << 16);
    *reinterpret_cast<uint4*>(b + kCodeBytes + lane * 16) = mv;
  }
}

__global__ void tiles_unpack_kernel(const uint8_t* __restrict__ tiles, int64_t rows, int64_t cols,
                                    int ni, int which, int64_t GP, uint8_t* __restrict__ out) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= rows * cols) return;
  const int64_t r = idx / cols, k = idx - r * cols;
  const int64_t t = r / 16;
  const int rr = static_cast<int>(r % 16), gid = rr & 7, rs = rr >> 3;
  const int64_t g = k / 64, q = g / 2;
  const int h = static_cast<int>(g & 1), w = static_cast<int>(k % 64);
  const int kw = 2 * (w / 32) + (w % 32) / 16, tid = (w % 16) / 4, bb = w % 4;
  const int lane = gid * 4 + tid;
  const uint8_t* b = tiles + ((t * GP + q) * ni + which) * kBlk;
  const uint32_t word = reinterpret_cast<const uint32_t*>(b + lane * 16)[kw];
  out[idx] = static_cast<uint8_t>((word >> (8 * bb + 2 * (2 * h + rs))) & 3u);
}

// -------------------------------------------------------- PTX primitives ---
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Weight tiles are read exactly once per step: stream them with an L2
// evict-first policy so they do not evict the small hot state every kernel of
// the layer touches (code, parameters, gate, activations, the pair plan).
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol, bool hint) {
  if (hint)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
template <int NW>
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(NW * 32) : "memory");
}
__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ uint2 lds64(const void* p) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(smem_u32(p)));
  return v;
}
// D += A (u8, 16x32) . B (s8, 32x8), s32 accumulators
__device__ __forceinline__ void mma_u8s8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// D = A . B (zero accumulator: the first MMA of a chain reads RZ)
__device__ __forceinline__ void mma_u8s8_z(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                           uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%10,%10,%10};"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "r"(0));
}
constexpr int kMagicBits = 0x4B400000;   // 1.5 * 2^23: integer v added to its bits reads as 1.5*2^23 + v
constexpr float kMagic = 12582912.0f;

// ------------------------------------------------------------- LR tiles ---
// Stream of a 16-row tile of factor rows: element (rr, j) at index rr*r + j
// (LSB-first, the factor's own bit width).  One thread per output byte.
template <typename F>
__device__ void fill_stream(uint8_t* dst, int nbytes, int bits, int count, F code_of) {
  for (int b = threadIdx.x; b < nbytes; b += blockDim.x) {
    uint32_t v = 0;
    for (int t = 0; t < 8; ++t) {
      const int gbit = b * 8 + t;
      const int idx = gbit / bits;
      if (idx < count) v |= ((code_of(idx) >> (gbit - idx * bits)) & 1u) << t;
    }
    dst[b] = static_cast<uint8_t>(v);
  }
}

__device__ void fill_u_meta(uint8_t* dst, const lrc_qmat& u, int64_t row0) {
  const int gpu = (u.cols + u.group_size - 1) / u.group_size;
  uint16_t* d = reinterpret_cast<uint16_t*>(dst);
  for (int i = threadIdx.x; i < 16 * gpu; i += blockDim.x) {
    const int rr = i / gpu, g = i - rr * gpu;
    const int64_t R = row0 + rr;
    const bool ok = R < u.rows;
    d[2 * i] = ok ? u.scales[R * gpu + g] : 0;
    d[2 * i + 1] = ok ? u.zeros[R * gpu + g] : 0;
  }
}

__device__ void fill_u_codes(uint8_t* dst, const lrc_qmat& u, int64_t row0) {
  const int r = u.cols;
  const int64_t nb = (static_cast<int64_t>(u.rows) * r * u.bits + 7) >> 3;
  fill_stream(dst, (16 * r * 4 + 7) / 8, 4, 16 * r, [&](int idx) -> uint32_t {
    const int rr = idx / r, j = idx - rr * r;
    const int64_t R = row0 + rr;
    return R < u.rows ? read_code(u.packed, R * r + j, u.bits, nb) : 0u;
  });
}

__global__ void build_lr_up_kernel(lrc_expert e, LrLayout L, uint8_t* __restrict__ out) {
  const int64_t t = blockIdx.x;
  uint8_t* base = out + t * L.up_total;
  const int64_t row0 = t * 16;
  if (factor_present(e.u1)) {
    fill_u_codes(base + L.u1c, e.u1, row0);
    fill_u_meta(base + L.u1m, e.u1, row0);
  }
  if (factor_present(e.u3)) {
    fill_u_codes(base + L.u3c, e.u3, row0);
    fill_u_meta(base + L.u3m, e.u3, row0);
  }
  if (factor_present(e.v2)) {
    // V2^T tile, j-major: element (j, rr) = V2[j, row0 + rr] at index j*16 + rr
    // (one lane per rank index j reads 16 consecutive codes); group along ffn
    const lrc_qmat& v = e.v2;
    const int r2 = v.rows;
    const int64_t nb = (static_cast<int64_t>(v.rows) * v.cols * v.bits + 7) >> 3;
    fill_stream(base + L.v2c, (16 * r2 * 4 + 7) / 8, 4, 16 * r2, [&](int idx) -> uint32_t {
      const int j = idx / 16, rr = idx - j * 16;
      const int64_t f = row0 + rr;
      return f < v.cols ? read_code(v.packed, static_cast<int64_t>(j) * v.cols + f, v.bits, nb) : 0u;
    });
    const int gpr = (v.cols + v.group_size - 1) / v.group_size;
    const int64_t gv = row0 / v.group_size;
    uint16_t* d = reinterpret_cast<uint16_t*>(base + L.v2m);
    for (int j = threadIdx.x; j < r2; j += blockDim.x) {
      d[2 * j] = v.scales[static_cast<int64_t>(j) * gpr + gv];
      d[2 * j + 1] = v.zeros[static_cast<int64_t>(j) * gpr + gv];
    }
  }
}

__global__ void build_lr_down_kernel(lrc_expert e, LrLayout L, uint8_t* __restrict__ out, int half) {
  const int64_t t = blockIdx.x;
  uint8_t* base = out + t * L.down_total;
  if (factor_present(e.u2)) {  // tile t of the top half and of the bottom half
    fill_u_codes(base + L.u2c, e.u2, t * 16);
    fill_u_codes(base + L.u2bc, e.u2, half + t * 16);
    fill_u_meta(base + L.u2m, e.u2, t * 16);
    fill_u_meta(base + L.u2bm, e.u2, half + t * 16);
  }
}

__device__ __forceinline__ float lr_deq(const uint8_t* codes, int idx, int bits, const uint8_t* meta,
                                        int midx) {
  const uint32_t c = read_code(codes, idx, bits, 1 << 30);
  const uint32_t sz = *reinterpret_cast<const uint32_t*>(meta + midx * 4);
  return fmaf(static_cast<float>(c), h2f(sz & 0xffff), h2f(sz >> 16));
}

// --------------------------------------------------------- tiled kernel ---
// Work item = (active expert, token pass, K chunk, 16-row tile).  One CTA per
// SM: warp kNW + kNEpi (producer) streams items with cp.async.bulk into a
// ring of shared-memory stages; kNW consumer warps each own a 4-group-pair
// (512-column) span of the item, unpack the codes in registers and issue
// mma.sync m16n8k32 u8 x s8 with the activation digits from shared memory.
struct TiledParams {
  ExpertArgs a;
  int M, K;             // rows / cols of the streamed matrix (per interleaved matrix)
  int64_t GP, RT;       // group pairs per row, row tiles
  int NS, SPC, nchunk;  // spans, spans per chunk, chunks
  int stage_bytes;      // weight bytes per stage
  int lr_slot;          // low-rank tile bytes per stage (max over experts; 0 = none)
  int nstage;
  int xs_stride;        // bytes per x-digit row (stride % 128 == 32: conflict-free B-fragment loads)
  int xs_rows;          // x-digit rows held in shared memory (<= TPP)
  int prebuilt;         // UP with B <= TPP: digit rows = tokens, built before the grid-dependency wait
  int debug;            // LRC_TILED_DEBUG: bit0 skip MMA core, bit1 skip epilogue math
};

constexpr int kNRed = 2;  // partial-sum ring depth (consumers -> epilogue warps)
static_assert(kNRed == kNEpi, "partial slot k % kNRed belongs to epilogue warp k % kNEpi");

struct SmemMap {
  int xs, sums, red, ts, act, lrs, bars, total;
};

__host__ __device__ inline int align16(int x) { return (x + 15) & ~15; }

// NQ token quads per pass: TPP = 4 NQ tokens, partials in NT = ceil(TPP / 8)
// 16x8 tiles (token n -> tile n / 8, column n % 8)
template <int NQ>
struct Tpp {
  static constexpr int TPP = 4 * NQ;
  static constexpr int NT = (TPP + 7) / 8;
};

template <int NI, int NQ>
__host__ __device__ inline SmemMap smem_map(const TiledParams& p) {
  constexpr int TPP = Tpp<NQ>::TPP, NT = Tpp<NQ>::NT, NW = KCfg<NQ>::NW, SPAN = KCfg<NQ>::SPAN;
  SmemMap m;
  int o = p.nstage * (p.stage_bytes + p.lr_slot);
  m.xs = o;
  o = align16(o + p.xs_rows * p.xs_stride);
  m.sums = o;
  o = align16(o + p.SPC * SPAN * 2 * TPP * 8);
  m.red = o;
  o = align16(o + kNRed * NW * NI * NT * 128 * 4);
  m.ts = o;
  o = align16(o + kNEpi * TPP * NI * (p.a.maxr > 0 ? p.a.maxr : 1) * 4);
  m.act = o;
  o = align16(o + kNEpi * 16 * TPP * 4);
  m.lrs = o;
  o = align16(o + kNEpi * NI * 16 * TPP * 4);
  m.bars = o;
  m.total = o + (2 * p.nstage + 2 * kNRed) * 8;
  return m;
}

__device__ __forceinline__ void griddep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ float2 h2f2(uint32_t w) {
  return __half22float2(*reinterpret_cast<const __half2*>(&w));
}

// exact float of a small unsigned code without the XU pipe: 2^23 + c, minus 2^23
__device__ __forceinline__ float code_f(uint32_t c) {
  return __uint_as_float(0x4B000000u | c) - 8388608.0f;
}

// code at bit offset `bit` of a shared-memory bitstream (4-byte aligned base)
__device__ __forceinline__ uint32_t smem_code(const uint32_t* w, int bit, uint32_t mask) {
  return __funnelshift_r(w[bit >> 5], w[(bit >> 5) + 1], bit & 31) & mask;
}

// (w & m) | c in one lop3
__device__ __forceinline__ uint32_t lop3_and_or(uint32_t w, uint32_t m, uint32_t c) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(w), "r"(m), "r"(c));
  return r;
}
// nibble Q of w as the float 1 + c/16 (no int->float conversion): c*t = 16*(v*t - t)
template <int Q>
__device__ __forceinline__ float nib_f(uint32_t w) {
  const uint32_t sh = (4 * Q <= 19) ? (w << (19 - 4 * Q)) : (w >> (4 * Q - 19));
  return __uint_as_float(lop3_and_or(sh, 0x00780000u, 0x3F800000u));
}

// Per-pass state of one epilogue warp.
template <int TPP>
struct EpiPass {
  int epair[TPP], etok[TPP], ecomp_of[TPP], ecomp_n[TPP], ecomp_tok[TPP];
  float ew[TPP];
  int encomp, r[3], ub[3], ugs[3], vb;
  LrLayout L;
};

// does pass `pass` (pairs [pass TPP, pass TPP + TPP)) hold a compensated pair?
// (ActiveRec::cmask bit q: pairs [8q, 8q + 8))
__device__ __forceinline__ bool pass_has_comp(uint32_t m, int pass, int tpp) {
  bool c = false;
  for (int q = (pass * tpp) >> 3; q <= ((pass + 1) * tpp - 1) >> 3; ++q) c |= ((m >> min(q, 31)) & 1u) != 0;
  return c;
}


// x-digit rows and per-(group, row) {2^-S, sum x} for `nrows` rows over
// columns [k0, k0 + 64 ng) of the chunk.  Row n reads x row rowsrc[n] (token,
// UP) or a16 row rowsrc[n] (pair, DOWN); rowsrc == nullptr: row n is token n.
// Group gl of a row is 128 bytes: digit d (0: high, 1: low) of column
// kk = 32m + 16h + 4t + b at byte 64d + 8(4m + t) + 4h + b (the m16n8k32
// B-fragment order: lane (t, column) loads 8 bytes per m).  One 16-byte load
// per thread-task (8 columns), two tasks in flight per thread; the 8 lanes of
// a (row, group) reduce its max |x| and sum by shuffles (nthr % 32 == 0).
template <bool UP, int TPP>
__device__ __forceinline__ void build_xdigits(const ExpertArgs& A, const TiledParams& P, uint8_t* xs,
                                              float2* sums, const int* rowsrc, int nrows, int k0, int ng,
                                              int t0, int nthr) {
  const int ntask = nrows * ng * 8;
  const int c8 = t0 & 7;  // == task & 7 (base is a multiple of 8)
  // byte offset of columns 8 c8 .. 8 c8 + 3 within a digit half (+8 for the next 4)
  const int off = ((c8 >> 2) * 4 + 2 * (c8 & 1)) * 8 + ((c8 >> 1) & 1) * 4;
  for (int base = 0; base < ntask; base += 2 * nthr) {
    uint4 raw[2];
    int tn[2], tg[2];
    bool ok[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int task = base + u * nthr + t0;
      ok[u] = task < ntask;
      const int ng8 = ok[u] ? (task >> 3) : 0;
      tn[u] = ng8 / ng;
      tg[u] = ng8 - tn[u] * ng;
      raw[u] = make_uint4(0u, 0u, 0u, 0u);
      if (ok[u]) {
        const int src = rowsrc ? rowsrc[tn[u]] : tn[u];
        const uint16_t* row = UP ? A.x + static_cast<int64_t>(src) * A.hidden
                                 : A.a16 + static_cast<int64_t>(src) * A.ffn;
        const int kk = k0 + tg[u] * 64 + c8 * 8;
        if (kk + 8 <= P.K && (reinterpret_cast<uintptr_t>(row + kk) & 15) == 0) {
          raw[u] = __ldg(reinterpret_cast<const uint4*>(row + kk));
        } else {
          uint16_t h[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) h[j] = (kk + j < P.K) ? row[kk + j] : 0;
          raw[u] = make_uint4(h[0] | (uint32_t(h[1]) << 16), h[2] | (uint32_t(h[3]) << 16),
                              h[4] | (uint32_t(h[5]) << 16), h[6] | (uint32_t(h[7]) << 16));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const uint32_t w4[4] = {raw[u].x, raw[u].y, raw[u].z, raw[u].w};
      float xv[8];
      float xsum = 0.f, amax = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        xv[j] = bf2f((j & 1) ? (w4[j >> 1] >> 16) : (w4[j >> 1] & 0xffff));
        xsum += xv[j];
        amax = fmaxf(amax, fabsf(xv[j]));
      }
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        xsum += __shfl_xor_sync(0xffffffffu, xsum, o);
        amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      }
      // amax < 2^(E - 126) for exponent field E: S = 138 - E puts |x| 2^S < 2^12
      const int S = min(138 - static_cast<int>((__float_as_uint(amax) >> 23) & 255u), 126);
      const float sc = __uint_as_float(static_cast<uint32_t>(S + 127) << 23);
      if (ok[u]) {
        uint32_t d0w[2] = {0u, 0u}, d1w[2] = {0u, 0u};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int X = __float2int_rn(xv[j] * sc);  // exact scaling, |X| <= 2^12
          d0w[j >> 2] |= (static_cast<uint32_t>(X >> 7) & 0xffu) << (8 * (j & 3));
          d1w[j >> 2] |= (static_cast<uint32_t>(X) & 0x7fu) << (8 * (j & 3));
        }
        uint8_t* g = xs + tn[u] * P.xs_stride + tg[u] * 128 + off;
        *reinterpret_cast<uint32_t*>(g) = d0w[0];
        *reinterpret_cast<uint32_t*>(g + 8) = d0w[1];
        *reinterpret_cast<uint32_t*>(g + 64) = d1w[0];
        *reinterpret_cast<uint32_t*>(g + 72) = d1w[1];
        if (c8 == 0) sums[tg[u] * TPP + tn[u]] = make_float2(__uint_as_float(static_cast<uint32_t>(127 - S) << 23), xsum);
      }
    }
  }
}

struct ItemDesc {
  int ai, pass, chunk, tile, lr, gp0, gp1, pad;
};
constexpr int kMaxStages = 8;

// Warp roles: warps [0, kNW) consume (MMA over a K span of each item), warp
// kNW is the epilogue warp (cross-warp reduction, low-rank terms, SwiGLU /
// combine), warp kNW+1 produces (cp.async.bulk).  Consumers never block on the
// epilogue: partials go through a kNRed-deep mbarrier ring.
// LRC_TILED_DEBUG bit 3: %globaltimer stamps per CTA (lrc_debug_stamps)
constexpr int kTStampCtas = 256;
__device__ unsigned long long g_tiled_stamps[2][kTStampCtas][8];
// CTA 0 per item: issue, consumer pre-wait, data, MMA core done, partials posted, epi done
__device__ unsigned long long g_item_stamps[2][64][6];
#define ISTAMP(k, j)                                                      \
  do {                                                                    \
    if ((P.debug & 8) && blockIdx.x == 0 && (k) < 64) {                   \
      unsigned long long t_;                                              \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));              \
      g_item_stamps[UP][k][j] = t_;                                       \
    }                                                                     \
  } while (0)
#define TSTAMP(k)                                                          \
  do {                                                                     \
    if (P.debug & 8) {                                                     \
      unsigned long long t_;                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));               \
      if (blockIdx.x < kTStampCtas) g_tiled_stamps[UP][blockIdx.x][k] = t_; \
    }                                                                      \
  } while (0)

template <bool UP, int NQ>
__global__ void __launch_bounds__(KCfg<NQ>::THREADS, 1) tiled_kernel(const __grid_constant__ TiledParams P) {
  // two interleaved matrices per tile: w1|w3 (UP) or the two row halves of W2
  // (DOWN: two independent accumulator chains, as for the up projection)
  constexpr int NI = 2;
  constexpr int TPP = Tpp<NQ>::TPP;  // tokens per pass
  constexpr int NT = Tpp<NQ>::NT;    // 16x8 partial tiles per (warp, matrix)
  constexpr int kNW = KCfg<NQ>::NW, kSpanGP = KCfg<NQ>::SPAN;
  constexpr int kEpi0 = kNW, kProd = kNW + kNEpi;
  extern __shared__ __align__(128) uint8_t smem[];
  const SmemMap SM = smem_map<NI, NQ>(P);
  uint8_t* stages = smem;
  const int slot_bytes = P.stage_bytes + P.lr_slot;
  uint8_t* xs = smem + SM.xs;                                 // [row][group] x digits
  float2* sums = reinterpret_cast<float2*>(smem + SM.sums);  // [g_local][TPP] (2^-S, sum x)
  float* red = reinterpret_cast<float*>(smem + SM.red);      // [ring][warp][NI][NT][16][8]
  float* ts = reinterpret_cast<float*>(smem + SM.ts);        // [comp c][NI][maxr]
  float* act_s = reinterpret_cast<float*>(smem + SM.act);    // [TPP][16]
  float* lrs = reinterpret_cast<float*>(smem + SM.lrs);      // [NI][16][TPP(comp idx)]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SM.bars);
  uint64_t* empty = full + P.nstage;
  uint64_t* rfull = empty + P.nstage;
  uint64_t* rempty = rfull + kNRed;
  __shared__ ItemDesc s_desc[kMaxStages];
  __shared__ int s_prefix[LRC_MAX_EXPERTS + 1];
  __shared__ int s_range[2];
  __shared__ int s_aoff[LRC_MAX_EXPERTS], s_acnt[LRC_MAX_EXPERTS], s_ae[LRC_MAX_EXPERTS];
  __shared__ const uint8_t* s_wsrc[LRC_MAX_EXPERTS];
  __shared__ const uint8_t* s_lsrc[LRC_MAX_EXPERTS];
  __shared__ int s_lbytes[LRC_MAX_EXPERTS];
  __shared__ uint32_t s_acmask[LRC_MAX_EXPERTS];
  __shared__ int s_cpair[TPP], s_ctok[TPP];  // consumer-owned pass data
  __shared__ EpiPass<TPP> s_ep[kNEpi];       // epilogue-owned pass data (per warp)

  const ExpertArgs& A = P.a;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int maxr = A.maxr;
  // The up kernel consumes the router's plan: wait for it.  The down kernel's
  // plan is two launches old (complete before the up kernel passed its own
  // wait), so its producer may start streaming W2 while the up kernel drains;
  // its consumers / epilogue wait before touching the up kernel's outputs.
  if (threadIdx.x == 0) {
    TSTAMP(0);
    // the stage barriers do not depend on the plan: initialise them before the
    // wait (the __syncthreads after the plan loads publishes them)
    for (int s = 0; s < P.nstage; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kNW + 1);  // consumers + the item's epilogue warp (LR slot)
    }
    for (int r = 0; r < kNRed; ++r) {
      mbar_init(&rfull[r], kNW);
      mbar_init(&rempty[r], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (UP && P.prebuilt) {
    // the router releases this grid only after the previous layer finished,
    // so x is final: build the digits of all B tokens while the routing completes
    build_xdigits<UP, TPP>(A, P, xs, sums, nullptr, P.xs_rows, 0, static_cast<int>(2 * P.GP), threadIdx.x,
                           blockDim.x);
  }
  if (UP) griddep_wait();
  griddep_launch_dependents();
  if (threadIdx.x == 0) TSTAMP(1);
  // one round trip: the active count and every active-expert record (records
  // past n_active are stale and ignored) are loaded concurrently
  const int n_active = A.plan.counts[0];
  for (int ai = threadIdx.x; ai < min(A.ne, LRC_MAX_EXPERTS); ai += blockDim.x) {
    const ActiveRec R = A.plan.arec[ai];
    s_aoff[ai] = R.off;
    s_acnt[ai] = R.cnt;
    s_ae[ai] = R.e;
    s_wsrc[ai] = UP ? R.up_tiles : R.down_tiles;
    s_lbytes[ai] = UP ? R.up_lr_bytes : R.down_lr_bytes;
    s_lsrc[ai] = UP ? R.up_lr_tiles : R.down_lr_tiles;
    s_acmask[ai] = R.cmask;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int ai = 0; ai < n_active; ++ai) {
      s_prefix[ai] = acc;
      acc += ((s_acnt[ai] + TPP - 1) / TPP) * P.nchunk * static_cast<int>(P.RT);
    }
    s_prefix[n_active] = acc;
    const int64_t total = acc;
    s_range[0] = static_cast<int>(total * blockIdx.x / gridDim.x);
    s_range[1] = static_cast<int>(total * (blockIdx.x + 1) / gridDim.x);
  }
  __syncthreads();
  if (threadIdx.x == 0) TSTAMP(2);
  const int beg = s_range[0], end = s_range[1];
  if (beg >= end) return;
  const int nitems = end - beg;

  if (warp == kProd) {
    // ===================== producer: one elected lane streams work items ====
    if (lane == 0) {
      const bool hint = (P.debug & 4) == 0;  // LRC_TILED_DEBUG bit 2: plain L2 policy
      const uint64_t pol = l2_evict_first_policy();
      int ai = 0, s = 0, ph = 0;
      for (int it = beg; it < end; ++it) {
        const int k = it - beg;
        if (k >= P.nstage) mbar_wait(&empty[s], ph ^ 1);
        while (s_prefix[ai + 1] <= it) ++ai;
        int r = it - s_prefix[ai];
        const int tile = r % static_cast<int>(P.RT);
        r /= static_cast<int>(P.RT);
        const int chunk = r % P.nchunk, pass = r / P.nchunk;
        const bool c_comp = pass_has_comp(s_acmask[ai], pass, TPP);
        const int gp0 = chunk * P.SPC * kSpanGP;
        const int gp1 = static_cast<int>(min(P.GP, static_cast<int64_t>(gp0) + P.SPC * kSpanGP));
        const uint8_t* src = s_wsrc[ai] + ((static_cast<int64_t>(tile) * P.GP + gp0) * NI) * kBlk;
        const uint32_t bytes = static_cast<uint32_t>((gp1 - gp0) * NI * kBlk);
        const bool lr = P.lr_slot > 0 && c_comp && (UP || chunk == 0) && s_lbytes[ai] > 0;
        const uint32_t lr_bytes = lr ? static_cast<uint32_t>(s_lbytes[ai]) : 0u;
        s_desc[s] = ItemDesc{ai, pass, chunk, tile, lr ? 1 : 0, gp0, gp1, 0};
        uint8_t* dst = stages + static_cast<size_t>(s) * slot_bytes;
        mbar_expect_tx(&full[s], bytes + lr_bytes);  // release: orders the descriptor store
        bulk_g2s(dst, src, bytes, &full[s], pol, hint);
        if (lr) bulk_g2s(dst + P.stage_bytes, s_lsrc[ai] + static_cast<int64_t>(tile) * lr_bytes,
                         lr_bytes, &full[s], pol, hint);
        if (k == 0) TSTAMP(3);
        ISTAMP(k, 0);
        if (++s == P.nstage) {
          s = 0;
          ph ^= 1;
        }
      }
      TSTAMP(4);
    }
    return;
  }

  if (warp >= kEpi0 && warp < kEpi0 + kNEpi) {
    // ====== epilogue warps: reduce, low-rank terms, SwiGLU / combine ========
    // Item k belongs to warp kEpi0 + k % kNEpi and partial slot k % kNRed.  The
    // pass setup of an item (pair lists, t vectors) is done from the item index
    // before its partials are awaited, off the critical path.
    const int ew = warp - kEpi0;
    EpiPass<TPP>& EP = s_ep[ew];
    float* tsw = ts + ew * TPP * NI * (maxr > 0 ? maxr : 1);
    float* actw = act_s + ew * 16 * TPP;
    float* lrsw = lrs + ew * NI * 16 * TPP;
    if (!UP) griddep_wait();  // t2 comes from the up kernel
    int cur_ai = -1, cur_pass = -1, pass_tok = 0, cur_e = -1, ai = 0;
    int s = ew % P.nstage;
    for (int k = ew; k < nitems; k += kNEpi) {
      const int rs = k % kNRed;
      const int it = beg + k;
      while (s_prefix[ai + 1] <= it) ++ai;
      const int pass = ((it - s_prefix[ai]) / static_cast<int>(P.RT)) / P.nchunk;
      if (ai != cur_ai || pass != cur_pass) {
        cur_ai = ai;
        cur_pass = pass;
        cur_e = s_ae[ai];
        pass_tok = min(TPP, s_acnt[ai] - cur_pass * TPP);
        const int off = s_aoff[ai];
        if (lane < TPP) {
          int p = -1, tok = 0, cmp = 0;
          float w = 0.0f;
          if (lane < pass_tok) {
            p = A.plan.pair_list[off + cur_pass * TPP + lane];
            tok = A.plan.pair_token[p];
            w = A.plan.pair_w[p];
            cmp = A.plan.pair_comp[p] >= 0;
          }
          EP.epair[lane] = p;
          EP.etok[lane] = tok;
          EP.ew[lane] = w;
          EP.ecomp_of[lane] = cmp;
        } else if (lane == 31) {
          const lrc_expert& E = A.experts[cur_e];
          EP.L = lr_layout(E);
          const lrc_qmat* us[3] = {&E.u1, &E.u3, &E.u2};
          for (int i = 0; i < 3; ++i) {
            EP.r[i] = factor_present(*us[i]) ? us[i]->cols : 0;
            EP.ub[i] = us[i]->bits;
            EP.ugs[i] = us[i]->group_size;
          }
          EP.vb = E.v2.bits;
        }
        __syncwarp();
        if (lane == 0) {
          int nc = 0;
          for (int n = 0; n < TPP; ++n) {
            if (EP.ecomp_of[n]) {
              EP.ecomp_of[n] = nc;
              EP.ecomp_n[nc] = n;
              EP.ecomp_tok[nc] = EP.etok[n];
              ++nc;
            } else {
              EP.ecomp_of[n] = -1;
            }
          }
          EP.encomp = nc;
        }
        __syncwarp();
        if (maxr > 0) {  // low-rank input vectors (t1/t3 up, t2 down) of the comp tokens
          const int ntask = EP.encomp * NI * maxr;
          for (int task = lane; task < ntask; task += 32) {
            const int j = task % maxr, ci = task / maxr;
            const int i = ci % NI, c = ci / NI;
            const int proj = UP ? i : 2;
            tsw[task] = __ldcg(A.t + ((static_cast<int64_t>(EP.ecomp_tok[c]) * A.ne + cur_e) * 3 + proj) * maxr + j);
          }
        }
        __syncwarp();
      }
      mbar_wait(&rfull[rs], (k / kNRed) & 1);
      const ItemDesc dsc = s_desc[s];
      const uint8_t* st = stages + static_cast<size_t>(s) * slot_bytes;
      const int nw = min((dsc.gp1 - dsc.gp0 + kSpanGP - 1) / kSpanGP, kNW);
      const float* rb = red + static_cast<size_t>(rs) * kNW * NI * NT * 128;
      const int rr = lane & 15, il = lane >> 4;  // lane -> (matrix, row)
      const bool lane_on = il < NI;
      // ---- E1: low-rank up-projection U.t for this tile's rows (ref/lowrank.py:165)
      if (dsc.lr && lane_on && !(P.debug & 2)) {
        const int pi = UP ? il : 2;
        const int r = EP.r[pi];
        const uint8_t* lr = st + P.stage_bytes;
        const uint32_t* cw = reinterpret_cast<const uint32_t*>(
            lr + (UP ? (il ? EP.L.u3c : EP.L.u1c) : (il ? EP.L.u2bc : EP.L.u2c)));
        const uint8_t* meta = lr + (UP ? (il ? EP.L.u3m : EP.L.u1m) : (il ? EP.L.u2bm : EP.L.u2m));
        const int gsu = EP.ugs[pi];  // LR tile codes are 4-bit nibbles
        const int gpu = (r + gsu - 1) / gsu;
        const bool fast = (r % 8) == 0 && (gsu % 8) == 0;
        for (int c = 0; c < EP.encomp; ++c) {
          const float* tv = tsw + (c * NI + il) * maxr;
          float v = 0.0f;
          for (int g = 0; g < gpu; ++g) {
            const float2 f = h2f2(*reinterpret_cast<const uint32_t*>(meta + (rr * gpu + g) * 4));
            float cx = 0.0f, sx = 0.0f;
            const int j0 = g * gsu, j1 = min(r, (g + 1) * gsu);
            if (fast) {
              float vx = 0.0f;
              for (int j = j0; j < j1; j += 8) {
                const uint32_t w = cw[(rr * r + j) >> 3];
                const float4 t0 = *reinterpret_cast<const float4*>(tv + j);
                const float4 t1 = *reinterpret_cast<const float4*>(tv + j + 4);
                vx = fmaf(nib_f<0>(w), t0.x, vx);
                vx = fmaf(nib_f<1>(w), t0.y, vx);
                vx = fmaf(nib_f<2>(w), t0.z, vx);
                vx = fmaf(nib_f<3>(w), t0.w, vx);
                vx = fmaf(nib_f<4>(w), t1.x, vx);
                vx = fmaf(nib_f<5>(w), t1.y, vx);
                vx = fmaf(nib_f<6>(w), t1.z, vx);
                vx = fmaf(nib_f<7>(w), t1.w, vx);
                sx += (t0.x + t0.y) + (t0.z + t0.w) + (t1.x + t1.y) + (t1.z + t1.w);
              }
              cx = 16.0f * (vx - sx);
            } else {
              for (int j = j0; j < j1; ++j) {
                cx = fmaf(code_f(smem_code(cw, (rr * r + j) * 4, 0xFu)), tv[j], cx);
                sx += tv[j];
              }
            }
            v = fmaf(f.x, cx, fmaf(f.y, sx, v));
          }
          lrsw[(il * 16 + rr) * TPP + c] = v;
        }
      }
      __syncwarp();
      // ---- E2: reduce the consumer partials per (matrix, row, token) and finish
      for (int n = 0; n < ((P.debug & 2) ? 0 : pass_tok); ++n) {
        const int nt = n >> 3, col = n & 7;
        float v = 0.0f;
        if (lane_on) {
#pragma unroll
          for (int w = 0; w < kNW; ++w)
            if (w < nw) v += rb[((w * NI + il) * NT + nt) * 128 + rr * 8 + col];
          const int c = EP.ecomp_of[n];
          if (dsc.lr && c >= 0) v += lrsw[(il * 16 + rr) * TPP + c];
        }
        const int row = dsc.tile * 16 + rr;
        if (UP) {
          const float h3 = __shfl_down_sync(0xffffffffu, v, 16);
          if (lane < 16) {
            const float act = (row < P.M) ? silu_f(v) * h3 : 0.0f;
            actw[n * 16 + rr] = act;
            if (row < P.M) A.a16[static_cast<int64_t>(EP.epair[n]) * A.ffn + row] = f2bf(act);
          }
        } else if (lane_on && row < P.M) {  // row half il of W2
          atomicAdd(&A.y[static_cast<int64_t>(EP.etok[n]) * A.hidden + il * P.M + row], EP.ew[n] * v);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&rempty[rs]);  // partial slot free for the consumers
      // ---- E3 (up): partial t2 = V2[:, tile rows] . act for the comp tokens
      if (UP && dsc.lr && EP.r[2] > 0 && !(P.debug & 2)) {
        const int r2 = EP.r[2];
        const uint8_t* lr = st + P.stage_bytes;
        const uint32_t* vw = reinterpret_cast<const uint32_t*>(lr + EP.L.v2c);
        for (int j = lane; j < r2; j += 32) {
          const float2 f = h2f2(*reinterpret_cast<const uint32_t*>(lr + EP.L.v2m + j * 4));
          // V2^T tile is j-major nibbles: codes (j, rl), rl = 0..15, in words 2j, 2j+1
          const uint32_t w0 = vw[2 * j], w1 = vw[2 * j + 1];
          for (int c = 0; c < EP.encomp; ++c) {
            const float4* an = reinterpret_cast<const float4*>(actw + EP.ecomp_n[c] * 16);
            const float4 a0 = an[0], a1 = an[1], a2 = an[2], a3 = an[3];
            float vx = nib_f<0>(w0) * a0.x;
            vx = fmaf(nib_f<1>(w0), a0.y, vx);
            vx = fmaf(nib_f<2>(w0), a0.z, vx);
            vx = fmaf(nib_f<3>(w0), a0.w, vx);
            vx = fmaf(nib_f<4>(w0), a1.x, vx);
            vx = fmaf(nib_f<5>(w0), a1.y, vx);
            vx = fmaf(nib_f<6>(w0), a1.z, vx);
            vx = fmaf(nib_f<7>(w0), a1.w, vx);
            vx = fmaf(nib_f<0>(w1), a2.x, vx);
            vx = fmaf(nib_f<1>(w1), a2.y, vx);
            vx = fmaf(nib_f<2>(w1), a2.z, vx);
            vx = fmaf(nib_f<3>(w1), a2.w, vx);
            vx = fmaf(nib_f<4>(w1), a3.x, vx);
            vx = fmaf(nib_f<5>(w1), a3.y, vx);
            vx = fmaf(nib_f<6>(w1), a3.z, vx);
            vx = fmaf(nib_f<7>(w1), a3.w, vx);
            const float sx = ((a0.x + a0.y) + (a0.z + a0.w)) + ((a1.x + a1.y) + (a1.z + a1.w)) +
                             ((a2.x + a2.y) + (a2.z + a2.w)) + ((a3.x + a3.y) + (a3.z + a3.w));
            const float cx = 16.0f * (vx - sx);
            atomicAdd(&A.t[((static_cast<int64_t>(EP.ecomp_tok[c]) * A.ne + cur_e) * 3 + 2) * maxr + j],
                      fmaf(f.x, cx, f.y * sx));
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // LR slot read: stage may be refilled
      if (lane == 0) ISTAMP(k, 5);
      s += kNEpi;
      while (s >= P.nstage) s -= P.nstage;
    }
    if (lane == 0) TSTAMP(7);
    return;
  }

  // ============================ consumers ====================================
  const int gid = lane >> 2, tid = lane & 3;
  const int ctid = threadIdx.x;  // consumer thread id, 0 .. kNW*32-1
  if (!UP) griddep_wait();  // a16 comes from the up kernel
  int cur_ai = -1, cur_pass = -1, cur_chunk = -1, pass_tok = 0;
  int s = 0, ph = 0;
  for (int k = 0; k < nitems; ++k) {
    if (ctid == 0) ISTAMP(k, 1);
    mbar_wait(&full[s], ph);  // acquire: descriptor + bytes visible
    if (k == 0 && ctid == 0) TSTAMP(5);
    if (ctid == 0) ISTAMP(k, 2);
    const ItemDesc dsc = s_desc[s];
    const int gp0 = dsc.gp0, gp1 = dsc.gp1;
    if (dsc.ai != cur_ai || dsc.pass != cur_pass || dsc.chunk != cur_chunk) {
      // ---- (re)build the activation digits (consumers only)
      consumer_sync<kNW>();  // every consumer is past the previous item's MMA
      const bool new_pass = (dsc.ai != cur_ai || dsc.pass != cur_pass);
      cur_ai = dsc.ai;
      cur_pass = dsc.pass;
      cur_chunk = dsc.chunk;
      pass_tok = min(TPP, s_acnt[dsc.ai] - cur_pass * TPP);
      if (new_pass) {
        if (ctid < TPP) {
          int p = -1, tok = 0;
          if (ctid < pass_tok) {
            p = A.plan.pair_list[s_aoff[dsc.ai] + cur_pass * TPP + ctid];
            tok = A.plan.pair_token[p];
          }
          s_cpair[ctid] = p;
          s_ctok[ctid] = tok;
        }
        consumer_sync<kNW>();
      }
      if (!P.prebuilt) {
        // only real token rows are built (empty MMA columns read row 0: their
        // accumulators are never read -- MMA columns are independent)
        build_xdigits<UP, TPP>(A, P, xs, sums, UP ? s_ctok : s_cpair, pass_tok, gp0 * 128, (gp1 - gp0) * 2,
                               ctid, kNW * 32);
      }
      consumer_sync<kNW>();
    }
    const uint8_t* st = stages + static_cast<size_t>(s) * slot_bytes;

    // ---------------------------------------------------------- MMA core ----
    // acc[i][nq][r]: matrix i, token nq*4 + tid, row gid (r = 0) / gid + 8 (r = 1)
    float acc[NI][NQ][2];
#pragma unroll
    for (int i = 0; i < NI; ++i)
#pragma unroll
      for (int nq = 0; nq < NQ; ++nq) acc[i][nq][0] = acc[i][nq][1] = 0.0f;

    const int ngp = gp1 - gp0;
    const int nspan = (ngp + kSpanGP - 1) / kSpanGP;
    // B-fragment column gid of quad nq = digit gid & 1 of token nq*4 + gid/2
    // (empty columns read row 0: MMA columns are independent and the lanes
    // holding them are never read); the digit / sums row of a token is its pass
    // position, or (prebuilt) the token itself
    const uint8_t* brow[NQ];
    int srow[NQ];
#pragma unroll
    for (int nq = 0; nq < NQ; ++nq) {
      const int nb = nq * 4 + (gid >> 1), nc = nq * 4 + tid;
      brow[nq] = xs + (nb < pass_tok ? (P.prebuilt ? s_ctok[nb] : nb) : 0) * P.xs_stride + (gid & 1) * 64 + tid * 8;
      srow[nq] = nc < pass_tok ? (P.prebuilt ? s_ctok[nc] : nc) : 0;
    }
    constexpr uint32_t kM = 0x03030303u, kM4 = kM << 2;
    for (int sp = warp; sp < ((P.debug & 1) ? 0 : nspan); sp += kNW) {
      const int q0 = sp * kSpanGP, q1 = min(ngp, q0 + kSpanGP);
#pragma unroll kQUnroll
      for (int q = q0; q < q1; ++q) {
        const uint8_t* blk = st + q * NI * kBlk;
        uint4 cw[NI], mw[NI];
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          cw[i] = *reinterpret_cast<const uint4*>(blk + i * kBlk + lane * 16);
          mw[i] = *reinterpret_cast<const uint4*>(blk + i * kBlk + kCodeBytes + gid * 16);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gl = q * 2 + h;  // group index within the chunk
          uint2 b0[NQ], b1[NQ];
          float2 sx[NQ];
          float nm[NQ], inv4[NQ], nm4[NQ];
#pragma unroll
          for (int nq = 0; nq < NQ; ++nq) {
            b0[nq] = lds64(brow[nq] + gl * 128);       // m = 0
            b1[nq] = lds64(brow[nq] + gl * 128 + 32);  // m = 1
            sx[nq] = sums[gl * TPP + srow[nq]];          // (2^-S, sum x) of token nq*4 + tid
            nm[nq] = -kMagic * sx[nq].x;
            inv4[nq] = 0.25f * sx[nq].x;  // B-row codes carry a factor 4
            nm4[nq] = 0.25f * nm[nq];
          }
#pragma unroll
          for (int i = 0; i < NI; ++i) {
            // group h's planes: 2h (row gid) and 2h + 1 (row gid+8, x4)
            const uint32_t w0 = h ? cw[i].x >> 4 : cw[i].x, w1 = h ? cw[i].y >> 4 : cw[i].y;
            const uint32_t w2 = h ? cw[i].z >> 4 : cw[i].z, w3 = h ? cw[i].w >> 4 : cw[i].w;
            const float2 mA = h2f2(h ? mw[i].y : mw[i].x);  // {s, z} row gid
            const float2 mB = h2f2(h ? mw[i].w : mw[i].z);  // {s, z} row gid+8
#pragma unroll
            for (int nq = 0; nq < NQ; ++nq) {
              int d[4];
              mma_u8s8_z(d, w0 & kM, w0 & kM4, w1 & kM, w1 & kM4, b0[nq].x, b0[nq].y);
              mma_u8s8(d, w2 & kM, w2 & kM4, w3 & kM, w3 & kM4, b1[nq].x, b1[nq].y);
              // 2^-S sum c X, exact: (1.5*2^23 + v) 2^-S - 1.5*2^23 2^-S
              const float ta = fmaf(__int_as_float(d[0] * 128 + (d[1] + kMagicBits)), sx[nq].x, nm[nq]);
              const float tb = fmaf(__int_as_float(d[2] * 128 + (d[3] + kMagicBits)), inv4[nq], nm4[nq]);
              acc[i][nq][0] = fmaf(mA.x, ta, fmaf(mA.y, sx[nq].y, acc[i][nq][0]));
              acc[i][nq][1] = fmaf(mB.x, tb, fmaf(mB.y, sx[nq].y, acc[i][nq][1]));
            }
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // weights consumed
    if (ctid == 0) ISTAMP(k, 3);
    if (++s == P.nstage) {
      s = 0;
      ph ^= 1;
    }
    // ---- partials to the epilogue ring (slot reused every kNRed items)
    const int rs = k % kNRed;
    mbar_wait(&rempty[rs], ((k / kNRed) & 1) ^ 1);
    if (warp < nspan) {
      float* rb = red + (static_cast<size_t>(rs) * kNW + warp) * NI * NT * 128;
#pragma unroll
      for (int i = 0; i < NI; ++i)
#pragma unroll
        for (int nq = 0; nq < NQ; ++nq) {
          const int n = nq * 4 + tid;  // token column of this lane
          float* q = rb + (i * NT + (n >> 3)) * 128 + (n & 7);
          q[gid * 8] = acc[i][nq][0];
          q[(gid + 8) * 8] = acc[i][nq][1];
        }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&rfull[rs]);
    if (ctid == 0) ISTAMP(k, 4);
  }
  if (ctid == 0) TSTAMP(6);
}

void tiled_stamps_copy(uint64_t* host, int n) {
  const int n0 = 2 * kTStampCtas * 8;
  if (n > n0) {
    cudaMemcpyFromSymbol(host + n0, g_item_stamps, sizeof(uint64_t) * (n - n0));
    void* dev = nullptr;
    if (cudaGetSymbolAddress(&dev, g_item_stamps) == cudaSuccess) cudaMemset(dev, 0, sizeof(g_item_stamps));
    n = n0;
  }
  if (cudaMemcpyFromSymbol(host, g_tiled_stamps, sizeof(uint64_t) * n) == cudaSuccess) {
    void* dev = nullptr;
    if (cudaGetSymbolAddress(&dev, g_tiled_stamps) == cudaSuccess) cudaMemset(dev, 0, sizeof(g_tiled_stamps));
  }
}

template <bool UP, int NQ>
static lrc_status launch_one(const TiledParams& P, int num_sms, cudaStream_t st, bool pdl) {
  constexpr int NI = 2;
  const SmemMap m = smem_map<NI, NQ>(P);
  auto fn = tiled_kernel<UP, NQ>;
  static int configured[2][5] = {{0, 0, 0, 0, 0}, {0, 0, 0, 0, 0}};
  if (configured[UP][NQ] < m.total) {
    cudaFuncAttributes fa{};
    LRC_CUDA_TRY(cudaFuncGetAttributes(&fa, fn));
    int dev = 0, optin = 0;
    LRC_CUDA_TRY(cudaGetDevice(&dev));
    LRC_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (m.total + static_cast<int>(fa.sharedSizeBytes) > optin)
      return fail(LRC_ERR_UNSUPPORTED, "tiled kernel: shared memory budget");
    LRC_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      optin - static_cast<int>(fa.sharedSizeBytes)));
    configured[UP][NQ] = optin - static_cast<int>(fa.sharedSizeBytes);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(num_sms);
  cfg.blockDim = dim3(KCfg<NQ>::THREADS);
  cfg.dynamicSmemBytes = m.total;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  LRC_CUDA_TRY(cudaLaunchKernelEx(&cfg, fn, P));
  return LRC_OK;
}

template <bool UP>
static lrc_status launch_tiled(const ExpertArgs& a, int num_sms, int max_tok, int lr_max,
                               cudaStream_t st, bool pdl) {
  constexpr int NI = 2;  // w1|w3, or the two row halves of W2
  TiledParams P{};
  P.a = a;
  P.M = UP ? a.ffn : a.hidden / 2;  // rows per interleaved matrix
  P.K = UP ? a.hidden : a.ffn;
  P.GP = (P.K + 127) / 128;
  P.RT = (P.M + 15) / 16;
  P.lr_slot = lr_max;
  P.debug = getenv("LRC_TILED_DEBUG") ? atoi(getenv("LRC_TILED_DEBUG")) : 0;
  const int budget = 227 * 1024 - 12 * 1024;  // static shared (~10 KB) + slack
  auto fits = [&](int nq) {
    const int nw = nq == 1 ? KCfg<1>::NW : KCfg<2>::NW, span = nq == 1 ? KCfg<1>::SPAN : KCfg<2>::SPAN;
    P.NS = static_cast<int>((P.GP + span - 1) / span);
    if (UP) {  // the SwiGLU needs complete h1/h3: one chunk covers all of K
      P.nchunk = 1;
      P.SPC = P.NS;
    } else {  // split K into <= nw-span chunks; partial outputs combine with atomics
      P.nchunk = (P.NS + nw - 1) / nw;
      P.SPC = (P.NS + P.nchunk - 1) / P.nchunk;
    }
    P.xs_stride = P.SPC * span * 2 * 128 + 32;
    P.stage_bytes = P.SPC * span * NI * kBlk;
    P.xs_rows = min(4 * nq, max(max_tok, 1));  // digit rows actually needed
    const int tot = nq == 1 ? smem_map<NI, 1>(P).total : nq == 2 ? smem_map<NI, 2>(P).total
                                                                  : smem_map<NI, 4>(P).total;
    return tot <= budget;
  };
  // token quads per pass: the fewest that hold the largest expert batch (<= 4)
  int nq = max_tok <= 4 ? 1 : (max_tok <= 8 ? 2 : 4);
  for (;; nq >>= 1) {
    for (P.nstage = 4; P.nstage >= 2; --P.nstage)
      if (fits(nq)) break;
    if (P.nstage >= 2 || nq == 1) break;
  }
  if (P.nstage < 2) return fail(LRC_ERR_UNSUPPORTED, "tiled kernel: K too large for smem");
  fits(nq);  // final digit-row count for the chosen pass width
  P.prebuilt = (UP && max_tok >= 1 && max_tok <= 4 * nq) ? 1 : 0;
  return nq == 1 ? launch_one<UP, 1>(P, num_sms, st, pdl)
                 : nq == 2 ? launch_one<UP, 2>(P, num_sms, st, pdl) : launch_one<UP, 4>(P, num_sms, st, pdl);
}

lrc_status launch_up_tiled(const ExpertArgs& a, int num_sms, int max_tok, int lr_max,
                           cudaStream_t st, bool pdl) {
  return launch_tiled<true>(a, num_sms, max_tok, lr_max, st, pdl);
}
lrc_status launch_down_tiled(const ExpertArgs& a, int num_sms, int max_tok, int lr_max,
                             cudaStream_t st, bool pdl) {
  return launch_tiled<false>(a, num_sms, max_tok, lr_max, st, pdl);
}

}  // namespace lrc

using namespace lrc;

extern "C" int64_t lrc_tiles_bytes(int64_t rows, int64_t cols, int interleave) {
  return tiles_bytes(rows, cols, interleave);
}

extern "C" lrc_status lrc_build_tiles(const lrc_qmat* mats, int interleave, uint8_t* tiles,
                                      void* stream) {
  if (!mats || !tiles || interleave < 1 || interleave > 2)
    return fail(LRC_ERR_INVALID, "build_tiles: bad arguments");
  for (int i = 0; i < interleave; ++i) {
    if (mats[i].bits != 2 || mats[i].group_size != 64 || mats[i].packed == nullptr)
      return fail(LRC_ERR_UNSUPPORTED, "build_tiles: tiled layout needs 2-bit codes, group 64");
    if (mats[i].rows != mats[0].rows || mats[i].cols != mats[0].cols)
      return fail(LRC_ERR_INVALID, "build_tiles: interleaved matrices differ in shape");
  }
  const int64_t RT = (mats[0].rows + 15) / 16, GP = (mats[0].cols + 127) / 128;
  const int64_t threads = RT * GP * interleave * 32;
  build_tiles_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, as_stream(stream)>>>(
      mats[0], mats[interleave - 1], interleave, RT, GP, tiles);
  LRC_CHECK_LAUNCH();
  return LRC_OK;
}

static lrc_status lr_tiles_check(const lrc_expert* e, int hidden, int ffn) {
  const lrc_qmat* fs[6] = {&e->u1, &e->v1, &e->u3, &e->v3, &e->u2, &e->v2};
  for (auto f : fs) {
    if (!factor_present(*f)) continue;
    if (f->dense != nullptr)
      return fail(LRC_ERR_UNSUPPORTED, "lr tiles: raw (unquantized) factors use the generic path");
    if (f->bits < 1 || f->bits > 4)
      return fail(LRC_ERR_UNSUPPORTED, "lr tiles: factor codes wider than 4 bits use the generic path");
  }
  if (factor_present(e->v2) && (e->v2.group_size % 16) != 0)
    return fail(LRC_ERR_UNSUPPORTED, "lr tiles: V2 group size must be a multiple of 16");
  (void)hidden;
  (void)ffn;
  return LRC_OK;
}

extern "C" lrc_status lrc_lr_tiles_bytes(const lrc_expert* e, int hidden, int ffn,
                                         int64_t* up_bytes, int64_t* down_bytes) {
  if (!e || !up_bytes || !down_bytes) return fail(LRC_ERR_INVALID, "lr_tiles_bytes: null");
  lrc_status s = lr_tiles_check(e, hidden, ffn);
  if (s != LRC_OK) return s;
  const LrLayout L = lr_layout(*e);
  *up_bytes = static_cast<int64_t>(L.up_total) * ((ffn + 15) / 16);
  *down_bytes = static_cast<int64_t>(L.down_total) * ((hidden / 2 + 15) / 16);
  return LRC_OK;
}

extern "C" lrc_status lrc_build_lr_tiles(const lrc_expert* e, int hidden, int ffn, uint8_t* up_lr,
                                         uint8_t* down_lr, void* stream) {
  if (!e) return fail(LRC_ERR_INVALID, "build_lr_tiles: null");
  lrc_status s = lr_tiles_check(e, hidden, ffn);
  if (s != LRC_OK) return s;
  const LrLayout L = lr_layout(*e);
  cudaStream_t st = as_stream(stream);
  if (L.up_total > 0 && up_lr) {
    build_lr_up_kernel<<<(ffn + 15) / 16, 256, 0, st>>>(*e, L, up_lr);
    LRC_CHECK_LAUNCH();
  }
  if (L.down_total > 0 && down_lr) {
    build_lr_down_kernel<<<(hidden / 2 + 15) / 16, 256, 0, st>>>(*e, L, down_lr, hidden / 2);
    LRC_CHECK_LAUNCH();
  }
  return LRC_OK;
}

extern "C" lrc_status lrc_tiles_unpack(const uint8_t* tiles, int64_t rows, int64_t cols,
                                       int interleave, int which, uint8_t* codes, void* stream) {
  if (!tiles || !codes || rows <= 0 || cols <= 0 || which < 0 || which >= interleave)
    return fail(LRC_ERR_INVALID, "tiles_unpack: bad arguments");
  const int64_t GP = (cols + 127) / 128;
  tiles_unpack_kernel<<<static_cast<unsigned>((rows * cols + 255) / 256), 256, 0,
                        as_stream(stream)>>>(tiles, rows, cols, interleave, which, GP, codes);
  LRC_CHECK_LAUNCH();
  return LRC_OK;
}
