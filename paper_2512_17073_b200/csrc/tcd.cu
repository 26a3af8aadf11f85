// Tensor-core decode engine ("tcd") for small batches: one persistent kernel
// per MoE layer step (ref/moe.py:217-259 forward, mode "compensated", for
// B <= 8 tokens), one CTA per SM.
//
// Per CTA (15 warps):
//   all warps   x digit images (below) for a share of the (token, group)s,
//               cooperatively over the grid; routing: fp32 gate GEMV from
//               shared memory (the gate is prefetched before the
//               grid-dependency wait), softmax, stable top-k/top-n with a
//               proven fp32 error bound -- tokens whose ranking margin is
//               inside it are re-routed in fp64, so the selection equals the
//               fp64 reference ranking (ref/moe.py:165-193); every CTA
//               derives the same plan;
//   warp 9      producer: per stage (<= 4 consecutive 64-code groups of one
//               128-row tile) one cp.async.bulk of the codes + fp16 metadata
//               and the B operand: digit images of x (phase U) or of the
//               activations (phase D, after the grid barrier);
//   warps 0-7   decode: codes -> u8 bytes in registers ((w >> 2j) & 0x03..
//               for 2-bit; byte-aligned repacked 3-bit) -> tcgen05.st into a
//               TMEM A block per stage; epilogue one stage later: tcgen05.ld
//               of the int32 group dot products, per-group fp16 scale/zero
//               (ref/quant.py:216-224) in fp32;
//   warp 8      MMA: tcgen05.mma.kind::i8, A from TMEM (128 rows x 32 codes),
//               B = digits (8 rows per token), 2 MMAs per (group, matrix) unit;
//   warps 11-14 low-rank V.x jobs, up-tile finalisation (U1.t1, U3.t3,
//               SwiGLU, t2 = V2.a partials; ref/lowrank.py:153-165 factored;
//               the activations' digit images), the grid barrier, U2.t2.
// Work is split stream-K over (expert, tile, group) for phase U (w1|w3) and
// phase D (w2); the producer keeps streaming W2 codes across the grid barrier.
// B operand: every value of a 64-value group is scaled by 2^S (S from the
// group's max |value|) and rounded to a 21-bit integer, stored as three
// signed 7-bit digits in rows 0..2 of a 512-byte core-matrix image (K order =
// the decoded codes' order); group dot products are then exact int32, and the
// fp16 scale/zero, 2^-S and fp32 accumulation follow -- the layer output is
// within the 1e-2 contract.
#include <cuda_bf16.h>

#include "tcd.cuh"
#include "umma.cuh"

namespace lrc {
namespace tcd {

constexpr int kDec = 8;  // decode warps: 2 per TMEM lane quarter, each <= 4 units of a stage
constexpr int kNEpi = 4;     // epilogue warps: one per lane quarter, every unit of a stage
constexpr int kEpi0 = kDec;
constexpr int kMmaWarp = kDec + kNEpi, kProdWarp = kMmaWarp + 1, kAux0 = kMmaWarp + 2;
constexpr int kWarps = kAux0 + 4, kThreads = kWarps * 32;
#ifndef TCD_ONE_NAS
#define TCD_ONE_NAS 3
#endif
// B == 1 (N = 8, D block 64 columns): TMEM = kOneNAS x 128 A columns + kOneNDS x 64 D columns
constexpr int kOneNAS = TCD_ONE_NAS, kOneNDS = (512 - 128 * kOneNAS) / 64 > 4 ? 4 : (512 - 128 * kOneNAS) / 64;
constexpr int kNAS = 3;   // A ring (max): stages x 8 units x 16 TMEM columns
constexpr int kGPS = 4;   // groups per stage (2 when an expert has > 4 tokens)

constexpr int kMaxNST = 8;
constexpr int kMaxNDS = 4;
constexpr int kMaxE = LRC_MAX_EXPERTS;
constexpr int kMaxStages = 512;
constexpr int kTresBytes = 2 * 2 * kMaxTok * 128 * 4;  // 2 slots x {w1, w3}
constexpr int kEaccBytes = 2 * kMaxTok * 128 * 4;     // epilogue segment sums (B > 1)

__device__ uint64_t g_stamps[148 * 16];
__device__ uint64_t g_trace[4][256];  // CTA 0: producer stage codes, producer stage B, MMA stage, decode-w0 stage
__device__ __forceinline__ void trace(const Args& A, int w, int i) {
  if (A.stamp && blockIdx.x == 0 && i < 256) g_trace[w][i] = clock64();
}
__device__ uint64_t g_trace2[4][256];  // CTA 0: -, epilogue-w0 stage, -, -
__device__ __forceinline__ void trace2(const Args& A, int w, int i) {
  if (A.stamp && blockIdx.x == 0 && i < 256) g_trace2[w][i] = clock64();
}

// ---------------------------------------------------------------- plan ----
struct Plan {
  int n_act, NT, N, np, n_comp, epoch, par, fallback, gps;
  long long lo[2], hi[2];
  int act_e[kMaxAct], act_n[kMaxAct], act_p0[kMaxAct];
  const uint8_t* act_pack[kMaxAct][2];  // tcd packs (up, down) of the active experts
  int pair_tok[kMaxP], pair_comp[kMaxP], comp_pair[kMaxP];
  float pair_w[kMaxP];
  float xmax[kMaxTok];
};

// -------------------------------------------------------- ptx helpers ----
using umma::smem_u32;
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) { umma::bar_init(b, n); }
__device__ __forceinline__ void arrive(uint64_t* b) { umma::bar_arrive(b); }
__device__ __forceinline__ void arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
// spin wait (no suspend hint: these are latency-critical hand-offs); traps
// after ~4 s instead of hanging the GPU

__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{.reg .pred P; mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2; selp.b32 %0, 1, 0, P;}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Inline wait (no call: a call from a hot loop spills to the stack, and local
// memory misses L1 here -- ~200 KB of shared memory leaves L1 almost nothing).
// try_wait with a suspend-time hint parks the warp until the phase completes,
// so waiting warps do not take issue slots from the working ones.
__device__ __forceinline__ bool try_wait_sleep(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{.reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2, %3; selp.b32 %0, 1, 0, P;}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity), "r"(0x100000u)
      : "memory");
  return ok != 0;
}
#ifndef TCD_WAIT
#define TCD_WAIT 1
#endif
__device__ __forceinline__ bool try_wait_hw(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{.reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2; selp.b32 %0, 1, 0, P;}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t parity) {
  if (try_wait(b, parity)) return;
  uint64_t t0 = 0;
#if TCD_WAIT == 2
  uint32_t ns = 32;
#endif
  for (uint32_t spin = 1;; ++spin) {
#if TCD_WAIT == 1
    if (try_wait_hw(b, parity)) return;
#elif TCD_WAIT == 3
    if (try_wait_sleep(b, parity)) return;
#else
    if (try_wait(b, parity)) return;
#endif
#if TCD_WAIT == 0
#ifndef TCD_SPIN
    __nanosleep(20);
#endif
#elif TCD_WAIT == 2
    __nanosleep(ns);
    ns = min(ns * 2, 512u);
#endif
    if ((spin & 0xFF) == 0) {
      const uint64_t t = umma::globaltimer();
      if (t0 == 0) t0 = t;
      else if (t - t0 > 4000000000ull) __trap();
    }
  }
}
// debug (-DTCD_WSTAT and A.stamp): waits with the cycles spent accumulated per
// warp (CTA 0 -> g_wstat; tools/tcd_stamps.py prints them)
__device__ unsigned long long g_wstat[24][8];
#ifdef TCD_WSTAT
struct WStat {
  long long t0, c[8];
};
__device__ __forceinline__ void wstat_init(const Args& A, WStat& w) {
  if (A.stamp) {
    w.t0 = clock64();
#pragma unroll
    for (int i = 0; i < 8; ++i) w.c[i] = 0;
  }
}
template <int K>
__device__ __forceinline__ void wait_s(const Args& A, WStat& w, uint64_t* b, uint32_t parity) {
  if (!A.stamp) {
    wait(b, parity);
    return;
  }
  const long long t = clock64();
  wait(b, parity);
  w.c[K] += clock64() - t;
}
template <int K>
__device__ __forceinline__ void wstat_add(const Args& A, WStat& w, long long v) {
  if (A.stamp) w.c[K] += v;
}
__device__ __forceinline__ long long wstat_clock(const Args& A) { return A.stamp ? clock64() : 0; }
__device__ __forceinline__ void wstat_done(const Args& A, WStat& w) {
  if (A.stamp && blockIdx.x == 0 && (threadIdx.x & 31) == 0) {
    w.c[7] = clock64() - w.t0;
#pragma unroll
    for (int i = 0; i < 8; ++i) g_wstat[threadIdx.x >> 5][i] = w.c[i];
  }
}
#else
struct WStat {};
__device__ __forceinline__ void wstat_init(const Args&, WStat&) {}
template <int K>
__device__ __forceinline__ void wait_s(const Args&, WStat&, uint64_t* b, uint32_t parity) {
  wait(b, parity);
}
template <int K>
__device__ __forceinline__ void wstat_add(const Args&, WStat&, long long) {}
__device__ __forceinline__ long long wstat_clock(const Args&) { return 0; }
__device__ __forceinline__ void wstat_done(const Args&, WStat&) {}
#endif
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{.reg .pred P; elect.sync _|P, 0xffffffff; selp.b32 %0, 1, 0, P;}" : "=r"(p));
  return p != 0;
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{.reg .pred p; setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
  return (2u << 4) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) | (8u << 24);  // s32 D, u8 A, s8 B, M=128
}
__device__ __forceinline__ uint64_t bdesc(uint32_t saddr) {  // no swizzle, K-major: LBO 128 (K), SBO 256 (N)
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>(128 >> 4) << 16) |
         (static_cast<uint64_t>(256 >> 4) << 32) | (static_cast<uint64_t>(1) << 46);
}
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}
__device__ __forceinline__ void ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void ld4(uint32_t taddr, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
__device__ __forceinline__ void ld3(uint32_t taddr, uint32_t (&r)[3]) {  // columns c, c+1, c+2
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(taddr));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[2]) : "r"(taddr + 2));
}
__device__ __forceinline__ void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_plain(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float4 ldsf4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void red_add(float* p, float v) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void stamp(const Args& A, int i) {
  if (A.stamp && threadIdx.x % 32 == 0) g_stamps[blockIdx.x * 16 + i] = umma::globaltimer();
}

// ---------------------------------------------------- code layouts ----
// MMA K position k (0..63 within a group) -> code index in the group.
// 2-bit (reference bytes): TMEM column 4w+j byte b = code 16w + 4b + j.
// 3-bit (repacked): identity.
__device__ __forceinline__ int kcode(int bits, int k) {
  if (bits == 3) return k;
  const int reg = k >> 2, b = k & 3;
  return 16 * (reg >> 2) + 4 * b + (reg & 3);
}
__device__ __forceinline__ void decode2(const uint4 c, uint32_t (&r)[16]) {
  const uint32_t w4[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
  for (int w = 0; w < 4; ++w)
#pragma unroll
    for (int j = 0; j < 4; ++j) r[4 * w + j] = (w4[w] >> (2 * j)) & 0x03030303u;
}
// 3-bit repack (build_pack): word w < 6, byte b: bits 0-2 = code 8w+b, bits 3-5 = code 8w+4+b;
// bits 6-7 of word 3s (3s+1) byte b = low bits of code 48+8s+b (48+8s+4+b); word 3s+2 byte b
// bit 6 / 7 = bit 2 of those codes.  Register r byte b = code 4r + b.
__device__ __forceinline__ void decode3(const uint32_t (&w)[6], uint32_t (&r)[16]) {
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    r[2 * i] = w[i] & 0x07070707u;
    r[2 * i + 1] = (w[i] >> 3) & 0x07070707u;
  }
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    r[12 + 2 * s] = ((w[3 * s] >> 6) & 0x03030303u) | ((w[3 * s + 2] >> 4) & 0x04040404u);
    r[13 + 2 * s] = ((w[3 * s + 1] >> 6) & 0x03030303u) | ((w[3 * s + 2] >> 5) & 0x04040404u);
  }
}


// ------------------------------------------------------- factor access ----
// element (r, c) of a quantized factor (reference bitstream, fp16 meta)
__device__ __forceinline__ float fac(const lrc_qmat& m, int r, int c) { return qmat_elem(m, r, c); }

// sum_k (c_k s + z) t[k] over a row of nibble codes (16-byte chunks)
__device__ __noinline__ float nib_dot(const uint8_t* codes, int r, float s, float z, const float* t) {
  float acc = 0.f;
  for (int k0 = 0; k0 < r; k0 += 32) {
    const uint4 v = *reinterpret_cast<const uint4*>(codes + k0 / 2);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        const int k = k0 + 8 * q + n;
        if (k < r) acc = fmaf(fmaf(static_cast<float>((w[q] >> (4 * n)) & 15u), s, z), t[k], acc);
      }
  }
  return acc;
}

// Digit image of one 64-value group (one warp; lane l holds values 2l, 2l+1):
// scale 2^S with S from the group's max |value| (21-bit integers), three
// signed 7-bit digits at the value's K position in rows 0..2 of a 512-byte
// no-swizzle K-major core-matrix image (rows 3..7 stay zero); sum of the
// integers and 2^-S -> *sum.  kpos = the position of code i in the A operand.
__device__ __forceinline__ int kpos(int bits, int i) {
  return bits == 3 ? i : 16 * (i >> 4) + 4 * (i & 3) + ((i >> 2) & 3);
}
__device__ __forceinline__ void digit_image(int bits, float v0, float v1, uint8_t* img, float4* sum, int lane) {
  float m = fmaxf(fabsf(v0), fabsf(v1));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  int e = 0;
  frexpf(m, &e);
  const int S = m > 0.f ? 20 - e : 0;
  const float sc = ldexpf(1.f, S);
  const int x[2] = {__float2int_rn(v0 * sc), __float2int_rn(v1 * sc)};
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int k = kpos(bits, 2 * lane + i);
    const int base = (k >> 5) * 256 + ((k >> 4) & 1) * 128 + (k & 15);
    const int d0 = x[i] >> 14, rr = x[i] - (d0 << 14);
    img[base] = static_cast<uint8_t>(d0);
    img[base + 16] = static_cast<uint8_t>(rr >> 7);
    img[base + 32] = static_cast<uint8_t>(rr & 127);
  }
  int t = x[0] + x[1];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) *sum = make_float4(ldexpf(1.f, -S), static_cast<float>(t), 0.f, 0.f);
}

// -------------------------------------------------------------- kernel ----
// Static shared state.  The hot loops of the roles live in separate
// non-inlined functions so that each warp's steady-state code stays small:
// the kernel runs 15 warps through 6 different loops at once, and an earlier
// fully-inlined version (21K instructions) was bound by instruction fetch.
struct Shared {
  Plan P;
  uint64_t full[kMaxNST], bopf[kMaxNST], empty[kMaxNST];
  uint64_t afull[kNAS], aempty[kNAS], dfull[kMaxNDS], dempty[kMaxNDS], xrdy;
  int NAS, dcol;  // A ring depth, first D column
  uint64_t tfull[2], tempty[2], dready, gbarr;
  uint32_t tmem_base;
  int N, SB, NST, NDS, bop_off, xs_off, BG;
  uint8_t* ring;
  float* tres;
  float* eacc;  // B > 1 epilogue segment sums [2][kMaxTok][128]
  float red[kWarps][40];
  double lg64[kMaxTok][kFuseMaxE];
  float pw[kMaxTok][kMaxE];
  uint8_t pc[kMaxTok][kMaxE];
  uint32_t mark[kMaxE];
  int last_flag;
  float t13s[2][2 * kRMax];
  float gred[4];
  int nstage, nstage_u;       // this CTA's stages (phase U first)
  // resident B operand (B == 1): the token's x images (phase U), then the
  // activation images of this CTA's phase-D groups, loaded once per phase
  int res, bimg_off, bsum_off;
  uint64_t bimgf;
  uint16_t doff[kMaxStages];  // per stage: image index of its first group in the resident buffer
  int2 stab[kMaxStages];      // per stage: {g | tile << 16, a | ph << 8 | ns << 9 | seg_end << 13 | seg_ng << 16}
  float t2red[4][kRMax];
};

template <int BITS>
struct Geo {
  static constexpr int CB = BITS == 2 ? 16 : 24;  // code bytes per row-group
  static constexpr int UB = 128 * CB + 512;       // unit: codes + {s, z} per row
};

// ---- routing: record a selected (token, expert) pair
__device__ __forceinline__ void select_pair(const Args& A, Shared& S, int t, int i, int e, float w) {
  S.pw[t][e] = w;
  S.pc[t][e] = (i < A.top_n) ? 1 : 0;
  atomicOr(&S.mark[e], 1u << t);
  if (blockIdx.x == 0) {
    A.topk_idx[t * A.top_k + i] = e;
    A.topk_w[t * A.top_k + i] = w;
  }
}

// warp-wide argmax over lanes (value, index), ties -> lower index
__device__ __forceinline__ int warp_argmax(float v, int idx) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
    if (v2 > v || (v2 == v && i2 < idx)) {
      v = v2;
      idx = i2;
    }
  }
  return idx;
}

// Fused routing (E <= 16): fp32 gate GEMV from shared memory, warp-parallel
// stable top-k per token.  The ranking is exact unless an adjacent gap of the
// top-(k+1) logits is inside the fp32 error bound 256 u ||x|| ||g_e||
// (Cauchy-Schwarz bound on sum |x_i g_i|, gate rounding included); those
// tokens are re-routed in fp64 (route_fallback).
__device__ __noinline__ void route_fused(const Args& A, Shared& S, const float* gs) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int H = A.hidden, B = A.B;
  const int wpt = max(1, kWarps / B);
  const int t = warp / wpt, wi = warp % wpt;
  float acc[kFuseMaxE], xx = 0.f, xm = 0.f;
#pragma unroll
  for (int e = 0; e < kFuseMaxE; ++e) acc[e] = 0.f;
  if (t < B) {
    for (int c = wi * 32 + lane; c < H / 8; c += wpt * 32) {
      const uint4 xv = __ldg(reinterpret_cast<const uint4*>(A.x + static_cast<size_t>(t) * H) + c);
      const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
      float xf[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        xf[2 * q] = bf2f(xw[q] & 0xffff);
        xf[2 * q + 1] = bf2f(xw[q] >> 16);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        xm = fmaxf(xm, fabsf(xf[q]));
        xx = fmaf(xf[q], xf[q], xx);
      }
#pragma unroll
      for (int e = 0; e < kFuseMaxE; ++e) {
        if (e < A.E) {
          const float4 g0 = *reinterpret_cast<const float4*>(gs + static_cast<size_t>(e) * H + 8 * c);
          const float4 g1 = *reinterpret_cast<const float4*>(gs + static_cast<size_t>(e) * H + 8 * c + 4);
          acc[e] = fmaf(xf[0], g0.x, fmaf(xf[1], g0.y, fmaf(xf[2], g0.z, fmaf(xf[3], g0.w, acc[e]))));
          acc[e] = fmaf(xf[4], g1.x, fmaf(xf[5], g1.y, fmaf(xf[6], g1.z, fmaf(xf[7], g1.w, acc[e]))));
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < kFuseMaxE; ++e)
    if (e < A.E) acc[e] = warp_sum(acc[e]);
  xx = warp_sum(xx);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) xm = fmaxf(xm, __shfl_xor_sync(0xffffffffu, xm, o));
  if (lane == 0) {
#pragma unroll
    for (int e = 0; e < kFuseMaxE; ++e)
      if (e < A.E) S.red[warp][e] = acc[e];
    S.red[warp][32] = xm;
    S.red[warp][33] = xx;
  }
  __syncthreads();
  if (warp < B) {  // warp tt selects for token tt; lane e holds logit e
    const int tt = warp;
    float l = -INFINITY, m = 0.f, s2 = 0.f;
    if (lane < A.E) l = 0.f;
    for (int w = tt * wpt; w < tt * wpt + wpt; ++w) {
      if (lane < A.E) l += S.red[w][lane];
      m = fmaxf(m, S.red[w][32]);
      s2 += S.red[w][33];
    }
    if (lane == 0) S.P.xmax[tt] = m;
    const float xn = sqrtf(s2) * 1.001f;
    const float gn = lane < A.E ? A.gnorm[lane] : 0.f;
    const int kk = min(A.top_k + 1, A.E);
    bool used = false, ok = true;
    float prev_l = 0.f, prev_g = 0.f, lmax = 0.f;
    int sel_i = -1;  // rank of this lane's expert among the selected (-1: not selected)
    for (int i = 0; i < kk; ++i) {
      const int b = warp_argmax(used || lane >= A.E ? -INFINITY : l, lane);
      const float lb = __shfl_sync(0xffffffffu, l, b), gb = __shfl_sync(0xffffffffu, gn, b);
      if (i == 0) lmax = lb;
      if (i > 0 && !(prev_l - lb > 256.f * 5.9604645e-8f * xn * (prev_g + gb))) ok = false;
      if (lane == b) {
        used = true;
        if (i < A.top_k) sel_i = i;
      }
      prev_l = lb;
      prev_g = gb;
    }
    if (!ok) {
      if (lane == 0) atomicOr(&S.P.fallback, 1 << tt);
    } else {
      const float ex = lane < A.E ? __expf(l - lmax) : 0.f;
      const float den = warp_sum(ex);
      const float w = ex / den;
      const float wsum = warp_sum(sel_i >= 0 ? w : 0.f);
      if (sel_i >= 0) select_pair(A, S, tt, sel_i, lane, (A.renorm && wsum > 0.f) ? w / wsum : w);
    }
  }
  __syncthreads();
}

// exact fp64 routing of the tokens flagged by route_fused (rare)
__device__ __noinline__ void route_fallback(const Args& A, Shared& S) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int H = A.hidden;
  for (int t = 0; t < A.B; ++t) {
    if (!(S.P.fallback >> t & 1)) continue;
    double accd[kFuseMaxE];
#pragma unroll
    for (int e = 0; e < kFuseMaxE; ++e) accd[e] = 0.0;
    for (int c = tid; c < H; c += kThreads) {
      const double xv = bf2f(A.x[static_cast<size_t>(t) * H + c]);
#pragma unroll
      for (int e = 0; e < kFuseMaxE; ++e)
        if (e < A.E) accd[e] = fma(xv, A.gate64[static_cast<size_t>(e) * H + c], accd[e]);
    }
#pragma unroll
    for (int e = 0; e < kFuseMaxE; ++e)
      if (e < A.E) accd[e] = warp_sum_d(accd[e]);
    __syncthreads();
    if (lane == 0) {
#pragma unroll
      for (int e = 0; e < kFuseMaxE; ++e)
        if (e < A.E) reinterpret_cast<double*>(&S.red[warp][0])[e] = accd[e];
    }
    __syncthreads();
    if (tid < A.E) {
      double sd = 0.0;
      for (int w = 0; w < kWarps; ++w) sd += reinterpret_cast<double*>(&S.red[w][0])[tid];
      S.lg64[t][tid] = sd;
    }
    __syncthreads();
  }
  if (warp == 0 && lane < A.B && (S.P.fallback >> lane & 1)) {
    const int tt = lane;
    uint32_t used = 0u;
    int sel[8];
    for (int i = 0; i < A.top_k; ++i) {
      int b = -1;
      for (int e = 0; e < A.E; ++e)
        if (!(used >> e & 1u) && (b < 0 || S.lg64[tt][e] > S.lg64[tt][b])) b = e;
      used |= 1u << b;
      sel[i] = b;
    }
    const double mx = S.lg64[tt][sel[0]];
    double den = 0.0, wsum = 0.0, w[8];
    for (int e = 0; e < A.E; ++e) den += exp(S.lg64[tt][e] - mx);
    for (int i = 0; i < A.top_k; ++i) {
      w[i] = exp(S.lg64[tt][sel[i]] - mx) / den;
      wsum += w[i];
    }
    for (int i = 0; i < A.top_k; ++i)
      select_pair(A, S, tt, i, sel[i], static_cast<float>((A.renorm && wsum > 0.0) ? w[i] / wsum : w[i]));
  }
  __syncthreads();
}

// routing given (router kernel / pairs mode), shared experts, token max |x|
__device__ __noinline__ void route_rest(const Args& A, Shared& S, bool fused) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int B = A.B, H = A.hidden;
  if (!A.pairs_mode) {
    if (!fused && tid < B * A.top_k) {
      const int t = tid / A.top_k, i = tid % A.top_k;
      const int e = A.given_idx[tid];
      S.pw[t][e] = A.given_w[tid];
      S.pc[t][e] = (i < A.top_n) ? 1 : 0;
      atomicOr(&S.mark[e], 1u << t);
    }
    if (tid < B * A.S) {  // shared experts: every token, weight 1 (ref/moe.py:249-258)
      const int t = tid / A.S, sx = tid % A.S;
      S.pw[t][A.E + sx] = 1.0f;
      S.pc[t][A.E + sx] = A.comp_shared ? 1 : 0;
      atomicOr(&S.mark[A.E + sx], 1u << t);
    }
  } else if (tid < B) {  // pairs mode: row b -> one (token b, expert) pair
    const int e = A.given_idx[tid];
    S.pw[tid][e] = A.given_w[tid];
    S.pc[tid][e] = A.given_comp[tid] ? 1 : 0;
    atomicOr(&S.mark[e], 1u << tid);
  }
  if (!fused) {  // token max |x| (the fused path computed it with the logits)
    for (int t = 0; t < B; ++t) {
      float xm = 0.f;
      for (int c = tid; c < H; c += kThreads) xm = fmaxf(xm, fabsf(bf2f(A.x[static_cast<size_t>(t) * H + c])));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) xm = fmaxf(xm, __shfl_xor_sync(0xffffffffu, xm, o));
      if (lane == 0) S.red[warp][0] = xm;
      __syncthreads();
      if (tid == 0) {
        float m = 0.f;
        for (int w = 0; w < kWarps; ++w) m = fmaxf(m, S.red[w][0]);
        S.P.xmax[t] = m;
      }
      __syncthreads();
    }
  }
  __syncthreads();
}

// plan (warp 0): active experts ascending, pairs by (expert, token), spans
template <int BITS>
__device__ __noinline__ void build_plan(const Args& A, Shared& S) {
  const int lane = threadIdx.x & 31;
  const int NE = A.E + A.S, H = A.hidden, F = A.ffn;
  Plan& P = S.P;
  int n_act = 0, np = 0, nt = 0;
  for (int e0 = 0; e0 < NE; e0 += 32) {
    const int e = e0 + lane;
    const uint32_t m = e < NE ? S.mark[e] : 0u;
    const uint32_t bal = __ballot_sync(0xffffffffu, m != 0u);
    const int cnt = __popc(m);
    int pre = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, pre, o);
      if (lane >= o) pre += v;
    }
    if (m != 0u) {
      const int a = n_act + __popc(bal & ((1u << lane) - 1u));
      if (a < kMaxAct) {
        P.act_e[a] = e;
        P.act_n[a] = cnt;
        P.act_pack[a][0] = A.ex[e].up;
        P.act_pack[a][1] = A.ex[e].down;
        P.act_p0[a] = np + pre - cnt;
        uint32_t mm = m;
        for (int j = 0; mm; ++j) {
          const int t = __ffs(mm) - 1;
          mm &= mm - 1u;
          const int p = np + pre - cnt + j;
          if (p < kMaxP) {
            P.pair_tok[p] = t;
            P.pair_w[p] = S.pw[t][e];
            P.pair_comp[p] = (S.pc[t][e] && A.ex[e].rank > 0) ? 1 : 0;
          }
        }
      }
    }
    nt = max(nt, cnt);
    n_act += __popc(bal);
    np += __shfl_sync(0xffffffffu, pre, 31);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nt = max(nt, __shfl_xor_sync(0xffffffffu, nt, o));
  __syncwarp();
  if (lane == 0) {
    P.n_act = min(n_act, kMaxAct);
    P.np = min(np, kMaxP);
    P.NT = nt;
    P.N = nt == 1 ? 8 : (8 * nt + 15) / 16 * 16;
    int nc = 0;
    for (int p = 0; p < P.np; ++p) {
      if (P.pair_comp[p]) {
        P.comp_pair[nc] = p;
        P.pair_comp[p] = nc++;
      } else {
        P.pair_comp[p] = -1;
      }
    }
    P.n_comp = nc;
    const long long G0 = H / 64, T0 = F / 128, G1 = F / 64, T1 = H / 128;
    const long long tot0 = static_cast<long long>(P.n_act) * T0 * G0, tot1 = static_cast<long long>(P.n_act) * T1 * G1;
    const long long c = blockIdx.x, ncta = gridDim.x;
    if ((ncta + 1) * (tot0 > tot1 ? tot0 : tot1) < (1ll << 32)) {  // 32-bit divisions (the common case)
      const unsigned cu = static_cast<unsigned>(c), nu = static_cast<unsigned>(ncta);
      const unsigned t0u = static_cast<unsigned>(tot0), t1u = static_cast<unsigned>(tot1);
      P.lo[0] = cu * t0u / nu;
      P.hi[0] = (cu + 1) * t0u / nu;
      P.lo[1] = cu * t1u / nu;
      P.hi[1] = (cu + 1) * t1u / nu;
    } else {
      P.lo[0] = c * tot0 / ncta;
      P.hi[0] = (c + 1) * tot0 / ncta;
      P.lo[1] = c * tot1 / ncta;
      P.hi[1] = (c + 1) * tot1 / ncta;
    }
    // stage layout: [codes + meta of <= gps groups x 2 matrices][B operand: per
    // group NT x 512-byte digit images][per token x group: {2^-S, sum}]
    // B operand rows: 8 per token (digits in rows 0..2), N = 8 NT
    // (tcgen05.mma M=128 takes N = 8 or a multiple of 16)
    const int N = nt == 1 ? 8 : (8 * nt + 15) / 16 * 16;
    P.gps = nt <= 4 ? kGPS : kGPS / 2;  // D block per stage: 2 gps x N <= 256 columns
    S.N = N;
    S.BG = nt * 512;
    S.bop_off = P.gps * 2 * Geo<BITS>::UB;
    S.xs_off = S.bop_off + P.gps * S.BG;
    S.SB = S.xs_off + kMaxTok * P.gps * 16;
    S.res = A.B == 1 ? 1 : 0;
    int bimg_bytes = 0;
    if (S.res) {
      const int nimg = max(static_cast<int>(G0), static_cast<int>(P.hi[1] - P.lo[1]));
      S.SB = S.bop_off;  // stages carry only codes + metadata
      bimg_bytes = nimg * (512 + 16);
    }
    uint32_t dyn;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    S.NST = min(kMaxNST, static_cast<int>((dyn - kTresBytes - kEaccBytes - bimg_bytes) / S.SB));
    if (S.res) {
      S.bimg_off = S.NST * S.SB;
      S.bsum_off = S.bimg_off + (bimg_bytes / (512 + 16)) * 512;
    }
    // D ring after the A ring (256 columns): stages x 2 gps units x N columns;
    // NDS = 2 lets the epilogue trail the decode by one stage
    // TMEM: A ring (NAS x 128 columns) then the D ring (NDS x 2 gps x N columns)
    const int dblk = 2 * P.gps * N;
    S.NAS = A.B == 1 ? kOneNAS : (3 * 128 + dblk <= 512 ? 3 : 2);
    S.dcol = S.NAS * 128;
    S.NDS = max(1, min(kMaxNDS, (512 - S.dcol) / dblk));
  }
}

// ---- this CTA's stages (a stage = <= gps consecutive groups of one tile)
struct Stg {
  int g, tile, a, ph, ns, seg_end, seg_ng;
};
__device__ __forceinline__ Stg stg(const Shared& S, int s) {
  const int2 r = S.stab[s];
  Stg t;
  t.g = r.x & 0xffff;
  t.tile = r.x >> 16;
  t.a = r.y & 0xff;
  t.ph = (r.y >> 8) & 1;
  t.ns = (r.y >> 9) & 15;
  t.seg_end = (r.y >> 13) & 1;
  t.seg_ng = r.y >> 16;
  return t;
}
// warp 0: the span [lo, hi) of (expert, tile, group) of each phase -> tile parts
// (one lane each) -> stages of <= gps groups
__device__ __noinline__ void build_stages(const Args& A, Shared& S) {
  const int lane = threadIdx.x & 31;
  const Plan& P = S.P;
  int base = 0;
  for (int ph = 0; ph < 2; ++ph) {
    int gbase = 0;
    // units per stage: phase U gps groups x (w1, w3); phase D gps groups of w2, or
    // 2 gps with the resident B operand (B == 1: the stage carries 2 gps units either way)
    const int gps = (ph == 1 && S.res) ? 2 * P.gps : P.gps;
    const int G = ph == 0 ? A.hidden / 64 : A.ffn / 64, T = ph == 0 ? A.ffn / 128 : A.hidden / 128;
    const int lo = static_cast<int>(P.lo[ph]), hi = static_cast<int>(P.hi[ph]);
    if (hi > lo) {
      const int t0 = lo / G, t1 = (hi - 1) / G;
      for (int tp0 = t0; tp0 <= t1; tp0 += 32) {
        const int tl = tp0 + lane;
        int n = 0, g0 = 0, g1 = 0;
        if (tl <= t1) {
          g0 = tl == t0 ? lo % G : 0;
          g1 = tl == t1 ? (hi - 1) % G + 1 : G;
          n = (g1 - g0 + gps - 1) / gps;
        }
        int pre = n, gpre = g1 - g0;  // inclusive prefixes: stages, groups
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, pre, o), w = __shfl_up_sync(0xffffffffu, gpre, o);
          if (lane >= o) {
            pre += v;
            gpre += w;
          }
        }
        const int at = base + pre - n, gat = gbase + gpre - (g1 - g0);
        // the tile parts one after another (a CTA has 1-3 per phase), each
        // part's stages written by the lanes in parallel
        for (unsigned m = __ballot_sync(0xffffffffu, n > 0); m; m &= m - 1) {
          const int j = __ffs(m) - 1;
          const int nj = __shfl_sync(0xffffffffu, n, j), g0j = __shfl_sync(0xffffffffu, g0, j);
          const int g1j = __shfl_sync(0xffffffffu, g1, j), atj = __shfl_sync(0xffffffffu, at, j);
          const int gatj = __shfl_sync(0xffffffffu, gat, j), tlj = tp0 + j;
          const int hi_word = (tlj / T) | (ph << 8) | ((g1j - g0j) << 16), lo_word = (tlj % T) << 16;
          for (int k = lane; k < nj && atj + k < kMaxStages; k += 32) {
            const int g = g0j + k * gps, ns = min(gps, g1j - g);
            const int segend = g + ns == g1j ? 1 : 0;
            S.stab[atj + k] = make_int2(g | lo_word, hi_word | (ns << 9) | (segend << 13));
            // resident-B image index: U = the group's K index; D = position in this CTA's D groups
            S.doff[atj + k] = static_cast<uint16_t>(ph == 0 ? g : gatj + k * gps);
          }
        }
        base += __shfl_sync(0xffffffffu, pre, 31);
        gbase += __shfl_sync(0xffffffffu, gpre, 31);
      }
    }
    if (ph == 0 && lane == 0) S.nstage_u = min(base, kMaxStages);
  }
  if (lane == 0) S.nstage = min(base, kMaxStages);
}

// ---- producer: per stage one cp.async.bulk of the codes + metadata (ring
// slot free -> issue; phase D codes stream ahead across the grid barrier) and
// the B operand copies: digit images + group sums (phase U once the grid's x
// images are done; phase D once the grid barrier has passed).
template <int BITS>
__device__ __noinline__ void role_producer(const Args& A, Shared& S) {
  constexpr int UB = Geo<BITS>::UB;
  const int lane = threadIdx.x & 31;
  const int NST = S.NST, SB = S.SB, BG = S.BG, G0 = A.hidden / 64, G1 = A.ffn / 64, nst = S.nstage;
  const Plan& P = S.P;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const uint32_t ring = smem_u32(S.ring);
  int sc = 0, sb = 0;  // next stage for codes / for the B operand (sb < sc)
  int cslot = 0, cph = 0, bslot = 0;
  bool xready = false, dready = false;
  uint64_t t0 = 0;
  while (sb < nst || sc < nst) {
    bool progress = false;
    // codes + metadata: one bulk copy (lane 0) once the ring slot is free
    if (sc < nst && (sc < NST || try_wait(&S.empty[cslot], cph ^ 1))) {
      if (lane == 0) {
        const Stg t = stg(S, sc);
        const int nm = 2 - t.ph, G = t.ph == 0 ? G0 : G1;
        const size_t off = (static_cast<size_t>(t.tile) * G + t.g) * nm * UB;
        const uint32_t bytes = static_cast<uint32_t>(t.ns * nm * UB);
        arrive_tx(&S.full[cslot], bytes);
        bulk_g2s(ring + cslot * SB, P.act_pack[t.a][t.ph] + off, bytes, &S.full[cslot], pol);
        trace(A, 0, sc);
      }
      ++sc;
      if (++cslot == NST) {
        cslot = 0;
        cph ^= 1;
      }
      progress = true;
    }
    if (S.res) {  // resident B operand: x images once (phase U), activation images once (phase D)
      if (sb == 0 && (xready || (xready = try_wait(&S.xrdy, 0)))) {
        if (lane == 0) {
          const int G0b = A.hidden / 64;
          arrive_tx(&S.bimgf, G0b * (512 + 16));
          bulk_g2s_plain(ring + S.bimg_off, A.xdig, G0b * 512, &S.bimgf);
          bulk_g2s_plain(ring + S.bsum_off, A.xsum, G0b * 16, &S.bimgf);
        }
        sb = 1;
        progress = true;
      } else if (sb == 1 && (dready || (dready = try_wait(&S.dready, 0)))) {
        if (lane == 0) {
          int bytes = 0;
          for (int k = S.nstage_u; k < nst; ++k) bytes += stg(S, k).ns * (512 + 16);
          arrive_tx(&S.bimgf, static_cast<uint32_t>(bytes));
          for (int k = S.nstage_u; k < nst; ++k) {
            const Stg t = stg(S, k);
            const int p = P.act_p0[t.a], dof = S.doff[k];
            bulk_g2s_plain(ring + S.bimg_off + dof * 512, A.adig + (static_cast<size_t>(p) * G1 + t.g) * 512,
                           t.ns * 512, &S.bimgf);
            bulk_g2s_plain(ring + S.bsum_off + dof * 16, A.asum + static_cast<size_t>(p) * G1 + t.g, t.ns * 16,
                           &S.bimgf);
          }
        }
        sb = nst;
        progress = true;
      }
      if (sc >= nst && sb >= nst) break;
    } else if (sb < sc) {
      // B operand (digit images + group sums): 16-byte cp.async by all lanes
      // (LDGSTS: not queued behind the ring's bulk copies), completion tracked
      // by one arrive.noinc per lane on the stage's bopf barrier
      const Stg t = stg(S, sb);
      if (t.ph == 0 && !xready) xready = try_wait(&S.xrdy, 0);
      if (t.ph == 1 && !dready) dready = try_wait(&S.dready, 0);
      if (t.ph == 0 ? xready : dready) {
        const int na = P.act_n[t.a], p0 = P.act_p0[t.a], ns = t.ns;
        const uint32_t st = ring + bslot * SB;
        const int G = t.ph == 0 ? G0 : G1;
        for (int j = 0; j < na; ++j) {
          const int p = p0 + j;
          const int row = t.ph == 0 ? P.pair_tok[p] : p;  // image row: token (U) or pair (D)
          const uint8_t* img = (t.ph == 0 ? A.xdig : A.adig) + (static_cast<size_t>(row) * G + t.g) * 512;
          const float4* sm = (t.ph == 0 ? A.xsum : A.asum) + static_cast<size_t>(row) * G + t.g;
          // group sg, K half hs, 16-byte chunk c (16 per half) -> sg * BG + hs * na * 256 + j * 256 + 16 c
          for (int k = lane; k < ns * 32; k += 32) {
            const int sg = k >> 5, hs = (k >> 4) & 1, cidx = k & 15;
            umma::cp_async16(st + S.bop_off + sg * BG + hs * na * 256 + j * 256 + cidx * 16,
                             img + sg * 512 + hs * 256 + cidx * 16, 16);
          }
          if (lane < ns) umma::cp_async16(st + S.xs_off + (j * P.gps + lane) * 16, sm + lane, 16);
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&S.bopf[bslot]))
                     : "memory");
        if (lane == 0) trace(A, 1, sb);
        ++sb;
        if (++bslot == NST) bslot = 0;
        progress = true;
      }
    }
    if (!progress) {
      const uint64_t t = umma::globaltimer();
      if (t0 == 0) t0 = t;
      else if (t - t0 > 4000000000ull) __trap();
    } else {
      t0 = 0;
    }
  }
}

// ---- MMA issuer: per stage, 2 x tcgen05.mma.kind::i8 (K = 32 each) per
// (group, matrix) unit with N = 8 x the expert's tokens, one commit for the
// stage's D block and one for its ring slot
// 8 units x 2 MMAs of a full B == 1 stage; unit u: D columns 8u (N = 8), A
// columns 16u, B image (u >> SH) (512 bytes = 32 descriptor address units),
// second K half 256 bytes on
template <int SH>
__device__ __forceinline__ void mma_stage8(uint32_t d0, uint32_t a0, uint64_t b0, uint32_t id) {
  const uint32_t blo = static_cast<uint32_t>(b0), bhi = static_cast<uint32_t>(b0 >> 32);
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const uint32_t bl = blo + (u >> SH) * 32;
    asm volatile(
        "{.reg .b64 bd0, bd1; mov.b64 bd0, {%2, %4}; mov.b64 bd1, {%3, %4};\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], bd0, %5, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%6], bd1, %5, 1;}" ::"r"(d0 + u * 8),
        "r"(a0 + u * 16), "r"(bl), "r"(bl + 16), "r"(bhi), "r"(id), "r"(a0 + u * 16 + 8));
  }
}

template <bool ONE>
__device__ __noinline__ void role_mma(const Args& A, Shared& S, int bop_off) {
  // ONE (B == 1): one token per expert, N = 8, resident B operand, A ring 3, D ring 2
  const int NST = S.NST, SB = S.SB, nst = S.nstage, nsu = S.nstage_u;
  const int N = ONE ? 8 : S.N, NDS = ONE ? kOneNDS : S.NDS, NAS = ONE ? kOneNAS : S.NAS, BG = ONE ? 512 : S.BG;
  const uint32_t tm = S.tmem_base, dcol = S.dcol;
  const uint32_t ring = smem_u32(S.ring);
  const int dstride = 2 * S.P.gps * N;
  int slot = 0, sph = 0, as = 0, aph = 0, ds = 0, dph = 0;
  WStat ws;
  wstat_init(A, ws);
  for (int s = 0; s < nst; ++s) {
    const Stg t = stg(S, s);
    if (!ONE) {
      wait(&S.bopf[slot], sph);
    } else {
      if (s == 0) wait_s<6>(A, ws, &S.bimgf, 0);    // x images
      if (s == nsu) wait_s<6>(A, ws, &S.bimgf, 1);  // activation images
    }
    wait_s<4>(A, ws, &S.afull[as], aph);
    if (s >= NDS) wait_s<5>(A, ws, &S.dempty[ds], dph ^ 1);
    fence_after();
    const long long tm0 = wstat_clock(A);
    if (elect_one()) {
      const int na = ONE ? 1 : S.P.act_n[t.a], nm = 2 - t.ph, nu = t.ns * nm;
      const uint32_t id = idesc_i8(na == 1 ? 8 : (8 * na + 15) / 16 * 16);
      const uint32_t bop0 = ONE ? ring + S.bimg_off + S.doff[s] * 512 : ring + slot * SB + bop_off;
      if (ONE && nu == 8) {
        // full B == 1 stage, fully unrolled: descriptors are the stage bases plus constants
        const uint32_t d0 = tm + dcol + ds * (8 * 8), a0 = tm + as * 128;
        const uint64_t b0 = bdesc(bop0);
        if (t.ph == 0) mma_stage8<1>(d0, a0, b0, id);
        else mma_stage8<0>(d0, a0, b0, id);
      } else
      for (int u = 0; u < nu; ++u) {
        const uint32_t bop = bop0 + (u >> (nm - 1)) * BG;
        const uint32_t d = tm + dcol + ds * dstride + u * N, a = tm + as * 128 + u * 16;
        mma_i8(d, a, bdesc(bop), id, 0u);
        mma_i8(d, a + 8, bdesc(bop + na * 256), id, 1u);
      }
      wstat_add<2>(A, ws, wstat_clock(A) - tm0);
      commit(&S.aempty[as]);
      commit(&S.dfull[ds]);
      commit(&S.empty[slot]);
      wstat_add<3>(A, ws, wstat_clock(A) - tm0);
      trace(A, 2, s);
      if (A.dbg & 32) {  // debug: MMA completion latency seen by the issuer
        wait(&S.dfull[ds], dph);
        trace(A, 1, s);
      }
    }
    __syncwarp();
    if (++slot == NST) { slot = 0; sph ^= 1; }
    if (++as == NAS) { as = 0; aph ^= 1; }
    if (++ds == NDS) { ds = 0; dph ^= 1; }
  }
  wstat_done(A, ws);
}

// one decode warp's units u = sub + 2 i (i < 4) of a stage: codes (shared) ->
// 8-bit A operand (TMEM); the ring slot's codes are released after the loads
template <int BITS, bool FULL>
__device__ __forceinline__ void dec_units(uint32_t st, uint32_t ta, int sub, int nu, int lane, uint64_t* empty) {
  constexpr int UB = Geo<BITS>::UB;
  uint32_t cw[4][6];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int u = sub + 2 * i;
    if (FULL || u < nu) {
      const uint32_t cp = st + u * UB;
      if (BITS == 2) {
        const uint4 v = lds128(cp);
        cw[i][0] = v.x; cw[i][1] = v.y; cw[i][2] = v.z; cw[i][3] = v.w;
      } else {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const uint2 v = lds64(cp + 8 * k);
          cw[i][2 * k] = v.x;
          cw[i][2 * k + 1] = v.y;
        }
      }
    }
  }
  __syncwarp();
  if (lane == 0) arrive(empty);  // codes read
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int u = sub + 2 * i;
    if (FULL || u < nu) {
      uint32_t r[16];
      if (BITS == 2) {
        decode2(make_uint4(cw[i][0], cw[i][1], cw[i][2], cw[i][3]), r);
      } else {
        uint32_t w[6] = {cw[i][0], cw[i][1], cw[i][2], cw[i][3], cw[i][4], cw[i][5]};
        decode3(w, r);
      }
      st16(ta + u * 16, r);
    }
  }
}

// ---- decode warps, per stage: codes -> TMEM A block; epilogue of the
// previous stage (NDS = 2) or of this stage (NDS = 1, N = 24).
// Phase U: half h decodes matrix h (w1 / w3) of the stage's groups; phase D:
// half h decodes the groups sg with sg % 2 == h.
template <int BITS, bool ONE>
__device__ __noinline__ void role_decode(const Args& A, Shared& S) {
  constexpr int CB = Geo<BITS>::CB, UB = Geo<BITS>::UB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = warp >> 2, q = warp & 3, row = q * 32 + lane;  // units u = sub + 2 i of a stage
  const int NST = S.NST, SB = S.SB, nst = S.nstage, NAS = ONE ? kOneNAS : S.NAS;
  const uint32_t tl = S.tmem_base + (static_cast<uint32_t>(q * 32) << 16);
  const uint32_t ring = smem_u32(S.ring) + row * CB;
  int slot = 0, sph = 0, as = 0, aph = 0;
  WStat ws;
  wstat_init(A, ws);
  for (int s = 0; s < nst; ++s) {
    const Stg t = stg(S, s);
    wait_s<0>(A, ws, &S.full[slot], sph);
    if (s >= NAS) wait_s<1>(A, ws, &S.aempty[as], aph ^ 1);  // MMAs of stage s - NAS read this A block
    fence_after();
    if (lane == 0 && warp == 0) trace2(A, 3, s);
    const uint32_t st = ring + slot * SB;
    const int nu = t.ns * (2 - t.ph);
    // full stage (the common case): no per-unit predicates, so the loads and
    // the decode chains of the four units interleave
    if (nu == 8) dec_units<BITS, true>(st, tl + as * 128, sub, nu, lane, &S.empty[slot]);
    else dec_units<BITS, false>(st, tl + as * 128, sub, nu, lane, &S.empty[slot]);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    fence_before();
    __syncwarp();
    if (lane == 0) {
      arrive(&S.afull[as]);
      if (warp == 0) trace(A, 3, s);
    }
    if (++slot == NST) { slot = 0; sph ^= 1; }
    if (++as == NAS) { as = 0; aph ^= 1; }
  }
  wstat_done(A, ws);
}

// B == 1 epilogue of one stage (N = 8: unit u's D block = columns 8u..8u+2,
// the x digits' dot products): TMEM loads, then the group metadata and x
// sums while they are in flight, then per unit s * dot + z * sum(x) scaled
// by 2^-S.  Phase U: unit u = (group u / 2, matrix u % 2); phase D: group u.
template <int UB, bool FULL, int PH>
__device__ __forceinline__ void epi_one(uint32_t td, uint32_t meta, uint32_t xs4, int nu, int lane, uint64_t* dempty,
                                        float& acc0, float& acc1) {
  uint32_t D[8][3];
#pragma unroll
  for (int u = 0; u < 8; ++u)
    if (FULL || u < nu) ld3(td + u * 8, D[u]);
  ld_wait();
  fence_before();
  __syncwarp();
  if (lane == 0) arrive(dempty);
  uint32_t sz[8];
#pragma unroll
  for (int u = 0; u < 8; ++u)
    if (FULL || u < nu) sz[u] = lds32(meta + u * UB);
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    if (FULL || u < nu) {
      const uint2 xv = lds64(xs4 + (PH == 0 ? u >> 1 : u) * 16);
      const float2 sf = __half22float2(*reinterpret_cast<const __half2*>(&sz[u]));
      const int v = (static_cast<int>(D[u][0]) << 14) + (static_cast<int>(D[u][1]) << 7) + static_cast<int>(D[u][2]);
      const float r = fmaf(sf.x, static_cast<float>(v), sf.y * __uint_as_float(xv.y)) * __uint_as_float(xv.x);
      if (PH == 0 && (u & 1)) acc1 += r;
      else acc0 += r;
    }
  }
}

// B > 1 epilogue of one stage: NA (>= na) tokens per unit, UC units per chunk
// (stage sums in registers, segment sums in shared memory: eacc + (m kMaxTok + j) 512)
template <int UB, int NA, int UC>
__device__ __forceinline__ void epi_multi(uint32_t td, int N, uint32_t meta, uint32_t xs, int gps, int nu, int sh,
                                          int na, uint32_t eacc, bool fresh) {
  float rs[2][NA];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int j = 0; j < NA; ++j) rs[m][j] = 0.f;
#pragma unroll 1
  for (int c = 0; c < nu; c += UC) {
    uint32_t D[UC][NA][3];
#pragma unroll
    for (int i = 0; i < UC; ++i)
#pragma unroll
      for (int j = 0; j < NA; ++j)
        if (c + i < nu && j < na) ld3(td + (c + i) * N + 8 * j, D[i][j]);
    uint32_t sz[UC];
#pragma unroll
    for (int i = 0; i < UC; ++i)
      if (c + i < nu) sz[i] = lds32(meta + (c + i) * UB);
    ld_wait();
#pragma unroll
    for (int i = 0; i < UC; ++i) {
      if (c + i < nu) {
        const float2 sf = __half22float2(*reinterpret_cast<const __half2*>(&sz[i]));
        const bool mat = ((c + i) & sh) != 0;
        const int sg = (c + i) >> sh;
#pragma unroll
        for (int j = 0; j < NA; ++j) {
          if (j < na) {
            const uint2 xv = lds64(xs + (j * gps + sg) * 16);
            const float2 xq = make_float2(__uint_as_float(xv.x), __uint_as_float(xv.y));
            const int v = (static_cast<int>(D[i][j][0]) << 14) + (static_cast<int>(D[i][j][1]) << 7) +
                          static_cast<int>(D[i][j][2]);
            const float r = fmaf(sf.x, static_cast<float>(v), sf.y * xq.y) * xq.x;
            // both sums updated (selects): a branch here is merged by the compiler
            // into rs[mat][j], a dynamic index that moves rs to local memory
            rs[0][j] += mat ? 0.f : r;
            rs[1][j] += mat ? r : 0.f;
          }
        }
      }
    }
  }
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    if (m <= sh) {
#pragma unroll
      for (int j = 0; j < NA; ++j) {
        if (j < na) {
          const uint32_t a = eacc + (m * kMaxTok + j) * 512;
          float v = rs[m][j];
          if (!fresh) v += __uint_as_float(lds32(a));
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
        }
      }
    }
  }
}

// ---- epilogue warps (one per TMEM lane quarter; thread = tile row): every
// unit of a stage -> per-group scale/zero and 2^-S, accumulated per matrix;
// segment ends: w1|w3 results to the finalisers (phase U) or the weighted
// combine into y (phase D)
template <int BITS, bool ONE>
__device__ __noinline__ void role_epilogue(const Args& A, Shared& S) {
  constexpr int CB = Geo<BITS>::CB, UB = Geo<BITS>::UB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, row = q * 32 + lane;
  const int NST = S.NST, SB = S.SB, nst = S.nstage, H = A.hidden;
  const int N = ONE ? 8 : S.N, NDS = ONE ? kOneNDS : S.NDS;
  const Plan& P = S.P;
  const uint32_t tl = S.tmem_base + (static_cast<uint32_t>(q * 32) << 16) + S.dcol;
  uint8_t* const ring = S.ring;
  const uint32_t sring = smem_u32(S.ring);
  const int dstride = 2 * P.gps * N;
  const uint32_t bsum = sring + S.bsum_off;
  float acc0 = 0.f, acc1 = 0.f;  // B == 1: this row's w1 (or w2) and w3 sums of the segment
  const uint32_t eacc = smem_u32(S.eacc) + row * 4;  // B > 1: [2][kMaxTok][128] segment sums
  bool fresh = true;
  int useg = 0;
  int slot = 0, sph = 0, ds = 0, dph = 0;
  WStat ws;
  wstat_init(A, ws);
  for (int s = 0; s < nst; ++s) {
    const Stg t = stg(S, s);
    const int nm = 2 - t.ph;
    const uint8_t* st = ring + static_cast<size_t>(slot) * SB;
    const int na = ONE ? 1 : P.act_n[t.a], p0 = P.act_p0[t.a];
    const int nu = t.ns * nm;
    wait_s<2>(A, ws, &S.dfull[ds], dph);
    if (!ONE) wait(&S.bopf[slot], sph);
    fence_after();
    if (lane == 0 && warp == kEpi0) trace2(A, 2, s);
    if (ONE) {
      const uint32_t xs4 = bsum + S.doff[s] * 16;
      const uint32_t meta = sring + slot * SB + 128 * CB + row * 4;
      const uint32_t td = tl + ds * dstride;
      if (nu == 8) {
        if (t.ph == 0) epi_one<UB, true, 0>(td, meta, xs4, nu, lane, &S.dempty[ds], acc0, acc1);
        else epi_one<UB, true, 1>(td, meta, xs4, nu, lane, &S.dempty[ds], acc0, acc1);
      } else {
        if (t.ph == 0) epi_one<UB, false, 0>(td, meta, xs4, nu, lane, &S.dempty[ds], acc0, acc1);
        else epi_one<UB, false, 1>(td, meta, xs4, nu, lane, &S.dempty[ds], acc0, acc1);
      }
    } else {
      // several tokens per expert: D block of unit u, token j = columns u N + 8 j;
      // units in chunks whose TMEM loads are all in flight together
      const uint32_t td = tl + ds * dstride, meta = sring + slot * SB + 128 * CB + row * 4;
      const uint32_t xs = sring + slot * SB + S.xs_off;
      const int sh = nm - 1;
      // reloaded per stage (volatile): keeps the compiler from hoisting every
      // instance's gps / N derived offsets out of the stage loop (register spills)
      const int gps = static_cast<int>(lds32(smem_u32(&S.P.gps))), N = static_cast<int>(lds32(smem_u32(&S.N)));
      if (na == 1) epi_multi<UB, 1, 2>(td, N, meta, xs, gps, nu, sh, na, eacc, fresh);
      else if (na == 2) epi_multi<UB, 2, 1>(td, N, meta, xs, gps, nu, sh, na, eacc, fresh);
      else if (na <= 4) epi_multi<UB, 4, 1>(td, N, meta, xs, gps, nu, sh, na, eacc, fresh);
      else epi_multi<UB, 8, 1>(td, N, meta, xs, gps, nu, sh, na, eacc, fresh);
      fence_before();
      __syncwarp();
      if (lane == 0) arrive(&S.dempty[ds]);
    }
    __syncwarp();
    if (lane == 0) arrive(&S.empty[slot]);  // metadata and sums read
    if (lane == 0 && warp == kEpi0) trace2(A, 1, s);
    if (warp == kEpi0 && s == S.nstage_u - 1) stamp(A, 12);  // last phase-U stage through the epilogue
    fresh = false;
    if (t.seg_end) {  // segment end: flush
      fresh = true;
      if (t.ph == 0) {
        const int ts = useg & 1;
        if (useg >= 2) wait_s<3>(A, ws, &S.tempty[ts], ((useg >> 1) - 1) & 1);
        const uint32_t tr = smem_u32(S.tres) + ts * (2 * kMaxTok * 128) * 4;
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
          for (int j = 0; j < kMaxTok; ++j)
            if (j < na) {
              const float v = ONE ? (m == 0 ? acc0 : acc1) : __uint_as_float(lds32(eacc + (m * kMaxTok + j) * 512));
              asm volatile("st.shared.f32 [%0], %1;" ::"r"(tr + ((m * kMaxTok + j) * 128 + row) * 4), "f"(v)
                           : "memory");
            }
        __syncwarp();
        if (lane == 0) arrive(&S.tfull[ts]);
        ++useg;
      } else {
        const int rg = t.tile * 128 + row;
#pragma unroll
        for (int j = 0; j < kMaxTok; ++j) {
          if (j < na) {
            const int p = p0 + j;
            const float v = ONE ? acc0 : __uint_as_float(lds32(eacc + j * 512));
            red_add(A.y + static_cast<size_t>(P.pair_tok[p]) * H + rg, v * P.pair_w[p]);
          }
        }
      }
      acc0 = acc1 = 0.f;
    }
    if (++slot == NST) { slot = 0; sph ^= 1; }
    if (++ds == NDS) { ds = 0; dph ^= 1; }
  }
  wstat_done(A, ws);
}

// ---- aux warps (128 threads = tile rows)
// V.x jobs: one warp per (compensated pair, factor row), spread over the grid
__device__ __noinline__ void vx_jobs(const Args& A, Shared& S) {
  const int lane = threadIdx.x & 31, aw = (threadIdx.x >> 5) - kAux0;
  const Plan& P = S.P;
  const int njobs = P.n_comp * 2 * kRMax;
  for (int jb = blockIdx.x * 4 + aw; jb < njobs; jb += gridDim.x * 4) {
    const int cs = jb / (2 * kRMax), rr = jb % (2 * kRMax);
    const int p = P.comp_pair[cs];
    int a = 0;
    while (a + 1 < P.n_act && P.act_p0[a + 1] <= p) ++a;
    const Expert& ex = A.ex[P.act_e[a]];
    if (rr % kRMax >= ex.rank) continue;
    const lrc_qmat& V = rr < kRMax ? ex.v1 : ex.v3;
    float acc1[1];
    const uint16_t* xt = A.x + static_cast<size_t>(P.pair_tok[p]) * A.hidden;
    if (A.fb == 3)
      vrow_dot_tokens<3, 1>(V, rr % kRMax, xt, A.hidden, 1, acc1);
    else if (A.fb == 2)
      vrow_dot_tokens<2, 1>(V, rr % kRMax, xt, A.hidden, 1, acc1);
    else
      vrow_dot_tokens<4, 1>(V, rr % kRMax, xt, A.hidden, 1, acc1);
    if (lane == 0) {
      A.t13[cs * 2 * kRMax + rr] = acc1[0];
      __threadfence();
      atomicAdd(&A.tcnt[S.P.par * kMaxP + cs], 1u);
    }
  }
}

// finalise one up tile: low-rank terms, SwiGLU, bf16 activations, t2 partials
__device__ __noinline__ void finalize_up(const Args& A, Shared& S, int a, int tile, const float* h1v,
                                         const float* h3v) {
  const int f = threadIdx.x - kAux0 * 32, lane = f & 31, aw = f >> 5;
  const Plan& P = S.P;
  const int par = P.par, F = A.ffn;
  const Expert& ex = A.ex[P.act_e[a]];
  const int i = tile * 128 + f, na = P.act_n[a], p0 = P.act_p0[a];
  for (int j = 0; j < na; ++j) {
    const int p = p0 + j, cs = P.pair_comp[p];
    float hj1 = h1v[j], hj3 = h3v[j];
    const int rk = ex.rank, RB = lr_rb(rk);
    const uint8_t* lt = cs >= 0 ? ex.lr_up + static_cast<size_t>(tile) * lr_up_tile_bytes(rk) : nullptr;
    if (cs >= 0) {
      if (f == 0) {
        const uint64_t t0 = umma::globaltimer();
        while (ld_acquire(&A.tcnt[par * kMaxP + cs]) < static_cast<unsigned>(2 * rk)) {
          __nanosleep(64);
          if (umma::globaltimer() - t0 > 2000000000ull) __trap();
        }
      }
      named_sync(2, 128);
      for (int q2 = f; q2 < 2 * kRMax; q2 += 128) S.t13s[0][q2] = __ldcg(A.t13 + cs * 2 * kRMax + q2);
      named_sync(2, 128);
      const uint32_t* lm = reinterpret_cast<const uint32_t*>(lt + 3 * 128 * RB);
      const uint32_t m1 = lm[f], m3 = lm[128 + f];
      hj1 += nib_dot(lt + f * RB, rk, h2f(m1 & 0xffff), h2f(m1 >> 16), S.t13s[0]);
      hj3 += nib_dot(lt + (128 + f) * RB, rk, h2f(m3 & 0xffff), h2f(m3 >> 16), S.t13s[0] + kRMax);
    }
    const float act = silu_f(hj1) * hj3;
    const uint16_t ab = f2bf(act);  // activations are bf16 (the W2 input), as on the tiled path
    const float av = bf2f(ab);
    // digit image of this row's phase-D group (rows 64 gl .. 64 gl + 63 = warps 2 gl, 2 gl + 1)
    {
      const int gl = f >> 6, G1 = F / 64;
      float m = fabsf(av);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) S.gred[aw] = m;
      named_sync(2, 128);
      m = fmaxf(S.gred[2 * gl], S.gred[2 * gl + 1]);
      int e2 = 0;
      frexpf(m, &e2);
      const int sc = m > 0.f ? 20 - e2 : 0;
      const int X = __float2int_rn(av * ldexpf(1.f, sc));
      const int k = kpos(A.bits, f & 63);
      uint8_t* img = A.adig + (static_cast<size_t>(p) * G1 + 2 * tile + gl) * 512 + (k >> 5) * 256 + ((k >> 4) & 1) * 128 + (k & 15);
      const int d0 = X >> 14, rr = X - (d0 << 14);
      img[0] = static_cast<uint8_t>(d0);
      img[16] = static_cast<uint8_t>(rr >> 7);
      img[32] = static_cast<uint8_t>(rr & 127);
      int t = X;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      named_sync(2, 128);
      if (lane == 0) S.gred[aw] = __int_as_float(t);
      named_sync(2, 128);
      if (f == 0 || f == 64)
        A.asum[static_cast<size_t>(p) * G1 + 2 * tile + gl] =
            make_float4(ldexpf(1.f, -sc), static_cast<float>(__float_as_int(S.gred[2 * gl]) + __float_as_int(S.gred[2 * gl + 1])), 0.f, 0.f);
    }
    if (cs >= 0) {  // t2 partial: V2[:, i] . a_i, reduced over the tile rows
      // (row words and group metadata loaded up front; per 32 factor columns one
      // butterfly reduce-scatter: 31 shuffles leave lane l the warp sum of column l)
      const uint32_t* vm = reinterpret_cast<const uint32_t*>(lt + 3 * 128 * RB) + 256 + (f / 64) * kRMax;
      for (int k0 = 0; k0 < rk; k0 += 32) {
        const uint4 wv = __ldg(reinterpret_cast<const uint4*>(lt + (256 + f) * RB + k0 / 2));
        const uint32_t ww[4] = {wv.x, wv.y, wv.z, wv.w};
        const uint32_t mzl = k0 + lane < rk ? __ldg(vm + k0 + lane) : 0u;
        float v[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const uint32_t mz = __shfl_sync(0xffffffffu, mzl, k);
          const float vk = fmaf(static_cast<float>((ww[k >> 3] >> (4 * (k & 7))) & 15u), h2f(mz & 0xffff), h2f(mz >> 16));
          v[k] = k0 + k < rk ? vk * av : 0.f;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const bool up = (lane & o) != 0;
#pragma unroll
          for (int i = 0; i < o; ++i) {
            const float send = up ? v[i] : v[i + o];
            const float keep = up ? v[i + o] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
        }
        if (k0 + lane < rk) S.t2red[aw][k0 + lane] = v[0];
      }
      named_sync(2, 128);
      if (f < rk)
        atomicAdd(A.t2 + (par * kMaxP + p) * kRMax + f, S.t2red[0][f] + S.t2red[1][f] + S.t2red[2][f] + S.t2red[3][f]);
      named_sync(2, 128);
    }
  }
}

// phase-U tile results -> (split tiles: accumulate, last contributor) finalise
__device__ __noinline__ void aux_phase_u(const Args& A, Shared& S) {
  const int f = threadIdx.x - kAux0 * 32, lane = f & 31;
  const Plan& P = S.P;
  const int G0 = A.hidden / 64, T0 = A.ffn / 128;
  int useg = 0;
  // the LR tile packs this CTA may finalise: pull them into L2 while the
  // stages stream (their first touch is otherwise on the critical path)
  for (int s = 0; s < S.nstage_u; ++s) {
    const Stg t = stg(S, s);
    if (!t.seg_end) continue;
    const Expert& ex = A.ex[P.act_e[t.a]];
    if (ex.rank > 0 && ex.lr_up != nullptr) {
      const int tb = lr_up_tile_bytes(ex.rank);
      const uint8_t* lt = ex.lr_up + static_cast<size_t>(t.tile) * tb;
      for (int o = f * 128; o < tb; o += 128 * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(lt + o));
    }
  }
  for (int s = 0; s < S.nstage_u; ++s) {
    const Stg t = stg(S, s);
    if (!t.seg_end) continue;
    const int a = t.a, tile = t.tile, na = P.act_n[a];
    const int ng = t.seg_ng;
    const int ts = useg & 1;
    wait(&S.tfull[ts], (useg >> 1) & 1);
    float h1[kMaxTok], h3[kMaxTok];
    const float* tr = S.tres + ts * (2 * kMaxTok * 128);  // [w1, w3][token][row]
#pragma unroll
    for (int j = 0; j < kMaxTok; ++j) {
      h1[j] = j < na ? tr[j * 128 + f] : 0.f;
      h3[j] = j < na ? tr[(kMaxTok + j) * 128 + f] : 0.f;
    }
    named_sync(2, 128);
    if (lane == 0) arrive(&S.tempty[ts]);
    ++useg;
    bool fin = ng == G0;
    if (!fin) {  // split tile: accumulate; the last contributor finalises
      float* ha = A.hacc + (static_cast<size_t>(a) * T0 + tile) * (2 * kMaxTok * 128);
#pragma unroll
      for (int j = 0; j < kMaxTok; ++j) {
        if (j < na) {
          red_add(ha + j * 128 + f, h1[j]);
          red_add(ha + (kMaxTok + j) * 128 + f, h3[j]);
        }
      }
      __threadfence();
      named_sync(2, 128);
      if (f == 0) {
        const unsigned old = atomicAdd(&A.hcnt[static_cast<size_t>(a) * T0 + tile], static_cast<unsigned>(ng));
        S.last_flag = ((old + ng) % G0) == 0;
      }
      named_sync(2, 128);
      fin = S.last_flag != 0;
      if (fin) {
        __threadfence();
#pragma unroll
        for (int j = 0; j < kMaxTok; ++j) {
          if (j < na) {
            h1[j] = __ldcg(ha + j * 128 + f);
            h3[j] = __ldcg(ha + (kMaxTok + j) * 128 + f);
            ha[j * 128 + f] = 0.f;
            ha[(kMaxTok + j) * 128 + f] = 0.f;
          }
        }
      }
    }
    if (fin) finalize_up(A, S, a, tile, h1, h3);
  }
}

// phase D: U2.t2 for the tiles whose group 0 this CTA owns
__device__ __noinline__ void aux_phase_d(const Args& A, Shared& S) {
  const int f = threadIdx.x - kAux0 * 32;
  const Plan& P = S.P;
  const int par = P.par, H = A.hidden;
  for (int s = S.nstage_u; s < S.nstage; ++s) {
    const Stg st = stg(S, s);
    if (st.g != 0) continue;
    const int a = st.a, tile = st.tile, na = P.act_n[a], p0 = P.act_p0[a];
    const Expert& ex = A.ex[P.act_e[a]];
    const int i = tile * 128 + f;
    for (int j = 0; j < na; ++j) {
      const int p = p0 + j;
      if (P.pair_comp[p] < 0) continue;
      const int rk = ex.rank, RB = lr_rb(rk);
      for (int k = f; k < rk; k += 128) S.t13s[1][k] = __ldcg(A.t2 + (par * kMaxP + p) * kRMax + k);
      named_sync(2, 128);
      const uint8_t* lt = ex.lr_down + static_cast<size_t>(tile) * lr_down_tile_bytes(rk);
      const uint32_t mz = reinterpret_cast<const uint32_t*>(lt + 128 * RB)[f];
      const float d = nib_dot(lt + f * RB, rk, h2f(mz & 0xffff), h2f(mz >> 16), S.t13s[1]);
      named_sync(2, 128);
      red_add(A.y + static_cast<size_t>(P.pair_tok[p]) * H + i, d * P.pair_w[p]);
    }
  }
}

__device__ __noinline__ void role_aux(const Args& A, Shared& S) {
  const int f = threadIdx.x - kAux0 * 32, aw = f >> 5;
  Plan& P = S.P;
  const int par = P.par;
  // scratch of the next launch (other parity) and this launch's y
  if (blockIdx.x == 0) {
    for (int i = f; i < kMaxP; i += 128) A.tcnt[(1 - par) * kMaxP + i] = 0u;
    if (f == 0) A.xcnt[1 - par] = 0u;
    for (int i = f; i < kMaxP * kRMax; i += 128) A.t2[(1 - par) * kMaxP * kRMax + i] = 0.f;
  }
  {
    const size_t n = static_cast<size_t>(A.B) * A.hidden;
    const size_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
    for (size_t i = lo + f; i < hi; i += 128) A.y[i] = 0.f;
  }
  if (f == 0) {  // the grid's x digit images -> the producer may copy phase-U B operands
    const unsigned xtarget = static_cast<unsigned>(A.B) * (A.hidden / 64);
    const uint64_t t0 = umma::globaltimer();
    while (ld_acquire(&A.xcnt[par]) < xtarget) {
      __nanosleep(64);
      if (umma::globaltimer() - t0 > 2000000000ull) __trap();
    }
    arrive(&S.xrdy);
  }
  vx_jobs(A, S);
  if (aw == 0) stamp(A, 2);
  aux_phase_u(A, S);
  if (aw == 0) stamp(A, 3);
  // grid barrier: every CTA's activation digit images and t2 partials written
  __threadfence();
  named_sync(2, 128);
  if (f == 0) {
    atomicAdd(A.gbar, 1ull);
    const unsigned long long target = static_cast<unsigned long long>(gridDim.x) * (P.epoch + 1);
    const uint64_t t0 = umma::globaltimer();
    while (ld_acquire64(A.gbar) < target) {
      __nanosleep(32);
      if (umma::globaltimer() - t0 > 2000000000ull) __trap();  // CTAs not co-resident
    }
    __threadfence();
  }
  named_sync(2, 128);
  if (f == 0) arrive(&S.dready);
  if (aw == 0) stamp(A, 4);
  aux_phase_d(A, S);
}

// ONE: the single-token specialisation (resident B operand, N = 8) -- a
// separate instantiation so each kernel carries one set of role loops (the
// code is one-shot per launch: its size is instruction-fetch latency)
template <int BITS, bool ONE>
__global__ void __launch_bounds__(kThreads, 1) tcd_kernel(const __grid_constant__ Args A) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ Shared S;
  const int tid = threadIdx.x, warp = tid >> 5;

  // ---------------- prologue (overlaps the previous kernel under PDL) ----
  if (tid == 0) {
    for (int i = 0; i < kMaxNST; ++i) {
      bar_init(&S.full[i], 1);
      bar_init(&S.bopf[i], 32);
      bar_init(&S.empty[i], kDec + kNEpi + 1);  // decode warps (codes), epilogue warps (meta, sums), MMA (B)
    }
    for (int i = 0; i < kNAS; ++i) {
      bar_init(&S.afull[i], kDec);
      bar_init(&S.aempty[i], 1);
    }
    for (int i = 0; i < kMaxNDS; ++i) bar_init(&S.dempty[i], kNEpi);
    for (int i = 0; i < kMaxNDS; ++i) bar_init(&S.dfull[i], 1);
    for (int i = 0; i < 2; ++i) {
      bar_init(&S.tfull[i], kNEpi);
      bar_init(&S.tempty[i], 4);
    }
    bar_init(&S.dready, 1);
    bar_init(&S.xrdy, 1);
    bar_init(&S.bimgf, 1);
    bar_init(&S.gbarr, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) umma::tmem_alloc<512>(&S.tmem_base);
  __syncthreads();
  const bool fused = A.gate32 != nullptr && !A.pairs_mode;
  if (fused && tid == 0) {  // gate rows -> shared memory (constant data)
    const uint32_t bytes = static_cast<uint32_t>(A.E) * A.hidden * 4;
    arrive_tx(&S.gbarr, bytes);
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    for (uint32_t o = 0; o < bytes; o += 32768)
      bulk_g2s(smem_u32(smem) + o, reinterpret_cast<const uint8_t*>(A.gate32) + o, min(32768u, bytes - o), &S.gbarr,
               pol);
  }
  fence_before();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (warp == 0) stamp(A, 0);

  // ---------------- routing + plan (all warps) ----------------------------
  if (tid == 0) {
    const unsigned long long gb = ld_acquire64(A.gbar);
    S.P.epoch = static_cast<int>(gb / gridDim.x);
    S.P.par = S.P.epoch & 1;
    S.P.fallback = 0;
    S.ring = smem;
    uint32_t dyn;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    S.tres = reinterpret_cast<float*>(smem + dyn - kTresBytes);
    S.eacc = reinterpret_cast<float*>(smem + dyn - kTresBytes - kEaccBytes);
  }
  for (int i = tid; i < kMaxE; i += kThreads) S.mark[i] = 0u;
  __syncthreads();
  {  // x digit images (phase-U B operand): (token, group) items spread over the grid's warps
    const int G0 = A.hidden / 64, n = A.B * G0, lane = tid & 31;
    for (int it = blockIdx.x * kWarps + warp; it < n; it += gridDim.x * kWarps) {
      const int t = it / G0, g = it % G0;
      const uint32_t v2 = __ldg(reinterpret_cast<const unsigned int*>(A.x + static_cast<size_t>(t) * A.hidden + g * 64) + lane);
      digit_image(BITS, bf2f(v2 & 0xffff), bf2f(v2 >> 16), A.xdig + static_cast<size_t>(it) * 512, A.xsum + it, lane);
      __threadfence();
      __syncwarp();
      if (lane == 0) atomicAdd(&A.xcnt[S.P.par], 1u);
    }
  }
  if (warp == 0) stamp(A, 13);
  if (fused) {
    wait(&S.gbarr, 0);
    if (warp == 0) stamp(A, 8);
    route_fused(A, S, reinterpret_cast<const float*>(smem));
    if (warp == 0) stamp(A, 9);
    if (S.P.fallback) route_fallback(A, S);
  }
  route_rest(A, S, fused);
  if (warp == 0) stamp(A, 11);
  if (warp == 0) {
    build_plan<BITS>(A, S);
    __syncwarp();
    stamp(A, 14);
    build_stages(A, S);
    stamp(A, 15);
  }
  __syncthreads();
  if (warp == 0) stamp(A, 1);

  if (warp == kProdWarp) {
    role_producer<BITS>(A, S);
  } else if (warp == kMmaWarp) {
    role_mma<ONE>(A, S, S.bop_off);
    stamp(A, 7);
  } else if (warp < kDec) {
    role_decode<BITS, ONE>(A, S);
  } else if (warp < kEpi0 + kNEpi) {
    role_epilogue<BITS, ONE>(A, S);
  } else {
    role_aux(A, S);
  }
  if (warp == 0) stamp(A, 5);
  fence_before();
  __syncthreads();
  if (warp == kMmaWarp) umma::tmem_dealloc<512>(S.tmem_base);
}

// ------------------------------------------------------------- packs ----
// One thread per (row, group, matrix): code bytes (2-bit: the reference row
// bytes; 3-bit: the byte-aligned repack above) + the {s, z} fp16 pair.
__global__ void build_pack_kernel(const lrc_qmat m0, const lrc_qmat m1, int nmat, int bits, uint8_t* out) {
  const int rows = m0.rows, cols = m0.cols, G = cols / 64;
  const int64_t n = static_cast<int64_t>(rows) * G * nmat;
  const int CB = bits == 2 ? 16 : 24, UB = 128 * CB + 512;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int mat = static_cast<int>(i % nmat);
    const int64_t rg = i / nmat;
    const int r = static_cast<int>(rg % rows), g = static_cast<int>(rg / rows);
    const lrc_qmat& m = mat == 0 ? m0 : m1;
    const int tile = r / 128, rl = r % 128;
    uint8_t* u = out + ((static_cast<int64_t>(tile) * G + g) * nmat + mat) * UB;
    const int64_t code0 = static_cast<int64_t>(r) * cols + 64 * g;
    if (bits == 2) {
      const uint4 v = *reinterpret_cast<const uint4*>(m.packed + code0 / 4);
      *reinterpret_cast<uint4*>(u + rl * 16) = v;
    } else {
      const int64_t nbytes = (static_cast<int64_t>(m.rows) * m.cols * 3 + 7) / 8;
      uint8_t c[64];
      for (int k = 0; k < 64; ++k) c[k] = static_cast<uint8_t>(read_code(m.packed, code0 + k, 3, nbytes));
      uint32_t w[6] = {0, 0, 0, 0, 0, 0};
      for (int wi = 0; wi < 6; ++wi)
        for (int b = 0; b < 4; ++b) {
          w[wi] |= static_cast<uint32_t>(c[8 * wi + b]) << (8 * b);
          w[wi] |= static_cast<uint32_t>(c[8 * wi + 4 + b]) << (8 * b + 3);
        }
      for (int s = 0; s < 2; ++s)
        for (int b = 0; b < 4; ++b) {
          const uint32_t X = c[48 + 8 * s + b], Y = c[48 + 8 * s + 4 + b];
          w[3 * s] |= (X & 3u) << (8 * b + 6);
          w[3 * s + 1] |= (Y & 3u) << (8 * b + 6);
          w[3 * s + 2] |= ((X >> 2) & 1u) << (8 * b + 6);
          w[3 * s + 2] |= ((Y >> 2) & 1u) << (8 * b + 7);
        }
      for (int wi = 0; wi < 6; ++wi) *reinterpret_cast<uint32_t*>(u + rl * 24 + 4 * wi) = w[wi];
    }
    const int gpr = (cols + m.group_size - 1) / m.group_size;
    const uint32_t s = m.scales[static_cast<int64_t>(r) * gpr + g], z = m.zeros[static_cast<int64_t>(r) * gpr + g];
    *reinterpret_cast<uint32_t*>(u + 128 * CB + rl * 4) = s | (z << 16);
  }
}

// LR packs.  Up tile: [U1 rows][U3 rows][V2^T rows] (128 x RB nibble bytes each),
// [U1 {s,z}][U3 {s,z}] per row, [V2 {s,z}] for the tile's 2 column groups x kRMax.
// Down tile: [U2 rows][U2 {s,z}].
__device__ __forceinline__ uint32_t qmeta(const lrc_qmat& m, int r, int g) {
  const int gpr = (m.cols + m.group_size - 1) / m.group_size;
  return static_cast<uint32_t>(m.scales[static_cast<int64_t>(r) * gpr + g]) |
         (static_cast<uint32_t>(m.zeros[static_cast<int64_t>(r) * gpr + g]) << 16);
}
__device__ __forceinline__ uint32_t qcode(const lrc_qmat& m, int r, int c) {
  const int64_t nbytes = (static_cast<int64_t>(m.rows) * m.cols * m.bits + 7) >> 3;
  return read_code(m.packed, static_cast<int64_t>(r) * m.cols + c, m.bits, nbytes);
}
__global__ void build_lr_up_kernel(const lrc_expert e, int ffn, uint8_t* out) {
  const int r = e.u1.cols, RB = lr_rb(r), TB = lr_up_tile_bytes(r);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // ffn row
  if (i >= ffn) return;
  const int tile = i / 128, f = i % 128;
  uint8_t* t = out + static_cast<int64_t>(tile) * TB;
  uint8_t nb[3][32];
  for (int k = 0; k < 32; ++k) nb[0][k] = nb[1][k] = nb[2][k] = 0;
  for (int k = 0; k < r; ++k) {
    const uint32_t c1 = qcode(e.u1, i, k), c3 = qcode(e.u3, i, k), c2 = qcode(e.v2, k, i);
    nb[0][k >> 1] |= static_cast<uint8_t>(c1 << (4 * (k & 1)));
    nb[1][k >> 1] |= static_cast<uint8_t>(c3 << (4 * (k & 1)));
    nb[2][k >> 1] |= static_cast<uint8_t>(c2 << (4 * (k & 1)));
  }
  for (int m = 0; m < 3; ++m)
    for (int b = 0; b < RB; ++b) t[(m * 128 + f) * RB + b] = nb[m][b];
  uint32_t* meta = reinterpret_cast<uint32_t*>(t + 3 * 128 * RB);
  meta[f] = qmeta(e.u1, i, 0);
  meta[128 + f] = qmeta(e.u3, i, 0);
  if (f < 2 * kRMax) {  // V2 {s,z}: column group cg of the tile, factor row k
    const int cg = f / kRMax, k = f % kRMax;
    meta[256 + f] = k < r ? qmeta(e.v2, k, (tile * 128) / 64 + cg) : 0u;
  }
}
__global__ void build_lr_down_kernel(const lrc_expert e, int hidden, uint8_t* out) {
  const int r = e.u2.cols, RB = lr_rb(r), TB = lr_down_tile_bytes(r);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // hidden row
  if (i >= hidden) return;
  const int tile = i / 128, f = i % 128;
  uint8_t* t = out + static_cast<int64_t>(tile) * TB;
  uint8_t nb[32];
  for (int k = 0; k < 32; ++k) nb[k] = 0;
  for (int k = 0; k < r; ++k) nb[k >> 1] |= static_cast<uint8_t>(qcode(e.u2, i, k) << (4 * (k & 1)));
  for (int b = 0; b < RB; ++b) t[f * RB + b] = nb[b];
  reinterpret_cast<uint32_t*>(t + 128 * RB)[f] = qmeta(e.u2, i, 0);
}
lrc_status build_lr_pack(const lrc_expert& e, int hidden, int ffn, uint8_t* up, uint8_t* down, cudaStream_t st) {
  build_lr_up_kernel<<<(ffn + 127) / 128, 128, 0, st>>>(e, ffn, up);
  LRC_CHECK_LAUNCH();
  build_lr_down_kernel<<<(hidden + 127) / 128, 128, 0, st>>>(e, hidden, down);
  LRC_CHECK_LAUNCH();
  return LRC_OK;
}

int64_t pack_bytes(int rows, int cols, int nmat, int bits) {
  const int CB = bits == 2 ? 16 : 24;
  return static_cast<int64_t>(rows / 128) * (cols / 64) * nmat * (128 * CB + 512);
}

lrc_status build_pack(const lrc_qmat* mats, int nmat, int bits, uint8_t* out, cudaStream_t st) {
  const lrc_qmat& m0 = mats[0];
  const int64_t n = static_cast<int64_t>(m0.rows) * (m0.cols / 64) * nmat;
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 32));
  build_pack_kernel<<<grid, 256, 0, st>>>(m0, nmat > 1 ? mats[1] : m0, nmat, bits, out);
  LRC_CHECK_LAUNCH();
  return LRC_OK;
}

static bool mat_ok(const lrc_qmat& m, int rows, int cols, int bits) {
  return m.packed && !m.dense && m.scales && m.zeros && m.rows == rows && m.cols == cols && m.bits == bits &&
         m.group_size == 64;
}

bool eligible(const lrc_expert* experts, int n, int hidden, int ffn, int* bits, int* fbits) {
  if (n <= 0 || hidden % 128 || ffn % 128) return false;
  const int b = experts[0].w1.bits;
  if (b != 2 && b != 3) return false;
  int fb = 0;
  for (int i = 0; i < n; ++i) {
    const lrc_expert& e = experts[i];
    if (!mat_ok(e.w1, ffn, hidden, b) || !mat_ok(e.w3, ffn, hidden, b) || !mat_ok(e.w2, hidden, ffn, b)) return false;
    const lrc_qmat* fs[6] = {&e.u1, &e.v1, &e.u3, &e.v3, &e.u2, &e.v2};
    const bool any = e.rank > 0;
    if (!any) continue;
    if (e.rank > kRMax) return false;
    for (auto f : fs) {
      if (!f->packed || f->dense || f->bits < 2 || f->bits > 4) return false;
      if (fb == 0) fb = f->bits;
      if (f->bits != fb) return false;
    }
    if (e.v1.group_size != 64 || e.v3.group_size != 64 || e.v1.cols != hidden || e.v3.cols != hidden) return false;
    if (e.u1.cols != e.rank || e.u3.cols != e.rank || e.u2.cols != e.rank || e.v2.rows != e.rank) return false;
    if (e.u1.group_size < e.rank || e.u3.group_size < e.rank || e.u2.group_size < e.rank) return false;
    if (e.v2.group_size != 64) return false;
  }
  *bits = b;
  *fbits = fb ? fb : 3;
  return true;
}

template <int BITS, bool ONE>
static lrc_status launch_t(const Args& a, int num_sms, cudaStream_t st, bool pdl) {
  static int smem = 0;
  if (smem == 0) {  // dynamic shared memory: everything the static state leaves
    cudaFuncAttributes fa{};
    LRC_CUDA_TRY(cudaFuncGetAttributes(&fa, tcd_kernel<BITS, ONE>));
    int dev = 0, optin = 0;
    LRC_CUDA_TRY(cudaGetDevice(&dev));
    LRC_CUDA_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    smem = (optin - static_cast<int>(fa.sharedSizeBytes) - 1024) & ~1023;
    LRC_CUDA_TRY(cudaFuncSetAttribute(tcd_kernel<BITS, ONE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(num_sms);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  LRC_CUDA_TRY(cudaLaunchKernelEx(&cfg, tcd_kernel<BITS, ONE>, a));
  return LRC_OK;
}

lrc_status launch(const Args& a, int num_sms, cudaStream_t st, bool pdl) {
  if (a.B < 1 || a.B > kMaxTok) return fail(LRC_ERR_UNSUPPORTED, "tcd: 1..8 tokens");
  // (the resident-B single-token layout is chosen on the device from A.B == 1)
  if (a.B == 1) return a.bits == 2 ? launch_t<2, true>(a, num_sms, st, pdl) : launch_t<3, true>(a, num_sms, st, pdl);
  return a.bits == 2 ? launch_t<2, false>(a, num_sms, st, pdl) : launch_t<3, false>(a, num_sms, st, pdl);
}

void set_wait_mode(int) {}
void wstat_copy(unsigned long long* host) {
  cudaMemcpyFromSymbol(host, g_wstat, sizeof(g_wstat));
  void* dev = nullptr;
  cudaGetSymbolAddress(&dev, g_wstat);
  cudaMemset(dev, 0, sizeof(g_wstat));
}
void trace_copy(uint64_t* host) {
  cudaMemcpyFromSymbol(host, g_trace, sizeof(g_trace));
  cudaMemcpyFromSymbol(host + 1024, g_trace2, sizeof(g_trace2));
  void* dev = nullptr;
  cudaGetSymbolAddress(&dev, g_trace);
  cudaMemset(dev, 0, sizeof(g_trace));
  cudaGetSymbolAddress(&dev, g_trace2);
  cudaMemset(dev, 0, sizeof(g_trace2));
}
void stamps_copy(uint64_t* host, int n) {
  cudaMemcpyFromSymbol(host, g_stamps, sizeof(uint64_t) * n);
  void* dev = nullptr;
  cudaGetSymbolAddress(&dev, g_stamps);
  cudaMemset(dev, 0, sizeof(g_stamps));
}

}  // namespace tcd
}  // namespace lrc
