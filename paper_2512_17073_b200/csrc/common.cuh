// Shared helpers for the lrc CUDA library (sm_100a).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/lrc.h"

namespace lrc {

// ---- error plumbing --------------------------------------------------------
void set_error(const std::string& msg);
lrc_status fail(lrc_status st, const std::string& msg);

#define LRC_CUDA_TRY(expr)                                                          \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess)                                                          \
      return ::lrc::fail(LRC_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define LRC_CHECK_LAUNCH()                                                          \
  do {                                                                              \
    cudaError_t _e = cudaGetLastError();                                            \
    if (_e != cudaSuccess)                                                          \
      return ::lrc::fail(LRC_ERR_CUDA, std::string("launch: ") + cudaGetErrorString(_e)); \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kWarp = 32;

// ---- fp16 metadata ---------------------------------------------------------
__device__ __forceinline__ float h2f(uint16_t h) {
  return __half2float(__ushort_as_half(h));
}

__device__ __forceinline__ float bf2f(uint16_t b) {
  return __uint_as_float(static_cast<uint32_t>(b) << 16);
}

// round-to-nearest-even fp32 -> bf16 bits
__device__ __forceinline__ uint16_t f2bf(float f) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

// ---- reference bitstream (ref/quant.py:243-262): code i at bits [i*b, i*b+b) --
// `nbytes` bounds the read so the last code never touches memory past the buffer.
__device__ __forceinline__ uint32_t read_code(const uint8_t* __restrict__ p, int64_t i, int bits,
                                              int64_t nbytes) {
  int64_t bit = i * bits;
  int64_t byte = bit >> 3;
  uint32_t v = p[byte];
  if (byte + 1 < nbytes) v |= static_cast<uint32_t>(p[byte + 1]) << 8;
  return (v >> (bit & 7)) & ((1u << bits) - 1u);
}

// Dequantized element of an lrc_qmat (fp32): code*scale + zero, or dense value.
__device__ __forceinline__ float qmat_elem(const lrc_qmat& m, int64_t r, int64_t c) {
  if (m.dense) return m.dense[r * m.cols + c];
  int64_t nbytes = (static_cast<int64_t>(m.rows) * m.cols * m.bits + 7) >> 3;
  uint32_t code = read_code(m.packed, r * m.cols + c, m.bits, nbytes);
  int gpr = (m.cols + m.group_size - 1) / m.group_size;
  int64_t g = r * gpr + c / m.group_size;
  return fmaf(static_cast<float>(code), h2f(m.scales[g]), h2f(m.zeros[g]));
}

__device__ __forceinline__ bool qmat_present(const lrc_qmat& m) {
  return m.dense != nullptr || m.packed != nullptr;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float silu_f(float v) { return v / (1.0f + __expf(-v)); }

}  // namespace lrc
