// Quantizer-side kernels: bit packing (K6), fp64 dequantize, fp64 quantize
// with half-quadratic zero refinement.  Reference: ref/quant.py.
#include <math.h>

#include "common.cuh"

namespace lrc {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
lrc_status fail(lrc_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

// ---------------------------------------------------------------- packing --
// One thread per output byte; byte j holds stream bits [8j, 8j+8).
__global__ void pack_kernel(const uint8_t* __restrict__ codes, int64_t count, int bits,
                            uint8_t* __restrict__ out, int64_t nbytes) {
  int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (j >= nbytes) return;
  uint32_t b = 0;
  int64_t bit0 = j * 8;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    int64_t bit = bit0 + t;
    int64_t i = bit / bits;
    if (i < count) b |= ((static_cast<uint32_t>(codes[i]) >> (bit - i * bits)) & 1u) << t;
  }
  out[j] = static_cast<uint8_t>(b);
}

__global__ void unpack_kernel(const uint8_t* __restrict__ packed, int64_t count, int bits,
                              uint8_t* __restrict__ out, int64_t nbytes) {
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= count) return;
  out[i] = static_cast<uint8_t>(read_code(packed, i, bits, nbytes));
}

// ------------------------------------------------------------- dequantize --
// ref/quant.py:216-224: deq = code * scale + zero evaluated as two separately
// rounded fp64 ops (numpy does not fuse), hence __dmul_rn / __dadd_rn.
__global__ void dequant_f64_kernel(const uint8_t* __restrict__ codes,
                                   const double* __restrict__ scales,
                                   const double* __restrict__ zeros, int64_t rows, int64_t cols,
                                   int gs, double* __restrict__ out) {
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= rows * cols) return;
  int64_t r = i / cols, c = i - r * cols;
  int64_t gpr = (cols + gs - 1) / gs;
  int64_t g = r * gpr + c / gs;
  out[i] = __dadd_rn(__dmul_rn(static_cast<double>(codes[i]), scales[g]), zeros[g]);
}

// ---------------------------------------------------------------- quantize --
// numpy's float64 add-reduce over a contiguous axis of n elements is
// 0 + pairwise_sum(n) with 8-way unrolled blocks of <= 128
// (numpy/_core/src/umath/loops_utils.h.src); replicated so nanmean matches.
template <typename F>
__device__ double np_pairwise(F v, int lo, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, v(lo + i));
    return r;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = v(lo + j);
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], v(lo + i + j));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, v(lo + i));
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise(v, lo, n2), np_pairwise(v, lo + n2, n - n2));
}

template <typename F>
__device__ __forceinline__ double np_sum(F v, int n) {
  return __dadd_rn(0.0, np_pairwise(v, 0, n));
}

__device__ __forceinline__ double round_half_away(double x) {
  return copysign(floor(__dadd_rn(fabs(x), 0.5)), x);
}

__device__ __forceinline__ double code_of(double w, double z, double s, double qmax) {
  double q = round_half_away(__ddiv_rn(__dsub_rn(w, z), s));
  return fmin(fmax(q, 0.0), qmax);
}

// One thread per (row, group).  ref/quant.py:146-213.
__global__ void quantize_f64_kernel(const double* __restrict__ w, int64_t rows, int64_t cols,
                                    int bits, int gs, int iters, double p,
                                    uint8_t* __restrict__ codes, double* __restrict__ scales,
                                    double* __restrict__ zeros) {
  int64_t gpr = (cols + gs - 1) / gs;
  int64_t tg = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (tg >= rows * gpr) return;
  int64_t r = tg / gpr, g = tg - r * gpr;
  const double* wr = w + r * cols + g * gs;
  int nv = static_cast<int>(gs < cols - g * gs ? (int64_t)gs : cols - g * gs);  // valid (non-NaN-pad) count
  const double qmax = static_cast<double>((1 << bits) - 1);

  double lo = wr[0], hi = wr[0];
  for (int j = 1; j < nv; ++j) {
    lo = fmin(lo, wr[j]);
    hi = fmax(hi, wr[j]);
  }
  const double s = (hi == lo) ? 1.0 : __ddiv_rn(__dsub_rn(hi, lo), qmax);
  double z = lo;

  if (iters > 0) {
    // objective: nanmean |w - (q*s + z)|^p with q from zero point zq
    auto objective = [&](double zq) {
      auto term = [&](int j) -> double {
        if (j >= nv) return 0.0;
        double q = code_of(wr[j], zq, s, qmax);
        return pow(fabs(__dsub_rn(wr[j], __dadd_rn(__dmul_rn(q, s), zq))), p);
      };
      return __ddiv_rn(np_sum(term, gs), static_cast<double>(nv));
    };
    double best = objective(z);
    double zbest = z;
    double beta = 10.0;
    for (int it = 0; it < iters; ++it) {
      const double zq = z;
      const double inv_beta = __ddiv_rn(1.0, beta);
      // err = shrink_lp(nan_to_num(w - deq)), zeros = nanmean(w - err - q*s)
      auto term = [&](int j) -> double {
        if (j >= nv) return 0.0;
        double q = code_of(wr[j], zq, s, qmax);
        double qs = __dmul_rn(q, s);
        double resid = __dsub_rn(wr[j], __dadd_rn(qs, zq));
        double a = fabs(resid);
        double thr = (p == 1.0) ? inv_beta : __dmul_rn(inv_beta, pow(a, p - 1.0));
        double sg = (resid > 0.0) ? 1.0 : ((resid < 0.0) ? -1.0 : 0.0);
        double err = __dmul_rn(sg, fmax(__dsub_rn(a, thr), 0.0));
        return __dsub_rn(__dsub_rn(wr[j], err), qs);
      };
      z = __ddiv_rn(np_sum(term, gs), static_cast<double>(nv));
      double obj = objective(z);
      if (obj < best) {
        best = obj;
        zbest = z;
      }
      beta = __dmul_rn(beta, 1.01);
    }
    z = zbest;
  }
  uint8_t* cr = codes + r * cols + g * gs;
  for (int j = 0; j < nv; ++j) cr[j] = static_cast<uint8_t>(code_of(wr[j], z, s, qmax));
  scales[tg] = s;
  zeros[tg] = z;
}

__global__ void add_lowrank_f64_kernel(const double* __restrict__ u, const double* __restrict__ v,
                                       int64_t m, int64_t n, int r, double* __restrict__ out) {
  int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= m * n) return;
  int64_t row = i / n, col = i - row * n;
  double acc = 0.0;
  for (int t = 0; t < r; ++t) acc = fma(u[row * r + t], v[t * n + col], acc);
  out[i] = __dadd_rn(out[i], acc);
}

static inline unsigned nblocks(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace lrc

using namespace lrc;

extern "C" int lrc_abi_version(void) { return LRC_ABI_VERSION; }
extern "C" const char* lrc_last_error(void) { return g_last_error.c_str(); }

extern "C" lrc_status lrc_pack_codes(const uint8_t* codes, int64_t count, int bits,
                                     uint8_t* packed, void* stream) {
  if (bits < 1 || bits > 8 || count < 0) return fail(LRC_ERR_INVALID, "pack_codes: bad bits/count");
  int64_t nbytes = (count * bits + 7) / 8;
  if (nbytes == 0) return LRC_OK;
  pack_kernel<<<nblocks(nbytes, 256), 256, 0, as_stream(stream)>>>(codes, count, bits, packed, nbytes);
  LRC_CHECK_LAUNCH();
  return LRC_OK;
}

extern "C" lrc_status lrc_unpack_codes(const uint8_t* packed, int64_t count, int bits,
                                       uint8_t* codes, void* stream) {
  if (bits < 1 || bits > 8 || count < 0) return fail(LRC_ERR_INVALID, "unpack_codes: bad bits/count");
  if (count == 0) return LRC_OK;
  int64_t nbytes = (count * bits + 7) / 8;
  unpack_kernel<<<nblocks(count, 256), 256, 0, as_stream(stream)>>>(packed, count, bits, codes, nbytes);
  LRC_CHECK_LAUNCH();
  return LRC_OK;
}

extern "C" lrc_status lrc_dequantize_f64(const uint8_t* codes, const double* scales,
                                         const double* zeros, int64_t rows, int64_t cols,
                                         int group_size, double* out, void* stream) {
  if (rows <= 0 || cols <= 0 || group_size < 1) return fail(LRC_ERR_INVALID, "dequantize: bad shape");
  dequant_f64_kernel<<<nblocks(rows * cols, 256), 256, 0, as_stream(stream)>>>(
      codes, scales, zeros, rows, cols, group_size, out);
  LRC_CHECK_LAUNCH();
  return LRC_OK;
}

extern "C" lrc_status lrc_quantize_f64(const double* w, int64_t rows, int64_t cols, int bits,
                                       int group_size, int hqq_iters, double shrink_p,
                                       uint8_t* codes, double* scales, double* zeros,
                                       void* stream) {
  if (rows <= 0 || cols <= 0) return fail(LRC_ERR_INVALID, "quantize: empty matrix");
  if (bits < 2 || bits > 4) return fail(LRC_ERR_INVALID, "quantize: bits must be 2, 3 or 4");
  if (group_size < 1 || hqq_iters < 0 || !(shrink_p > 0.0 && shrink_p <= 1.0))
    return fail(LRC_ERR_INVALID, "quantize: bad config");
  int64_t groups = rows * ((cols + group_size - 1) / group_size);
  quantize_f64_kernel<<<nblocks(groups, 128), 128, 0, as_stream(stream)>>>(
      w, rows, cols, bits, group_size, hqq_iters, shrink_p, codes, scales, zeros);
  LRC_CHECK_LAUNCH();
  return LRC_OK;
}

extern "C" lrc_status lrc_add_lowrank_f64(const double* u, const double* v, int64_t m, int64_t n,
                                          int r, double* out, void* stream) {
  if (m <= 0 || n <= 0 || r < 0) return fail(LRC_ERR_INVALID, "add_lowrank: bad shape");
  if (r == 0) return LRC_OK;
  add_lowrank_f64_kernel<<<nblocks(m * n, 256), 256, 0, as_stream(stream)>>>(u, v, m, n, r, out);
  LRC_CHECK_LAUNCH();
  return LRC_OK;
}
