// Compress: quantize_shard + lane encoding, written straight into the
// per-worker communication buffer.
//
//   reference: quantizer.cpp:8-48 (quantize_shard), levels.cpp:63-84
//              (bracket_index / random_round), rng.hpp:45-61 (dither
//              u01(Dither, worker, round, j)), algorithm.cpp:69-82
//              (encode_dense_std: lane = sign * (s - idx)),
//              exp_arith.cpp:126-160 (tokens_from_shard + pack_tokens:
//              lane = (idx + shift) | sign bit, idx == s -> 0).
//
// Bit-exactness strategy. The reference decides each element with IEEE f64
// arithmetic: y = |x|/norm, bracket by comparison with the level table,
// p = (y - lo)/(hi - lo), round up iff u < p. Two correctly rounded f64
// divisions per element would make this kernel FP64-bound, so each element
// first takes an f32 FAST PATH that computes an approximation of the
// fractional position f ~ p with a proven error bound M:
//   standard    t = |x| * fl32(s/norm), f = t - floor(t), |f - p| < M
//               with M = (s+1) 2^-21 (f32 product error s*2^-23 dominates)
//   exponential y = |x| * fl32(1/norm), bracket from the f32 exponent,
//               f = mantissa fraction (or y 2^(s-1) in the last bracket),
//               |f - p| < M = 2^-20
// and a 23-bit truncation uf <= u < uf + 2^-23 of the dither. The element
// rounds up iff uf + M + 2^-23 <= f, down iff uf >= f + M, and any element
// within M of a bracket edge or of the decision boundary (probability
// ~4M, <1e-4) falls to the SLOW PATH, which replays the reference's f64
// sequence literally (__ddiv_rn / __dsub_rn, exact level values), so every
// decision equals the reference's.
//
// Memory: thread-per-quad (4 elements) with 128-bit streaming loads; each
// quad emits 4 lanes (2/4/8/16 bytes for w = 4/8/16/32) with one coalesced
// store. HBM bytes per element: 4 (f32 in) + w/8 (lanes out).
#include <cuda_runtime.h>

#include "gq_common.cuh"
#include "gq_internal.h"

namespace gqb {

namespace {

constexpr int kQThreads = 256;
constexpr int kQUnroll = 4;

struct QuantArgs {
  const void* x[kMaxWorkers];
  void* lanes[kMaxWorkers];
  uint64_t h4[kMaxWorkers];
  uint64_t d;
  const double* norm;
  uint32_t* err;
  uint32_t s;
  uint32_t shift;
};

// Per-block constants derived from the device-resident norm.
struct QConst {
  double norm;
  float c;        // std: fl32(s / norm); exp: fl32(1 / norm)
  float thr;      // largest f32 <= norm: |x| > norm  <=>  |x| > thr (f32 |x|)
  float m_lo;     // M
  float m_up;     // M + 2^-23
  float one_m;    // 1 - M
  float pow_s1;   // exp: 2^(s-1)
  bool fast;      // fast path usable
};

template <int KIND>
__device__ __forceinline__ QConst make_const(double norm, uint32_t s) {
  QConst k;
  k.norm = norm;
  k.thr = __double2float_rd(norm);
  if (KIND == 0) {
    const double c = __ddiv_rn(static_cast<double>(s), norm);
    k.c = __double2float_rn(c);
    const float M = static_cast<float>(s + 1) * 0x1.0p-21f;
    k.m_lo = M;
    k.m_up = M + 0x1.0p-23f;
    k.one_m = 1.0f - M;
    k.pow_s1 = 0.0f;
    k.fast = (s <= 4096) && isfinite(k.c) && k.c >= 0x1.0p-100f && k.c <= 0x1.0p100f;
  } else {
    const double c = __drcp_rn(norm);
    k.c = __double2float_rn(c);
    k.m_lo = 0x1.0p-20f;
    k.m_up = 0x1.0p-20f + 0x1.0p-23f;
    k.one_m = 1.0f - 0x1.0p-20f;
    k.pow_s1 = (s >= 1 && s <= 120) ? __uint_as_float((126u + s) << 23) : 0.0f;  // 2^(s-1)
    k.fast = (s <= 120) && isfinite(k.c) && k.c >= 0x1.0p-100f && k.c <= 0x1.0p100f;
  }
  return k;
}

// Exact level value (levels.cpp:31-48).
template <int KIND>
__device__ __forceinline__ double level_of(uint32_t i, uint32_t s) {
  if (KIND == 0) return __ddiv_rn(static_cast<double>(s - i), static_cast<double>(s));
  return i < s ? ldexp(1.0, -static_cast<int>(i)) : 0.0;
}

// The reference's f64 decision, literally (levels.cpp:63-84 with
// quantizer.cpp:38-44). Returns the level index.
template <int KIND>
__device__ __noinline__ uint32_t slow_index(double ad, double norm, uint64_t bits,
                                            uint32_t s) {
  double y = __ddiv_rn(ad, norm);
  if (y > 1.0) y = 1.0;  // already flagged as EXCEEDS_SCALE; keep going
  int64_t g;
  if (KIND == 0) {
    g = static_cast<int64_t>(s) - 1 - static_cast<int64_t>(floor(__dmul_rn(y, static_cast<double>(s))));
  } else {
    if (y == 0.0) {
      g = static_cast<int64_t>(s) - 1;
    } else {
      int e;
      const double m = frexp(y, &e);  // y = m 2^e, m in [0.5, 1)
      g = (m == 0.5) ? -(e - 1) : -e;  // y == 2^(e-1) sits at level e-1... -(e-1)
    }
  }
  if (g < 0) g = 0;
  if (g > static_cast<int64_t>(s) - 1) g = static_cast<int64_t>(s) - 1;
  uint32_t i = static_cast<uint32_t>(g);
  // bracket_index: largest i <= s-1 with level(i) >= y.
  while (i > 0 && level_of<KIND>(i, s) < y) --i;
  while (i + 1 < s && level_of<KIND>(i + 1, s) >= y) ++i;
  const double hi = level_of<KIND>(i, s);
  const double lo = level_of<KIND>(i + 1, s);
  const double p_hi = __ddiv_rn(__dsub_rn(y, lo), __dsub_rn(hi, lo));
  return (u01_from_bits(bits) < p_hi) ? i : i + 1;
}

// One element -> its lane code (std: signed level count; exp: packed token).
template <int KIND, typename T>
__device__ __forceinline__ int32_t quant_elem(T v, uint64_t h4, uint64_t j,
                                              const QConst& K, uint32_t s,
                                              uint32_t shift, uint32_t sign_bit,
                                              uint32_t& flags) {
  float a;
  bool neg, zero;
  if constexpr (sizeof(T) == 4) {
    const uint32_t ab = __float_as_uint(v) & 0x7fffffffu;
    a = __uint_as_float(ab);
    neg = (__float_as_uint(v) >> 31) != 0;
    zero = ab == 0;
    if (ab >= 0x7f800000u) flags |= GQ_FLAG_NONFINITE;
    if (a > K.thr) flags |= GQ_FLAG_EXCEEDS_SCALE;
  } else {
    const double ad = fabs(static_cast<double>(v));
    a = __double2float_rn(ad);
    neg = signbit(static_cast<double>(v)) != 0;
    zero = ad == 0.0;
    if (!isfinite(ad)) flags |= GQ_FLAG_NONFINITE;
    if (ad > K.norm) flags |= GQ_FLAG_EXCEEDS_SCALE;
  }
  if (zero) return 0;  // y = 0: bracket s-1, p = 0 -> idx = s (lane 0)

  const uint64_t bits = mix64(h4 ^ j);
  const float uf = __uint_as_float(0x3f800000u | (static_cast<uint32_t>(bits >> 32) >> 9)) - 1.0f;

  int32_t idx_or_mag;
  bool slow;
  if constexpr (KIND == 0) {
    const float t = a * K.c;
    const float tm = __fadd_rd(t, 8388608.0f);
    const int fl = __float_as_int(tm) - 0x4b000000;
    const float f = t - (tm - 8388608.0f);
    const bool up = (uf + K.m_up) <= f;
    const bool down = uf >= (f + K.m_lo);
    slow = !K.fast || (f < K.m_lo) || (f > K.one_m) || !(up || down);
    idx_or_mag = fl + (up ? 1 : 0);  // magnitude s - idx
  } else {
    const float y = a * K.c;
    const uint32_t yb = __float_as_uint(y);
    int i = 126 - static_cast<int>(yb >> 23);  // -E - 1
    float f;
    if (i >= static_cast<int>(s) - 1) {
      i = static_cast<int>(s) - 1;
      f = y * K.pow_s1;
    } else {
      f = __uint_as_float((yb & 0x7fffffu) | 0x3f800000u) - 1.0f;
    }
    const bool up = (uf + K.m_up) <= f;
    const bool down = uf >= (f + K.m_lo);
    slow = !K.fast || (i < 0) || (f < K.m_lo) || (f > K.one_m) || !(up || down);
    idx_or_mag = i + (up ? 0 : 1);  // level index
  }
  if (slow) {
    double ad;
    if constexpr (sizeof(T) == 4) ad = static_cast<double>(a);
    else ad = fabs(static_cast<double>(v));
    const uint32_t idx = slow_index<KIND>(ad, K.norm, bits, s);
    idx_or_mag = KIND == 0 ? static_cast<int32_t>(s - idx) : static_cast<int32_t>(idx);
  }
  if constexpr (KIND == 0) {
    return neg ? -idx_or_mag : idx_or_mag;
  } else {
    const uint32_t idx = static_cast<uint32_t>(idx_or_mag);
    if (idx >= s) return 0;
    return static_cast<int32_t>((idx + shift) | (neg ? sign_bit : 0u));
  }
}

template <int W>
__device__ __forceinline__ void store_quad(void* lanes, uint64_t q, const int32_t (&c)[4]) {
  if constexpr (W == 4) {
    const uint32_t v = (c[0] & 0xf) | ((c[1] & 0xf) << 4) | ((c[2] & 0xf) << 8) | ((c[3] & 0xf) << 12);
    reinterpret_cast<uint16_t*>(lanes)[q] = static_cast<uint16_t>(v);
  } else if constexpr (W == 8) {
    const uint32_t v = (c[0] & 0xff) | ((c[1] & 0xff) << 8) | ((c[2] & 0xff) << 16) |
                       (static_cast<uint32_t>(c[3]) << 24);
    reinterpret_cast<uint32_t*>(lanes)[q] = v;
  } else if constexpr (W == 16) {
    uint2 v;
    v.x = (c[0] & 0xffff) | (static_cast<uint32_t>(c[1]) << 16);
    v.y = (c[2] & 0xffff) | (static_cast<uint32_t>(c[3]) << 16);
    reinterpret_cast<uint2*>(lanes)[q] = v;
  } else {
    uint4 v;
    v.x = c[0]; v.y = c[1]; v.z = c[2]; v.w = c[3];
    reinterpret_cast<uint4*>(lanes)[q] = v;
  }
}

template <typename T>
__device__ __forceinline__ void load_quad(const T* x, uint64_t q, T (&v)[4]) {
  if constexpr (sizeof(T) == 4) {
    const float4 f = __ldcs(reinterpret_cast<const float4*>(x) + q);
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
  } else {
    const double2 a = __ldcs(reinterpret_cast<const double2*>(x) + 2 * q);
    const double2 b = __ldcs(reinterpret_cast<const double2*>(x) + 2 * q + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
}

template <typename T, int KIND, int W>
__global__ void __launch_bounds__(kQThreads)
quantize_kernel(const __grid_constant__ QuantArgs args) {
  const uint32_t r = blockIdx.y;
  const T* x = static_cast<const T*>(args.x[r]);
  void* lanes = args.lanes[r];
  const uint64_t h4 = args.h4[r];
  const uint64_t d = args.d;
  const uint32_t s = args.s;
  const uint32_t shift = args.shift;
  const uint32_t sign_bit = 1u << (W - 1);
  const double norm = *args.norm;
  uint32_t flags = 0;

  const uint64_t nquad = d / 4;
  if (!(norm >= 0.0) || !isfinite(norm)) {
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) raise_flag(args.err, GQ_FLAG_BAD_SCALE);
    return;
  }
  if (norm == 0.0) {
    // quantizer.cpp:21-32: every element must be zero; all idx = s (lane 0).
    for (uint64_t q = blockIdx.x * kQThreads + threadIdx.x; q < nquad; q += gridDim.x * kQThreads) {
      T v[4];
      load_quad<T>(x, q, v);
#pragma unroll
      for (int e = 0; e < 4; ++e) if (v[e] != T(0)) flags |= GQ_FLAG_ZERO_SCALE;
      const int32_t c[4] = {0, 0, 0, 0};
      store_quad<W>(lanes, q, c);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      for (uint64_t j = nquad * 4; j < d; ++j) if (x[j] != T(0)) flags |= GQ_FLAG_ZERO_SCALE;
      uint8_t* lb = static_cast<uint8_t*>(lanes);
      const uint64_t b0 = nquad * 4 * W / 8, b1 = (d * W + 7) / 8;
      for (uint64_t b = b0; b < b1; ++b) lb[b] = 0;
    }
    raise_flags_warp(args.err, flags);
    return;
  }

  const QConst K = make_const<KIND>(norm, s);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kQThreads * kQUnroll;
  for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * kQThreads * kQUnroll + threadIdx.x;
       base < nquad; base += stride) {
    T v[kQUnroll][4];
#pragma unroll
    for (int u = 0; u < kQUnroll; ++u) {
      const uint64_t q = base + u * kQThreads;
      if (q < nquad) load_quad<T>(x, q, v[u]);
    }
#pragma unroll
    for (int u = 0; u < kQUnroll; ++u) {
      const uint64_t q = base + u * kQThreads;
      if (q < nquad) {
        int32_t c[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
          c[e] = quant_elem<KIND, T>(v[u][e], h4, 4 * q + e, K, s, shift, sign_bit, flags);
        store_quad<W>(lanes, q, c);
      }
    }
  }
  // Tail (d % 4 elements): one thread writes whole bytes, zero-padded.
  if (blockIdx.x == 0 && threadIdx.x == 0 && nquad * 4 < d) {
    int32_t c[4] = {0, 0, 0, 0};
    for (uint64_t j = nquad * 4; j < d; ++j)
      c[j - nquad * 4] = quant_elem<KIND, T>(x[j], h4, j, K, s, shift, sign_bit, flags);
    uint8_t* lb = static_cast<uint8_t*>(lanes);
    const uint64_t b0 = nquad * 4 * W / 8;
    const uint64_t nb = ((d - nquad * 4) * W + 7) / 8;
    uint64_t packed[2] = {0, 0};
    for (int e = 0; e < 4; ++e) {
      const uint64_t mask = (W == 64) ? ~0ull : ((1ull << W) - 1);
      const uint64_t bitpos = static_cast<uint64_t>(e) * W;
      const uint64_t val = static_cast<uint64_t>(static_cast<uint32_t>(c[e])) & mask;
      packed[bitpos / 64] |= val << (bitpos % 64);
    }
    for (uint64_t b = 0; b < nb; ++b) lb[b0 + b] = static_cast<uint8_t>(packed[b / 8] >> (8 * (b % 8)));
  }
  raise_flags_warp(args.err, flags);
}

template <typename T, int KIND>
cudaError_t launch_w(const QuantArgs& a, dim3 grid, uint32_t width, cudaStream_t st) {
  switch (width) {
    case 4: quantize_kernel<T, KIND, 4><<<grid, kQThreads, 0, st>>>(a); break;
    case 8: quantize_kernel<T, KIND, 8><<<grid, kQThreads, 0, st>>>(a); break;
    case 16: quantize_kernel<T, KIND, 16><<<grid, kQThreads, 0, st>>>(a); break;
    case 32: quantize_kernel<T, KIND, 32><<<grid, kQThreads, 0, st>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_quantize(const QuantLaunch& q, cudaStream_t stream) {
  QuantArgs a{};
  for (uint32_t i = 0; i < q.n_local; ++i) {
    a.x[i] = q.shards[i];
    a.lanes[i] = q.lanes[i];
    // RngStream::Dither = 1 (rng.hpp:31-37); keys (worker, round, j).
    a.h4[i] = hoist_prefix(q.seed, 1ull, q.worker_ids[i], q.round);
  }
  a.d = q.d;
  a.norm = q.norm;
  a.err = q.err;
  a.s = q.s;
  uint32_t shift = 0;
  for (uint64_t p = 1; p < 2ull * q.n_total; p <<= 1) ++shift;  // prescale_shift
  a.shift = shift;
  const uint64_t nquad = q.d / 4;
  const uint64_t per_block = static_cast<uint64_t>(kQThreads) * kQUnroll;
  uint64_t bx = (nquad + per_block - 1) / per_block;
  const uint64_t cap = (148ull * 8 * 2 + q.n_local - 1) / q.n_local;
  if (bx > cap) bx = cap;
  if (bx == 0) bx = 1;
  const dim3 grid(static_cast<uint32_t>(bx), q.n_local);
  if (q.dtype == GQ_DTYPE_F32) {
    return q.kind == 0 ? launch_w<float, 0>(a, grid, q.width, stream)
                       : launch_w<float, 1>(a, grid, q.width, stream);
  }
  return q.kind == 0 ? launch_w<double, 0>(a, grid, q.width, stream)
                     : launch_w<double, 1>(a, grid, q.width, stream);
}

}  // namespace gqb
