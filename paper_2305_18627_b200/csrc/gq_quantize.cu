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

#ifndef GQ_QUNROLL
#define GQ_QUNROLL 4
#endif
#ifndef GQ_QMINBLOCKS
#define GQ_QMINBLOCKS 1
#endif
constexpr int kQThreads = 256;
constexpr int kQUnroll = GQ_QUNROLL;
constexpr int kChunkQ = kQThreads * kQUnroll;  // quads per staged chunk (16 KiB of f32)
template <typename T>
struct QStages {
  static constexpr int value = sizeof(T) == 4 ? 4 : 3;  // 64 KiB (f32) / 96 KiB (f64) per block
};
template <typename T>
constexpr size_t qsmem_bytes() {
  return QStages<T>::value * (kChunkQ * 4 * sizeof(T)) + QStages<T>::value * sizeof(uint64_t);
}

struct QuantArgs {
  const void* x[kMaxWorkers];
  void* lanes[kMaxWorkers];
  uint64_t h4[kMaxWorkers];
  uint64_t d;
  const double* norm;
  uint32_t* err;
  uint32_t s;
  uint32_t shift;
  uint32_t n_local;
  MulConsts mk;
};

// Per-block constants derived from the device-resident norm.
struct QConst {
  double norm;
  float c;        // std: fl32(s / norm); exp: fl32(1 / norm)
  float half_m;   // 0.5 - M: slow iff |frac - 1/2| > 0.5 - M
  bool fast;      // fast path usable
};

template <int KIND>
__device__ __forceinline__ QConst make_const(double norm, uint32_t s) {
  QConst k;
  k.norm = norm;
  if (KIND == 0) {
    // error budget: t (2 roundings) s 2^-23, dither truncation 2^-23, z rounding
    // (s+1) 2^-24  ->  < (s+1) 1.5 2^-23;  M = (s+1) 2^-21 leaves 2.6x slack
    k.c = __double2float_rn(__ddiv_rn(static_cast<double>(s), norm));
    k.half_m = 0.5f - static_cast<float>(s + 1) * 0x1.0p-21f;
    k.fast = (s <= 4096) && isfinite(k.c) && k.c >= 0x1.0p-100f && k.c <= 0x1.0p100f;
  } else {
    // error budget: f (2 roundings of ys, +1 rounding) 2^-22 + 2^-24, dither
    // truncation 2^-23  ->  < 2^-21;  M = 2^-20
    k.c = (s <= 120) ? __double2float_rn(__ddiv_rn(ldexp(1.0, static_cast<int>(s) - 1), norm)) : 0.0f;
    k.half_m = 0.5f - 0x1.0p-20f;
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

// Absolute-value bit patterns; their running max gives both error checks
// (NaN/Inf: bits >= Inf pattern; |x| > norm: max magnitude > norm) with one
// integer max per element instead of per-element compares.
template <typename T>
struct Abs;
template <>
struct Abs<float> {
  using U = uint32_t;
  __device__ static U bits(float v) { return __float_as_uint(v) & 0x7fffffffu; }
  __device__ static float mag(U b) { return __uint_as_float(b); }
  __device__ static bool neg(float v) { return (__float_as_uint(v) >> 31) != 0; }
  __device__ static uint32_t hibits(float v) { return __float_as_uint(v); }
  __device__ static double dbl(U b) { return static_cast<double>(__uint_as_float(b)); }
  __device__ static bool nonfinite(U b) { return b >= 0x7f800000u; }
  // max of magnitudes that keeps NaN (max.NaN.f32 on the bit patterns of
  // non-negative floats; one FMNMX.NAN instead of an integer compare + select)
  __device__ static U vmax(U m, U b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(__uint_as_float(m)), "f"(__uint_as_float(b)));
    return __float_as_uint(r);
  }
};
template <>
struct Abs<double> {
  using U = unsigned long long;
  __device__ static U bits(double v) {
    return static_cast<U>(__double_as_longlong(v)) & 0x7fffffffffffffffull;
  }
  __device__ static float mag(U b) { return __double2float_rn(__longlong_as_double(static_cast<long long>(b))); }
  __device__ static bool neg(double v) { return __double_as_longlong(v) < 0; }
  __device__ static uint32_t hibits(double v) { return static_cast<uint32_t>(__double_as_longlong(v) >> 32); }
  __device__ static double dbl(U b) { return __longlong_as_double(static_cast<long long>(b)); }
  __device__ static bool nonfinite(U b) { return b >= 0x7ff0000000000000ull; }
  __device__ static U vmax(U m, U b) { return b > m ? b : m; }
};

// Fast path for one element. `H` is hi32 of the final mix64 state of the
// element's dither (see mix64_hi): X = 1 + uf with uf <= u < uf + 2^-23.
// Returns the lane code and sets `slow` when the decision is within the
// error margin M of a boundary.
//
// standard: the reference's result s - idx equals floor(t + 1 - u) with
//   t = s|x|/norm (fl + [u < f], continuous across brackets), so
//   z = t + (2 - X), mag = floor(z), slow iff frac(z) within M of 0 or 1.
// exponential: with ys = |x| 2^(s-1)/norm the bracket is i = s-1 when ys < 1
//   (f = ys), else i = s + 125 - exponent(ys) (f = mantissa fraction);
//   idx = i + [u >= f], slow iff u - f within M of 0 or of -1 (the latter is
//   where an approximate f could sit in the neighbouring bracket).
// y = 0 needs no special case: z = 1 - uf (std) or f = 0 (exp) round to the
// zero level exactly as the reference does.
template <int KIND>
__device__ __forceinline__ int32_t fast_code(float a, uint32_t vbits, uint32_t H, const QConst& K,
                                             const MulConsts& MK, uint32_t s, uint32_t shift,
                                             uint32_t sign_bit, bool& slow) {
  // X = 1 + uf: (H >> 9) | 0x3f800000 on the multiply pipe
  const float X = __uint_as_float(mulhi(H, MK.p23) | 0x3f800000u);
  const uint32_t neg = mulhi(vbits, MK.two);  // sign bit of x (0 / 1)
  if constexpr (KIND == 0) {
    const float t = a * K.c;
    const float z = t + (2.0f - X);
    const float zm = __fadd_rd(z, 8388608.0f);
    const float fr = z - (zm - 8388608.0f);
    slow = fabsf(fr - 0.5f) > K.half_m;
    // mag = bits(zm) - 0x4b000000;  lane = neg ? -mag : mag  =  mag * (1 - 2 neg)
    const uint32_t factor = mad_lo(neg, 0xfffffffeu, 1u);
    return static_cast<int32_t>(mad_lo(static_cast<uint32_t>(__float_as_int(zm)) - 0x4b000000u, factor, 0u));
  } else {
    const float ys = a * K.c;
    const uint32_t yb = __float_as_uint(ys);
    const uint32_t e8 = mulhi(yb, MK.p9);  // yb >> 23
    const bool last = yb < 0x3f800000u;
    const float f1 = last ? ys + 1.0f : __uint_as_float((yb & 0x7fffffu) | 0x3f800000u);
    // i1 = bracket + shift + 1 = min(s + 126 + shift - e8, s + shift)
    const int i1 = min(static_cast<int>(s + 126u + shift) - static_cast<int>(e8),
                       static_cast<int>(s + shift));
    const float dd = X - f1;  // uf - f
    slow = (fabsf(fabsf(dd) - 0.5f) > K.half_m) || i1 <= static_cast<int>(shift);  // i1 <= shift: y >= 1
    // idx + shift = i1 - [u < f] = i1 - signbit(dd); sign applied on the multiply pipe
    const uint32_t sdd = mulhi(__float_as_uint(dd), MK.two);
    const uint32_t code = mad_lo(sdd, 0xffffffffu, static_cast<uint32_t>(i1));
    return code >= s + shift ? 0 : static_cast<int32_t>(mad_lo(neg, sign_bit, code));
  }
}

// Exact decision for element j (the rare deferred elements).
template <int KIND>
__device__ __noinline__ int32_t slow_code(double ad, bool neg, uint64_t h4, uint64_t j, double norm,
                                          uint32_t s, uint32_t shift, uint32_t sign_bit) {
  const uint64_t bits = mix64(h4 ^ j);
  const uint32_t idx = slow_index<KIND>(ad, norm, bits, s);
  if constexpr (KIND == 0) {
    const int32_t mag = static_cast<int32_t>(s - idx);
    return neg ? -mag : mag;
  } else {
    return idx >= s ? 0 : static_cast<int32_t>((idx + shift) | (neg ? sign_bit : 0u));
  }
}

// Four consecutive elements j0..j0+3 (j0 % 4 == 0, or a scalar tail).
template <int KIND, typename T>
__device__ __forceinline__ void quant_quad(const T (&v)[4], int cnt, uint64_t h4, uint64_t j0,
                                           const QConst& K, const MulConsts& MK, uint32_t s,
                                           uint32_t shift, uint32_t sign_bit,
                                           typename Abs<T>::U& maxab, int32_t (&c)[4]) {
  const uint32_t xl0 = static_cast<uint32_t>(h4) ^ static_cast<uint32_t>(j0);
  const uint32_t xh = static_cast<uint32_t>(h4 >> 32) ^ static_cast<uint32_t>(j0 >> 32);
  bool slow[4];
  bool any = false;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const auto ab = Abs<T>::bits(v[e]);
    if (e < cnt) maxab = Abs<T>::vmax(maxab, ab);
    const uint32_t H = mix64_hi(xl0 ^ static_cast<uint32_t>(e), xh, MK);
    c[e] = fast_code<KIND>(Abs<T>::mag(ab), Abs<T>::hibits(v[e]), H, K, MK, s, shift, sign_bit, slow[e]);
    slow[e] = (slow[e] || !K.fast) && e < cnt;
    any |= slow[e];
  }
  if (any) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (slow[e]) {
        c[e] = slow_code<KIND>(Abs<T>::dbl(Abs<T>::bits(v[e])), Abs<T>::neg(v[e]), h4, j0 + e, K.norm,
                               s, shift, sign_bit);
      }
    }
  }
  if (cnt < 4) {
#pragma unroll
    for (int e = 0; e < 4; ++e) if (e >= cnt) c[e] = 0;
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
__global__ void __launch_bounds__(kQThreads, GQ_QMINBLOCKS)
quantize_kernel(const __grid_constant__ QuantArgs args) {
  const uint64_t d = args.d;
  const uint32_t s = args.s;
  const uint32_t shift = args.shift;
  const uint32_t nl = args.n_local;
  const uint32_t sign_bit = 1u << (W - 1);
  const double norm = *args.norm;
  uint32_t flags = 0;
  const uint64_t nquad = d / 4;

  if (!(norm >= 0.0) || !isfinite(norm)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_flag(args.err, GQ_FLAG_BAD_SCALE);
    return;
  }
  if (norm == 0.0) {
    // quantizer.cpp:21-32: every element must be zero; all idx = s (lane 0).
    const uint64_t total = nquad * nl;
    for (uint64_t g = blockIdx.x * static_cast<uint64_t>(kQThreads) + threadIdx.x; g < total;
         g += static_cast<uint64_t>(gridDim.x) * kQThreads) {
      const uint32_t r = static_cast<uint32_t>(g / nquad);
      const uint64_t q = g - r * nquad;
      T v[4];
      load_quad<T>(static_cast<const T*>(args.x[r]), q, v);
#pragma unroll
      for (int e = 0; e < 4; ++e) if (v[e] != T(0)) flags |= GQ_FLAG_ZERO_SCALE;
      const int32_t c[4] = {0, 0, 0, 0};
      store_quad<W>(args.lanes[r], q, c);
    }
    if (threadIdx.x == 0) {
      for (uint32_t r = blockIdx.x; r < nl; r += gridDim.x) {
        const T* x = static_cast<const T*>(args.x[r]);
        for (uint64_t j = nquad * 4; j < d; ++j) if (x[j] != T(0)) flags |= GQ_FLAG_ZERO_SCALE;
        uint8_t* lb = static_cast<uint8_t*>(args.lanes[r]);
        const uint64_t b0 = nquad * 4 * W / 8, b1 = (d * W + 7) / 8;
        for (uint64_t bb = b0; bb < b1; ++bb) lb[bb] = 0;
      }
    }
    raise_flags_warp(args.err, flags);
    return;
  }

  const QConst K = make_const<KIND>(norm, s);
  const MulConsts MK = args.mk;
  typename Abs<T>::U maxab = 0;

  // ---- TMA bulk-copy pipeline over a global list of (worker, chunk) pairs ----
  // Block b owns global chunks [g0, g0 + cnt); thread 0 issues one 1-D bulk
  // copy per chunk into one of kStages shared-memory stages; every thread
  // waits on that stage's mbarrier, quantizes its kQUnroll quads from shared
  // memory and stores its lanes; the stage is refilled after a block barrier.
  extern __shared__ __align__(128) uint8_t qsmem[];
  constexpr uint32_t kChunkB = kChunkQ * 4 * sizeof(T);
  constexpr int kStages = QStages<T>::value;
  uint64_t* bars = reinterpret_cast<uint64_t*>(qsmem + kStages * kChunkB);
  const uint64_t nch = nquad / kChunkQ;
  const uint64_t gtotal = nch * nl;
  const uint64_t per = (gtotal + gridDim.x - 1) / gridDim.x;
  const uint64_t g0 = min(gtotal, per * blockIdx.x);
  const uint64_t cnt = min(gtotal, g0 + per) - g0;
  auto chunk_src = [&](uint64_t g) -> const T* {
    const uint32_t r = static_cast<uint32_t>(g / nch);
    return static_cast<const T*>(args.x[r]) + (g - r * nch) * kChunkQ * 4;
  };
  if (threadIdx.x == 0) {
#pragma unroll
    for (int st = 0; st < kStages; ++st) mbar_init(&bars[st], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (uint64_t k = 0; k < kStages && k < cnt; ++k) {
      mbar_expect_tx(&bars[k], kChunkB);
      bulk_g2s(qsmem + k * kChunkB, chunk_src(g0 + k), kChunkB, &bars[k]);
    }
  }
  uint32_t r = nch ? static_cast<uint32_t>(g0 / nch) : 0;
  uint64_t cidx = g0 - static_cast<uint64_t>(r) * nch;
  for (uint64_t k = 0; k < cnt; ++k, ++cidx) {
    const int st = static_cast<int>(k % kStages);
    const uint64_t g = g0 + k;
    if (cidx == nch) {
      cidx = 0;
      ++r;
    }
    const uint64_t qbase = cidx * kChunkQ;
    const uint64_t h4 = args.h4[r];
    void* lanes = args.lanes[r];
    mbar_wait(&bars[st], static_cast<uint32_t>((k / kStages) & 1));
    const T* src = reinterpret_cast<const T*>(qsmem + st * kChunkB);
#pragma unroll
    for (int u = 0; u < kQUnroll; ++u) {
      const int ql = u * kQThreads + threadIdx.x;
      T v[4];
      if constexpr (sizeof(T) == 4) {
        const float4 f = reinterpret_cast<const float4*>(src)[ql];
        v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
      } else {
        const double2 a0 = reinterpret_cast<const double2*>(src)[2 * ql];
        const double2 a1 = reinterpret_cast<const double2*>(src)[2 * ql + 1];
        v[0] = a0.x; v[1] = a0.y; v[2] = a1.x; v[3] = a1.y;
      }
      int32_t c[4];
      quant_quad<KIND, T>(v, 4, h4, 4 * (qbase + ql), K, MK, s, shift, sign_bit, maxab, c);
      store_quad<W>(lanes, qbase + ql, c);
    }
    __syncthreads();  // every thread is done with stage st
    if (threadIdx.x == 0 && k + kStages < cnt) {
      mbar_expect_tx(&bars[st], kChunkB);
      bulk_g2s(qsmem + st * kChunkB, chunk_src(g + kStages), kChunkB, &bars[st]);
    }
  }

  // ---- per-worker remainder: quads past the last whole chunk + tail ----
  for (uint32_t r = blockIdx.x; r < nl; r += gridDim.x) {
    const T* x = static_cast<const T*>(args.x[r]);
    void* lanes = args.lanes[r];
    const uint64_t h4 = args.h4[r];
    for (uint64_t q = nch * kChunkQ + threadIdx.x; q < nquad; q += kQThreads) {
      T v[4];
      load_quad<T>(x, q, v);
      int32_t c[4];
      quant_quad<KIND, T>(v, 4, h4, 4 * q, K, MK, s, shift, sign_bit, maxab, c);
      store_quad<W>(lanes, q, c);
    }
    // d % 4 tail elements: one thread writes whole bytes, zero-padded
    if (threadIdx.x == 0 && nquad * 4 < d) {
      int32_t c[4] = {0, 0, 0, 0};
      T tv[4] = {T(0), T(0), T(0), T(0)};
      const int tc = static_cast<int>(d - nquad * 4);
      for (int e = 0; e < tc; ++e) tv[e] = x[nquad * 4 + e];
      quant_quad<KIND, T>(tv, tc, h4, nquad * 4, K, MK, s, shift, sign_bit, maxab, c);
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
      for (uint64_t bb = 0; bb < nb; ++bb) lb[b0 + bb] = static_cast<uint8_t>(packed[bb / 8] >> (8 * (bb % 8)));
    }
  }
  // quantizer.cpp:35-41: NaN/Inf, then |x| > norm (y > 1).
  if (Abs<T>::nonfinite(maxab)) flags |= GQ_FLAG_NONFINITE;
  else if (Abs<T>::dbl(maxab) > norm) flags |= GQ_FLAG_EXCEEDS_SCALE;
  raise_flags_warp(args.err, flags);
}

template <typename T, int KIND, int W>
cudaError_t launch_one(const QuantArgs& a, uint64_t work_chunks, cudaStream_t st) {
  auto* fn = quantize_kernel<T, KIND, W>;
  const size_t smem = qsmem_bytes<T>();
  // one-time per instantiation: opt in to >48 KiB smem, read the residency
  static int blocks_per_sm = 0;
  static int sms = 0;
  if (blocks_per_sm == 0) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, fn, kQThreads, smem);
    if (e != cudaSuccess) return e;
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  // persistent grid: exactly one wave of resident blocks (never a tail wave)
  uint64_t blocks = static_cast<uint64_t>(sms) * blocks_per_sm;
  if (blocks > work_chunks) blocks = work_chunks;
  if (blocks == 0) blocks = 1;
  fn<<<static_cast<uint32_t>(blocks), kQThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <typename T, int KIND>
cudaError_t launch_w(const QuantArgs& a, uint64_t work_chunks, uint32_t width, cudaStream_t st) {
  switch (width) {
    case 4: return launch_one<T, KIND, 4>(a, work_chunks, st);
    case 8: return launch_one<T, KIND, 8>(a, work_chunks, st);
    case 16: return launch_one<T, KIND, 16>(a, work_chunks, st);
    case 32: return launch_one<T, KIND, 32>(a, work_chunks, st);
    default: return cudaErrorInvalidValue;
  }
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
  a.mk = GQ_MULCONSTS_INIT;
  a.n_local = q.n_local;
  // work units for the grid: whole staged chunks over all local workers
  // (at least one per worker so the remainder/tail loop has an owner)
  uint64_t work = (q.d / 4 / kChunkQ) * q.n_local;
  if (work < q.n_local) work = q.n_local;
  if (q.dtype == GQ_DTYPE_F32) {
    return q.kind == 0 ? launch_w<float, 0>(a, work, q.width, stream)
                       : launch_w<float, 1>(a, work, q.width, stream);
  }
  return q.kind == 0 ? launch_w<double, 0>(a, work, q.width, stream)
                     : launch_w<double, 1>(a, work, q.width, stream);
}

}  // namespace gqb
