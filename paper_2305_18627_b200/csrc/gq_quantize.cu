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

int g_quant_ctas_per_sm = 0;

namespace {

#ifndef GQ_QBAL
#define GQ_QBAL 1
#endif
#ifndef GQ_QWAVES  // CTA waves: > 1 lets the block scheduler rebalance SMs that finish early
#define GQ_QWAVES 1
#endif
#ifndef GQ_QBAL_STD
#define GQ_QBAL_STD 0
#endif
#ifndef GQ_QSIGN_ALU
#define GQ_QSIGN_ALU 0
#endif
#ifndef GQ_QPACK
#define GQ_QPACK 1
#endif
#ifndef GQ_QUNROLL
#define GQ_QUNROLL 4
#endif
#ifndef GQ_QUPRAGMA  // unroll factor of the per-chunk quad loop (fewer live registers when < GQ_QUNROLL)
#define GQ_QUPRAGMA 4
#endif
#ifndef GQ_QMINBLOCKS
#define GQ_QMINBLOCKS 3
#endif
constexpr int kQThreads = 256;
constexpr int kQUnroll = GQ_QUNROLL;
constexpr int kQUPragma = GQ_QUPRAGMA;
#ifndef GQ_QSTAGES
#define GQ_QSTAGES 3
#endif
constexpr int kWarpQ = 32 * kQUnroll;  // quads per warp chunk (2 KiB of f32 at kQUnroll = 4)
// chunks per 2^32 elements: the high word of j = 4 kWarpQ cidx changes when cidx crosses a multiple
constexpr uint32_t kHiWordChunkMask = static_cast<uint32_t>((1ull << 32) / (4ull * kWarpQ)) - 1u;
template <typename T>
struct QStages {
  static constexpr int value = GQ_QSTAGES;  // per warp: 6 KiB (f32) / 12 KiB (f64) at 3 stages
};
template <typename T>
constexpr size_t qsmem_bytes() {
  return (kQThreads / 32) * (QStages<T>::value * (kWarpQ * 4 * sizeof(T)) + QStages<T>::value * sizeof(uint64_t));
}

struct QuantArgs {
  const void* x[kMaxWorkers];
  void* lanes[kMaxWorkers];
  uint64_t h4[kMaxWorkers];
  uint32_t wid[kMaxWorkers];    // worker ids (for the device-side prefixes)
  const uint64_t* round_ptr;    // non-null: round read on the device (graph replays)
  uint64_t seed;
  // scatter mode (one local worker): quad q goes to sdst[q / slice_quads] at
  // quad offset q % slice_quads - the lane slices land directly in their
  // owners' receive buffers (peer pointers over NVLink)
  void* sdst[kMaxPeers];
  uint64_t slice_quads;
  uint64_t row_bytes;  // scatter mode: local worker r's rows start r * row_bytes into each slice destination
  SignalArgs sig;      // n > 0: flag the peers when the whole grid is done (scatter mode)
  PeerWait pw;         // n > 0: wait for the peers' stats (folded exchange) ...
  StatsFold fold;      // ... and fold them into the norm (instead of reading *norm)
  uint32_t nslices;
  uint64_t d;
  const double* norm;
  uint32_t* err;
  uint32_t s;
  uint32_t shift;
  uint32_t n_local;
  MulConsts mk;
  uint32_t pk[3];  // lane-packing multipliers 2^W, 2^2W, 2^3W (runtime: kept on the FMA pipe)
};

// Per-block constants derived from the device-resident norm.
//
// Fast-path formulations (all decisions in integer form on fp32 bit patterns):
//   standard:    z = t + (2^k + 1 + (1 - u~)) with t = |x| fl32(s/norm), u~ the
//                top 23 - k dither bits; 2^k > s + 2 fixes z's exponent, so the
//                lane magnitude floor(t + 1 - u) is z's integer part read from
//                the mantissa, and frac(z) (the distance to the decision
//                boundary) is the rest of the mantissa.
//   exponential: ys = |x| fl32(2^(s-1)/norm); ys2 = max(ys, (ys + 1)/2) puts
//                the last bracket [0, 1) at exponent 126 with frac = ys; the
//                stochastic rounding between neighbouring levels is then the
//                carry of bits(ys2) + (2^23 - 1 - U) into the exponent field
//                (U = top 23 dither bits), and the low 23 bits of that sum are
//                (frac - U - 1) mod 2^23, the distance to the boundary.
// An element whose boundary distance is within Mq units (or whose input is
// NaN/Inf or |x| >= norm) is decided by slow_code, the reference's f64 rule.
struct QConst {
  double norm;
  float c;        // std: fl32(s / norm); exp: fl32(2^(s-1) / norm)
  bool fast;      // fast path usable at all
  // standard
  uint32_t ybase;  // bits of 2^k + 2 - 2^(k-23): Y = ybase - (H >> (9+k)) = 2^k + 1 + (1 - u~) - ulp
  uint32_t ysh;    // 9 + k: H >> ysh = the top 23 - k dither bits
  uint32_t zsh;    // 23 - k: zi >> zsh = the integer part of z (with the exponent above it)
  uint32_t zmul;   // 2^(9+k): zi * zmul = frac bits << (9+k)
  uint32_t cm;     // ((127 + k) << k) + 1
  uint32_t mq;     // margin, in the shifted frac word
  uint32_t s_lim;  // s: raw >= cm + s (magnitude s or more: y near 1 or above) defers to slow_code
  // exponential
  int32_t cc;      // s + 126 + shift
  uint32_t ythr;   // bits of 2^(s-1) (1 - 2^-19): ys at or above it defers to slow_code
};

template <int KIND>
__device__ __forceinline__ QConst make_const(double norm, uint32_t s, uint32_t shift) {
  QConst k{};
  k.norm = norm;
  if (KIND == 0) {
    // t error: c (1 rounding) + product (1) + f64->f32 input (1): 3 s 2^-24;
    // u~ truncation 2^(k-23); z rounding 2^(k-24): total < 3 units of 2^(k-23)
    int kk = 1;
    while ((1u << kk) < s + 3u) ++kk;
    k.c = __double2float_rn(__ddiv_rn(static_cast<double>(s), norm));
    k.fast = (kk <= 14) && isfinite(k.c) && k.c >= 0x1.0p-100f && k.c <= 0x1.0p100f;
    k.ybase = __float_as_uint(static_cast<float>((1u << kk) + 1u)) + ((1u << (23 - kk)) - 1u);
    k.ysh = 9u + kk;
    k.zsh = 23u - kk;
    k.zmul = 1u << (9 + kk);
    k.cm = ((127u + kk) << kk) + 1u;
    k.mq = 6u << (9 + kk);
    k.s_lim = s;
  } else {
    // frac error: ys (3 roundings) <= 3 units of 2^-23, ys2 rounding 1/2 unit,
    // U truncation 1 unit: < 5 units; margin 8 units
    k.c = (s <= 120) ? __double2float_rn(__ddiv_rn(ldexp(1.0, static_cast<int>(s) - 1), norm)) : 0.0f;
    k.fast = (s <= 120) && isfinite(k.c) && k.c >= 0x1.0p-100f && k.c <= 0x1.0p100f;
    k.mq = 8u << 9;
    k.cc = static_cast<int32_t>(s + 126u + shift);
    k.ythr = __float_as_uint(ldexpf(1.0f - 0x1.0p-19f, static_cast<int>(s) - 1));
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
__device__ __forceinline__ uint32_t slow_index(double ad, double norm, uint64_t bits, uint32_t s) {
  double y = __ddiv_rn(ad, norm);
  if (y > 1.0) y = 1.0;  // flagged as EXCEEDS_SCALE by the caller; keep going
  int64_t g;
  if (KIND == 0) {
    g = static_cast<int64_t>(s) - 1 - static_cast<int64_t>(floor(__dmul_rn(y, static_cast<double>(s))));
  } else {
    if (y == 0.0) {
      g = static_cast<int64_t>(s) - 1;
    } else {
      int e;
      const double m = frexp(y, &e);  // y = m 2^e, m in [0.5, 1)
      g = (m == 0.5) ? -(e - 1) : -e;
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

// Exact decision for element j (the rare deferred elements), including the
// reference's per-element checks (quantizer.cpp:35-41): NaN/Inf, |x| > norm.
template <int KIND>
__device__ __noinline__ int32_t slow_code(double ad, bool neg, uint64_t h4, uint64_t j, double norm,
                                          uint32_t s, uint32_t shift, uint32_t sign_bit,
                                          uint32_t* flags) {
  if (!isfinite(ad)) {
    *flags |= GQ_FLAG_NONFINITE;
    return 0;
  }
  if (ad > norm) *flags |= GQ_FLAG_EXCEEDS_SCALE;
  const uint64_t bits = mix64(h4 ^ j);
  const uint32_t idx = slow_index<KIND>(ad, norm, bits, s);
  if constexpr (KIND == 0) {
    const int32_t mag = static_cast<int32_t>(s - idx);
    return neg ? -mag : mag;
  } else {
    return idx >= s ? 0 : static_cast<int32_t>((idx + shift) | (neg ? sign_bit : 0u));
  }
}

template <typename T>
struct Abs;
template <>
struct Abs<float> {
  __device__ static float mag(float v) { return fabsf(v); }
  __device__ static uint32_t hibits(float v) { return __float_as_uint(v); }
  __device__ static double dbl(float v) { return fabs(static_cast<double>(v)); }
  __device__ static bool neg(float v) { return (__float_as_uint(v) >> 31) != 0; }
};
template <>
struct Abs<double> {
  __device__ static float mag(double v) { return __double2float_rn(fabs(v)); }
  __device__ static uint32_t hibits(double v) { return static_cast<uint32_t>(__double_as_longlong(v) >> 32); }
  __device__ static double dbl(double v) { return fabs(v); }
  __device__ static bool neg(double v) { return __double_as_longlong(v) < 0; }
};

// Quads of four consecutive elements use the group-shared mix64 of
// gq_common.cuh (QuadMix / elem_mix) with G = 4. Within one 512-element
// chunk the high word of x = h4 ^ j is fixed, so the two possible values of
// (zh << 2, K1) - carry 0 or 1 out of the low-word add - are computed once
// per chunk and selected per quad.
struct ChunkMix {
  uint32_t hl;          // h4lo & ~3
  uint32_t ce[4];       // e ^ (h4lo & 3)
  uint32_t zh2[2], K1[2];
};

__device__ __forceinline__ ChunkMix chunk_mix(uint64_t h4, uint64_t jc) {
  ChunkMix m;
  const uint32_t hl = static_cast<uint32_t>(h4);
  m.hl = hl & ~3u;
#pragma unroll
  for (int e = 0; e < 4; ++e) m.ce[e] = static_cast<uint32_t>(e) ^ (hl & 3u);
  const uint32_t xh = static_cast<uint32_t>(h4 >> 32) ^ static_cast<uint32_t>(jc >> 32);
#pragma unroll
  for (int cy = 0; cy < 2; ++cy) {
    const uint32_t zh = xh + 0x9e3779b9u + static_cast<uint32_t>(cy);
    m.zh2[cy] = zh << 2;
    m.K1[cy] = (zh ^ (zh >> 30)) * 0x1ce4e5b9u;
  }
  return m;
}

// j0lo: low word of the quad's first index (j0 % 4 == 0, same chunk as m)
__device__ __forceinline__ QuadMix quad_mix(const ChunkMix& m, uint32_t j0lo) {
  QuadMix q;
  const uint32_t b = m.hl ^ j0lo;
  q.B = b + 0x7f4a7c15u;
  const bool cy = q.B < b;
  q.ok = q.B <= 0xfffffffcu;
  q.zh2 = cy ? m.zh2[1] : m.zh2[0];
  q.K1 = cy ? m.K1[1] : m.K1[0];
  return q;
}

// Fast decision for one element from its dither word H. Sets `slow` when the
// element must take slow_code (boundary within the margin, NaN/Inf, y >= 1).
template <int KIND, int W>
__device__ __forceinline__ int32_t fast_code(float a, uint32_t vbits, uint32_t H, const QConst& K,
                                             const MulConsts& MK, uint32_t s, uint32_t shift,
                                             bool& slow) {
  if constexpr (KIND == 0) {
    const float t = a * K.c;
#if GQ_QBAL_STD >= 2
    const float z = t + __uint_as_float(mad_lo(H >> K.ysh, MK.neg1, K.ybase));
#else
    const float z = t + __uint_as_float(K.ybase - (H >> K.ysh));       // 2^k + 1 + t + (1 - u~)
#endif
    const uint32_t zi = __float_as_uint(z);
#if GQ_QBAL_STD >= 1  // (zi >> zsh) - cm as one multiply-add: hi32(zi * 2^(32 - zsh)) - cm
    const int32_t mag = static_cast<int32_t>(mad_hi(zi, K.zmul, 0u - K.cm));
#else
    const int32_t mag = static_cast<int32_t>((zi >> K.zsh) - K.cm);   // floor(t + 1 - u)
#endif
    slow = (mad_lo(zi, K.zmul, K.mq) <= 2u * K.mq) || mag >= static_cast<int32_t>(s);
#if GQ_QSIGN_ALU  // (mag ^ m) - m with m = 0 / -1: the sign on the ALU pipe
    const uint32_t sm = static_cast<uint32_t>(static_cast<int32_t>(vbits) >> 31);
    return static_cast<int32_t>((static_cast<uint32_t>(mag) ^ sm) - sm);
#else
    // two's complement sign on the multiply pipe: mag * (1 - 2 neg)
    const uint32_t factor = mad_lo(static_cast<uint32_t>(static_cast<int32_t>(vbits) >> 31), 2u, 1u);
    return static_cast<int32_t>(mad_lo(static_cast<uint32_t>(mag), factor, 0u));
#endif
  } else {
    const float ys = a * K.c;
    const float ys2 = fmaxf(ys, fmaf(ys, 0.5f, 0.5f));
    const uint32_t yb = __float_as_uint(ys2);
    const uint32_t R = yb + 0x7fffffu - mulhi(H, MK.p23);               // carry = round up
#if GQ_QBAL  // runtime multiplier operands keep these on the multiply pipe (ptxas would make them ALU LEA/IADD)
    const int32_t code = static_cast<int32_t>(mad_lo(mulhi(R, MK.p9), MK.neg1, static_cast<uint32_t>(K.cc)));
    slow = (mad_lo(R, MK.c512, K.mq) <= 2u * K.mq) || yb >= K.ythr;
#else
    const int32_t code = static_cast<int32_t>(mad_lo(mulhi(R, MK.p9), 0xffffffffu, static_cast<uint32_t>(K.cc)));
    // (ys2 >= ythr: y within 2^-19 of 1 or above, NaN/Inf) -> slow_code, which
    // applies the exact |x| > norm test; below it code >= shift always holds
    slow = (mad_lo(R, 512u, K.mq) <= 2u * K.mq) || yb >= K.ythr;
#endif
    // sign bit of x into lane bit W-1; the zero level (code == s + shift) is lane 0
    uint32_t nb;
    if constexpr (W == 32) nb = vbits & 0x80000000u;
    else nb = (vbits >> (32 - W)) & (1u << (W - 1));
    return code >= static_cast<int32_t>(s + shift) ? 0 : static_cast<int32_t>(static_cast<uint32_t>(code) | nb);
  }
}

// Four consecutive elements j0..j0+3 (j0 % 4 == 0); cnt < 4 only for a tail
// (the missing elements are zero-filled by the caller and forced to lane 0).
template <int KIND, int W, typename T>
__device__ __forceinline__ void quant_quad(const T (&v)[4], int cnt, uint64_t h4, const ChunkMix& m,
                                           uint64_t j0, const QConst& K, const MulConsts& MK, uint32_t s,
                                           uint32_t shift, uint32_t& flags, int32_t (&c)[4]) {
  const QuadMix q = quad_mix(m, static_cast<uint32_t>(j0));
  bool slow[4];
  bool any = !q.ok || !K.fast;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint32_t H = elem_mix(q, m.ce[e], MK);
    c[e] = fast_code<KIND, W>(Abs<T>::mag(v[e]), Abs<T>::hibits(v[e]), H, K, MK, s, shift, slow[e]);
    slow[e] = slow[e] && e < cnt;
    any |= slow[e];
  }
  if (any) {
    const uint32_t sign_bit = 1u << (W - 1);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (e < cnt && (slow[e] || !q.ok || !K.fast)) {
        c[e] = slow_code<KIND>(Abs<T>::dbl(v[e]), Abs<T>::neg(v[e]), h4, j0 + e, K.norm, s, shift,
                               sign_bit, &flags);
      }
    }
  }
  if (cnt < 4) {
#pragma unroll
    for (int e = 0; e < 4; ++e) if (e >= cnt) c[e] = 0;
  }
}

// Exponential lanes of 4 / 8 bits: after the carry, the f32 exponent field
// E = R >> 23 of the dithered ys2 names the level (E = 126: the zero level,
// E = 126 + i: code s + shift - i), so the lane - code | sign bit, or 0 for the
// zero level whatever the sign (exp_arith.cpp:126-160) - is one byte of a
// per-block table indexed by 2E + sign (E < 512 for any 32-bit R, so every
// index is in bounds; entries outside [126, 126 + s] belong to slow elements
// and are 0). 3 instructions (IMAD.HI, SHF, LDS) instead of the code /
// zero-select / sign chain's 6, 4 of them on the ALU pipe.
constexpr int kExpTab = 1024;
#ifndef GQ_QTAB
#define GQ_QTAB 1
#endif
template <int KIND, int W>
constexpr bool kUseQtab = GQ_QTAB && (W == 4 || W == 8);
template <int KIND>
constexpr int kQtabBytes = KIND == 1 ? kExpTab : 512;

template <int W>
__device__ __forceinline__ void build_exp_tab(uint8_t* tab, uint32_t s, uint32_t shift) {
  for (uint32_t i = threadIdx.x; i < kExpTab; i += blockDim.x) {
    const uint32_t E = i >> 1, neg = i & 1u;
    uint32_t lane = 0;
    if (E > 126 && E <= 126 + s) lane = (s + shift - (E - 126)) | (neg << (W - 1));
    tab[i] = static_cast<uint8_t>(lane);
  }
}

template <int W>
__device__ __forceinline__ int32_t fast_code_tab(float a, uint32_t vbits, uint32_t H, const QConst& K,
                                                 const MulConsts& MK, const uint8_t* tab, bool& slow) {
  const float ys = a * K.c;
  const float ys2 = fmaxf(ys, fmaf(ys, 0.5f, 0.5f));
  const uint32_t yb = __float_as_uint(ys2);
  const uint32_t R = yb + 0x7fffffu - mulhi(H, MK.p23);  // carry = round up
  slow = (mad_lo(R, MK.c512, K.mq) <= 2u * K.mq) || yb >= K.ythr;
  uint32_t idx;  // (E << 1) | sign(x)
  asm("shf.l.clamp.b32 %0, %1, %2, 1;" : "=r"(idx) : "r"(vbits), "r"(mulhi(R, MK.p9)));
  return tab[idx];
}

// Standard lanes of 4 / 8 bits, the same idea: z's bits above zsh are
// raw = ((127 + k) << k) + floor(t + 1 - u) (QConst), so the lane magnitude is
// raw - cm and the signed W-bit lane (encode_dense_std, algorithm.cpp:69-82;
// 0 for the zero level whatever the sign) is one byte of a 512-entry table
// indexed by ((raw mod 256) << 1) | sign - the magnitudes of the fast path are
// a window of s + 1 <= 128 consecutive raw values, so raw mod 256 names them
// uniquely, and the mask keeps every index (slow elements') in bounds.
template <int W>
__device__ __forceinline__ void build_std_tab(uint8_t* tab, uint32_t s, uint32_t cm) {
  for (uint32_t i = threadIdx.x; i < 512; i += blockDim.x) {
    const uint32_t mag = ((i >> 1) - cm) & 255u, neg = i & 1u;
    uint32_t lane = 0;
    if (mag <= s) lane = (neg ? 0u - mag : mag) & ((1u << W) - 1u);
    tab[i] = static_cast<uint8_t>(lane);
  }
}

template <int W>
__device__ __forceinline__ int32_t fast_code_tab_std(float a, uint32_t vbits, uint32_t H, const QConst& K,
                                                     const MulConsts& MK, const uint8_t* tab, bool& slow) {
  const float t = a * K.c;
  const float z = t + __uint_as_float(K.ybase - (H >> K.ysh));  // 2^k + 1 + t + (1 - u~)
  const uint32_t zi = __float_as_uint(z);
  const uint32_t raw = zi >> K.zsh;
  slow = (mad_lo(zi, K.zmul, K.mq) <= 2u * K.mq) || raw >= K.cm + K.s_lim;
  uint32_t idx;  // (raw << 1) | sign(x), mod 512
  asm("shf.l.clamp.b32 %0, %1, %2, 1;" : "=r"(idx) : "r"(vbits), "r"(raw));
  return tab[idx & 511u];
}

// Fast decisions only for a whole quad (the hot loop): `any` is raised when
// some element (or the quad's shared-carry hash) needs quant_quad's exact
// handling; the caller then redoes its quads with quant_quad (rare).
template <int KIND, int W>
__device__ __forceinline__ void fast_quad(const float (&v)[4], const ChunkMix& m, uint32_t j0lo, const QConst& K,
                                          const MulConsts& MK, uint32_t s, uint32_t shift, const uint8_t* tab,
                                          bool& any, int32_t (&c)[4]) {
  const QuadMix q = quad_mix(m, j0lo);
  any |= !q.ok;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    bool slow;
    const uint32_t H = elem_mix(q, m.ce[e], MK);
    if constexpr (kUseQtab<KIND, W> && KIND == 1)
      c[e] = fast_code_tab<W>(fabsf(v[e]), __float_as_uint(v[e]), H, K, MK, tab, slow);
    else if constexpr (kUseQtab<KIND, W>)
      c[e] = fast_code_tab_std<W>(fabsf(v[e]), __float_as_uint(v[e]), H, K, MK, tab, slow);
    else c[e] = fast_code<KIND, W>(fabsf(v[e]), __float_as_uint(v[e]), H, K, MK, s, shift, slow);
    any |= slow;
  }
}

// Pack a quad of W-bit lane values (each already < 2^W) with multiply-adds
// (runtime multipliers, so they stay on the FMA pipe) and store it.
template <int W>
__device__ __forceinline__ void store_quad_mad(void* lanes, uint64_t q, const int32_t (&c)[4], const uint32_t (&pk)[3]) {
  uint32_t v = mad_lo(static_cast<uint32_t>(c[1]), pk[0], static_cast<uint32_t>(c[0]));
  v = mad_lo(static_cast<uint32_t>(c[2]), pk[1], v);
  v = mad_lo(static_cast<uint32_t>(c[3]), pk[2], v);
  if constexpr (W == 4) reinterpret_cast<uint16_t*>(lanes)[q] = static_cast<uint16_t>(v);
  else reinterpret_cast<uint32_t*>(lanes)[q] = v;
}

template <int W, bool kNonNeg = false>
__device__ __forceinline__ void store_quad(void* lanes, uint64_t q, const int32_t (&c)[4]) {
  if constexpr (kNonNeg && GQ_QPACK && (W == 4 || W == 8)) {
    // token lanes are already W-bit values (sign bit | exponent): no masks
    const uint32_t v = static_cast<uint32_t>(c[0]) | (static_cast<uint32_t>(c[1]) << W) |
                       (static_cast<uint32_t>(c[2]) << (2 * W)) | (static_cast<uint32_t>(c[3]) << (3 * W));
    if constexpr (W == 4) reinterpret_cast<uint16_t*>(lanes)[q] = static_cast<uint16_t>(v);
    else reinterpret_cast<uint32_t*>(lanes)[q] = v;
  } else if constexpr (W == 4) {
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

// Base pointer that quad q of local worker r is stored relative to: the
// worker's lane buffer, or in scatter mode the destination of q's slice,
// rebased so store_quad(base, q) lands at the quad's offset in that slice.
template <int W>
__device__ __forceinline__ void* lane_base_for(const QuantArgs& a, uint32_t r, uint64_t q) {
  if (!a.nslices) return a.lanes[r];
  uint64_t j = q / a.slice_quads;
  if (j >= a.nslices) j = a.nslices - 1;  // the tail quad of the last slice
  return static_cast<uint8_t*>(a.sdst[j]) + r * a.row_bytes - j * a.slice_quads * (W / 2);
}

// Folded norm exchange (gq_comm graphs): thread 0 of every CTA waits for all
// ranks' stats flags, then folds the n stats in the reference's tree order
// (collectives.cpp:210-233, norms.cpp:64-75) - every CTA gets the identical
// norm; CTA 0 also stores it for the decode.
__device__ __noinline__ double wait_and_fold_norm(const PeerWait& pw, const StatsFold& f, uint32_t* err) {
  __shared__ double s_st[kMaxWorkers];
  __shared__ double s_norm;
  if (threadIdx.x == 0) {
    peer_wait_flags(pw.flags, pw.n, pw.ep_dev ? *pw.ep_dev : pw.epoch, err, pw.timeout_ns);
    for (uint32_t w = 0; w < f.n; ++w) s_st[w] = __ldcv(f.stats + w);  // peers' stores, not a stale L1 line
    const double nm = tree_fold_stats(s_st, f.n, f.p);
    s_norm = nm;
    if (blockIdx.x == 0 && f.norm_out) *f.norm_out = nm;
  }
  __syncthreads();
  return s_norm;
}

template <typename T, int KIND, int W>
__global__ void __launch_bounds__(kQThreads, GQ_QMINBLOCKS)
quantize_kernel(const __grid_constant__ QuantArgs args) {
  pdl_wait();     // the norm (and the previous step) are complete and visible
  pdl_trigger();  // the reduce may take SM slots as this grid's CTAs retire
  const uint64_t d = args.d;
  const uint32_t s = args.s;
  const uint32_t shift = args.shift;
  const uint32_t nl = args.n_local;
  const double norm = args.pw.n ? wait_and_fold_norm(args.pw, args.fold, args.err) : *args.norm;
  uint32_t flags = 0;
  const uint64_t nquad = d / 4;

  if (!(norm >= 0.0) || !isfinite(norm)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_flag(args.err, GQ_FLAG_BAD_SCALE);
    grid_done_signal(args.sig);  // peers must not wait for the timeout: the error travels via gq_sync
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
      store_quad<W>(lane_base_for<W>(args, r, q), q, c);
    }
    if (threadIdx.x == 0) {
      for (uint32_t r = blockIdx.x; r < nl; r += gridDim.x) {
        const T* x = static_cast<const T*>(args.x[r]);
        for (uint64_t j = nquad * 4; j < d; ++j) if (x[j] != T(0)) flags |= GQ_FLAG_ZERO_SCALE;
        uint8_t* lb = static_cast<uint8_t*>(lane_base_for<W>(args, r, nquad));
        const uint64_t b0 = nquad * 4 * W / 8, b1 = (d * W + 7) / 8;
        for (uint64_t bb = b0; bb < b1; ++bb) lb[bb] = 0;
      }
    }
    raise_flags_warp(args.err, flags);
    grid_done_signal(args.sig);
    return;
  }

  const QConst K = make_const<KIND>(norm, s, shift);
  const MulConsts MK = args.mk;
  __shared__ uint8_t s_qtab[kUseQtab<KIND, W> ? kQtabBytes<KIND> : 4];
  if constexpr (kUseQtab<KIND, W> && KIND == 1) build_exp_tab<W>(s_qtab, s, shift);
  else if constexpr (kUseQtab<KIND, W>) build_std_tab<W>(s_qtab, s, K.cm);
  // per-worker RNG prefixes mix64^4(seed, Dither, worker, round): from the
  // launch (host-computed) or, in graph replays, from the device round
  __shared__ uint64_t s_h4[kMaxWorkers];
  for (uint32_t i = threadIdx.x; i < nl; i += kQThreads)
    s_h4[i] = args.round_ptr ? hoist_prefix(args.seed, 1ull, args.wid[i], *args.round_ptr) : args.h4[i];
  __syncthreads();

  // ---- per-warp TMA bulk-copy pipelines over a global list of (worker, chunk) pairs ----
  // Warp w owns global warp-chunks [g0, g0 + cnt) (kWarpQ quads each). Its
  // lane 0 issues one 1-D bulk copy per chunk into one of the warp's kStages
  // shared-memory stages (cp.async.bulk, completion on the stage's mbarrier);
  // the warp waits on the mbarrier, quantizes kQUnroll quads per lane from
  // shared memory, stores its lanes, and lane 0 refills the stage after a
  // __syncwarp. No block-wide barrier: a warp delayed by a slow-path element
  // never stalls the others.
  extern __shared__ __align__(128) uint8_t qsmem[];
  constexpr uint32_t kChunkB = kWarpQ * 4 * sizeof(T);
  constexpr int kStages = QStages<T>::value;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // all warps' stage buffers first (each 128-byte aligned), then the mbarriers
  uint8_t* wsm = qsmem + warp * (kStages * kChunkB);
  uint64_t* bars = reinterpret_cast<uint64_t*>(qsmem + (kQThreads / 32) * kStages * kChunkB) + warp * kStages;
  // Chunk cursors are 32-bit (d < 2^41) and advance incrementally: no
  // division in the loop. The chunk-shared hash constants depend only on the
  // worker's prefix and the high word of the element index, so they are
  // rebuilt when the worker changes or j crosses a multiple of 2^32.
  const uint32_t nch = static_cast<uint32_t>(nquad / kWarpQ);
  const uint64_t gtotal = static_cast<uint64_t>(nch) * nl;
  const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * (kQThreads / 32);
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * (kQThreads / 32) + warp;
  const uint64_t per = (gtotal + nwarps - 1) / nwarps;
  const uint64_t g0 = min(gtotal, per * gw);
  const uint32_t cnt = static_cast<uint32_t>(min(gtotal, g0 + per) - g0);
  uint32_t r = nch ? static_cast<uint32_t>(g0 / nch) : 0;
  uint32_t cidx = static_cast<uint32_t>(g0 - static_cast<uint64_t>(r) * nch);
  auto chunk_src = [&](uint32_t wr, uint32_t c) -> const T* {
    return static_cast<const T*>(args.x[wr]) + static_cast<uint64_t>(c) * (kWarpQ * 4);
  };
  uint32_t pr = r, pc = cidx;  // producer cursor (lane 0): the next chunk to load
  if (lane == 0) {
#pragma unroll
    for (int st = 0; st < kStages; ++st) mbar_init(&bars[st], 1);
    mbar_fence_init();
    for (uint32_t k = 0; k < static_cast<uint32_t>(kStages) && k < cnt; ++k) {
      mbar_expect_tx(&bars[k], kChunkB);
      bulk_g2s(wsm + k * kChunkB, chunk_src(pr, pc), kChunkB, &bars[k]);
      if (++pc == nch) { pc = 0; ++pr; }
    }
  }
  __syncwarp();
  uint64_t h4 = 0;
  void* lanes = nullptr;
  ChunkMix cm{};
  uint64_t slice_end = 0;  // scatter mode: first quad past the current slice
  uint32_t slice_j = 0;
  for (uint32_t k = 0; k < cnt; ++k) {
    const int st = static_cast<int>(k % kStages);
    const uint64_t qbase = static_cast<uint64_t>(cidx) * kWarpQ;
    if (k == 0 || (cidx & kHiWordChunkMask) == 0) {  // new worker, or a new 2^32 block of j
      h4 = s_h4[r];
      cm = chunk_mix(h4, 4 * qbase);
      if (args.nslices) {
        slice_j = static_cast<uint32_t>(min(qbase / args.slice_quads, static_cast<uint64_t>(args.nslices - 1)));
        slice_end = (slice_j + 1 == args.nslices) ? ~0ull : (slice_j + 1) * args.slice_quads;
        lanes = lane_base_for<W>(args, r, qbase);
      } else {
        lanes = args.lanes[r];
      }
    } else if (args.nslices && qbase >= slice_end) {  // chunks never straddle slices
      ++slice_j;
      slice_end = (slice_j + 1 == args.nslices) ? ~0ull : (slice_j + 1) * args.slice_quads;
      lanes = lane_base_for<W>(args, r, qbase);
    }
    mbar_wait(&bars[st], (k / kStages) & 1u);
    const T* src = reinterpret_cast<const T*>(wsm + st * kChunkB);
    if constexpr (sizeof(T) == 4) {
      bool any = !K.fast;
#pragma unroll kQUPragma
      for (int u = 0; u < kQUnroll; ++u) {
        const int ql = u * 32 + lane;
        const float4 f = reinterpret_cast<const float4*>(src)[ql];
        const float v[4] = {f.x, f.y, f.z, f.w};
        int32_t c[4];
        fast_quad<KIND, W>(v, cm, static_cast<uint32_t>(4 * (qbase + ql)), K, MK, s, shift, s_qtab, any, c);
        if constexpr (kUseQtab<KIND, W>) store_quad_mad<W>(lanes, qbase + ql, c, args.pk);
        else store_quad<W, KIND == 1>(lanes, qbase + ql, c);
      }
      if (__builtin_expect(any, 0)) {  // exact handling of this lane's quads, stored over the fast ones
#pragma unroll 1
        for (int u = 0; u < kQUnroll; ++u) {
          const int ql = u * 32 + lane;
          const float4 f = reinterpret_cast<const float4*>(src)[ql];
          const T v[4] = {f.x, f.y, f.z, f.w};
          int32_t c[4];
          quant_quad<KIND, W, T>(v, 4, h4, cm, 4 * (qbase + ql), K, MK, s, shift, flags, c);
          store_quad<W, KIND == 1>(lanes, qbase + ql, c);
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < kQUnroll; ++u) {
        const int ql = u * 32 + lane;
        const double2 a0 = reinterpret_cast<const double2*>(src)[2 * ql];
        const double2 a1 = reinterpret_cast<const double2*>(src)[2 * ql + 1];
        const T v[4] = {a0.x, a0.y, a1.x, a1.y};
        int32_t c[4];
        quant_quad<KIND, W, T>(v, 4, h4, cm, 4 * (qbase + ql), K, MK, s, shift, flags, c);
        store_quad<W, KIND == 1>(lanes, qbase + ql, c);
      }
    }
    __syncwarp();  // every lane is done with stage st
    if (lane == 0 && k + kStages < cnt) {
      mbar_expect_tx(&bars[st], kChunkB);
      bulk_g2s(wsm + st * kChunkB, chunk_src(pr, pc), kChunkB, &bars[st]);
      if (++pc == nch) { pc = 0; ++pr; }
    }
    if (++cidx == nch) {
      cidx = 0;
      ++r;
    }
  }

  // ---- per-worker remainder: quads past the last whole chunk + tail ----
  for (uint32_t r = blockIdx.x; r < nl; r += gridDim.x) {
    const T* x = static_cast<const T*>(args.x[r]);
    const uint64_t h4 = s_h4[r];
    for (uint64_t q = nch * kWarpQ + threadIdx.x; q < nquad; q += kQThreads) {
      T v[4];
      load_quad<T>(x, q, v);
      int32_t c[4];
      quant_quad<KIND, W, T>(v, 4, h4, chunk_mix(h4, 4 * q), 4 * q, K, MK, s, shift, flags, c);
      store_quad<W>(lane_base_for<W>(args, r, q), q, c);
    }
    // d % 4 tail elements: one thread writes whole bytes, zero-padded
    if (threadIdx.x == 0 && nquad * 4 < d) {
      int32_t c[4] = {0, 0, 0, 0};
      T tv[4] = {T(0), T(0), T(0), T(0)};
      const int tc = static_cast<int>(d - nquad * 4);
      for (int e = 0; e < tc; ++e) tv[e] = x[nquad * 4 + e];
      quant_quad<KIND, W, T>(tv, tc, h4, chunk_mix(h4, nquad * 4), nquad * 4, K, MK, s, shift, flags, c);
      uint8_t* lb = static_cast<uint8_t*>(lane_base_for<W>(args, r, nquad));
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
  raise_flags_warp(args.err, flags);
  grid_done_signal(args.sig);
}

// 64-bit standard lanes (standard_lane_width, algorithm.cpp:22-29: the
// reference moves to int64 lanes when n(s+1) > 2^31, or when 64 bits are
// asked for). Every element takes the reference's f64 decision (slow_index:
// the f32 fast path needs s < 2^14, and s may be up to 2^32 - 1 here), the
// lane is sign * (s - idx) as a little-endian int64 (encode_dense_std,
// algorithm.cpp:69-82). One quad (32 lane bytes) per thread iteration; scatter
// mode and the grid-completion signal work as in quantize_kernel.
template <typename T>
__global__ void __launch_bounds__(kQThreads)
quantize64_kernel(const __grid_constant__ QuantArgs args) {
  pdl_wait();
  pdl_trigger();
  const uint64_t d = args.d;
  const uint32_t s = args.s;
  const uint32_t nl = args.n_local;
  const double norm = *args.norm;
  uint32_t flags = 0;
  if (!(norm >= 0.0) || !isfinite(norm)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_flag(args.err, GQ_FLAG_BAD_SCALE);
    grid_done_signal(args.sig);
    return;
  }
  __shared__ uint64_t s_h4[kMaxWorkers];
  for (uint32_t i = threadIdx.x; i < nl; i += kQThreads)
    s_h4[i] = args.round_ptr ? hoist_prefix(args.seed, 1ull, args.wid[i], *args.round_ptr) : args.h4[i];
  __syncthreads();
  const uint64_t nq = (d + 3) / 4;  // quads, the last one possibly partial
  const uint64_t total = nq * nl;
  for (uint64_t g = blockIdx.x * static_cast<uint64_t>(kQThreads) + threadIdx.x; g < total;
       g += static_cast<uint64_t>(gridDim.x) * kQThreads) {
    const uint32_t r = static_cast<uint32_t>(g / nq);
    const uint64_t q = g - static_cast<uint64_t>(r) * nq;
    const T* x = static_cast<const T*>(args.x[r]);
    const uint64_t h4 = s_h4[r];
    int64_t c[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint64_t j = 4 * q + e;
      c[e] = 0;
      if (j >= d) continue;
      const T v = x[j];
      if (norm == 0.0) {  // quantizer.cpp:21-32: all idx = s (lane 0); every element must be zero
        if (v != T(0)) flags |= GQ_FLAG_ZERO_SCALE;
        continue;
      }
      const double ad = Abs<T>::dbl(v);
      if (!isfinite(ad)) {
        flags |= GQ_FLAG_NONFINITE;
        continue;
      }
      if (ad > norm) flags |= GQ_FLAG_EXCEEDS_SCALE;
      const uint32_t idx = slow_index<0>(ad, norm, mix64(h4 ^ j), s);
      const int64_t mag = static_cast<int64_t>(s) - static_cast<int64_t>(idx);
      c[e] = Abs<T>::neg(v) ? -mag : mag;
    }
    int64_t* out = static_cast<int64_t*>(lane_base_for<64>(args, r, q)) + 4 * q;
    if (4 * q + 4 <= d) {
      reinterpret_cast<longlong2*>(out)[0] = make_longlong2(c[0], c[1]);
      reinterpret_cast<longlong2*>(out)[1] = make_longlong2(c[2], c[3]);
    } else {
      for (int e = 0; 4 * q + e < d; ++e) out[e] = c[e];
    }
  }
  raise_flags_warp(args.err, flags);
  grid_done_signal(args.sig);
}

template <typename T>
cudaError_t launch_q64(const QuantArgs& a, cudaStream_t st) {
  const uint64_t units = (a.d + 3) / 4 * a.n_local;
  uint64_t blocks = (units + kQThreads - 1) / kQThreads;
  if (blocks > 148ull * 8) blocks = 148ull * 8;
  if (blocks == 0) blocks = 1;
  const cudaError_t e = launch_maybe_pdl(quantize64_kernel<T>, static_cast<uint32_t>(blocks), kQThreads, 0, st, a);
  return e != cudaSuccess ? e : cudaGetLastError();
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
  const int per_sm = (g_quant_ctas_per_sm > 0 && g_quant_ctas_per_sm < blocks_per_sm) ? g_quant_ctas_per_sm
                                                                                     : blocks_per_sm;
  uint64_t blocks = static_cast<uint64_t>(sms) * per_sm * GQ_QWAVES;
  if (blocks > work_chunks) blocks = work_chunks;
  if (blocks == 0) blocks = 1;
  const cudaError_t e = launch_maybe_pdl(fn, static_cast<uint32_t>(blocks), kQThreads, smem, st, a);
  return e != cudaSuccess ? e : cudaGetLastError();
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
    a.wid[i] = q.worker_ids[i];
  }
  a.round_ptr = q.round_ptr;
  a.seed = q.seed;
  a.nslices = q.nslices;
  a.slice_quads = q.slice_lanes / 4;
  a.row_bytes = q.row_bytes;
  if (q.wait) {
    a.pw = *q.wait;
    a.fold = q.fold;
  }
  if (q.signal) {
    for (uint32_t i = 0; i < q.signal->n; ++i) a.sig.slots[i] = q.signal->slots[i];
    a.sig.n = q.signal->n;
    a.sig.epoch = q.signal->epoch;
    a.sig.ep_dev = q.signal->ep_dev;
    a.sig.ticket = q.signal->ticket;
  }
  for (uint32_t i = 0; i < q.nslices; ++i) a.sdst[i] = q.slice_dst[i];
  a.d = q.d;
  a.norm = q.norm;
  a.err = q.err;
  a.s = q.s;
  uint32_t shift = 0;
  for (uint64_t p = 1; p < 2ull * q.n_total; p <<= 1) ++shift;  // prescale_shift
  a.shift = shift;
  a.mk = GQ_MULCONSTS_INIT;
  if (q.width < 32) {
    a.pk[0] = 1u << q.width;
    a.pk[1] = 1u << (2 * q.width);
    a.pk[2] = q.width < 16 ? 1u << (3 * q.width) : 0u;
  }
  a.n_local = q.n_local;
  // work units for the grid: whole staged chunks over all local workers
  // (at least one per worker so the remainder/tail loop has an owner)
#ifndef GQ_QMIN_CHUNKS
#define GQ_QMIN_CHUNKS 4  // staged chunks per warp at least (small d: fewer, fuller CTAs)
#endif
  uint64_t work = ((q.d / 4 / kWarpQ) * q.n_local + (kQThreads / 32) * GQ_QMIN_CHUNKS - 1) /
                  ((kQThreads / 32) * GQ_QMIN_CHUNKS);
  if (work < q.n_local) work = q.n_local;
  if (q.width == 64) {
    if (q.kind != 0 || a.pw.n) return cudaErrorInvalidValue;
    return q.dtype == GQ_DTYPE_F32 ? launch_q64<float>(a, stream) : launch_q64<double>(a, stream);
  }
  if (q.dtype == GQ_DTYPE_F32) {
    return q.kind == 0 ? launch_w<float, 0>(a, work, q.width, stream)
                       : launch_w<float, 1>(a, work, q.width, stream);
  }
  return q.kind == 0 ? launch_w<double, 0>(a, work, q.width, stream)
                     : launch_w<double, 1>(a, work, q.width, stream);
}

}  // namespace gqb
