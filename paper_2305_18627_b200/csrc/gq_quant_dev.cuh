// Device-side pieces of the quantizer (quantize_shard + lane encoding), shared
// by the quantize kernels (gq_quantize.cu) and the fused small-d sync kernel
// (gq_reduce.cu). Reference semantics and the fast / exact decision scheme are
// described in gq_quantize.cu and DESIGN.md §4.
#pragma once

#include <cuda_runtime.h>

#include "gq_common.cuh"
#include "gq_internal.h"

namespace gqb {
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
#ifndef GQ_QUNROLL  // quads per lane per staged chunk (default geometry; see gq_quantize.cu launch_w)
#define GQ_QUNROLL 4
#endif
#ifndef GQ_QSTAGES  // TMA stages per warp (default geometry): 3 x 2 KiB (f32)
#define GQ_QSTAGES 3
#endif
#ifndef GQ_QMINBLOCKS
#define GQ_QMINBLOCKS 3
#endif
constexpr int kQThreads = 256;

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
#ifndef GQ_QTAB_SHR  // 1: the dither shift H >> 9 on the ALU pipe (an IMAD.HI otherwise): C2 175 -> 169 us
#define GQ_QTAB_SHR 1
#endif
#ifndef GQ_QTAB_ESHR  // 1: the exponent field R >> 23 on the ALU pipe (an IMAD.HI otherwise)
#define GQ_QTAB_ESHR 0
#endif
  const uint32_t R = yb + 0x7fffffu - (GQ_QTAB_SHR ? (H >> 9) : mulhi(H, MK.p23));  // carry = round up
#ifndef GQ_QTAB_LEA  // 1: the boundary-distance word (R << 9) + mq on the ALU pipe (an IMAD otherwise)
#define GQ_QTAB_LEA 0
#endif
  slow = ((GQ_QTAB_LEA ? (R << 9) + K.mq : mad_lo(R, MK.c512, K.mq)) <= 2u * K.mq) || yb >= K.ythr;
  uint32_t idx;  // (E << 1) | sign(x)
  asm("shf.l.clamp.b32 %0, %1, %2, 1;" : "=r"(idx) : "r"(vbits), "r"(GQ_QTAB_ESHR ? (R >> 23) : mulhi(R, MK.p9)));
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
#ifndef GQ_QSTD_RAWMUL  // 1: raw = zi >> (23 - k) as an IMAD.HI by 2^(9 + k) (multiply pipe)
#define GQ_QSTD_RAWMUL 0
#endif
  const float t = a * K.c;
  const float z = t + __uint_as_float(K.ybase - (H >> K.ysh));  // 2^k + 1 + t + (1 - u~)
  const uint32_t zi = __float_as_uint(z);
  const uint32_t raw = GQ_QSTD_RAWMUL ? mulhi(zi, K.zmul) : zi >> K.zsh;
#ifndef GQ_QSTD_SHL  // 1: the boundary-distance word zi << (9 + k) on the ALU pipe (an IMAD otherwise)
#define GQ_QSTD_SHL 0
#endif
  slow = ((GQ_QSTD_SHL ? (zi << K.ysh) + K.mq : mad_lo(zi, K.zmul, K.mq)) <= 2u * K.mq) || raw >= K.cm + K.s_lim;
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

}  // namespace
}  // namespace gqb
