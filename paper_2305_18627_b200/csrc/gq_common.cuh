// Shared device helpers for the Global-QSGD sm_100a kernels.
//
// Reference semantics cited per helper (paths under /root/reference/proj).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "gq_b200.h"

namespace gqb {

// ---------------------------------------------------------------------------
// Counter RNG (rng.hpp:20-61). bits(stream,a,b,c) = mix64 applied five times;
// the first four depend only on (seed, stream, a, b) and are hoisted to the
// host (hoist_prefix below), so each element pays one mix64.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// mix64(mix64(mix64(mix64(seed ^ K) ^ stream) ^ a) ^ b): the prefix shared by
// every draw of one (stream, a, b) triple (rng.hpp:45-53).
__host__ __device__ __forceinline__ uint64_t hoist_prefix(uint64_t seed,
                                                          uint64_t stream,
                                                          uint64_t a,
                                                          uint64_t b) {
  uint64_t h = mix64(seed ^ 0x517cc1b727220a95ull);
  h = mix64(h ^ stream);
  h = mix64(h ^ a);
  return mix64(h ^ b);
}

// ---------------------------------------------------------------------------
// Issue-balanced mix64 for the hot loops. Both hot kernels are bound by the
// integer ALU pipe (LOP3/SHF/IADD3 issue at half rate), so the 64-bit
// xor-shifts are rewritten as multiplies by 2^(32-r), which run on the
// multiply (FMA-heavy) pipe:
//   (hi:lo) >> r  =  ( hi*2^(32-r) + umulhi(lo, 2^(32-r)) ,  umulhi(hi, 2^(32-r)) )
// The multipliers come from a runtime struct so ptxas cannot strength-reduce
// them back into shifts. Only the high word of the final state is formed:
// (bits >> 32) = H ^ (H >> 31) with H = hi32(z * C2), so
//   bits >> 41 == H >> 9      (the 23 dither bits the fast path uses)
//   clz(bits >> 32) == clz(H) (the geometric k draw, exp_arith.cpp:43-50)
// Verified against the reference mix64 by tests/test_gpu_rng.py (gq_rng_draws).
// ---------------------------------------------------------------------------
struct MulConsts {
  uint32_t one, four, thirtytwo, two;  // runtime 1, 4, 32, 2
  uint32_t p9, p23, c512, neg1;        // runtime 2^9, 2^23, 512, 0xffffffff
};
#define GQ_MULCONSTS_INIT MulConsts{1u, 4u, 32u, 2u, 1u << 9, 1u << 23, 512u, 0xffffffffu}

// Multiply-pipe forms of shifts by constants (operands from MulConsts so
// ptxas keeps them as IMAD.HI): (a * k) >> 32.
__device__ __forceinline__ uint32_t mulhi(uint32_t a, uint32_t k) {
  uint32_t r;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(k));
  return r;
}
__device__ __forceinline__ uint32_t mad_hi(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
__device__ __forceinline__ uint32_t mad_lo(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}

__device__ __forceinline__ void shr_xor32(uint32_t& lo, uint32_t& hi, uint32_t mul) {
  const uint64_t w = static_cast<uint64_t>(lo) * mul;
  const uint32_t slo = hi * mul + static_cast<uint32_t>(w >> 32);
  const uint32_t shi = __umulhi(hi, mul);
  lo ^= slo;
  hi ^= shi;
}

// H = hi32 of (state before the last xor-shift) of mix64(x), x = (xh:xl).
// Written in PTX so every step is one IMAD-class or LOP3 instruction:
// 4 wide multiplies, 9 32-bit multiply(-add)s, 1 add, 4 xors.
__device__ __forceinline__ uint32_t mix64_hi(uint32_t xl, uint32_t xh, const MulConsts& K) {
  uint32_t h;
  asm("{\n\t"
      ".reg .u64 t, w, p;\n\t"
      ".reg .u32 lo, hi, th, wl, wh, s1, s2, pl, ph;\n\t"
      // z = x + 0x9e3779b97f4a7c15
      "mad.wide.u32 t, %1, %3, 0x9e3779b97f4a7c15;\n\t"
      "mov.b64 {lo, th}, t;\n\t"
      "add.u32 hi, %2, th;\n\t"
      // z ^= z >> 30   (multiplies by 4)
      "mul.wide.u32 w, lo, %4;\n\t"
      "mov.b64 {wl, wh}, w;\n\t"
      "mad.lo.u32 s1, hi, %4, wh;\n\t"
      "mul.hi.u32 s2, hi, %4;\n\t"
      "xor.b32 lo, lo, s1;\n\t"
      "xor.b32 hi, hi, s2;\n\t"
      // z *= 0xbf58476d1ce4e5b9
      "mul.wide.u32 p, lo, 0x1ce4e5b9;\n\t"
      "mov.b64 {pl, ph}, p;\n\t"
      "mad.lo.u32 ph, lo, 0xbf58476d, ph;\n\t"
      "mad.lo.u32 ph, hi, 0x1ce4e5b9, ph;\n\t"
      // z ^= z >> 27   (multiplies by 32)
      "mul.wide.u32 w, pl, %5;\n\t"
      "mov.b64 {wl, wh}, w;\n\t"
      "mad.lo.u32 s1, ph, %5, wh;\n\t"
      "mul.hi.u32 s2, ph, %5;\n\t"
      "xor.b32 lo, pl, s1;\n\t"
      "xor.b32 hi, ph, s2;\n\t"
      // hi32(z * 0x94d049bb133111eb)
      "mul.hi.u32 %0, lo, 0x133111eb;\n\t"
      "mad.lo.u32 %0, lo, 0x94d049bb, %0;\n\t"
      "mad.lo.u32 %0, hi, 0x133111eb, %0;\n\t"
      "}"
      : "=r"(h)
      : "r"(xl), "r"(xh), "r"(K.one), "r"(K.four), "r"(K.thirtytwo));
  return h;
}

// ---------------------------------------------------------------------------
// mix64 of a group of G consecutive keys x = key ^ (j0 + i), j0 % G == 0,
// sharing the high word: with b = (keylo & ~(G-1)) ^ j0lo and B = b + C0lo,
// member i has z0lo = B + (i ^ (keylo & (G-1))), and while B <= 2^32 - G all
// members share the carry into z0hi, hence z0hi, (z0 ^ z0 >> 30)hi and its
// product with C1lo (K1). elem_mix then costs 13 instructions per member.
// Measured pipe costs (profiles/r1/pipes_microbench.txt): ALU ops and IMAD
// 64/clk/SM, IMAD.HI 32/clk/SM; GQ_T30_ALU / GQ_T27_ALU pick the pipe of the
// two constant shifts. Returns H = hi32 of the last product (see mix64_hi).
// ---------------------------------------------------------------------------
#ifndef GQ_T30_ALU
#define GQ_T30_ALU 1
#endif
#ifndef GQ_T27_ALU
#define GQ_T27_ALU 1
#endif
#ifndef GQ_ADD_IMAD
#define GQ_ADD_IMAD 0
#endif
struct QuadMix {
  uint32_t B, zh2, K1;
  bool ok;
};

// Per (worker, 512-element chunk) constants of the quad-shared mix64: the
// high word of x = h4 ^ j is fixed within a chunk, so z0hi, (z0 ^ z0 >> 30)hi
// and its product with C1lo take one of two values, selected per quad by the
// carry out of the low-word add.
__device__ __forceinline__ uint32_t elem_mix(const QuadMix& q, uint32_t ce, const MulConsts& MK) {
  uint32_t h;
  // 13 instructions: 7 ALU-pipe (IADD, 2 SHF, 4 LOP3 fused to 3) and
  // IMAD, IMAD.HI(+K1), IMAD, IMAD.HI, 2 IMAD on the multiply pipe.
  asm("{\n\t"
      ".reg .u32 zl, t, pl, ph, f, ql, qh;\n\t"
#if GQ_ADD_IMAD
      "mad.lo.u32 zl, %2, %7, %1;\n\t"       // B + ce on the multiply pipe (runtime 1)
#else
      "add.u32 zl, %1, %2;\n\t"
#endif
#if GQ_T30_ALU
      "shr.u32 t, zl, 30;\n\t"                 // zl >> 30 (ALU pipe)
#else
      "mul.hi.u32 t, zl, %5;\n\t"              // zl >> 30 (multiply pipe)
#endif
      "xor.b32 zl, zl, t;\n\t"
      "xor.b32 zl, zl, %3;\n\t"                // ^ (zh << 2)
      "mul.lo.u32 pl, zl, 0x1ce4e5b9;\n\t"     // z *= C1: low word
      "mad.hi.u32 ph, zl, 0x1ce4e5b9, %4;\n\t" //          high word, + zh' * C1lo
      "mad.lo.u32 ph, zl, 0xbf58476d, ph;\n\t"
      "shf.r.clamp.b32 f, pl, ph, 27;\n\t"
      "xor.b32 ql, pl, f;\n\t"
#if GQ_T27_ALU
      "shr.u32 t, ph, 27;\n\t"                 // ph >> 27 (ALU pipe)
#else
      "mul.hi.u32 t, ph, %6;\n\t"              // ph >> 27 (multiply pipe)
#endif
      "xor.b32 qh, ph, t;\n\t"
      "mul.hi.u32 %0, ql, 0x133111eb;\n\t"
      "mad.lo.u32 %0, ql, 0x94d049bb, %0;\n\t"
      "mad.lo.u32 %0, qh, 0x133111eb, %0;\n\t"
      "}"
      : "=r"(h)
      : "r"(q.B), "r"(ce), "r"(q.zh2), "r"(q.K1), "r"(MK.four), "r"(MK.thirtytwo), "r"(MK.one));
  return h;
}

// Setup for a group of G consecutive indices (G a power of two <= 8).
template <int G>
__device__ __forceinline__ QuadMix group_mix(uint64_t key, uint64_t j0, uint32_t& lo) {
  QuadMix q;
  const uint32_t kl = static_cast<uint32_t>(key);
  lo = kl & (G - 1u);
  const uint32_t b = (kl & ~(G - 1u)) ^ static_cast<uint32_t>(j0);
  q.B = b + 0x7f4a7c15u;
  const uint32_t cy = q.B < b ? 1u : 0u;
  q.ok = q.B <= 0xffffffffu - (G - 1u);
  const uint32_t zh = (static_cast<uint32_t>(key >> 32) ^ static_cast<uint32_t>(j0 >> 32)) + 0x9e3779b9u + cy;
  q.zh2 = zh << 2;
  q.K1 = (zh ^ (zh >> 30)) * 0x1ce4e5b9u;
  return q;
}

// Out-of-line k draws for the (probability ~G 2^-32) word whose lanes do not
// share the mix64 carry; kept out of the hot loop so it is never if-converted.
static __device__ __noinline__ uint32_t mix64_hi_generic(uint32_t kl, uint32_t kh, const MulConsts& MK) {
  return mix64_hi(kl, kh, MK);
}

template <int W>
__device__ __noinline__ uint32_t k_word_generic(uint32_t kl, uint32_t kh, int kcap, const MulConsts& MK) {
  constexpr int G = 32 / W;
  uint32_t kw = 0;
  for (int i = 0; i < G; ++i) {
    const int kc = __clz(mix64_hi(kl ^ static_cast<uint32_t>(i), kh, MK)) + 1;
    kw |= static_cast<uint32_t>(kc < kcap ? kc : kcap) << (i * W);
  }
  return kw;
}

// The packed k draws of one lane word for one TokenReduceOps event
// (collectives.cpp:132-146): field i = min(m, clz(H_i) + 1) capped to the
// field (k > diff only matters for diff <= 2^(W-1) - 2), H_i the high word of
// mix64(key ^ (j0 + i)), key = the event's prefix mix64^4(seed, ReduceDraw,
// round, step<<32|dst). A pure function of (key, lane): the reduce kernel
// evaluates it in place, or reads it from a buffer the norm pass filled.
#ifndef GQ_KW_MAD
#define GQ_KW_MAD 1
#endif
#ifndef GQ_KW_LEA
#define GQ_KW_LEA 0
#endif
template <int W>
struct Swar1 {  // one in every W-bit field
  static constexpr uint32_t v() {
    uint32_t x = 0;
    for (int i = 0; i < 32 / W; ++i) x |= 1u << (i * W);
    return x;
  }
  static constexpr uint32_t value = v();
};

template <int W>
__device__ __forceinline__ uint32_t token_kword(uint64_t key, uint64_t j0, uint32_t m, const MulConsts& MK) {
  constexpr int G = 32 / W;
  const int kcap = static_cast<int>(m) < (1 << (W - 1)) - 1 ? static_cast<int>(m) : (1 << (W - 1)) - 1;
  uint32_t lo;
  const QuadMix q = group_mix<G>(key, j0, lo);
  if (__builtin_expect(q.ok, 1)) {
#if GQ_KW_MAD
    // k = min(clz(H) + 1, kcap) = 32 - bfind(H | 2^(32 - kcap)), so the packed
    // word is sum_i (32 - p_i) 2^(iW) = 32 ONE - sum_i p_i 2^(iW): one
    // multiply-add per lane on the IMAD pipe instead of min / shift / or.
    // (kcap > 32: no cap bit; H = 0 then gives p = -1, k = 33 = clz(0) + 1 as the reference)
    const uint32_t capbit = kcap <= 32 ? 1u << (32 - kcap) : 0u;
    uint32_t kw = 32u * Swar1<W>::value;  // mod 2^32; the true result fits
#pragma unroll
    for (int i = 0; i < G; ++i) {
      uint32_t p;
      asm("bfind.u32 %0, %1;" : "=r"(p) : "r"(elem_mix(q, static_cast<uint32_t>(i) ^ lo, MK) | capbit));
      kw = mad_lo(p, 0u - (1u << (i * W)), kw);
    }
    return kw;
#else
    uint32_t kw = 0;
#pragma unroll
    for (int i = 0; i < G; ++i) {
      const int kc = __clz(elem_mix(q, static_cast<uint32_t>(i) ^ lo, MK)) + 1;
      kw |= static_cast<uint32_t>(kc < kcap ? kc : kcap) << (i * W);
    }
    return kw;
#endif
  }
  return k_word_generic<W>(static_cast<uint32_t>(key) ^ static_cast<uint32_t>(j0),
                           static_cast<uint32_t>(key >> 32) ^ static_cast<uint32_t>(j0 >> 32), kcap, MK);
}

// token_kword for a run of words under one event key: the key's part of
// group_mix (its low bits, and for each carry the high-word products, which
// depend on the key and on the lane index's high word only) is formed once
// per run, so a word costs its G element hashes plus a handful of selects.
template <int W>
struct KeyMix {
  uint32_t klm, lo, jh;       // key low word & ~(G-1), key low word & (G-1), j0 >> 32 of the run
  uint32_t zh2[2], K1[2];
  uint64_t key;
};

template <int W>
__device__ __forceinline__ KeyMix<W> key_mix(uint64_t key, uint32_t jh) {
  constexpr int G = 32 / W;
  KeyMix<W> k;
  const uint32_t kl = static_cast<uint32_t>(key);
  k.key = key;
  k.klm = kl & ~(G - 1u);
  k.lo = kl & (G - 1u);
  k.jh = jh;
#pragma unroll
  for (int cy = 0; cy < 2; ++cy) {
    const uint32_t zh = (static_cast<uint32_t>(key >> 32) ^ jh) + 0x9e3779b9u + static_cast<uint32_t>(cy);
    k.zh2[cy] = zh << 2;
    k.K1[cy] = (zh ^ (zh >> 30)) * 0x1ce4e5b9u;
  }
  return k;
}

// token_kword(k.key, (k.jh << 32) | j0lo, m) bit for bit (j0lo % G == 0).
template <int W>
__device__ __forceinline__ uint32_t token_kword_km(const KeyMix<W>& k, uint32_t j0lo, uint32_t m,
                                                   const MulConsts& MK) {
  constexpr int G = 32 / W;
  const int kcap = static_cast<int>(m) < (1 << (W - 1)) - 1 ? static_cast<int>(m) : (1 << (W - 1)) - 1;
  QuadMix q;
  const uint32_t b = k.klm ^ j0lo;
  q.B = b + 0x7f4a7c15u;
  const bool cy = q.B < b;
  q.ok = q.B <= 0xffffffffu - (G - 1u);
  q.zh2 = cy ? k.zh2[1] : k.zh2[0];
  q.K1 = cy ? k.K1[1] : k.K1[0];
  if (__builtin_expect(q.ok, 1)) {
    const uint32_t capbit = kcap <= 32 ? 1u << (32 - kcap) : 0u;
#if GQ_KW_LEA  // sum_i p_i 2^(iW) with shift-adds on the ALU pipe, then one subtract
    uint32_t sp = 0;
#pragma unroll
    for (int i = 0; i < G; ++i) {
      uint32_t p;
      asm("bfind.u32 %0, %1;" : "=r"(p) : "r"(elem_mix(q, static_cast<uint32_t>(i) ^ k.lo, MK) | capbit));
      sp += p << (i * W);
    }
    return 32u * Swar1<W>::value - sp;
#else
    uint32_t kw = 32u * Swar1<W>::value;
#pragma unroll
    for (int i = 0; i < G; ++i) {
      uint32_t p;
      asm("bfind.u32 %0, %1;" : "=r"(p) : "r"(elem_mix(q, static_cast<uint32_t>(i) ^ k.lo, MK) | capbit));
      kw = mad_lo(p, 0u - (1u << (i * W)), kw);
    }
    return kw;
#endif
  }
  return k_word_generic<W>(static_cast<uint32_t>(k.key) ^ j0lo, static_cast<uint32_t>(k.key >> 32) ^ k.jh, kcap,
                           MK);
}

// Items it = e * kwords + wi, it in [it0, it1) with stride `stride` (wi < 2^32):
// buf[it] = token_kword(keys[e], (w0 + wi) G, m). keys may be in shared memory.
template <int W>
__device__ __forceinline__ void kdraw_run(uint32_t* buf, uint64_t kwords, uint64_t w0, uint32_t m,
                                          const uint64_t* keys, uint64_t it0, uint64_t it1, uint32_t stride,
                                          const MulConsts& MK) {
  constexpr int G = 32 / W;
  if (it0 >= it1) return;
  if (kwords + stride >= (1ull << 32)) {  // 32-bit word cursor would wrap: the plain loop
    for (uint64_t it = it0; it < it1; it += stride) {
      const uint32_t e = static_cast<uint32_t>(it / kwords);
      buf[it] = token_kword<W>(keys[e], (w0 + (it - static_cast<uint64_t>(e) * kwords)) * G, m, MK);
    }
    return;
  }
  uint32_t e = static_cast<uint32_t>(it0 / kwords);
  uint32_t wi = static_cast<uint32_t>(it0 - static_cast<uint64_t>(e) * kwords);
  uint64_t j0 = (w0 + wi) * G;
  KeyMix<W> k = key_mix<W>(keys[e], static_cast<uint32_t>(j0 >> 32));
  const uint32_t kw32 = static_cast<uint32_t>(kwords);
  uint32_t* out = buf + it0;
  for (uint64_t left = (it1 - it0 + stride - 1) / stride; left > 0; --left) {
    *out = token_kword_km<W>(k, static_cast<uint32_t>(j0), m, MK);
    out += stride;
    wi += stride;
    j0 += static_cast<uint64_t>(stride) * G;
    if (wi >= kw32) {  // the next event (or events, for a stride above kwords)
      do {
        wi -= kw32;
        ++e;
      } while (wi >= kw32);
      if (left > 1) {
        j0 = (w0 + wi) * G;
        k = key_mix<W>(keys[e], static_cast<uint32_t>(j0 >> 32));
      }
    } else if (static_cast<uint32_t>(j0 >> 32) != k.jh) {
      k = key_mix<W>(k.key, static_cast<uint32_t>(j0 >> 32));
    }
  }
}

// The 53-bit uniform of rng.hpp:58-61 as an exact double.
__device__ __forceinline__ double u01_from_bits(uint64_t bits) {
  return __dmul_rn(__ull2double_rn(bits >> 11), 0x1.0p-53);
}

// sample_k (exp_arith.cpp:43-50) straight from the raw bits:
// u = (bits >> 11) 2^-53, ilogb(u) = 10 - clz64(bits >> 11), so
// k = min(m, clz64(bits) + 1), and u == 0 (bits >> 11 == 0) gives m.
__device__ __forceinline__ uint32_t sample_k_bits(uint64_t bits, uint32_t m) {
  if ((bits >> 11) == 0) return m;
  const uint32_t k = static_cast<uint32_t>(__clzll(static_cast<long long>(bits))) + 1u;
  return k < m ? k : m;
}

// ---------------------------------------------------------------------------
// Device error flags (mapped to the reference's exception classes by the
// host; see include/gq_b200.h).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void raise_flag(uint32_t* err, uint32_t flag) {
  if (err) atomicOr(err, flag);
}

// Warp-aggregated flag raise: one atomic per warp that saw any flag.
__device__ __forceinline__ void raise_flags_warp(uint32_t* err, uint32_t flags) {
  const uint32_t any = __reduce_or_sync(0xffffffffu, flags);
  if (any && (threadIdx.x & 31) == 0 && err) atomicOr(err, any);
}

// ---------------------------------------------------------------------------
// Token arithmetic (exp_arith.cpp:82-109) on packed lanes
// [sign bit w-1][e in bits 0..w-2]. Returns the packed result lane.
// Zero operands pass the other through; two zeros give the canonical zero.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t reduce_pair_lane(uint32_t la, uint32_t lb,
                                                     uint32_t k, uint32_t sign_bit,
                                                     uint32_t& flags) {
  const uint32_t emask = sign_bit - 1u;
  const uint32_t ea = la & emask, eb = lb & emask;
  if (eb == 0) return ea == 0 ? 0u : la;
  if (ea == 0) return lb;
  const bool opposite = ((la ^ lb) & sign_bit) != 0;
  const int gap = ea > eb ? static_cast<int>(ea - eb) : static_cast<int>(eb - ea);
  const int diff = gap - (opposite ? 1 : 0);
  if (diff < 0) return 0u;  // equal magnitude, opposite sign: exact cancel
  const uint32_t sign_out = (ea <= eb ? la : lb) & sign_bit;
  const int e_min = static_cast<int>(ea <= eb ? ea : eb);
  const int bump = static_cast<int>(k) > diff ? 1 : 0;
  const int e_out = opposite ? e_min + bump : e_min - bump;
  if (e_out < 1 || e_out > static_cast<int>(emask)) {
    flags |= GQ_FLAG_TOKEN_RANGE;
    return 0u;
  }
  return static_cast<uint32_t>(e_out) | sign_out;
}

// ---------------------------------------------------------------------------
// Lane words. A 32-bit word holds 32/W lanes of W bits, lane i in bits
// [i*W, (i+1)*W) (little-endian; 4-bit lanes are nibbles, element 2i low).
// ---------------------------------------------------------------------------
template <int W>
__device__ __forceinline__ uint32_t lane_get(uint32_t word, int i) {
  if constexpr (W == 32) return word;
  else return (word >> (i * W)) & ((1u << W) - 1u);
}

template <int W>
__device__ __forceinline__ int32_t lane_sext(uint32_t lane) {
  if constexpr (W == 32) return static_cast<int32_t>(lane);
  else return static_cast<int32_t>(lane << (32 - W)) >> (32 - W);
}

// ---------------------------------------------------------------------------
// Bulk-copy (TMA 1-D, cp.async.bulk) + mbarrier helpers for staging streamed
// inputs through shared memory.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  while (!mbar_try_wait(bar, phase)) {
  }
}

// global -> shared bulk copy completing on `bar` (bytes % 16 == 0, 16 B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Host-visible limits.
constexpr int kMaxWorkers = GQ_MAX_WORKERS;

// Programmatic dependent launch: wait for the predecessor grid (and its
// memory) / let the successor grid be scheduled. No-ops without PDL.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

struct PtrArray {
  const void* p[kMaxWorkers];
};

// Device copy of a PeerSignal (gq_internal.h) and the grid-completion signal.
struct SignalArgs {
  uint32_t* slots[16];
  uint32_t n, epoch;
  const uint32_t* ep_dev;
  unsigned int* ticket;
};
__device__ __forceinline__ void grid_done_signal(const SignalArgs& sg) {
  if (sg.n == 0) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();  // this CTA's stores (peer memory included) before its ticket
    if (atomicAdd(sg.ticket, 1u) == gridDim.x - 1) {
      *sg.ticket = 0u;
      __threadfence_system();
      const uint32_t e = sg.ep_dev ? *sg.ep_dev : sg.epoch;
      for (uint32_t p = 0; p < sg.n; ++p)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(sg.slots[p]), "r"(e) : "memory");
    }
  }
}

// Spin (one thread) until every flag reached `epoch` (system-scope acquire),
// giving up after timeout_ns with GQ_FLAG_P2P_TIMEOUT; see PeerWait.
__device__ __forceinline__ void peer_wait_flags(const uint32_t* flags, uint32_t n, uint32_t epoch, uint32_t* err,
                                                uint64_t timeout_ns) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (uint32_t p = 0; p < n; ++p) {
    uint32_t v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + p) : "memory");
      if (static_cast<int32_t>(v - epoch) >= 0) break;
      uint64_t now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > timeout_ns) {
        raise_flag(err, GQ_FLAG_P2P_TIMEOUT);
        return;
      }
    }
  }
}

}  // namespace gqb
