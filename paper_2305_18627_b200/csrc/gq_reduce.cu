// Aggregate (+ fused decompress / SGD): replay the reference's allreduce
// schedule over n workers' lane buffers, per lane, on the device.
//
//   reference: collectives.cpp:155-190 (allreduce_inproc: walk the events,
//              dst = combine(dst, src) on chunk_lane_range), IntSumOps
//              (collectives.cpp:60-81: signed lanes, overflow throws),
//              TokenReduceOps (collectives.cpp:125-153: k from
//              u01(ReduceDraw, round, step<<32|dst, lane), sample_k,
//              reduce_pair exp_arith.cpp:43-50,82-109), tree/ring schedules
//              topology.cpp:19-72, decode algorithm.cpp:84-110, SGD
//              trainer.cpp:335.
//
// Every event of the reference touches whole chunks, and every lane's value
// depends only on that lane's inputs and keys, so the schedule can be
// evaluated lane by lane ("virtual schedule replay"):
//   tree: the reference's recursive halving is rebuilt with a binary-counter
//         stack over workers 0..n-1 (merge at step L into dst = left start);
//   ring: lane j's chunk c folds workers c, c+1, ... in ring order, step t
//         keyed (t, dst = c+t+1 mod n); the finished value is what the
//         allgather phase copies everywhere.
// Both give the bits of the sequential interpreter exactly; the integer sum
// also checks every partial sum for overflow as IntSumOps does.
//
// Work unit: one 32-bit lane word (32/w lanes) per worker per thread
// iteration, coalesced across the warp. Per-event RNG prefixes
// mix64^4(seed, ReduceDraw, round, step<<32|dst) live in shared memory, so a
// token reduce costs one mix64 per lane per event. The decode epilogue uses
// a shared-memory table of all 2^w lane codes (w <= 8) computed in f64 with
// the reference's formula, so the fp32 mean equals fl32(reference f64).
#include <cuda_runtime.h>

#include <cstdio>

#include "gq_common.cuh"
#include "gq_internal.h"
#include "gq_quant_dev.cuh"

namespace gqb {

int g_reduce_ctas_per_sm = 0;
int g_comm_wait = 0;
int g_comm_timeout_s = 60;
#ifndef GQ_PDL_DEFAULT
#define GQ_PDL_DEFAULT 0
#endif
int g_pdl = GQ_PDL_DEFAULT;
int g_small_path = 1;
int g_fused_path = 0;  // measured slower than the quantize + reduce kernels (scripts/fused_probe.py)
int g_comm_fold = 1;

namespace {

constexpr int kRThreads = 256;
constexpr int kMaxStack = 9;  // ceil(log2 128) + 2

struct ReduceArgs {
  const void* lanes[kMaxWorkers];
  uint32_t n;          // schedule workers
  uint32_t n_scale;    // decode divisor (job worker count)
  uint32_t s, m, shift;
  uint32_t topo;
  uint64_t d;
  uint64_t w_begin, w_end;  // word range
  uint64_t lane_end;
  uint64_t hround;     // mix64^3(seed, ReduceDraw, round)
  const double* norm;
  void* out_lanes;
  float* out_mean;
  float* param;
  float lr;
  bool param_vec;      // param 16-byte aligned: float4 SGD epilogue
  uint32_t* err;
  uint32_t key_mode;   // 0: none (int), 1: smem table, 2: on the fly
  MulConsts mk;
  const uint32_t* kpre;  // precomputed k words (KDrawJob layout, global word index) or null
  uint64_t kstride;      // words per event in kpre
  const uint64_t* round_ptr;  // non-null: hround from the device round (graph replays)
  uint64_t seed;
  void* out_peers[kMaxPeers];  // result lanes also stored to every peer (fused all_gather)
  uint32_t npeers;
  // graph replays: the last block to finish adds round_step to *round_inc
  // (every block has read the round by then), saving a one-thread launch
  uint64_t* round_inc;
  uint64_t round_step;
  unsigned int* ticket;  // zero-initialised; the last block resets it
  SignalArgs sig;        // n > 0: flag the peers when the whole grid is done (multicast mode)
  PeerWait pw;           // n > 0: folded exchange - wait for these flags before reading any lane
};

template <int W>
struct LaneOps {
  static constexpr int G = 32 / W;
  static constexpr uint32_t kSignBit = 1u << (W - 1);
};

// Token pair reduction for m <= 32 (exp_arith.cpp:82-109, branch-free):
// k = min(m, clz(H) + 1) where H is mix64_hi of the draw (sample_k from the
// raw bits, see gq_common.cuh), zero operands pass through, equal magnitude
// and opposite sign cancel, and a same-sign carry below e = 1 is the range
// error of exp_arith.cpp:103-107.
template <int W>
__device__ __forceinline__ uint32_t token_pair(uint32_t a, uint32_t b, uint32_t H, int m,
                                               uint32_t& flags) {
  constexpr uint32_t SB = 1u << (W - 1), EM = SB - 1u;
  const uint32_t ea = a & EM, eb = b & EM;
  const uint32_t emin = ea < eb ? ea : eb;
  const uint32_t emax = ea < eb ? eb : ea;
  const bool opp = ((a ^ b) & SB) != 0;
  const int diff = static_cast<int>(emax - emin) - (opp ? 1 : 0);
  const int kc = __clz(H) + 1;
  const int k = kc < m ? kc : m;
  const uint32_t bump = k > diff ? 1u : 0u;
  const uint32_t e_out = opp ? emin + bump : emin - bump;
  const uint32_t sign_out = (ea <= eb ? a : b) & SB;
  uint32_t out = diff < 0 ? 0u : (e_out | sign_out);
  if (!opp && e_out == 0 && emin != 0) flags |= GQ_FLAG_TOKEN_RANGE;
  out = (ea == 0) ? b : out;
  out = (eb == 0) ? (ea == 0 ? 0u : a) : out;
  return out;
}

// ---------------------------------------------------------------------------
// SWAR (SIMD within a register) forms of the two PayloadOps, operating on all
// 32/W fields of a lane word at once. Field layout [bit W-1: sign][e or value].
// Every intermediate is built so no field ever carries or borrows into its
// neighbour (each step is annotated with its per-field range).
// ---------------------------------------------------------------------------
template <int W>
#ifndef GQ_RBAL
#define GQ_RBAL 1
#endif
#ifndef GQ_TAB2
#define GQ_TAB2 0  // 4-bit decode: one lookup per lane pair
#endif
#ifndef GQ_NEGZ_SWAR
#define GQ_NEGZ_SWAR 1
#endif

struct Swar {
  static constexpr uint32_t field_ones() {
    uint32_t v = 0;
    for (int i = 0; i < 32 / W; ++i) v |= 1u << (i * W);
    return v;
  }
  static constexpr uint32_t ONE = field_ones();            // 0x11111111 / 0x01010101 / 0x00010001
  static constexpr uint32_t SM = ONE << (W - 1);           // sign bits
  static constexpr uint32_t EM = ~SM;                      // exponent / magnitude bits
  static constexpr uint32_t FIELD = (W == 32) ? 0xffffffffu : ((1u << W) - 1u);
};

// IntSumOps::combine (collectives.cpp:60-81) on all fields: signed W-bit add,
// overflow flagged per field (same-sign operands, result sign differs).
template <int W>
__device__ __forceinline__ uint32_t int_word_swar(uint32_t a, uint32_t b, uint32_t& flags) {
  using S = Swar<W>;
  // low W-1 bits add without crossing a field (max 2^W - 2), then the sign bits
  const uint32_t sum = ((a & S::EM) + (b & S::EM)) ^ ((a ^ b) & S::SM);
  if ((~(a ^ b) & (a ^ sum) & S::SM) != 0) flags |= GQ_FLAG_LANE_OVERFLOW;
  return sum;
}

// TokenReduceOps / reduce_pair (exp_arith.cpp:82-109) on all fields, given
// the per-field k draws packed in kw (1 <= k <= 2^(W-1) - 1).
template <int W>
__device__ __forceinline__ uint32_t token_word_swar(uint32_t a, uint32_t b, uint32_t kw,
                                                    uint32_t& flags, const MulConsts& MK = GQ_MULCONSTS_INIT) {
  using S = Swar<W>;
  // x - y on the multiply pipe (runtime -1 operand: ptxas keeps IMAD), to
  // offload the ALU pipe this SWAR code otherwise saturates
#if GQ_RBAL
  auto sub = [&](uint32_t x, uint32_t y) { return mad_lo(y, MK.neg1, x); };
#else
  auto sub = [](uint32_t x, uint32_t y) { return x - y; };
#endif
#if GQ_RBAL >= 2
  auto dec = [&](uint32_t x) { return mad_lo(x, MK.one, 0u - S::ONE); };  // x - ONE
#else
  auto dec = [](uint32_t x) { return x - S::ONE; };
#endif
  const uint32_t ea = a & S::EM, eb = b & S::EM;
  // ge: sign bit set where ea >= eb          (2^(W-1) + ea - eb in [1, 2^W - 1])
  const uint32_t ge = sub(ea | S::SM, eb) & S::SM;
  const uint32_t mge = (ge >> (W - 1)) * S::FIELD;
  const uint32_t emax = (ea & mge) | (eb & ~mge);
  const uint32_t emin = (eb & mge) | (ea & ~mge);
  const uint32_t gap = sub(emax, emin);                      // [0, 2^(W-1) - 1]
  const uint32_t opp = (a ^ b) & S::SM;                      // signs differ
  // bump = k > gap - opp  <=>  sign bit of 2^(W-1) - 1 + k + opp - gap
  const uint32_t t = sub(kw + (opp >> (W - 1)) + (S::SM - S::ONE), gap);  // [1, 2^W - 1]
  // gapnz: gap >= 1 (cancel = opp && gap == 0 gets no bump)
  const uint32_t gapnz = dec(gap | S::SM) & S::SM;
  const uint32_t bump_o = (t & opp & gapnz) >> (W - 1);
  const uint32_t bump_s = (t & ~opp & S::SM) >> (W - 1);
  const uint32_t eout = sub((emin | S::SM) + bump_o, bump_s);  // 2^(W-1) + e_out, e_out in [-1, emax]
  // sign of the operand with the smaller exponent (ties: same sign unless cancelled)
  uint32_t out = (eout & S::EM) | (((b & mge) | (a & ~mge)) & S::SM);
  const uint32_t cancel = opp & ~gapnz;
  out &= ~((cancel >> (W - 1)) * S::FIELD);
  // zero operands pass the other through; two zeros give the canonical zero
  const uint32_t nza = dec(ea | S::SM) & S::SM;
  const uint32_t nzb = dec(eb | S::SM) & S::SM;
  const uint32_t ma = (nza >> (W - 1)) * S::FIELD;
  const uint32_t mb = (nzb >> (W - 1)) * S::FIELD;
  uint32_t r = (out & mb) | (a & ~mb);
  r = (r & ma) | (b & ~ma);
  r &= (ma | mb);
  // exp_arith.cpp:103-107: same-sign carry below e = 1 (both operands nonzero)
  const uint32_t eo = eout & S::EM;
  const uint32_t eonz = dec(eo | S::SM) & S::SM;
  if ((nza & nzb & ~opp & ~eonz & ~cancel) != 0) flags |= GQ_FLAG_TOKEN_RANGE;
  return r;
}

// Combine two packed words lane-wise (acc = dst, in = src).
template <int KIND, int W, bool SMALLM>
__device__ __forceinline__ uint32_t combine_word(uint32_t acc, uint32_t in, uint64_t key,
                                                 uint64_t j0, uint32_t m, const MulConsts& MK,
                                                 uint32_t& flags) {
  constexpr int G = 32 / W;
  if constexpr (KIND == 0 && W < 32) {
    return int_word_swar<W>(acc, in, flags);
  } else if constexpr (KIND == 0) {
    const int64_t sum = static_cast<int64_t>(static_cast<int32_t>(acc)) + static_cast<int32_t>(in);
    if (sum > 2147483647ll || sum < -2147483648ll) flags |= GQ_FLAG_LANE_OVERFLOW;
    return static_cast<uint32_t>(sum);
  } else if constexpr (SMALLM) {
    // the G lanes of the word share the high word of their mix64 inputs
    // (group_mix, gq_common.cuh); the rare group whose low-word add straddles
    // 2^32 takes the generic per-lane hash
    if constexpr (W < 32) {
      return token_word_swar<W>(acc, in, token_kword<W>(key, j0, m, MK), flags, MK);
    } else {
      uint32_t lo;
      const QuadMix q = group_mix<G>(key, j0, lo);
      const uint32_t kl = static_cast<uint32_t>(key) ^ static_cast<uint32_t>(j0);
      const uint32_t kh = static_cast<uint32_t>(key >> 32) ^ static_cast<uint32_t>(j0 >> 32);
      const uint32_t H = __builtin_expect(q.ok, 1) ? elem_mix(q, lo, MK) : mix64_hi_generic(kl, kh, MK);
      return token_pair<W>(acc, in, H, static_cast<int>(m), flags);
    }
  } else {
    uint32_t out = 0;
#pragma unroll
    for (int i = 0; i < G; ++i) {
      const uint32_t a = lane_get<W>(acc, i), b = lane_get<W>(in, i);
      const uint64_t bits = mix64(key ^ (j0 + i));
      const uint32_t r = reduce_pair_lane(a, b, sample_k_bits(bits, m), 1u << (W - 1), flags);
      if constexpr (W == 32) out = r;
      else out |= (r & ((1u << W) - 1u)) << (i * W);
    }
    return out;
  }
}

__device__ __forceinline__ uint64_t event_key(const uint64_t* keys, uint32_t key_mode,
                                              uint64_t hround, uint32_t stride, uint32_t step,
                                              uint32_t dst) {
  if (key_mode == 1) return keys[step * stride + dst];
  return mix64(hround ^ ((static_cast<uint64_t>(step) << 32) | dst));
}

__host__ __device__ constexpr int ceil_log2_c(int v) { return v <= 1 ? 0 : 1 + ceil_log2_c((v + 1) / 2); }

// Index of tree event (step t, dst) in the reference's order (topology.cpp:28-35):
// all events of earlier steps, then dst / 2^(t+1) within step t.
__host__ __device__ constexpr int tree_events_before(int nt, int t) {
  int c = 0;
  for (int tt = 0; tt < t; ++tt)
    for (int r = 1 << tt; r < nt; r += 2 << tt) ++c;
  return c;
}
__host__ __device__ constexpr int tree_event_index(int nt, int t, int dst) {
  return tree_events_before(nt, t) + dst / (2 << t);
}

// Compile-time tree (NT workers): node [a, a + 2^L) merges its right half
// [a + 2^(L-1), ...) into a at step L-1 when that half is non-empty
// (topology.cpp:28-35: step t, span 2^t, src r, dst r - span). With KP the k
// draws of each event come from the precomputed buffer (KDrawJob).
template <int KIND, int W, bool SM, int NT, bool KP, int A0, int L>
__device__ __forceinline__ uint32_t tree_rec(const uint32_t (&words)[NT], const uint32_t (&kws)[NT],
                                             const ReduceArgs& A, const uint64_t* keys, uint64_t j0,
                                             uint32_t& flags) {
  if constexpr (L == 0) {
    return words[A0];
  } else {
    constexpr int HALF = 1 << (L - 1);
    if constexpr (A0 + HALF >= NT) {
      return tree_rec<KIND, W, SM, NT, KP, A0, L - 1>(words, kws, A, keys, j0, flags);
    } else {
      const uint32_t left = tree_rec<KIND, W, SM, NT, KP, A0, L - 1>(words, kws, A, keys, j0, flags);
      const uint32_t right = tree_rec<KIND, W, SM, NT, KP, A0 + HALF, L - 1>(words, kws, A, keys, j0, flags);
      if constexpr (KP && KIND == 1 && W < 32) {
        constexpr int E = tree_event_index(NT, L - 1, A0);
        return token_word_swar<W>(left, right, kws[E], flags, A.mk);
      } else {
        const uint64_t key = KIND == 1 ? event_key(keys, A.key_mode, A.hround, NT, L - 1, A0) : 0;
        return combine_word<KIND, W, SM>(left, right, key, j0, A.m, A.mk, flags);
      }
    }
  }
}

// Tree replay of one word position (topology.cpp:19-43 dataflow).
template <int KIND, int W, bool SM, int NT, bool KP = false>
__device__ __forceinline__ uint32_t tree_word(const ReduceArgs& A, uint64_t wi, const uint64_t* keys,
                                              uint32_t& flags) {
  constexpr int G = 32 / W;
  const uint64_t j0 = wi * G;
  if constexpr (NT > 0) {
    uint32_t words[NT], kws[NT];
#pragma unroll
    for (int r = 0; r < NT; ++r) words[r] = __ldg(static_cast<const uint32_t*>(A.lanes[r]) + wi);
    if constexpr (KP && KIND == 1 && W < 32) {
#pragma unroll
      for (int e = 0; e + 1 < NT; ++e) kws[e] = __ldcs(A.kpre + static_cast<uint64_t>(e) * A.kstride + wi);
    }
    return tree_rec<KIND, W, SM, NT, KP, 0, ceil_log2_c(NT)>(words, kws, A, keys, j0, flags);
  }
  const uint32_t n = A.n;
  uint32_t val[kMaxStack];
  uint32_t lvl[kMaxStack];
  uint32_t start[kMaxStack];
  int sp = 0;
  auto push = [&](uint32_t r, uint32_t word) {
    val[sp] = word;
    lvl[sp] = 0;
    start[sp] = r;
    ++sp;
    while (sp >= 2 && lvl[sp - 1] == lvl[sp - 2]) {
      const uint32_t L = lvl[sp - 2];
      const uint64_t key = KIND == 1 ? event_key(keys, A.key_mode, A.hround, n, L, start[sp - 2]) : 0;
      val[sp - 2] = combine_word<KIND, W, SM>(val[sp - 2], val[sp - 1], key, j0, A.m, A.mk, flags);
      lvl[sp - 2] = L + 1;
      --sp;
    }
  };
  for (uint32_t r = 0; r < n; ++r) push(r, __ldg(static_cast<const uint32_t*>(A.lanes[r]) + wi));
  while (sp >= 2) {
    const uint32_t L = lvl[sp - 2];
    const uint64_t key = KIND == 1 ? event_key(keys, A.key_mode, A.hround, n, L, start[sp - 2]) : 0;
    val[sp - 2] = combine_word<KIND, W, SM>(val[sp - 2], val[sp - 1], key, j0, A.m, A.mk, flags);
    lvl[sp - 2] = L + 1;
    --sp;
  }
  return val[0];
}

// V consecutive words (wi0 % V == 0, every buffer 16-byte aligned) of a
// compile-time tree: one V-word vector load per worker (and per k-draw event),
// then the per-word replay.
template <int V>
struct VecT;
template <>
struct VecT<2> {
  using type = uint2;
};
template <>
struct VecT<4> {
  using type = uint4;
};
template <int V>
__device__ __forceinline__ void load_vec(const uint32_t* p, uint32_t (&out)[V], bool stream) {
  using T = typename VecT<V>::type;
  const T t = stream ? __ldcs(reinterpret_cast<const T*>(p)) : __ldg(reinterpret_cast<const T*>(p));
  if constexpr (V == 2) {
    out[0] = t.x; out[1] = t.y;
  } else {
    out[0] = t.x; out[1] = t.y; out[2] = t.z; out[3] = t.w;
  }
}
template <int V>
__device__ __forceinline__ void store_vec(uint32_t* p, const uint32_t (&v)[V]) {
  if constexpr (V == 2) reinterpret_cast<uint2*>(p)[0] = make_uint2(v[0], v[1]);
  else reinterpret_cast<uint4*>(p)[0] = make_uint4(v[0], v[1], v[2], v[3]);
}

template <int KIND, int W, bool SM, int NT, bool KP, int V>
__device__ __forceinline__ void tree_group(const ReduceArgs& A, uint64_t wi0, const uint64_t* keys,
                                           uint32_t& flags, uint32_t (&res)[V]) {
  constexpr int G = 32 / W;
  uint32_t words[V][NT], kws[V][NT];
#pragma unroll
  for (int r = 0; r < NT; ++r) {
    uint32_t t[V];
    load_vec<V>(static_cast<const uint32_t*>(A.lanes[r]) + wi0, t, true);
#pragma unroll
    for (int v = 0; v < V; ++v) words[v][r] = t[v];
  }
  if constexpr (KP && KIND == 1 && W < 32) {
#pragma unroll
    for (int e = 0; e + 1 < NT; ++e) {
      uint32_t t[V];
      load_vec<V>(A.kpre + static_cast<uint64_t>(e) * A.kstride + wi0, t, true);
#pragma unroll
      for (int v = 0; v < V; ++v) kws[v][e] = t[v];
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v)
    res[v] = tree_rec<KIND, W, SM, NT, KP, 0, ceil_log2_c(NT)>(words[v], kws[v], A, keys, (wi0 + v) * G, flags);
}

// Ring replay (topology.cpp:45-72 dataflow) for lanes whose chunk is c.
template <int KIND, int W, bool SM>
__device__ __forceinline__ uint32_t ring_fold(const ReduceArgs& A, uint64_t wi, uint32_t c,
                                              const uint64_t* keys, uint32_t& flags) {
  constexpr int G = 32 / W;
  const uint32_t n = A.n;
  const uint64_t j0 = wi * G;
  uint32_t acc = __ldg(static_cast<const uint32_t*>(A.lanes[c]) + wi);
  uint32_t w = c;
  for (uint32_t t = 0; t + 1 < n; ++t) {
    w = (w + 1 == n) ? 0 : w + 1;
    const uint32_t dst_word = __ldg(static_cast<const uint32_t*>(A.lanes[w]) + wi);
    const uint64_t key = KIND == 1 ? event_key(keys, A.key_mode, A.hround, n, t, w) : 0;
    acc = combine_word<KIND, W, SM>(dst_word, acc, key, j0, A.m, A.mk, flags);
  }
  return acc;
}

// chunk_lane_range (topology.cpp:99-106) inverse: the chunk holding lane j
// when d lanes are cut into n chunks, c = ceil((j+1) n / d) - 1.
__device__ __forceinline__ uint32_t chunk_of(uint64_t j, uint32_t n, uint64_t d) {
  return static_cast<uint32_t>(((j + 1) * n - 1) / d);
}

// Decode + SGD epilogue of one result word (lanes j0 .. j0+G-1): the fp32
// mean from the 2^W-entry table (W <= 8, fl32 of the reference's f64 decode)
// or per lane, and x[j] -= eta * mean[j] (trainer.cpp:335).
template <int KIND, int W, bool kTab2>
__device__ __forceinline__ void decode_word(const ReduceArgs& A, uint64_t wi, uint32_t res, const float* tab,
                                            const float2* tab2, double norm, uint32_t& flags) {
  constexpr int G = 32 / W;
  const uint64_t j0 = wi * G;
  float v[G];
#if GQ_NEGZ_SWAR
  if constexpr (KIND == 1 && W < 32) {
    // any field == 2^(W-1) (negative zero, exp_arith.cpp:178-179): a zero
    // field of res ^ SM, by the borrow test on all fields at once
    using S = Swar<W>;
    const uint32_t z = res ^ S::SM;
    if (((z - S::ONE) & ~z & S::SM) != 0) flags |= GQ_FLAG_NEG_ZERO;
  }
#endif
  if constexpr (kTab2) {  // two lanes per lookup
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const float2 t = tab2[(res >> (8 * b)) & 0xffu];
      v[2 * b] = t.x;
      v[2 * b + 1] = t.y;
    }
  }
#pragma unroll
  for (int i = 0; i < G; ++i) {
    if constexpr (kTab2) break;
    const uint32_t c = lane_get<W>(res, i);
    if constexpr (KIND == 1 && (!GQ_NEGZ_SWAR || W == 32)) {
      if (c == (1u << (W - 1))) flags |= GQ_FLAG_NEG_ZERO;
    }
    if constexpr (W <= 8) {
      v[i] = tab[c];
    } else if constexpr (KIND == 0) {
      const double scale = __ddiv_rn(norm, __dmul_rn(static_cast<double>(A.n_scale), static_cast<double>(A.s)));
      v[i] = __double2float_rn(__dmul_rn(scale, static_cast<double>(lane_sext<W>(c))));
    } else {
      const uint32_t e = c & ((1u << (W - 1)) - 1u);
      const bool neg = (c >> (W - 1)) & 1u;
      v[i] = 0.0f;
      if (e != 0) {
        const double tv = ldexp(neg ? -1.0 : 1.0, static_cast<int>(A.shift) - static_cast<int>(e));
        v[i] = __double2float_rn(__ddiv_rn(__dmul_rn(norm, tv), static_cast<double>(A.n_scale)));
      }
    }
  }
  const bool full = j0 + G <= A.lane_end;
  if (A.out_mean) {
    if (full && (G % 4) == 0) {
#pragma unroll
      for (int i = 0; i < G; i += 4)
        __stcs(reinterpret_cast<float4*>(A.out_mean + j0) + i / 4, make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]));
    } else if (full && G == 2) {
      reinterpret_cast<float2*>(A.out_mean + j0)[0] = make_float2(v[0], v[1]);
    } else {
#pragma unroll
      for (int i = 0; i < G; ++i) if (j0 + i < A.lane_end) A.out_mean[j0 + i] = v[i];
    }
  }
  if (A.param) {
    // x[j] -= eta * estimate[j] (trainer.cpp:335), separate mul then sub.
    if ((G % 4) == 0 && full && A.param_vec) {
#pragma unroll
      for (int i = 0; i < G; i += 4) {
        float4* pp = reinterpret_cast<float4*>(A.param + j0) + i / 4;
        float4 p = *pp;
        p.x = __fsub_rn(p.x, __fmul_rn(A.lr, v[i]));
        p.y = __fsub_rn(p.y, __fmul_rn(A.lr, v[i + 1]));
        p.z = __fsub_rn(p.z, __fmul_rn(A.lr, v[i + 2]));
        p.w = __fsub_rn(p.w, __fmul_rn(A.lr, v[i + 3]));
        *pp = p;
      }
    } else {
#pragma unroll
      for (int i = 0; i < G; ++i) {
        if (j0 + i < A.lane_end) {
          const float p = A.param[j0 + i];
          A.param[j0 + i] = __fsub_rn(p, __fmul_rn(A.lr, v[i]));
        }
      }
    }
  }
}

// Warp-transposed decode (+ SGD) of 32·V consecutive result words starting
// at word wb, thread t holding words wb + V t .. wb + V t + V - 1 (4- and
// 8-bit lanes: F = G/4 float4s of output per word). One word per thread
// would make each float4 store cover only 1/(V F) of the sectors it touches;
// here store k of the V F stores has thread t write float4 32k + t of the
// warp's output, fetching that float4's word by shuffle, so every store
// (and SGD load) instruction covers 512 contiguous bytes. Values are the
// decode_word table entries, the same fp32 bits.
template <int KIND, int W, int V>
__device__ __forceinline__ void decode_warp(const ReduceArgs& A, uint64_t wb, const uint32_t (&res)[V],
                                            const float* tab, uint32_t& flags) {
  static_assert(W == 4 || W == 8, "warp decode: 4- and 8-bit lanes");
  constexpr int G = 32 / W, F = G / 4;
  const uint32_t lane = threadIdx.x & 31u;
  if constexpr (KIND == 1) {
    using S = Swar<W>;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const uint32_t z = res[v] ^ S::SM;
      if (((z - S::ONE) & ~z & S::SM) != 0) flags |= GQ_FLAG_NEG_ZERO;
    }
  }
#pragma unroll
  for (int k = 0; k < V * F; ++k) {
    const uint32_t f = 32u * k + lane;       // float4 of the warp's output
    const uint32_t q = f / F;                // its word, within the warp
    const uint32_t src = q / V, comp = q % V;
    uint32_t ww = 0;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const uint32_t x = __shfl_sync(0xffffffffu, res[v], src);
      if (comp == static_cast<uint32_t>(v)) ww = x;
    }
    if constexpr (F == 2) ww >>= (f & 1u) * 16u;
    constexpr uint32_t M = (1u << W) - 1u;
    const float4 val = make_float4(tab[ww & M], tab[(ww >> W) & M], tab[(ww >> (2 * W)) & M], tab[(ww >> (3 * W)) & M]);
    const uint64_t f4 = wb * F + f;
    if (A.out_mean) __stcs(reinterpret_cast<float4*>(A.out_mean) + f4, val);
    if (A.param) {
      // x[j] -= eta * estimate[j] (trainer.cpp:335), separate mul then sub.
      if (A.param_vec) {
        float4* pp = reinterpret_cast<float4*>(A.param) + f4;
        float4 p = *pp;
        p.x = __fsub_rn(p.x, __fmul_rn(A.lr, val.x));
        p.y = __fsub_rn(p.y, __fmul_rn(A.lr, val.y));
        p.z = __fsub_rn(p.z, __fmul_rn(A.lr, val.z));
        p.w = __fsub_rn(p.w, __fmul_rn(A.lr, val.w));
        *pp = p;
      } else {
        float* pp = A.param + f4 * 4;
        pp[0] = __fsub_rn(pp[0], __fmul_rn(A.lr, val.x));
        pp[1] = __fsub_rn(pp[1], __fmul_rn(A.lr, val.y));
        pp[2] = __fsub_rn(pp[2], __fmul_rn(A.lr, val.z));
        pp[3] = __fsub_rn(pp[3], __fmul_rn(A.lr, val.w));
      }
    }
  }
}

#ifndef GQ_RMINBLOCKS
#define GQ_RMINBLOCKS 4
#endif
#ifndef GQ_RVEC_INT  // words per thread group, integer lanes (1, 2 or 4)
#define GQ_RVEC_INT 2
#endif
#ifndef GQ_RDEC_ILP  // grid-stride words in flight per thread in the decode of summed lanes (n = 1, V = 1)
#define GQ_RDEC_ILP 8
#endif
#ifndef GQ_RDEC_WARP  // decode of summed 4/8-bit lanes: warp-shuffled words, each float4 store 512 contiguous bytes
#define GQ_RDEC_WARP 1
#endif
#ifndef GQ_RVEC_WARP  // the same in the V-word-group reduce (measured slower there: 0.0500 -> 0.0513 ms C2)
#define GQ_RVEC_WARP 0
#endif
#ifndef GQ_RVEC_DEC  // words per thread group, token-lane decode of summed lanes (n = 1)
#define GQ_RVEC_DEC 1
#endif
#ifndef GQ_RVEC_KP   // words per thread group, token lanes with precomputed k draws (1 or 2)
#define GQ_RVEC_KP 2
#endif
template <int KIND, int W, bool SM, int NT, int TOPO, bool KP = false, int V = 1>
__global__ void __launch_bounds__(kRThreads, GQ_RMINBLOCKS)
reduce_kernel(const __grid_constant__ ReduceArgs A) {
  pdl_wait();
  pdl_trigger();
  // folded exchange: the lanes come from peers (the __syncthreads below
  // orders every thread's reads after thread 0's system-scope acquire)
  if (A.pw.n && threadIdx.x == 0)
    peer_wait_flags(A.pw.flags, A.pw.n, A.pw.ep_dev ? *A.pw.ep_dev : A.pw.epoch, A.err, A.pw.timeout_ns);
  constexpr int G = 32 / W;
  extern __shared__ uint64_t smem[];
  float* tab = reinterpret_cast<float*>(smem);               // 2^W floats (W <= 8)
  // + a 256-entry table of lane pairs (the per-lane negative-zero test then
  // comes from the word-level check)
  constexpr bool kTab2 = GQ_TAB2 && W == 4 && (KIND == 0 || GQ_NEGZ_SWAR);
  float2* tab2 = reinterpret_cast<float2*>(smem + ((W <= 8) ? (1 << W) / 2 : 0));
  uint64_t* keys = smem + ((W <= 8) ? (1 << W) / 2 : 0) + (kTab2 ? 256 : 0);  // event prefixes
  uint32_t flags = 0;

  const bool decode = A.out_mean != nullptr || A.param != nullptr;
  double norm = 0.0;
  if (decode) norm = *A.norm;
  // ---- prologue: decode table + event keys ----
  if constexpr (W <= 8) {
    if (decode) {
      for (uint32_t c = threadIdx.x; c < (1u << W); c += blockDim.x) {
        float v;
        if constexpr (KIND == 0) {
          const double scale = __ddiv_rn(norm, __dmul_rn(static_cast<double>(A.n_scale), static_cast<double>(A.s)));
          v = __double2float_rn(__dmul_rn(scale, static_cast<double>(lane_sext<W>(c))));
        } else {
          const uint32_t e = c & ((1u << (W - 1)) - 1u);
          const bool neg = (c >> (W - 1)) & 1u;
          v = 0.0f;
          if (e != 0) {
            const double tv = ldexp(neg ? -1.0 : 1.0, static_cast<int>(A.shift) - static_cast<int>(e));
            v = __double2float_rn(__ddiv_rn(__dmul_rn(norm, tv), static_cast<double>(A.n_scale)));
          }
        }
        tab[c] = v;
      }
      if constexpr (kTab2) {
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < 256; b += blockDim.x) tab2[b] = make_float2(tab[b & 15], tab[b >> 4]);
      }
    }
  }
  if (KIND == 1 && A.key_mode == 1) {
    const uint64_t hround = A.round_ptr ? reduce_round_prefix(A.seed, *A.round_ptr) : A.hround;
    const uint32_t n = A.n;
    const uint32_t steps = TOPO == 0 ? 8 : (n > 1 ? n - 1 : 0);
    for (uint32_t i = threadIdx.x; i < steps * n; i += blockDim.x) {
      const uint32_t step = i / n, dst = i % n;
      keys[i] = mix64(hround ^ ((static_cast<uint64_t>(step) << 32) | dst));
    }
  }
  __syncthreads();

  auto epilogue = [&](uint64_t wi, uint32_t res) {
    decode_word<KIND, W, kTab2>(A, wi, res, tab, tab2, norm, flags);
  };

  // One word through the schedule (any topology), padding cleared, stored and decoded.
  auto one_word = [&](uint64_t wi) {
    const uint64_t j0 = wi * G;
    uint32_t res;
    if constexpr (TOPO == 0) {
      res = tree_word<KIND, W, SM, NT, KP>(A, wi, keys, flags);
    } else {
      const uint32_t c0 = chunk_of(j0, A.n, A.d);
      const uint64_t jl = (j0 + G - 1 < A.d) ? j0 + G - 1 : A.d - 1;
      const uint32_t c1 = chunk_of(jl, A.n, A.d);
      if (c0 == c1) {
        res = ring_fold<KIND, W, SM>(A, wi, c0, keys, flags);
      } else {
        // Word straddles a chunk boundary: fold each chunk's lanes apart.
        res = 0;
        for (uint32_t c = c0; c <= c1; ++c) {
          const uint32_t part = ring_fold<KIND, W, SM>(A, wi, c, keys, flags);
#pragma unroll
          for (int i = 0; i < G; ++i) {
            const uint64_t j = j0 + i;
            if (j < A.d && chunk_of(j, A.n, A.d) == c) {
              if constexpr (W == 32) res = part;
              else res |= lane_get<W>(part, i) << (i * W);
            }
          }
        }
      }
    }
    // Lanes past the end of the payload are padding: force them to zero.
    if (j0 + G > A.lane_end) {
#pragma unroll
      for (int i = 0; i < G; ++i)
        if (j0 + i >= A.lane_end) res &= ~(((W == 32) ? 0xffffffffu : ((1u << W) - 1u)) << (i * W));
    }
    if (A.out_lanes) static_cast<uint32_t*>(A.out_lanes)[wi] = res;
    for (uint32_t p = 0; p < A.npeers; ++p) static_cast<uint32_t*>(A.out_peers[p])[wi] = res;
    if (decode) epilogue(wi, res);
  };

  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * kRThreads + threadIdx.x;
  const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * kRThreads;
  if constexpr (V > 1 && TOPO == 0 && NT > 0) {
    // Whole V-word groups with vector loads/stores; the last group (it may
    // hold the payload's padding lanes) and the unaligned head words go
    // one word at a time.
    const uint64_t vb = min(A.w_end, (A.w_begin + V - 1) / V * V);
    const uint64_t last_full = A.lane_end / G;  // words below this hold no padding lanes
    const uint64_t ve = max(vb, min(A.w_end, last_full) / V * V);
    for (uint64_t g = vb / V + tid; g < ve / V; g += nthreads) {
      const uint64_t wi0 = g * V;
      uint32_t res[V];
      tree_group<KIND, W, SM, NT, KP, V>(A, wi0, keys, flags, res);
      if (A.out_lanes) store_vec<V>(static_cast<uint32_t*>(A.out_lanes) + wi0, res);
      for (uint32_t p = 0; p < A.npeers; ++p) store_vec<V>(static_cast<uint32_t*>(A.out_peers[p]) + wi0, res);
      if (decode) {
        if constexpr ((W == 4 || W == 8) && GQ_RVEC_WARP) {
          // the warp's 32 groups are all whole (warp-uniform test): the
          // shuffle-transposed epilogue
          const uint64_t g0 = g - (threadIdx.x & 31u);
          if (g0 + 32 <= ve / V) {
            decode_warp<KIND, W, V>(A, g0 * V, res, tab, flags);
            continue;
          }
        }
#pragma unroll
        for (int v = 0; v < V; ++v) epilogue(wi0 + v, res[v]);
      }
    }
    const uint64_t nhead = vb - A.w_begin, ntail = A.w_end - ve;
    for (uint64_t t = tid; t < nhead + ntail; t += nthreads) one_word(t < nhead ? A.w_begin + t : ve + (t - nhead));
  } else if constexpr (NT == 1 && TOPO == 0 && !KP && GQ_RDEC_ILP > 1) {
    // the decode of summed lanes (n = 1): one word per thread keeps the fp32
    // stores coalesced (a full 32-byte sector per thread for 4-bit lanes),
    // GQ_RDEC_ILP grid-stride iterations per pass put that many word loads in
    // flight before the table lookups
    constexpr int kU = GQ_RDEC_ILP;
    const uint32_t* src = static_cast<const uint32_t*>(A.lanes[0]);
    for (uint64_t wi = A.w_begin + tid; wi < A.w_end; wi += kU * nthreads) {
      uint32_t wv[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint64_t w = wi + u * nthreads;
        wv[u] = w < A.w_end ? __ldcs(src + w) : 0u;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint64_t w = wi + u * nthreads;
        if (w >= A.w_end) break;
        uint32_t res = wv[u];
        const uint64_t j0 = w * G;
        if (j0 + G > A.lane_end) {
#pragma unroll
          for (int i = 0; i < G; ++i)
            if (j0 + i >= A.lane_end) res &= ~(((W == 32) ? 0xffffffffu : ((1u << W) - 1u)) << (i * W));
        }
        if (A.out_lanes) static_cast<uint32_t*>(A.out_lanes)[w] = res;
        for (uint32_t p = 0; p < A.npeers; ++p) static_cast<uint32_t*>(A.out_peers[p])[w] = res;
        if (!decode) continue;
        if constexpr ((W == 4 || W == 8) && GQ_RDEC_WARP) {
          // whole warps of whole words: the shuffle-transposed epilogue
          const uint64_t wb = w - (threadIdx.x & 31u);
          if (wb + 32 <= A.w_end && (wb + 32) * G <= A.lane_end) {
            const uint32_t r1[1] = {res};
            decode_warp<KIND, W, 1>(A, wb, r1, tab, flags);
            continue;
          }
        }
        epilogue(w, res);
      }
    }
  } else {
    for (uint64_t wi = A.w_begin + tid; wi < A.w_end; wi += nthreads) one_word(wi);
  }
  raise_flags_warp(A.err, flags);
  if (A.round_inc) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(A.ticket, 1u) == gridDim.x - 1) {
        *A.round_inc += A.round_step;
        *A.ticket = 0;
      }
    }
  }
  grid_done_signal(A.sig);
}

// 64-bit IntSumOps lanes (collectives.cpp:60-81 with width_bits == 64: the
// int64 add itself must not overflow). One lane per thread; the schedule's
// partial sums are formed in the reference's order (tree: binary-counter
// stack, topology.cpp:28-35; ring: chunk c folds c+1, c+2, ...), so an
// overflow is detected exactly where the reference detects one.
__device__ __forceinline__ int64_t add64_checked(int64_t a, int64_t b, uint32_t& flags) {
  const int64_t sum = static_cast<int64_t>(static_cast<uint64_t>(a) + static_cast<uint64_t>(b));
  if (((a ^ sum) & (b ^ sum)) < 0) flags |= GQ_FLAG_LANE_OVERFLOW;
  return sum;
}

template <int TOPO>
__global__ void __launch_bounds__(kRThreads) reduce64_kernel(const __grid_constant__ ReduceArgs A) {
  pdl_wait();
  pdl_trigger();
  if (A.pw.n) {
    if (threadIdx.x == 0)
      peer_wait_flags(A.pw.flags, A.pw.n, A.pw.ep_dev ? *A.pw.ep_dev : A.pw.epoch, A.err, A.pw.timeout_ns);
    __syncthreads();
  }
  uint32_t flags = 0;
  const bool decode = A.out_mean != nullptr || A.param != nullptr;
  // decode_dense_std (algorithm.cpp:84-100): scale = norm / (double(n) s)
  const double scale =
      decode ? __ddiv_rn(*A.norm, __dmul_rn(static_cast<double>(A.n_scale), static_cast<double>(A.s))) : 0.0;
  const uint32_t n = A.n;
  for (uint64_t j = A.w_begin + static_cast<uint64_t>(blockIdx.x) * kRThreads + threadIdx.x; j < A.w_end;
       j += static_cast<uint64_t>(gridDim.x) * kRThreads) {
    auto lane = [&](uint32_t r) { return __ldg(static_cast<const long long*>(A.lanes[r]) + j); };
    int64_t res;
    if constexpr (TOPO == 0) {
      int64_t val[kMaxStack];
      uint32_t lvl[kMaxStack];
      int sp = 0;
      for (uint32_t r = 0; r < n; ++r) {
        val[sp] = lane(r);
        lvl[sp] = 0;
        ++sp;
        while (sp >= 2 && lvl[sp - 1] == lvl[sp - 2]) {
          val[sp - 2] = add64_checked(val[sp - 2], val[sp - 1], flags);
          ++lvl[sp - 2];
          --sp;
        }
      }
      while (sp >= 2) {
        val[sp - 2] = add64_checked(val[sp - 2], val[sp - 1], flags);
        --sp;
      }
      res = val[0];
    } else {
      uint32_t w = chunk_of(j, n, A.d);
      res = lane(w);
      for (uint32_t t = 0; t + 1 < n; ++t) {
        w = (w + 1 == n) ? 0 : w + 1;
        res = add64_checked(lane(w), res, flags);
      }
    }
    if (A.out_lanes) static_cast<long long*>(A.out_lanes)[j] = res;
    for (uint32_t p = 0; p < A.npeers; ++p) static_cast<long long*>(A.out_peers[p])[j] = res;
    if (decode) {
      const float v = __double2float_rn(__dmul_rn(scale, static_cast<double>(res)));
      if (A.out_mean) A.out_mean[j] = v;
      if (A.param) A.param[j] = __fsub_rn(A.param[j], __fmul_rn(A.lr, v));  // trainer.cpp:335
    }
  }
  raise_flags_warp(A.err, flags);
  if (A.round_inc) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(A.ticket, 1u) == gridDim.x - 1) {
        *A.round_inc += A.round_step;
        *A.ticket = 0;
      }
    }
  }
  grid_done_signal(A.sig);
}

// Persistent grid: one wave of resident blocks per launch (queried once per
// instantiation), grid-striding over the lane words.
template <typename F>
cudaError_t launch_persistent(F* fn, const ReduceArgs& a, uint64_t words, size_t smem, cudaStream_t st) {
  static int blocks_per_sm = 0;
  static int sms = 0;
  if (blocks_per_sm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, fn, kRThreads, 48 * 1024);
    if (e != cudaSuccess) return e;
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  uint64_t blocks = (words + kRThreads - 1) / kRThreads;
  const int per_sm = (g_reduce_ctas_per_sm > 0 && g_reduce_ctas_per_sm < blocks_per_sm) ? g_reduce_ctas_per_sm
                                                                                       : blocks_per_sm;
  const uint64_t wave = static_cast<uint64_t>(sms) * per_sm;
  if (blocks > wave) blocks = wave;
  if (blocks == 0) blocks = 1;
  const cudaError_t e = launch_maybe_pdl(fn, static_cast<uint32_t>(blocks), kRThreads, smem, st, a);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int KIND, int W>
cudaError_t launch_kind_w(const ReduceArgs& a, uint64_t words, size_t smem, cudaStream_t st) {
  if (KIND == 1 && a.m > 32) {  // wide k draws: generic 64-bit sample_k, dynamic paths
    if (a.topo == GQ_TOPO_RING) return launch_persistent(reduce_kernel<KIND, W, false, 0, 1>, a, words, smem, st);
    return launch_persistent(reduce_kernel<KIND, W, false, 0, 0>, a, words, smem, st);
  }
  if (a.topo == GQ_TOPO_RING) return launch_persistent(reduce_kernel<KIND, W, true, 0, 1>, a, words, smem, st);
  // vector groups: the lane / result / mean pointers are
  // 16-byte aligned by the API; precomputed k words also need an aligned base
  // and event stride
  constexpr int VI = GQ_RVEC_INT;
  if constexpr (KIND == 1 && W <= 8) {
    if (a.kpre) {  // k draws precomputed by the norm pass
      const bool kv = (reinterpret_cast<uintptr_t>(a.kpre) % 8) == 0 && a.kstride % 2 == 0;
      switch (a.n) {
        case 2: return kv ? launch_persistent(reduce_kernel<KIND, W, true, 2, 0, true, GQ_RVEC_KP>, a, words, smem, st)
                          : launch_persistent(reduce_kernel<KIND, W, true, 2, 0, true>, a, words, smem, st);
        case 4: return kv ? launch_persistent(reduce_kernel<KIND, W, true, 4, 0, true, GQ_RVEC_KP>, a, words, smem, st)
                          : launch_persistent(reduce_kernel<KIND, W, true, 4, 0, true>, a, words, smem, st);
        case 8: return kv ? launch_persistent(reduce_kernel<KIND, W, true, 8, 0, true, GQ_RVEC_KP>, a, words, smem, st)
                          : launch_persistent(reduce_kernel<KIND, W, true, 8, 0, true>, a, words, smem, st);
        default: break;
      }
    }
  }
  constexpr int VN = KIND == 0 ? VI : 1;
  switch (a.n) {
    // n = 1 (the decode of already-summed lanes): no k draws, vector groups for both kinds
    case 1: return launch_persistent(reduce_kernel<KIND, W, true, 1, 0, false, (KIND == 0 ? VI : GQ_RVEC_DEC)>, a,
                                     words, smem, st);
    case 2: return launch_persistent(reduce_kernel<KIND, W, true, 2, 0, false, VN>, a, words, smem, st);
    case 4: return launch_persistent(reduce_kernel<KIND, W, true, 4, 0, false, VN>, a, words, smem, st);
    case 8: return launch_persistent(reduce_kernel<KIND, W, true, 8, 0, false, VN>, a, words, smem, st);
    default: return launch_persistent(reduce_kernel<KIND, W, true, 0, 0>, a, words, smem, st);
  }
}

template <int KIND>
cudaError_t launch_kind(const ReduceArgs& a, uint32_t width, uint64_t words, size_t smem, cudaStream_t st) {
  switch (width) {
    case 4: return launch_kind_w<KIND, 4>(a, words, smem, st);
    case 8: return launch_kind_w<KIND, 8>(a, words, smem, st);
    case 16: return launch_kind_w<KIND, 16>(a, words, smem, st);
    case 32: return launch_kind_w<KIND, 32>(a, words, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_generic(ReduceArgs& a, uint32_t kind, uint32_t width, uint64_t lane_begin,
                           uint64_t lane_end, cudaStream_t stream) {
  if (width == 64) {  // one int64 lane per "word"
    if (kind != 0) return cudaErrorInvalidValue;
    a.w_begin = lane_begin;
    a.w_end = lane_end;
    a.lane_end = lane_end;
    if (lane_end <= lane_begin) return cudaSuccess;
    a.key_mode = 0;
    a.mk = GQ_MULCONSTS_INIT;
    return a.topo == GQ_TOPO_RING ? launch_persistent(reduce64_kernel<1>, a, lane_end - lane_begin, 0, stream)
                                  : launch_persistent(reduce64_kernel<0>, a, lane_end - lane_begin, 0, stream);
  }
  const uint32_t G = 32 / width;
  a.w_begin = lane_begin / G;
  a.w_end = (lane_end + G - 1) / G;
  a.lane_end = lane_end;
  if (a.w_end <= a.w_begin) return cudaSuccess;
  size_t smem = (width <= 8) ? (size_t{1} << width) * sizeof(float) : 0;
  smem = (smem + 7) & ~size_t{7};
  if (GQ_TAB2 && width == 4) smem += 256 * sizeof(float2);
  a.key_mode = 0;
  a.mk = GQ_MULCONSTS_INIT;
  if (kind == 1) {
    const uint32_t steps = a.topo == GQ_TOPO_TREE ? 8 : (a.n > 1 ? a.n - 1 : 0);
    const size_t kbytes = size_t{steps} * a.n * sizeof(uint64_t);
    if (kbytes <= 40 * 1024) {
      a.key_mode = 1;
      smem += kbytes;
    } else {
      if (a.round_ptr) return cudaErrorInvalidValue;  // device rounds need the shared key table
      a.key_mode = 2;
    }
  }
  const uint64_t words = a.w_end - a.w_begin;
  return kind == 0 ? launch_kind<0>(a, width, words, smem, stream)
                   : launch_kind<1>(a, width, words, smem, stream);
}

// ---- the whole in-process sync for small d, one cooperative launch ----
// For small gradients (C1: 4 x 2^20) the three-kernel step is bound by
// launch ramps and short per-kernel grids, not by HBM or the integer pipes.
// mean_small_kernel runs the same phases in one resident grid separated by
// grid barriers: (1) L-inf shard norms (max of |x| bit patterns, exact in any
// order) into per-worker atomics; (2) every CTA folds the n stats in the
// reference's tree order (collectives.cpp:210-233); (3) quantize_shard +
// encode of every quad (gq_quant_dev.cuh, the same decisions as
// quantize_kernel); (4) the schedule replay + decode (+ SGD) of every lane
// word (tree_word, decode_word). Results are bit-identical to the
// multi-kernel path.
struct SmallArgs {
  const float* x[16];
  uint64_t h4[16];            // quantize RNG prefixes mix64^4(seed, Dither, w, round) (host rounds)
  const uint64_t* round_ptr;  // non-null: the round from the device (graph replays) ...
  uint64_t* round_inc;        // ... advanced by 1 once the grid is done
  uint64_t seed;
  uint32_t p;                 // norm p (combine: max or L2)
  double* stats_out;
  double* norm_out;
  unsigned int* bar;          // zeroed grid-barrier counter; the last CTA resets it
  unsigned int* done;         // zeroed completion ticket
  uint32_t* maxbits;          // zeroed per-worker max |x| bits (16)
  MulConsts mk;
  uint32_t pk[3];
  ReduceArgs R;               // lanes, schedule, decode / SGD outputs (n, s, m, shift, hround, ...)
};

__device__ __forceinline__ void small_grid_barrier(unsigned int* bar, unsigned int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

#ifndef GQ_SMALL_TIMING
#define GQ_SMALL_TIMING 0
#endif
#ifndef GQ_SMALL_ILP  // quantize items per thread iteration in mean_small_kernel
#define GQ_SMALL_ILP 4
#endif
#if GQ_SMALL_TIMING
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

#ifndef GQ_SMALL_MINB  // resident CTAs per SM asked of the register allocator
#define GQ_SMALL_MINB 1
#endif
template <int KIND, int W, int NT>
__global__ void __launch_bounds__(256, GQ_SMALL_MINB) mean_small_kernel(const __grid_constant__ SmallArgs A) {
  constexpr int G = 32 / W;
#if GQ_SMALL_TIMING
  uint64_t tm[6];
  tm[0] = gtimer();
#endif
  const ReduceArgs& R = A.R;
  const uint32_t n = R.n;
  const uint64_t d = R.d;
  const uint64_t nquad = d / 4;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint32_t flags = 0;
  __shared__ uint32_t s_red[8];
  __shared__ double s_norm;
  __shared__ double s_st[16];
  __shared__ uint64_t s_h4[16];
  __shared__ uint8_t s_qtab[kQtabBytes<KIND>];
  __shared__ float s_tab[1 << W];
  __shared__ uint64_t s_keys[8 * 8];

  // ---- (1) per-worker max |x| bit patterns (NaN/Inf sort above every finite) ----
  {
    const uint32_t bpw = gridDim.x / n;  // blocks per worker (gridDim.x >= n)
    const uint32_t r = blockIdx.x % n, part = blockIdx.x / n;
    uint32_t mb = 0;
    if (part < bpw) {
      const float4* xv = reinterpret_cast<const float4*>(A.x[r]);
#pragma unroll 4
      for (uint64_t q = static_cast<uint64_t>(part) * blockDim.x + threadIdx.x; q < nquad;
           q += static_cast<uint64_t>(bpw) * blockDim.x) {
        const float4 f = __ldg(xv + q);
        mb = max(mb, max(max(__float_as_uint(f.x) & 0x7fffffffu, __float_as_uint(f.y) & 0x7fffffffu),
                         max(__float_as_uint(f.z) & 0x7fffffffu, __float_as_uint(f.w) & 0x7fffffffu)));
      }
      if (part == 0)
        for (uint64_t j = nquad * 4 + threadIdx.x; j < d; j += blockDim.x)
          mb = max(mb, __float_as_uint(A.x[r][j]) & 0x7fffffffu);
    }
    mb = __reduce_max_sync(0xffffffffu, mb);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = mb;
    __syncthreads();
    if (threadIdx.x == 0 && part < bpw) {
      uint32_t m = 0;
      for (int w = 0; w < 8; ++w) m = max(m, s_red[w]);
      atomicMax(A.maxbits + r, m);
    }
  }
#if GQ_SMALL_TIMING
  tm[1] = gtimer();
#endif
  small_grid_barrier(A.bar, gridDim.x);
#if GQ_SMALL_TIMING
  tm[2] = gtimer();
#endif

  // ---- (2) stats (local_norm_stat, norms.cpp:52-62) and the tree fold ----
  if (threadIdx.x == 0) {
    bool bad = false;
    for (uint32_t w = 0; w < n; ++w) {
      const uint32_t m = __ldcg(A.maxbits + w);
      bad |= m >= 0x7f800000u;
      const double nq = static_cast<double>(__uint_as_float(m));
      s_st[w] = (A.p == GQ_NORM_INF) ? nq : __dmul_rn(nq, nq);
      if (blockIdx.x == 0 && A.stats_out) A.stats_out[w] = s_st[w];
    }
    if (bad && blockIdx.x == 0) raise_flag(R.err, GQ_FLAG_NONFINITE);
    const double nm = tree_fold_stats(s_st, n, A.p);
    s_norm = nm;
    if (blockIdx.x == 0 && A.norm_out) *A.norm_out = nm;
  }
  const uint64_t round = A.round_ptr ? *A.round_ptr : 0;
  __shared__ ChunkMix s_cm[16];
  if (threadIdx.x < n) {
    const uint64_t h = A.round_ptr ? hoist_prefix(A.seed, 1ull, threadIdx.x, round) : A.h4[threadIdx.x];
    s_h4[threadIdx.x] = h;
    s_cm[threadIdx.x] = chunk_mix(h, 0);  // j < 2^32 on this path
  }
  __syncthreads();
  const double norm = s_norm;

  // ---- (3) quantize + encode (quantizer.cpp:8-48, algorithm.cpp:69-82 / exp_arith.cpp:126-160) ----
  const uint32_t s = R.s, shift = R.shift;
  const MulConsts MK = A.mk;
  const bool zero_norm = norm == 0.0, bad_norm = !(norm >= 0.0) || !isfinite(norm);
  const QConst K = make_const<KIND>(zero_norm || bad_norm ? 1.0 : norm, s, shift);
  if constexpr (KIND == 1) build_exp_tab<W>(s_qtab, s, shift);
  else build_std_tab<W>(s_qtab, s, K.cm);
  __syncthreads();
  if (bad_norm) {
    if (tid == 0) raise_flag(R.err, GQ_FLAG_BAD_SCALE);
  } else {
    // the same partition as phase 1: CTA b quantizes a contiguous range of
    // worker (b mod n)'s quads (that CTA just read them, so they sit in L2),
    // kIl quads per thread iteration with their loads issued together; the
    // worker's pointers and hash constants stay in registers
    constexpr int kIl = GQ_SMALL_ILP;
    const uint32_t bpw = gridDim.x / n, r = blockIdx.x % n, part = blockIdx.x / n;
    if (part < bpw) {
      const uint64_t per = (nquad + bpw - 1) / bpw;
      const uint64_t q0 = min(nquad, per * part), q1 = min(nquad, q0 + per);
      const float4* xv = reinterpret_cast<const float4*>(A.x[r]);
      void* lanes = const_cast<void*>(R.lanes[r]);
      const uint64_t h4 = s_h4[r];
      const ChunkMix cm = s_cm[r];
      for (uint64_t base = q0 + threadIdx.x; base < q1; base += kIl * blockDim.x) {
        float4 f[kIl];
#pragma unroll
        for (int k = 0; k < kIl; ++k) {
          const uint64_t q = base + k * blockDim.x;
          f[k] = q < q1 ? __ldg(xv + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < kIl; ++k) {
          const uint64_t q = base + k * blockDim.x;
          if (q >= q1) break;
          const float v[4] = {f[k].x, f[k].y, f[k].z, f[k].w};
          int32_t c[4];
          if (zero_norm) {  // quantizer.cpp:21-32: all idx = s; a nonzero element is an error
            for (int e = 0; e < 4; ++e) {
              c[e] = 0;
              if (v[e] != 0.0f) flags |= GQ_FLAG_ZERO_SCALE;
            }
            store_quad_mad<W>(lanes, q, c, A.pk);
          } else {
            bool any = !K.fast;
            fast_quad<KIND, W>(v, cm, static_cast<uint32_t>(4 * q), K, MK, s, shift, s_qtab, any, c);
            if (!any) {
              store_quad_mad<W>(lanes, q, c, A.pk);  // table lanes: W-bit values, packed with multiply-adds
            } else {  // exact decisions; signed standard lanes need the masked pack
              quant_quad<KIND, W, float>(v, 4, h4, cm, 4 * q, K, MK, s, shift, flags, c);
              store_quad<W, KIND == 1>(lanes, q, c);
            }
          }
        }
      }
    }
    for (uint32_t r = 0; r < n; ++r) {
      const float* x = A.x[r];
      void* lanes = const_cast<void*>(R.lanes[r]);
      const uint64_t h4 = s_h4[r];
      if (tid == 0 && nquad * 4 < d) {  // d % 4 tail: whole bytes, zero-padded
        int32_t c[4] = {0, 0, 0, 0};
        float tv[4] = {0.f, 0.f, 0.f, 0.f};
        const int tc = static_cast<int>(d - nquad * 4);
        for (int e = 0; e < tc; ++e) tv[e] = x[nquad * 4 + e];
        if (zero_norm) {
          for (int e = 0; e < tc; ++e) if (tv[e] != 0.0f) flags |= GQ_FLAG_ZERO_SCALE;
        } else {
          quant_quad<KIND, W, float>(tv, tc, h4, chunk_mix(h4, nquad * 4), nquad * 4, K, MK, s, shift, flags, c);
        }
        uint8_t* lb = static_cast<uint8_t*>(lanes);
        const uint64_t b0 = nquad * 4 * W / 8, nb = ((d - nquad * 4) * W + 7) / 8;
        uint32_t packed = 0;
        for (int e = 0; e < 4; ++e) packed |= (static_cast<uint32_t>(c[e]) & ((1u << W) - 1u)) << (e * W);
        for (uint64_t bb = 0; bb < nb; ++bb) lb[b0 + bb] = static_cast<uint8_t>(packed >> (8 * bb));
      }
    }
  }
#if GQ_SMALL_TIMING
  tm[3] = gtimer();
#endif
  small_grid_barrier(A.bar, 2 * gridDim.x);
#if GQ_SMALL_TIMING
  tm[4] = gtimer();
#endif

  // ---- (4) schedule replay (collectives.cpp:155-190) + decode (+ SGD) ----
  const bool decode = R.out_mean != nullptr || R.param != nullptr;
  if (decode) {
    for (uint32_t c = threadIdx.x; c < (1u << W); c += blockDim.x) {
      float v;
      if constexpr (KIND == 0) {
        const double scale = __ddiv_rn(norm, __dmul_rn(static_cast<double>(R.n_scale), static_cast<double>(R.s)));
        v = __double2float_rn(__dmul_rn(scale, static_cast<double>(lane_sext<W>(c))));
      } else {
        const uint32_t e = c & ((1u << (W - 1)) - 1u);
        const bool neg = (c >> (W - 1)) & 1u;
        v = 0.0f;
        if (e != 0) {
          const double tv = ldexp(neg ? -1.0 : 1.0, static_cast<int>(R.shift) - static_cast<int>(e));
          v = __double2float_rn(__ddiv_rn(__dmul_rn(norm, tv), static_cast<double>(R.n_scale)));
        }
      }
      s_tab[c] = v;
    }
  }
  if constexpr (KIND == 1) {
    const uint64_t hround = A.round_ptr ? reduce_round_prefix(A.seed, round) : R.hround;
    for (uint32_t i = threadIdx.x; i < 8 * n; i += blockDim.x)
      s_keys[i] = mix64(hround ^ ((static_cast<uint64_t>(i / n) << 32) | (i % n)));
  }
  __syncthreads();
  // whole groups of kSV words with one 16-byte load per worker (the grid is
  // small, so per-thread memory parallelism sets this phase's time); the
  // words past the last whole group, padding lanes included, one at a time
  // (integer lanes only: a token word's seven hashed events are already a
  // thread's worth of work, and grouping them starves the small grids)
  constexpr int kSV = KIND == 0 ? 4 : 1;
  const uint64_t last_full = R.lane_end / G;
  const uint64_t w_vec_end = kSV == 1 ? 0 : (R.w_end < last_full ? R.w_end : last_full) / kSV * kSV;
  const bool vec_out = (reinterpret_cast<uintptr_t>(R.out_lanes) & 15) == 0;
  for (uint64_t wi0 = tid * kSV; kSV > 1 && wi0 < w_vec_end; wi0 += nthreads * kSV) {
    uint32_t res[kSV > 1 ? kSV : 2];
    tree_group<KIND, W, true, NT, false, (kSV > 1 ? kSV : 2)>(R, wi0, s_keys, flags, res);
    if (R.out_lanes) {
      if (vec_out) {
        store_vec<(kSV > 1 ? kSV : 2)>(static_cast<uint32_t*>(R.out_lanes) + wi0, res);
      } else {
#pragma unroll
        for (int v = 0; v < kSV; ++v) static_cast<uint32_t*>(R.out_lanes)[wi0 + v] = res[v];
      }
    }
    if (decode) {
#pragma unroll
      for (int v = 0; v < kSV; ++v) decode_word<KIND, W, false>(R, wi0 + v, res[v], s_tab, nullptr, norm, flags);
    }
  }
  for (uint64_t wi = w_vec_end + tid; wi < R.w_end; wi += nthreads) {
    const uint64_t j0 = wi * G;
    uint32_t res = tree_word<KIND, W, true, NT>(R, wi, s_keys, flags);
    if (j0 + G > R.lane_end) {
#pragma unroll
      for (int i = 0; i < G; ++i)
        if (j0 + i >= R.lane_end) res &= ~(((1u << W) - 1u) << (i * W));
    }
    if (R.out_lanes) static_cast<uint32_t*>(R.out_lanes)[wi] = res;
    if (decode) decode_word<KIND, W, false>(R, wi, res, s_tab, nullptr, norm, flags);
  }
  raise_flags_warp(R.err, flags);
#if GQ_SMALL_TIMING
  tm[5] = gtimer();
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1))
    printf("small cta %u: t0 %llu norm %.2f bar1 %.2f quant %.2f bar2 %.2f reduce %.2f us\n", blockIdx.x,
           static_cast<unsigned long long>(tm[0] % 1000000000ull),
           (tm[1] - tm[0]) * 1e-3, (tm[2] - tm[1]) * 1e-3, (tm[3] - tm[2]) * 1e-3, (tm[4] - tm[3]) * 1e-3,
           (tm[5] - tm[4]) * 1e-3);
#endif

  // ---- the last CTA leaves the workspace zeroed and advances a device round ----
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(A.done, 1u) == gridDim.x - 1) {
      for (uint32_t w = 0; w < n; ++w) A.maxbits[w] = 0;
      *A.bar = 0;
      *A.done = 0;
      if (A.round_inc) *A.round_inc += 1;
      __threadfence();
    }
  }
}

template <int KIND, int W, int NT>
cudaError_t launch_small_nt(const SmallArgs& a, uint64_t work_threads, cudaStream_t st) {
  auto* fn = mean_small_kernel<KIND, W, NT>;
  static int per_sm = 0, sms = 0;
  if (per_sm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
#ifdef GQ_SMALL_CTAS_PER_SM
    if (per_sm > GQ_SMALL_CTAS_PER_SM) per_sm = GQ_SMALL_CTAS_PER_SM;
#endif
  }
  uint64_t grid = (work_threads + 255) / 256;
  const uint64_t cap = static_cast<uint64_t>(sms) * per_sm;  // every CTA resident (grid barriers)
  if (grid > cap) grid = cap;
  if (grid < a.R.n) grid = a.R.n;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<uint32_t>(grid));
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, fn, a);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int KIND, int W>
cudaError_t launch_small_w(const SmallArgs& a, uint64_t work, cudaStream_t st) {
  switch (a.R.n) {
    case 2: return launch_small_nt<KIND, W, 2>(a, work, st);
    case 4: return launch_small_nt<KIND, W, 4>(a, work, st);
    case 8: return launch_small_nt<KIND, W, 8>(a, work, st);
    default: return cudaErrorInvalidValue;
  }
}

// ---- uncompressed fp32 baseline (algorithm.cpp:303-340, tree order) ----
// Vectorised form for a compile-time worker count: one float4 of every
// worker per thread (N 128-bit streaming loads in flight), the same tree
// order per element, a 128-bit store.
template <int N>
__global__ void __launch_bounds__(256) baseline_tree_v4_kernel(PtrArray x, uint64_t d4, float* out) {
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < d4;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    float4 v[N];
#pragma unroll
    for (int r = 0; r < N; ++r) v[r] = __ldcs(static_cast<const float4*>(x.p[r]) + j);
#pragma unroll
    for (int span = 1; span < N; span <<= 1)
#pragma unroll
      for (int r = span; r < N; r += 2 * span) {
        v[r - span].x = __fadd_rn(v[r - span].x, v[r].x);
        v[r - span].y = __fadd_rn(v[r - span].y, v[r].y);
        v[r - span].z = __fadd_rn(v[r - span].z, v[r].z);
        v[r - span].w = __fadd_rn(v[r - span].w, v[r].w);
      }
    const double dn = static_cast<double>(N);
    float4 o;
    o.x = static_cast<float>(static_cast<double>(v[0].x) / dn);
    o.y = static_cast<float>(static_cast<double>(v[0].y) / dn);
    o.z = static_cast<float>(static_cast<double>(v[0].z) / dn);
    o.w = static_cast<float>(static_cast<double>(v[0].w) / dn);
    __stcs(reinterpret_cast<float4*>(out) + j, o);
  }
}

__global__ void baseline_tree_kernel(PtrArray x, uint32_t n, uint64_t d, float* out) {
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < d;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    float v[kMaxWorkers];
    for (uint32_t r = 0; r < n; ++r) v[r] = static_cast<const float*>(x.p[r])[j];
    for (uint32_t span = 1; span < n; span <<= 1)
      for (uint32_t r = span; r < n; r += 2 * span) v[r - span] = __fadd_rn(v[r - span], v[r]);
    out[j] = static_cast<float>(static_cast<double>(v[0]) / n);
  }
}

// ---- one PayloadOps::combine event on device lanes (collectives.hpp:39-48) ----
// acc = acc (+) in for `lanes` lanes whose first lane has global index
// elem_offset, as IntSumOps::combine (collectives.cpp:60-81) or
// TokenReduceOps::combine (collectives.cpp:125-153) for event (step, dst).
// One thread per byte of 4-bit lanes (two lanes), else one thread per lane;
// the pointers may sit at any lane (byte) offset.
template <int KIND, int W>
__global__ void combine_kernel(uint8_t* acc, const uint8_t* in, uint64_t lanes, uint64_t elem_offset,
                               uint32_t m, uint64_t key, uint32_t* err) {
  uint32_t flags = 0;
  constexpr int PER = W == 4 ? 2 : 1;  // lanes per thread
  const uint64_t units = (lanes + PER - 1) / PER;
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < units;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint32_t a, b;
    if constexpr (W == 4 || W == 8) {
      a = acc[t];
      b = in[t];
    } else if constexpr (W == 16) {
      a = acc[2 * t] | (static_cast<uint32_t>(acc[2 * t + 1]) << 8);
      b = in[2 * t] | (static_cast<uint32_t>(in[2 * t + 1]) << 8);
    } else {
      a = b = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a |= static_cast<uint32_t>(acc[4 * t + i]) << (8 * i);
        b |= static_cast<uint32_t>(in[4 * t + i]) << (8 * i);
      }
    }
    uint32_t out = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const uint64_t j = t * PER + i;
      const uint32_t la = W == 4 ? (a >> (4 * i)) & 0xfu : a;
      const uint32_t lb = W == 4 ? (b >> (4 * i)) & 0xfu : b;
      uint32_t r;
      if (j >= lanes) {
        r = la;  // the other nibble of a half-used byte is left as it was
      } else if constexpr (KIND == 0) {
        const int64_t sum = static_cast<int64_t>(lane_sext<W>(la)) + lane_sext<W>(lb);
        const int64_t hi = (W == 32) ? 2147483647ll : (1ll << (W - 1)) - 1;
        if (sum > hi || sum < -hi - 1) flags |= GQ_FLAG_LANE_OVERFLOW;
        r = static_cast<uint32_t>(sum) & ((W == 32) ? 0xffffffffu : ((1u << W) - 1u));
      } else {
        constexpr uint32_t SB = 1u << (W - 1);
        // TokenReduceOps decodes -0 as zero and re-encodes canonically
        const uint32_t ca = (la & (SB - 1u)) ? la : 0u;
        const uint32_t cb = (lb & (SB - 1u)) ? lb : 0u;
        const uint64_t bits = mix64(key ^ (elem_offset + j));
        r = reduce_pair_lane(ca, cb, sample_k_bits(bits, m), SB, flags);
      }
      out |= W == 4 ? (r << (4 * i)) : r;
    }
    if constexpr (W == 4 || W == 8) {
      acc[t] = static_cast<uint8_t>(out);
    } else if constexpr (W == 16) {
      acc[2 * t] = static_cast<uint8_t>(out);
      acc[2 * t + 1] = static_cast<uint8_t>(out >> 8);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[4 * t + i] = static_cast<uint8_t>(out >> (8 * i));
    }
  }
  raise_flags_warp(err, flags);
}

// ---- f64 decode, exactly the reference's doubles (algorithm.cpp:84-110) ----
template <int KIND, int W>
__global__ void dequant_f64_kernel(const uint8_t* lanes, uint64_t lane_begin, uint64_t lane_end,
                                   const double* normp, uint32_t s, uint32_t n, uint32_t shift,
                                   double* out, uint32_t* err) {
  uint32_t flags = 0;
  const double norm = *normp;
  for (uint64_t j = lane_begin + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < lane_end;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint32_t c;
    if constexpr (W == 4) c = (lanes[j >> 1] >> (4 * (j & 1))) & 0xfu;
    else if constexpr (W == 8) c = lanes[j];
    else if constexpr (W == 16) c = lanes[2 * j] | (static_cast<uint32_t>(lanes[2 * j + 1]) << 8);
    else if constexpr (W == 64) c = 0;
    else c = lanes[4 * j] | (static_cast<uint32_t>(lanes[4 * j + 1]) << 8) |
             (static_cast<uint32_t>(lanes[4 * j + 2]) << 16) | (static_cast<uint32_t>(lanes[4 * j + 3]) << 24);
    double v;
    if constexpr (W == 64) {
      uint64_t u = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) u |= static_cast<uint64_t>(lanes[8 * j + i]) << (8 * i);
      const double scale = __ddiv_rn(norm, __dmul_rn(static_cast<double>(n), static_cast<double>(s)));
      v = __dmul_rn(scale, static_cast<double>(static_cast<int64_t>(u)));
    } else if constexpr (KIND == 0) {
      // scale = norm / (double(n) * s); out = scale * double(int64(lane))
      const double scale = __ddiv_rn(norm, __dmul_rn(static_cast<double>(n), static_cast<double>(s)));
      v = __dmul_rn(scale, static_cast<double>(lane_sext<W>(c)));
    } else {
      const uint32_t e = c & ((1u << (W - 1)) - 1u);
      const bool neg = (c >> (W - 1)) & 1u;
      if (e == 0 && neg) flags |= GQ_FLAG_NEG_ZERO;
      // token_contribution(t, norm) / n = norm * ldexp(sign 2^-e, shift) / n
      v = e == 0 ? 0.0
                 : __ddiv_rn(__dmul_rn(norm, ldexp(neg ? -1.0 : 1.0, static_cast<int>(shift) - static_cast<int>(e))),
                             static_cast<double>(n));
    }
    out[j - lane_begin] = v;
  }
  raise_flags_warp(err, flags);
}

// IntSumOps::combine on 64-bit lanes at any byte offset (byte-assembled).
__global__ void combine64_kernel(uint8_t* acc, const uint8_t* in, uint64_t lanes, uint32_t* err) {
  uint32_t flags = 0;
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < lanes;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t a = 0, b = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      a |= static_cast<uint64_t>(acc[8 * t + i]) << (8 * i);
      b |= static_cast<uint64_t>(in[8 * t + i]) << (8 * i);
    }
    const uint64_t sum = static_cast<uint64_t>(add64_checked(static_cast<int64_t>(a), static_cast<int64_t>(b), flags));
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[8 * t + i] = static_cast<uint8_t>(sum >> (8 * i));
  }
  raise_flags_warp(err, flags);
}

template <int KIND>
cudaError_t launch_combine_w(uint8_t* acc, const uint8_t* in, uint64_t lanes, uint64_t off,
                             uint32_t width, uint32_t m, uint64_t key, uint32_t* err, cudaStream_t st) {
  const uint64_t per = width == 4 ? 2 : 1;
  uint64_t blocks = ((lanes + per - 1) / per + 255) / 256;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  if (blocks == 0) return cudaSuccess;
  const dim3 g(static_cast<uint32_t>(blocks));
  switch (width) {
    case 4: combine_kernel<KIND, 4><<<g, 256, 0, st>>>(acc, in, lanes, off, m, key, err); break;
    case 8: combine_kernel<KIND, 8><<<g, 256, 0, st>>>(acc, in, lanes, off, m, key, err); break;
    case 16: combine_kernel<KIND, 16><<<g, 256, 0, st>>>(acc, in, lanes, off, m, key, err); break;
    case 32: combine_kernel<KIND, 32><<<g, 256, 0, st>>>(acc, in, lanes, off, m, key, err); break;
    case 64:
      if (KIND != 0) return cudaErrorInvalidValue;
      combine64_kernel<<<g, 256, 0, st>>>(acc, in, lanes, err);
      break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_reduce(const ReduceLaunch& r, cudaStream_t stream) {
  ReduceArgs a{};
  for (uint32_t i = 0; i < r.n; ++i) a.lanes[i] = r.worker_lanes[i];
  a.n = r.n;
  a.n_scale = r.n;
  a.s = r.s;
  a.m = r.s + 1;
  uint32_t shift = 0;
  for (uint64_t p = 1; p < 2ull * r.n; p <<= 1) ++shift;
  a.shift = shift;
  a.topo = r.topo;
  a.d = r.d;
  // RngStream::ReduceDraw = 2; keys (round, step<<32|dst, lane).
  a.hround = reduce_round_prefix(r.seed, r.round);
  a.round_ptr = r.round_ptr;
  a.seed = r.seed;
  a.npeers = r.npeers;
  for (uint32_t i = 0; i < r.npeers; ++i) a.out_peers[i] = r.out_peers[i];
  a.round_inc = r.round_inc;
  a.round_step = r.round_step;
  a.ticket = r.round_ticket;
  if (r.wait) a.pw = *r.wait;
  if (r.signal) {
    for (uint32_t i = 0; i < r.signal->n; ++i) a.sig.slots[i] = r.signal->slots[i];
    a.sig.n = r.signal->n;
    a.sig.epoch = r.signal->epoch;
    a.sig.ep_dev = r.signal->ep_dev;
    a.sig.ticket = r.signal->ticket;
  }
  a.norm = r.norm;
  a.out_lanes = r.out_lanes;
  a.out_mean = r.out_mean;
  a.param = r.param;
  a.param_vec = (reinterpret_cast<uintptr_t>(r.param) & 15) == 0;
  a.lr = r.lr;
  a.err = r.err;
  if (r.kdraws && r.kind == 1 && r.width <= 8 && r.topo == GQ_TOPO_TREE && r.s + 1 <= 32 &&
      (r.n == 2 || r.n == 4 || r.n == 8)) {
    a.kpre = r.kdraws;
    a.kstride = r.kstride;
  }
  return launch_generic(a, r.kind, r.width, r.lane_begin, r.lane_end, stream);
}

cudaError_t launch_dequant(const void* lanes, uint64_t lane_begin, uint64_t lane_end,
                           const double* norm, uint32_t kind, uint32_t s, uint32_t n,
                           uint32_t width, float* out, float* param, float lr,
                           uint32_t* err, cudaStream_t stream) {
  return launch_dequant_ex(lanes, lane_begin, lane_end, norm, kind, s, n, width, out, param, lr, err, stream,
                           nullptr, nullptr, 0, nullptr);
}

cudaError_t launch_dequant_ex(const void* lanes, uint64_t lane_begin, uint64_t lane_end, const double* norm,
                              uint32_t kind, uint32_t s, uint32_t n, uint32_t width, float* out, float* param,
                              float lr, uint32_t* err, cudaStream_t stream, const PeerWait* wait,
                              uint64_t* round_inc, uint64_t round_step, unsigned int* ticket) {
  ReduceArgs a{};
  if (wait) a.pw = *wait;
  a.round_inc = round_inc;
  a.round_step = round_step;
  a.ticket = ticket;
  a.lanes[0] = lanes;
  a.n = 1;  // identity schedule: the lanes are already aggregated
  a.n_scale = n;
  a.s = s;
  a.m = s + 1;
  uint32_t shift = 0;
  for (uint64_t p = 1; p < 2ull * n; p <<= 1) ++shift;
  a.shift = shift;
  a.topo = GQ_TOPO_TREE;
  a.d = lane_end;
  a.norm = norm;
  a.out_lanes = nullptr;
  a.out_mean = out;
  a.param = param;
  a.param_vec = (reinterpret_cast<uintptr_t>(param) & 15) == 0;
  a.lr = lr;
  a.err = err;
  return launch_generic(a, kind, width, lane_begin, lane_end, stream);
}

// ---- in-process quantize + schedule replay + decode, tile by tile ----
// With all n workers on one device the quantized lanes need not leave the
// SM: a CTA quantizes one tile (256 lane words) of every worker into shared
// memory (quantize_shard + encode, the quantize kernel's decisions), then
// replays the tree schedule on those words (the precomputed k draws for
// tokens) and decodes (+ SGD) - the per-worker lanes round trip through HBM
// (n·w/8 B per lane written and read back) is gone. Per-worker lanes are
// still stored when the caller asks for them. Bit-identical to the
// quantize + reduce kernels.
struct FusedArgs {
  const float* x[kMaxWorkers];
  void* lanes_out[kMaxWorkers];  // optional per-worker lanes (null: not kept)
  uint64_t h4[kMaxWorkers];      // quantize prefixes (host rounds)
  const uint64_t* round_ptr;     // non-null: prefixes from the device round
  uint64_t seed;
  uint64_t ntiles;
  MulConsts mk;
  uint32_t pk[3];
  ReduceArgs R;                  // n, s, m, shift, norm, outputs, kpre, round advance
};

#ifndef GQ_FUSED_MINB
#define GQ_FUSED_MINB 2
#endif
template <int KIND, int W, int NT>
__global__ void __launch_bounds__(kRThreads, GQ_FUSED_MINB) fused_qr_kernel(const __grid_constant__ FusedArgs F) {
  constexpr int G = 32 / W;
  constexpr uint32_t TW = kRThreads;        // lane words per tile: one per thread in the replay
  constexpr uint32_t TQ = TW * G / 4;       // quads per worker per tile
  constexpr int QPT = G / 4;                // quads per thread per worker
  constexpr bool KP = KIND == 1;
  static_assert(W == 4 || W == 8, "fused path: 4- and 8-bit lanes");
  pdl_wait();
  pdl_trigger();
  const ReduceArgs& R = F.R;
  const double norm = *R.norm;
  uint32_t flags = 0;
  const bool bad = !(norm >= 0.0) || !isfinite(norm);
  const bool zero = norm == 0.0;
  const uint32_t s = R.s, shift = R.shift;
  const QConst K = make_const<KIND>(bad || zero ? 1.0 : norm, s, shift);
  const MulConsts MK = F.mk;
  __shared__ uint8_t s_qtab[kQtabBytes<KIND>];
  __shared__ float s_tab[1 << W];
  __shared__ uint64_t s_h4[NT];
  __shared__ ChunkMix s_cm[NT];
  __shared__ __align__(16) uint32_t s_lanes[NT][TW];
  if constexpr (KIND == 1) build_exp_tab<W>(s_qtab, s, shift);
  else build_std_tab<W>(s_qtab, s, K.cm);
  for (uint32_t c = threadIdx.x; c < (1u << W); c += blockDim.x) {  // decode table (reduce_kernel)
    float v;
    if constexpr (KIND == 0) {
      const double scale = __ddiv_rn(norm, __dmul_rn(static_cast<double>(R.n_scale), static_cast<double>(R.s)));
      v = __double2float_rn(__dmul_rn(scale, static_cast<double>(lane_sext<W>(c))));
    } else {
      const uint32_t e = c & ((1u << (W - 1)) - 1u);
      const bool neg = (c >> (W - 1)) & 1u;
      v = 0.0f;
      if (e != 0) {
        const double tv = ldexp(neg ? -1.0 : 1.0, static_cast<int>(R.shift) - static_cast<int>(e));
        v = __double2float_rn(__ddiv_rn(__dmul_rn(norm, tv), static_cast<double>(R.n_scale)));
      }
    }
    s_tab[c] = v;
  }
  if (threadIdx.x < NT)
    s_h4[threadIdx.x] = F.round_ptr ? hoist_prefix(F.seed, 1ull, threadIdx.x, *F.round_ptr) : F.h4[threadIdx.x];
  __syncthreads();
  if (bad) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_flag(R.err, GQ_FLAG_BAD_SCALE);
  } else {
    uint32_t cm_hi = 0xffffffffu;
    for (uint64_t tile = blockIdx.x; tile < F.ntiles; tile += gridDim.x) {
      const uint64_t q0 = tile * TQ;
      const uint32_t hi = static_cast<uint32_t>((4 * q0) >> 32);
      if (hi != cm_hi) {  // chunk constants: the high word of j is fixed within a tile
        if (threadIdx.x < NT) s_cm[threadIdx.x] = chunk_mix(s_h4[threadIdx.x], 4 * q0);
        __syncthreads();
        cm_hi = hi;
      }
      // ---- quantize + encode the tile of every worker into shared memory ----
#pragma unroll
      for (int r = 0; r < NT; ++r) {
        const float4* xv = reinterpret_cast<const float4*>(F.x[r]) + q0;
        float4 f[QPT];
#pragma unroll
        for (int qq = 0; qq < QPT; ++qq) f[qq] = __ldcs(xv + qq * TW + threadIdx.x);
        const ChunkMix cm = s_cm[r];
#pragma unroll
        for (int qq = 0; qq < QPT; ++qq) {
          const uint32_t ql = qq * TW + threadIdx.x;
          const float v[4] = {f[qq].x, f[qq].y, f[qq].z, f[qq].w};
          int32_t c[4];
          uint32_t pkd;
          if (zero) {  // quantizer.cpp:21-32: all idx = s (lane 0); a nonzero element is an error
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              c[e] = 0;
              if (v[e] != 0.0f) flags |= GQ_FLAG_ZERO_SCALE;
            }
            pkd = 0;
          } else {
            bool any = !K.fast;
            fast_quad<KIND, W>(v, cm, static_cast<uint32_t>(4 * (q0 + ql)), K, MK, s, shift, s_qtab, any, c);
            if (__builtin_expect(any, 0)) {
              quant_quad<KIND, W, float>(v, 4, s_h4[r], cm, 4 * (q0 + ql), K, MK, s, shift, flags, c);
              pkd = 0;
#pragma unroll
              for (int e = 0; e < 4; ++e) pkd |= (static_cast<uint32_t>(c[e]) & ((1u << W) - 1u)) << (e * W);
            } else {
              pkd = mad_lo(static_cast<uint32_t>(c[1]), F.pk[0], static_cast<uint32_t>(c[0]));
              pkd = mad_lo(static_cast<uint32_t>(c[2]), F.pk[1], pkd);
              pkd = mad_lo(static_cast<uint32_t>(c[3]), F.pk[2], pkd);
            }
          }
          if constexpr (W == 4) {
            reinterpret_cast<uint16_t*>(s_lanes[r])[ql] = static_cast<uint16_t>(pkd);
            if (F.lanes_out[r]) static_cast<uint16_t*>(F.lanes_out[r])[q0 + ql] = static_cast<uint16_t>(pkd);
          } else {
            s_lanes[r][ql] = pkd;
            if (F.lanes_out[r]) static_cast<uint32_t*>(F.lanes_out[r])[q0 + ql] = pkd;
          }
        }
      }
      __syncthreads();
      // ---- schedule replay + decode (+ SGD) of word threadIdx.x ----
      const uint64_t wi = tile * TW + threadIdx.x;
      uint32_t words[NT], kws[NT];
#pragma unroll
      for (int r = 0; r < NT; ++r) words[r] = s_lanes[r][threadIdx.x];
      if constexpr (KP) {
#pragma unroll
        for (int e = 0; e + 1 < NT; ++e) kws[e] = __ldcs(R.kpre + static_cast<uint64_t>(e) * R.kstride + wi);
      }
      const uint32_t res = tree_rec<KIND, W, true, NT, KP, 0, ceil_log2_c(NT)>(words, kws, R, nullptr, wi * G, flags);
      if (R.out_lanes) static_cast<uint32_t*>(R.out_lanes)[wi] = res;
      decode_word<KIND, W, false>(R, wi, res, s_tab, nullptr, norm, flags);
      __syncthreads();  // s_lanes is refilled by the next tile
    }
  }
  raise_flags_warp(R.err, flags);
  if (R.round_inc) {  // graph replays: advance the device round once the grid is done
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(R.ticket, 1u) == gridDim.x - 1) {
        *R.round_inc += R.round_step;
        *R.ticket = 0;
      }
    }
  }
}

// Applies to f32 shards, tree schedule, n in {2, 4, 8}, 4/8-bit lanes, whole
// 256-word tiles (d a multiple of 256 G), tokens with the precomputed k draws.
bool fused_path_applies(uint32_t dtype, uint32_t n, uint64_t d, uint32_t kind, uint32_t width, uint32_t topo,
                        bool kdraws) {
  if (!g_fused_path) return false;
  if (dtype != GQ_DTYPE_F32 || topo != GQ_TOPO_TREE || (n != 2 && n != 4 && n != 8)) return false;
  if (width != 4 && width != 8) return false;
  if (kind == GQ_KIND_EXPONENTIAL && !kdraws) return false;
  const uint64_t tile = static_cast<uint64_t>(kRThreads) * (32 / width);
  return d > 0 && d % tile == 0;
}

template <int KIND, int W, int NT>
cudaError_t launch_fused_nt(const FusedArgs& a, cudaStream_t st) {
  auto* fn = fused_qr_kernel<KIND, W, NT>;
  static int per_sm = 0, sms = 0;
  if (per_sm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kRThreads, 0);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
  }
  uint64_t grid = static_cast<uint64_t>(sms) * per_sm;
  if (grid > a.ntiles) grid = a.ntiles;
  if (grid == 0) grid = 1;
  const cudaError_t e = launch_maybe_pdl(fn, static_cast<uint32_t>(grid), kRThreads, 0, st, a);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int KIND, int W>
cudaError_t launch_fused_w(const FusedArgs& a, cudaStream_t st) {
  switch (a.R.n) {
    case 2: return launch_fused_nt<KIND, W, 2>(a, st);
    case 4: return launch_fused_nt<KIND, W, 4>(a, st);
    case 8: return launch_fused_nt<KIND, W, 8>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_fused_qr(const void* const* shards, uint32_t n, uint64_t d, uint32_t kind, uint32_t s,
                            uint32_t width, uint64_t seed, uint64_t round, const uint64_t* round_ptr,
                            uint64_t* round_inc, unsigned int* ticket, void* const* lane_bufs, void* result_lanes,
                            float* mean_out, float* param, float lr, const double* norm, const uint32_t* kdraws,
                            uint32_t* err, cudaStream_t stream) {
  FusedArgs a{};
  for (uint32_t i = 0; i < n; ++i) {
    a.x[i] = static_cast<const float*>(shards[i]);
    a.lanes_out[i] = lane_bufs ? lane_bufs[i] : nullptr;
    a.h4[i] = hoist_prefix(seed, 1ull, i, round);
  }
  a.round_ptr = round_ptr;
  a.seed = seed;
  const uint32_t G = 32 / width;
  const uint64_t words = d / G;
  a.ntiles = words / kRThreads;
  a.mk = GQ_MULCONSTS_INIT;
  a.pk[0] = 1u << width;
  a.pk[1] = 1u << (2 * width);
  a.pk[2] = 1u << (3 * width);
  ReduceArgs& r = a.R;
  r.n = n;
  r.n_scale = n;
  r.s = s;
  r.m = s + 1;
  uint32_t shift = 0;
  for (uint64_t pp = 1; pp < 2ull * n; pp <<= 1) ++shift;  // prescale_shift (as the quantize launch)
  r.shift = shift;
  r.topo = GQ_TOPO_TREE;
  r.d = d;
  r.w_begin = 0;
  r.w_end = words;
  r.lane_end = d;
  r.norm = norm;
  r.out_lanes = result_lanes;
  r.out_mean = mean_out;
  r.param = param;
  r.param_vec = (reinterpret_cast<uintptr_t>(param) & 15) == 0;
  r.lr = lr;
  r.err = err;
  r.key_mode = 0;
  r.mk = GQ_MULCONSTS_INIT;
  r.kpre = kdraws;
  r.kstride = words;
  r.round_inc = round_inc;
  r.round_step = 1;
  r.ticket = ticket;
  if (kind == GQ_KIND_STANDARD) return width == 4 ? launch_fused_w<0, 4>(a, stream) : launch_fused_w<0, 8>(a, stream);
  return width == 4 ? launch_fused_w<1, 4>(a, stream) : launch_fused_w<1, 8>(a, stream);
}

bool small_path_applies(uint32_t dtype, uint32_t n, uint64_t d, uint32_t kind, uint32_t s, uint32_t width,
                        uint32_t topo, uint32_t q, uint32_t p) {
  if (g_small_path == 0) return false;
  const uint64_t cap = g_small_path == 2 ? (uint64_t{1} << 24) : kSmallPathElems;  // 2: experiments
  return dtype == GQ_DTYPE_F32 && (n == 2 || n == 4 || n == 8) && (width == 4 || width == 8) &&
         (kind == 0 || s + 1 <= 32) &&  // token k draws of the SWAR path (m <= 32)
         topo == GQ_TOPO_TREE && q == GQ_NORM_INF && (p == GQ_NORM_INF || p == 2) && d > 0 &&
         static_cast<uint64_t>(n) * d <= cap;
}

cudaError_t launch_mean_small(const void* const* shards, uint32_t n, uint64_t d, uint32_t kind, uint32_t s,
                              uint32_t width, uint32_t p, uint64_t seed, uint64_t round, const uint64_t* round_ptr,
                              uint64_t* round_inc, void* const* lane_bufs, void* result_lanes, float* mean_out,
                              float* param, float lr, double* stats_out, double* norm_out, void* workspace,
                              uint32_t* err, cudaStream_t stream) {
  SmallArgs a{};
  for (uint32_t i = 0; i < n; ++i) {
    a.x[i] = static_cast<const float*>(shards[i]);
    a.h4[i] = hoist_prefix(seed, 1ull, i, round);  // RngStream::Dither = 1 (rng.hpp:31-37)
    a.R.lanes[i] = lane_bufs[i];
  }
  a.round_ptr = round_ptr;
  a.round_inc = round_inc;
  a.seed = seed;
  a.p = p;
  a.stats_out = stats_out;
  a.norm_out = norm_out;
  char* ws = static_cast<char*>(workspace);
  a.bar = reinterpret_cast<unsigned int*>(ws + kWsSmallBar);
  a.done = reinterpret_cast<unsigned int*>(ws + kWsSmallDone);
  a.maxbits = reinterpret_cast<uint32_t*>(ws + kWsSmallMax);
  a.mk = GQ_MULCONSTS_INIT;
  a.pk[0] = 1u << width;
  a.pk[1] = 1u << (2 * width);
  a.pk[2] = 1u << (3 * width);
  ReduceArgs& r = a.R;
  r.n = n;
  r.n_scale = n;
  r.s = s;
  r.m = s + 1;
  uint32_t shift = 0;
  for (uint64_t pp = 1; pp < 2ull * n; pp <<= 1) ++shift;
  r.shift = shift;
  r.topo = GQ_TOPO_TREE;
  r.d = d;
  r.w_begin = 0;
  r.w_end = (d + 32 / width - 1) / (32 / width);
  r.lane_end = d;
  r.hround = reduce_round_prefix(seed, round);
  r.out_lanes = result_lanes;
  r.out_mean = mean_out;
  r.param = param;
  r.param_vec = (reinterpret_cast<uintptr_t>(param) & 15) == 0;
  r.lr = lr;
  r.err = err;
  r.key_mode = 1;
  r.mk = GQ_MULCONSTS_INIT;
  const uint64_t work = d / 4;
  if (kind == 0) return width == 4 ? launch_small_w<0, 4>(a, work, stream) : launch_small_w<0, 8>(a, work, stream);
  return width == 4 ? launch_small_w<1, 4>(a, work, stream) : launch_small_w<1, 8>(a, work, stream);
}

cudaError_t launch_baseline_mean(const float* const* shards, uint32_t n, uint64_t d,
                                 uint32_t topo, float* mean_out, cudaStream_t stream) {
  (void)topo;
  PtrArray a{};
  bool al = (reinterpret_cast<uintptr_t>(mean_out) & 15) == 0;
  for (uint32_t i = 0; i < n; ++i) {
    a.p[i] = shards[i];
    al = al && (reinterpret_cast<uintptr_t>(shards[i]) & 15) == 0;
  }
  const uint64_t d4 = d / 4;
  if (al && d4 > 0 && (n == 1 || n == 2 || n == 4 || n == 8 || n == 16)) {
    uint64_t blocks = (d4 + 255) / 256;
    const uint64_t cap = 148ull * (n <= 8 ? 8 : 4);
    if (blocks > cap) blocks = cap;
    const uint32_t g = static_cast<uint32_t>(blocks);
    switch (n) {
      case 1: baseline_tree_v4_kernel<1><<<g, 256, 0, stream>>>(a, d4, mean_out); break;
      case 2: baseline_tree_v4_kernel<2><<<g, 256, 0, stream>>>(a, d4, mean_out); break;
      case 4: baseline_tree_v4_kernel<4><<<g, 256, 0, stream>>>(a, d4, mean_out); break;
      case 8: baseline_tree_v4_kernel<8><<<g, 256, 0, stream>>>(a, d4, mean_out); break;
      default: baseline_tree_v4_kernel<16><<<g, 256, 0, stream>>>(a, d4, mean_out); break;
    }
    if (d4 * 4 == d) return cudaGetLastError();
    // the d % 4 tail: the scalar kernel on the last elements
    for (uint32_t i = 0; i < n; ++i) a.p[i] = shards[i] + d4 * 4;
    baseline_tree_kernel<<<1, 32, 0, stream>>>(a, n, d - d4 * 4, mean_out + d4 * 4);
    return cudaGetLastError();
  }
  uint64_t blocks = (d + 255) / 256;
  if (blocks > 148ull * 8) blocks = 148ull * 8;
  if (blocks == 0) return cudaSuccess;
  baseline_tree_kernel<<<static_cast<uint32_t>(blocks), 256, 0, stream>>>(a, n, d, mean_out);
  return cudaGetLastError();
}

cudaError_t launch_combine(void* acc, const void* in, uint64_t lanes, uint64_t elem_offset,
                           uint32_t kind, uint32_t width, uint32_t s, uint64_t seed,
                           uint64_t round, uint32_t step, uint32_t dst, uint32_t* err,
                           cudaStream_t stream) {
  // RngStream::ReduceDraw = 2; keys (round, step<<32|dst, lane) (collectives.cpp:132-146)
  uint64_t h = mix64(seed ^ 0x517cc1b727220a95ull);
  h = mix64(h ^ 2ull);
  h = mix64(h ^ round);
  const uint64_t key = mix64(h ^ ((static_cast<uint64_t>(step) << 32) | dst));
  auto* a = static_cast<uint8_t*>(acc);
  auto* b = static_cast<const uint8_t*>(in);
  return kind == 0 ? launch_combine_w<0>(a, b, lanes, elem_offset, width, s + 1, key, err, stream)
                   : launch_combine_w<1>(a, b, lanes, elem_offset, width, s + 1, key, err, stream);
}

cudaError_t launch_dequant_f64(const void* lanes, uint64_t lane_begin, uint64_t lane_end,
                               const double* norm, uint32_t kind, uint32_t s, uint32_t n,
                               uint32_t width, double* out, uint32_t* err, cudaStream_t stream) {
  uint32_t shift = 0;
  for (uint64_t p = 1; p < 2ull * n; p <<= 1) ++shift;
  const uint64_t cnt = lane_end - lane_begin;
  uint64_t blocks = (cnt + 255) / 256;
  if (blocks > 148ull * 16) blocks = 148ull * 16;
  if (blocks == 0) return cudaSuccess;
  const auto* l = static_cast<const uint8_t*>(lanes);
  const dim3 g(static_cast<uint32_t>(blocks));
#define GQ_DQ64(K, W) dequant_f64_kernel<K, W><<<g, 256, 0, stream>>>(l, lane_begin, lane_end, norm, s, n, shift, out, err)
  if (kind == 0) {
    switch (width) {
      case 4: GQ_DQ64(0, 4); break;
      case 8: GQ_DQ64(0, 8); break;
      case 16: GQ_DQ64(0, 16); break;
      case 32: GQ_DQ64(0, 32); break;
      case 64: GQ_DQ64(0, 64); break;
      default: return cudaErrorInvalidValue;
    }
  } else {
    switch (width) {
      case 4: GQ_DQ64(1, 4); break;
      case 8: GQ_DQ64(1, 8); break;
      case 16: GQ_DQ64(1, 16); break;
      case 32: GQ_DQ64(1, 32); break;
      default: return cudaErrorInvalidValue;
    }
  }
#undef GQ_DQ64
  return cudaGetLastError();
}

uint64_t comm_timeout_ns() { return static_cast<uint64_t>(g_comm_timeout_s) * 1000000000ull; }

// ---- device RNG known-answer kernel (gq_rng_draws) ----
namespace {
__global__ void rng_draws_kernel(uint64_t prefix, uint64_t c0, uint64_t count, uint32_t m, const uint64_t* bits_in,
                                 uint64_t* bits_out, uint32_t* hi_out, uint32_t* k_out) {
  const MulConsts MK = GQ_MULCONSTS_INIT;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t c = c0 + i;
    if (bits_out) bits_out[i] = mix64(prefix ^ c);
    // the quad-shared hot-loop form: group of 4 starting at c & ~3
    if (hi_out) {
      uint32_t lo;
      const uint64_t g0 = c & ~3ull;
      const QuadMix q = group_mix<4>(prefix, g0, lo);
      const uint32_t e = static_cast<uint32_t>(c - g0);
      hi_out[i] = q.ok ? elem_mix(q, e ^ lo, MK)
                       : mix64_hi_generic(static_cast<uint32_t>(prefix ^ c), static_cast<uint32_t>((prefix ^ c) >> 32), MK);
    }
    // the 8-bit token reduce's packed k word: field c % 4 of the word at c & ~3
    if (k_out) {
      if (bits_in) {
        k_out[i] = sample_k_bits(bits_in[i], m);
      } else if (m <= 32) {
        const uint64_t g0 = c & ~3ull;
        const uint32_t kw = token_kword<8>(prefix, g0, m, MK);
        k_out[i] = (kw >> (8 * (c - g0))) & 0xffu;
      } else {
        k_out[i] = sample_k_bits(mix64(prefix ^ c), m);
      }
    }
  }
}
}  // namespace

cudaError_t launch_rng_draws(uint64_t seed, uint64_t stream_id, uint64_t a, uint64_t b, uint64_t c0, uint64_t count,
                             uint32_t m, const uint64_t* bits_in, uint64_t* bits_out, uint32_t* hi_out,
                             uint32_t* k_out, cudaStream_t st) {
  const uint64_t prefix = hoist_prefix(seed, stream_id, a, b);
  uint64_t blocks = (count + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  if (blocks == 0) return cudaSuccess;
  rng_draws_kernel<<<static_cast<uint32_t>(blocks), 256, 0, st>>>(prefix, c0, count, m, bits_in, bits_out, hi_out,
                                                                   k_out);
  return cudaGetLastError();
}

// ---- cross-GPU flags for the peer-memory exchange ----
// signal: after this stream's prior work (the peer stores of the previous
// kernel) is visible system-wide, write `epoch` into slot[p] of every peer.
// wait: spin (one thread) until this GPU's n flags all reached `epoch`.
namespace {
__global__ void p2p_signal_kernel(PtrArray slots, uint32_t n, uint32_t epoch, const uint32_t* ep) {
  if (ep) epoch = *ep;
  __threadfence_system();
  for (uint32_t p = threadIdx.x; p < n; p += blockDim.x) {
    uint32_t* f = static_cast<uint32_t*>(const_cast<void*>(slots.p[p]));
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
  }
}

// put: copy nbytes (a multiple of 4, small: norm stats, error words) from this
// GPU to dst[p] on every peer, then signal slot[p] as p2p_signal does.
__global__ void p2p_put_signal_kernel(const uint32_t* src, uint32_t words, PtrArray dst, PtrArray slots,
                                      uint32_t n, uint32_t epoch, const uint32_t* ep, bool bump) {
  // bump: this step's epoch is the stored one + 1 (graph replays; stored back
  // below once every thread has read the old value)
  if (ep) epoch = *ep + (bump ? 1u : 0u);
  for (uint32_t p = 0; p < n; ++p) {
    uint32_t* d = static_cast<uint32_t*>(const_cast<void*>(dst.p[p]));
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) d[i] = src[i];
  }
  __threadfence_system();
  __syncthreads();
  if (bump && ep && threadIdx.x == 0) *const_cast<uint32_t*>(ep) = epoch;
  for (uint32_t p = threadIdx.x; p < n; p += blockDim.x) {
    uint32_t* f = static_cast<uint32_t*>(const_cast<void*>(slots.p[p]));
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
  }
}

// A peer that never signals (crashed rank, broken mapping) must not hang the
// GPU: give up after `timeout_ns` (globaltimer) and raise GQ_FLAG_P2P_TIMEOUT.
__global__ void p2p_wait_kernel(const uint32_t* flags, uint32_t n, uint32_t epoch, const uint32_t* ep,
                                uint32_t* err, uint64_t* round_inc, uint64_t round_step, uint64_t timeout_ns) {
  if (ep) epoch = *ep;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (uint32_t p = threadIdx.x; p < n; p += blockDim.x) {
    uint32_t v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + p) : "memory");
      uint64_t now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > timeout_ns) {
        raise_flag(err, GQ_FLAG_P2P_TIMEOUT);
        break;
      }
    } while (static_cast<int32_t>(v - epoch) < 0);
  }
  __syncthreads();
  __threadfence_system();
  // graph replays: the step's last wait also advances the round (every kernel
  // that reads it has run)
  if (round_inc && threadIdx.x == 0) *round_inc += round_step;
}
__global__ void epoch_inc_kernel(uint32_t* ep) { *ep += 1; }
__global__ void round_inc_kernel(uint64_t* r, uint64_t step) {
  pdl_wait();  // the step's kernels have read the round
  *r += step;
}
}  // namespace

cudaError_t launch_epoch_inc(uint32_t* ep_dev, cudaStream_t st) {
  epoch_inc_kernel<<<1, 1, 0, st>>>(ep_dev);
  return cudaGetLastError();
}

cudaError_t launch_round_inc(uint64_t* round_dev, uint64_t step, cudaStream_t st) {
  const cudaError_t e = launch_maybe_pdl(round_inc_kernel, 1, 1, 0, st, round_dev, step);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_p2p_signal(uint32_t* const* slots, uint32_t n, uint32_t epoch, const uint32_t* ep_dev,
                              cudaStream_t st) {
  PtrArray a{};
  for (uint32_t i = 0; i < n; ++i) a.p[i] = slots[i];
  p2p_signal_kernel<<<1, 32, 0, st>>>(a, n, epoch, ep_dev);
  return cudaGetLastError();
}

cudaError_t launch_p2p_put_signal(const void* src, uint32_t nbytes, void* const* dst, uint32_t* const* slots,
                                  uint32_t n, uint32_t epoch, const uint32_t* ep_dev, cudaStream_t st, bool bump) {
  PtrArray d{}, f{};
  for (uint32_t i = 0; i < n; ++i) {
    d.p[i] = dst[i];
    f.p[i] = slots[i];
  }
  p2p_put_signal_kernel<<<1, 128, 0, st>>>(static_cast<const uint32_t*>(src), nbytes / 4, d, f, n, epoch, ep_dev,
                                           bump);
  return cudaGetLastError();
}

cudaError_t launch_p2p_wait(const uint32_t* flags, uint32_t n, uint32_t epoch, const uint32_t* ep_dev, uint32_t* err,
                            cudaStream_t st, uint64_t* round_inc, uint64_t round_step) {
  p2p_wait_kernel<<<1, 32, 0, st>>>(flags, n, epoch, ep_dev, err, round_inc, round_step,
                                    static_cast<uint64_t>(g_comm_timeout_s) * 1000000000ull);
  return cudaGetLastError();
}

}  // namespace gqb
