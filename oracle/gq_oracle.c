/* TEST INFRASTRUCTURE ONLY — CPU oracle for the Global-QSGD hot path.
 * See gq_oracle.h for who may use it and how it is pinned. Every function
 * cites the reference file:line it restates (paths under
 * /root/reference/proj). Compiled with -ffp-contract=off so every double
 * operation rounds exactly as the reference's scalar code does.
 *
 * Extension over the reference (documented in DESIGN.md): 4-bit lanes.
 * The reference admits 8/16/32(/64) only (algorithm.cpp:25,
 * exp_arith.cpp:65-67,144-146); here width 4 is admitted whenever
 * check_width(kind, s, n, 4) holds. Token exponents never exceed the larger
 * operand (exp_arith.cpp:98-102), so 4-bit results equal the reference run at
 * width 8 lane for lane; tests check exactly that.
 */
#define _DEFAULT_SOURCE
#include <pthread.h>
#include <unistd.h>
#include "gq_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

enum { ST_OK = 0, ST_INVALID = 1, ST_OVERFLOW = 2, ST_DOMAIN = 3 };

/* rng.hpp:20-25 */
uint64_t gqo_mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/* rng.hpp:45-53 */
uint64_t gqo_rng_bits(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b,
                      uint64_t c) {
  uint64_t h = gqo_mix64(seed ^ 0x517cc1b727220a95ull);
  h = gqo_mix64(h ^ stream);
  h = gqo_mix64(h ^ a);
  h = gqo_mix64(h ^ b);
  h = gqo_mix64(h ^ c);
  return h;
}

/* rng.hpp:58-61 */
double gqo_rng_u01(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b,
                   uint64_t c) {
  return (double)(gqo_rng_bits(seed, stream, a, b, c) >> 11) * 0x1.0p-53;
}

/* rng.hpp:72-78 */
double gqo_rng_normal(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b,
                      uint64_t c) {
  const double u1 = gqo_rng_u01(seed, stream, a, b, c ^ 0x8000000000000000ull);
  const double u2 = gqo_rng_u01(seed, stream, a, b, c ^ 0x4000000000000000ull);
  const double r = sqrt(-2.0 * log1p(-u1));
  return r * cos(6.283185307179586476925286766559 * u2);
}

/* levels.cpp:31-48 (kind 0 standard, 1 exponential) */
int gqo_levels(uint32_t kind, uint32_t s, double* out) {
  if (s == 0) return ST_INVALID;
  if (kind == 0) {
    for (uint32_t i = 0; i <= s; ++i) out[i] = (double)(s - i) / (double)s;
  } else {
    for (uint32_t i = 0; i < s; ++i) out[i] = ldexp(1.0, -(int)i);
    out[s] = 0.0;
  }
  return ST_OK;
}

/* levels.cpp:63-76: largest i with levels[i] >= y (lower_bound over the
 * descending grid minus one), clamped to s - 1. Caller guarantees y in [0,1]. */
uint32_t gqo_bracket_index(const double* levels, uint32_t s, double y) {
  uint32_t lo = 0, hi = s + 1; /* first index with levels[i] < y */
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo) / 2;
    if (levels[mid] >= y) lo = mid + 1; else hi = mid;
  }
  if (lo == 0) return 0;
  uint32_t u = lo - 1;
  if (u > s - 1) u = s - 1;
  return u;
}

/* levels.cpp:78-84 */
uint32_t gqo_random_round(const double* levels, uint32_t s, double y, double u) {
  const uint32_t lo_idx = gqo_bracket_index(levels, s, y);
  const double hi = levels[lo_idx];
  const double lo = levels[lo_idx + 1];
  const double p_hi = (y - lo) / (hi - lo);
  return (u < p_hi) ? lo_idx : lo_idx + 1;
}

/* exp_arith.cpp:8-17 */
uint32_t gqo_ceil_log2(uint64_t v) {
  uint32_t bits = 0;
  uint64_t p = 1;
  while (p < v) { p <<= 1; ++bits; }
  return bits;
}

/* exp_arith.cpp:19-22 */
uint32_t gqo_prescale_shift(uint32_t n) { return gqo_ceil_log2(2ull * n); }

/* exp_arith.cpp:24-41 */
int gqo_check_width(uint32_t kind, uint32_t s, uint32_t n, uint32_t width) {
  if (s == 0 || n == 0 || width < 2 || width > 32) return 0;
  const uint64_t capacity = 1ull << (width - 1);
  if (kind == 0) return (uint64_t)n * (s + 1ull) <= capacity;
  return s + 1ull + gqo_ceil_log2(n) <= capacity;
}

/* algorithm.cpp:22-29, plus the 4-bit extension (see file header). */
uint32_t gqo_standard_lane_width(uint32_t s, uint32_t n, uint32_t at_least) {
  if (at_least == 4 && gqo_check_width(0, s, n, 4)) return 4;
  static const uint32_t ws[4] = {8, 16, 32, 64};
  for (int i = 0; i < 4; ++i) {
    if (ws[i] >= at_least && gqo_check_width(0, s, n, ws[i])) return ws[i];
  }
  return 0;
}

/* exp_arith.cpp:43-50 */
uint32_t gqo_sample_k(double u, uint32_t m) {
  if (u < ldexp(1.0, -(int)m)) return m;
  const int b = ilogb(u);
  const uint32_t k = (uint32_t)(-b);
  return k > m ? m : k;
}

/* exp_arith.cpp:82-109 */
int gqo_reduce_pair(int32_t sa, uint32_t ea, int32_t sb, uint32_t eb,
                    uint32_t k, uint32_t max_e, int32_t* so, uint32_t* eo) {
  if (ea > max_e || eb > max_e) return ST_OVERFLOW;
  if (ea == 0 && eb == 0) { *so = 1; *eo = 0; return ST_OK; }
  if (ea == 0) { *so = sb; *eo = eb; return ST_OK; }
  if (eb == 0) { *so = sa; *eo = ea; return ST_OK; }
  const int sign12 = sa * sb;
  const int64_t gap = ea > eb ? (int64_t)ea - eb : (int64_t)eb - ea;
  const int64_t diff = gap - (sign12 < 0 ? 1 : 0);
  if (diff < 0) { *so = 1; *eo = 0; return ST_OK; }
  const int32_t sign_out = ea <= eb ? sa : sb;
  const uint32_t e_min = ea <= eb ? ea : eb;
  const int bump = (int64_t)k > diff;
  const int64_t e_out = (int64_t)e_min - (sign12 > 0 ? bump : -bump);
  if (e_out < 1 || e_out > (int64_t)max_e) return ST_OVERFLOW;
  *so = sign_out;
  *eo = (uint32_t)e_out;
  return ST_OK;
}

/* norms.cpp:34-62 */
int gqo_local_norm_stat(const double* x, uint64_t d, uint32_t q, uint32_t p,
                        double* out) {
  for (uint64_t j = 0; j < d; ++j) {
    if (!isfinite(x[j])) return ST_INVALID;
  }
  double nq;
  if (q == GQO_NORM_INF) {
    double m = 0.0;
    for (uint64_t j = 0; j < d; ++j) m = fmax(m, fabs(x[j]));
    nq = m;
  } else if (q == 2) {
    double ss = 0.0;
    for (uint64_t j = 0; j < d; ++j) ss += x[j] * x[j];
    nq = sqrt(ss);
  } else {
    double acc = 0.0;
    for (uint64_t j = 0; j < d; ++j) acc += pow(fabs(x[j]), (double)q);
    nq = pow(acc, 1.0 / (double)q);
  }
  if (p == GQO_NORM_INF) *out = nq;
  else if (p == 2) *out = nq * nq;
  else *out = pow(nq, (double)p);
  return ST_OK;
}

/* topology.cpp:19-72 (topo 0 tree, 1 ring). Events as
 * (step, src, dst, op[0 reduce, 1 copy], chunk) quintuples. */
int64_t gqo_schedule(uint32_t topo, uint32_t n, uint32_t* out, uint64_t cap) {
  uint64_t count = 0;
#define GQO_EMIT(t, s_, d_, op, ch)                                      \
  do {                                                                   \
    if (count < cap) {                                                   \
      out[5 * count] = (t); out[5 * count + 1] = (s_);                   \
      out[5 * count + 2] = (d_); out[5 * count + 3] = (op);              \
      out[5 * count + 4] = (ch);                                         \
    }                                                                    \
    ++count;                                                             \
  } while (0)
  if (n <= 1) return 0;
  if (topo == 0) {
    const uint32_t height = gqo_ceil_log2(n);
    for (uint32_t t = 0; t < height; ++t) {
      const uint32_t span = 1u << t;
      for (uint32_t r = span; r < n; r += 2 * span) GQO_EMIT(t, r, r - span, 0, 0);
    }
    for (uint32_t t = 0; t < height; ++t) {
      const uint32_t span = 1u << (height - 1 - t);
      for (uint32_t r = 0; r + span < n; r += 2 * span) GQO_EMIT(height + t, r, r + span, 1, 0);
    }
  } else {
    for (uint32_t t = 0; t + 1 < n; ++t)
      for (uint32_t r = 0; r < n; ++r) GQO_EMIT(t, r, (r + 1) % n, 0, (r + n - t % n) % n);
    for (uint32_t t = 0; t + 1 < n; ++t)
      for (uint32_t r = 0; r < n; ++r) GQO_EMIT(n - 1 + t, r, (r + 1) % n, 1, (r + 1 + n - t % n) % n);
  }
#undef GQO_EMIT
  return (int64_t)count;
}

/* collectives.cpp:210-233 + norms.cpp:64-75: the scalar exchange always walks
 * the tree schedule (dst op= src), then applies the root. */
int gqo_norm_tree_combine(const double* stats, uint32_t n, uint32_t q,
                          uint32_t p, double* out) {
  (void)q;
  if (n == 0) return ST_INVALID;
  double* acc = (double*)malloc(sizeof(double) * n);
  uint32_t* ev = (uint32_t*)malloc(sizeof(uint32_t) * 5 * 4 * (size_t)(n + 1));
  memcpy(acc, stats, sizeof(double) * n);
  const int64_t ne = gqo_schedule(0, n, ev, 4 * (uint64_t)(n + 1));
  for (int64_t i = 0; i < ne; ++i) {
    const uint32_t src = ev[5 * i + 1], dst = ev[5 * i + 2], op = ev[5 * i + 3];
    if (op == 0) {
      if (p == GQO_NORM_INF) acc[dst] = acc[dst] < acc[src] ? acc[src] : acc[dst];
      else acc[dst] = acc[dst] + acc[src];
    } else {
      acc[dst] = acc[src];
    }
  }
  const double v = acc[0];
  free(acc);
  free(ev);
  if (p == GQO_NORM_INF) *out = v;      /* max of one value */
  else if (p == 2) *out = sqrt(v);
  else *out = pow(v, 1.0 / (double)p);
  return ST_OK;
}

/* quantizer.cpp:8-48 */
int gqo_quantize(const double* x, uint64_t d, double norm, uint32_t kind,
                 uint32_t s, uint64_t seed, uint32_t worker, uint64_t round,
                 int8_t* sign, uint32_t* level_idx) {
  if (!isfinite(norm) || norm < 0.0) return ST_INVALID;
  if (s == 0) return ST_INVALID;
  if (norm == 0.0) {
    for (uint64_t j = 0; j < d; ++j) if (x[j] != 0.0) return ST_INVALID;
    for (uint64_t j = 0; j < d; ++j) { sign[j] = 1; level_idx[j] = s; }
    return ST_OK;
  }
  double* levels = (double*)malloc(sizeof(double) * (s + 1));
  gqo_levels(kind, s, levels);
  /* The first four mixes depend only on (seed, stream, worker, round)
   * (rng.hpp:45-53); hoisting them leaves the value unchanged. */
  uint64_t h = gqo_mix64(seed ^ 0x517cc1b727220a95ull);
  h = gqo_mix64(h ^ 1ull); /* RngStream::Dither, rng.hpp:31-37 */
  h = gqo_mix64(h ^ worker);
  h = gqo_mix64(h ^ round);
  int st = ST_OK;
  for (uint64_t j = 0; j < d; ++j) {
    const double v = x[j];
    if (!isfinite(v)) { st = ST_INVALID; break; }
    const double y = fabs(v) / norm;
    if (y > 1.0) { st = ST_INVALID; break; }
    const double u = (double)(gqo_mix64(h ^ j) >> 11) * 0x1.0p-53;
    const uint32_t idx = gqo_random_round(levels, s, y, u);
    level_idx[j] = idx;
    sign[j] = (idx == s) ? 1 : (v < 0.0 ? -1 : 1);
  }
  free(levels);
  return st;
}

static uint64_t lane_bytes_total(uint64_t lanes, uint32_t width) {
  return (lanes * width + 7) / 8;
}

static uint64_t load_lane(const uint8_t* buf, uint64_t j, uint32_t width) {
  if (width == 4) return (buf[j >> 1] >> (4 * (j & 1))) & 0xf;
  const uint32_t lb = width / 8;
  uint64_t v = 0;
  for (uint32_t i = 0; i < lb; ++i) v |= (uint64_t)buf[j * lb + i] << (8 * i);
  return v;
}

static void store_lane(uint8_t* buf, uint64_t j, uint32_t width, uint64_t v) {
  if (width == 4) {
    const uint32_t sh = 4 * (uint32_t)(j & 1);
    buf[j >> 1] = (uint8_t)((buf[j >> 1] & ~(0xfu << sh)) | ((v & 0xf) << sh));
    return;
  }
  const uint32_t lb = width / 8;
  for (uint32_t i = 0; i < lb; ++i) buf[j * lb + i] = (uint8_t)((v >> (8 * i)) & 0xff);
}

static int64_t sext(uint64_t v, uint32_t width) {
  if (width < 64 && ((v >> (width - 1)) & 1)) v |= ~0ull << width;
  return (int64_t)v;
}

static int valid_width(uint32_t kind, uint32_t width) {
  if (kind == 0) return width == 4 || width == 8 || width == 16 || width == 32 || width == 64;
  return width == 4 || width == 8 || width == 16 || width == 32;
}

/* Standard: algorithm.cpp:69-82 (lane = sign * (s - idx)).
 * Exponential: exp_arith.cpp:126-136 (tokens_from_shard: e = idx + shift,
 * idx == s -> zero token) then exp_arith.cpp:143-160 (pack_tokens:
 * [sign bit][e]). 4-bit lanes are nibbles, element 2i in the low nibble. */
int gqo_encode(uint32_t kind, uint32_t s, uint32_t n, uint32_t width,
               const int8_t* sign, const uint32_t* level_idx, uint64_t d,
               uint8_t* lanes) {
  if (!valid_width(kind, width)) return ST_INVALID;
  memset(lanes, 0, lane_bytes_total(d, width));
  if (kind == 0) {
    for (uint64_t j = 0; j < d; ++j) {
      const int64_t v = (int64_t)sign[j] * ((int64_t)s - (int64_t)level_idx[j]);
      store_lane(lanes, j, width, (uint64_t)v);
    }
    return ST_OK;
  }
  if (!gqo_check_width(1, s, n, width)) return ST_INVALID;
  const uint32_t shift = gqo_prescale_shift(n);
  const uint32_t sign_bit = 1u << (width - 1);
  for (uint64_t j = 0; j < d; ++j) {
    const uint32_t idx = level_idx[j];
    if (idx > s) return ST_INVALID;
    uint32_t lane = 0;
    if (idx != s) {
      const uint32_t e = idx + shift;
      if (e >= sign_bit) return ST_OVERFLOW;
      lane = e | (sign[j] < 0 ? sign_bit : 0);
    }
    store_lane(lanes, j, width, lane);
  }
  return ST_OK;
}

/* collectives.cpp:155-190 walking topology.cpp's schedule with
 * IntSumOps::combine (collectives.cpp:60-81) or TokenReduceOps::combine
 * (collectives.cpp:125-153; k keyed by (round, step<<32|dst, lane)). */
int gqo_allreduce_inproc(uint8_t* lanes, uint32_t n, uint64_t lanes_per_worker,
                         uint32_t kind, uint32_t width, uint32_t s,
                         uint32_t topo, uint64_t seed, uint64_t round) {
  if (!valid_width(kind, width) || n == 0) return ST_INVALID;
  if (kind == 1 && !gqo_check_width(1, s, n, width)) return ST_INVALID;
  const uint64_t bytes = lane_bytes_total(lanes_per_worker, width);
  const uint64_t cap = 4ull * n * n + 16;
  uint32_t* ev = (uint32_t*)malloc(sizeof(uint32_t) * 5 * cap);
  const int64_t ne = gqo_schedule(topo, n, ev, cap);
  const uint32_t chunks = (topo == 0) ? 1 : n;
  const uint32_t max_e = (1u << (width - 1)) - 1;
  const uint32_t m = s + 1;
  const uint32_t sign_bit = 1u << (width - 1);
  int st = ST_OK;
  uint64_t h0 = gqo_mix64(seed ^ 0x517cc1b727220a95ull);
  h0 = gqo_mix64(h0 ^ 2ull); /* RngStream::ReduceDraw */
  h0 = gqo_mix64(h0 ^ round);
  for (int64_t i = 0; i < ne && st == ST_OK; ++i) {
    const uint32_t step = ev[5 * i], src = ev[5 * i + 1], dst = ev[5 * i + 2];
    const uint32_t op = ev[5 * i + 3], chunk = ev[5 * i + 4];
    /* topology.cpp:99-106 */
    const uint64_t lb = lanes_per_worker * chunk / chunks;
    const uint64_t le = lanes_per_worker * (chunk + 1) / chunks;
    uint8_t* a = lanes + (uint64_t)dst * bytes;
    const uint8_t* b = lanes + (uint64_t)src * bytes;
    if (op == 1) {
      for (uint64_t j = lb; j < le; ++j) store_lane(a, j, width, load_lane(b, j, width));
      continue;
    }
    if (kind == 0) {
      const int64_t hi = width == 64 ? INT64_MAX : ((int64_t)1 << (width - 1)) - 1;
      const int64_t lo = width == 64 ? INT64_MIN : -((int64_t)1 << (width - 1));
      for (uint64_t j = lb; j < le; ++j) {
        const int64_t x = sext(load_lane(a, j, width), width);
        const int64_t y = sext(load_lane(b, j, width), width);
        int64_t sum;
        if (__builtin_add_overflow(x, y, &sum) || sum > hi || sum < lo) { st = ST_OVERFLOW; break; }
        store_lane(a, j, width, (uint64_t)sum);
      }
    } else {
      const uint64_t hstep = gqo_mix64(h0 ^ (((uint64_t)step << 32) | dst));
      for (uint64_t j = lb; j < le; ++j) {
        const uint32_t la = (uint32_t)load_lane(a, j, width);
        const uint32_t lin = (uint32_t)load_lane(b, j, width);
        const double u = (double)(gqo_mix64(hstep ^ j) >> 11) * 0x1.0p-53;
        int32_t so;
        uint32_t eo;
        st = gqo_reduce_pair((la & sign_bit) ? -1 : 1, la & (sign_bit - 1),
                             (lin & sign_bit) ? -1 : 1, lin & (sign_bit - 1),
                             gqo_sample_k(u, m), max_e, &so, &eo);
        if (st != ST_OK) break;
        uint32_t lane = eo;
        if (so < 0 && eo != 0) lane |= sign_bit;
        store_lane(a, j, width, lane);
      }
    }
  }
  free(ev);
  return st;
}

/* Standard: algorithm.cpp:84-100. Exponential: algorithm.cpp:102-110 with
 * unpack_tokens (exp_arith.cpp:162-184, negative zero -> domain_error) and
 * token_contribution (exp_arith.cpp:138-141). */
int gqo_decode(uint32_t kind, const uint8_t* lanes, uint64_t d, double norm,
               uint32_t s, uint32_t n, uint32_t width, double* out) {
  if (!valid_width(kind, width)) return ST_INVALID;
  if (kind == 0) {
    const double scale = norm / ((double)n * s);
    for (uint64_t j = 0; j < d; ++j) out[j] = scale * (double)sext(load_lane(lanes, j, width), width);
    return ST_OK;
  }
  const uint32_t shift = gqo_prescale_shift(n);
  const uint32_t sign_bit = 1u << (width - 1);
  for (uint64_t j = 0; j < d; ++j) {
    const uint32_t lane = (uint32_t)load_lane(lanes, j, width);
    const uint32_t e = lane & (sign_bit - 1);
    const int neg = (lane & sign_bit) != 0;
    if (e == 0 && neg) return ST_DOMAIN;
    const double tv = e == 0 ? 0.0 : (neg ? -1.0 : 1.0) * ldexp(1.0, -(int)e);
    out[j] = norm * ldexp(tv, (int)shift) / n;
  }
  return ST_OK;
}

/* algorithm.cpp:127-228 (dense paths, Transport::Inproc). norm_override, when
 * non-NULL, replaces the exchanged norm (used to inject a GPU L2 norm). */
int gqo_mean(const double* shards, uint32_t n, uint64_t d, uint32_t kind,
             uint32_t s, uint32_t q, uint32_t p, uint32_t width, uint32_t topo,
             uint64_t seed, uint64_t round, const double* norm_override,
             double* mean_out, double* norm_out, uint32_t* lane_width_out,
             uint8_t* summed_lanes_out) {
  if (n == 0 || s == 0) return ST_INVALID;
  /* plan_path, algorithm.cpp:40-67 */
  uint32_t w;
  if (kind == 0) {
    w = gqo_standard_lane_width(s, n, width);
    if (w == 0) return ST_INVALID;
  } else {
    if (!valid_width(1, width) || !gqo_check_width(1, s, n, width)) return ST_INVALID;
    w = width;
  }
  if (lane_width_out) *lane_width_out = w;
  double* stats = (double*)malloc(sizeof(double) * n);
  int st = ST_OK;
  for (uint32_t r = 0; r < n && st == ST_OK; ++r) st = gqo_local_norm_stat(shards + (uint64_t)r * d, d, q, p, &stats[r]);
  double norm = 0.0;
  if (st == ST_OK) st = gqo_norm_tree_combine(stats, n, q, p, &norm);
  free(stats);
  if (st != ST_OK) return st;
  if (norm_override) norm = *norm_override;
  if (norm_out) *norm_out = norm;
  const uint64_t bytes = lane_bytes_total(d, w);
  if (norm == 0.0) {
    for (uint64_t j = 0; j < d; ++j) mean_out[j] = 0.0;
    if (summed_lanes_out) memset(summed_lanes_out, 0, bytes);
    return ST_OK;
  }
  int8_t* sign = (int8_t*)malloc(d ? d : 1);
  uint32_t* idx = (uint32_t*)malloc(sizeof(uint32_t) * (d ? d : 1));
  uint8_t* lanes = (uint8_t*)calloc((size_t)n * bytes + 1, 1);
  for (uint32_t r = 0; r < n && st == ST_OK; ++r) {
    st = gqo_quantize(shards + (uint64_t)r * d, d, norm, kind, s, seed, r, round, sign, idx);
    if (st == ST_OK) st = gqo_encode(kind, s, n, w, sign, idx, d, lanes + (uint64_t)r * bytes);
  }
  if (st == ST_OK) st = gqo_allreduce_inproc(lanes, n, d, kind, w, s, topo, seed, round);
  if (st == ST_OK) st = gqo_decode(kind, lanes, d, norm, s, n, w, mean_out);
  if (st == ST_OK && summed_lanes_out) memcpy(summed_lanes_out, lanes, bytes);
  free(sign);
  free(idx);
  free(lanes);
  return st;
}

/* verify.cpp:118-128 */
int gqo_gaussian_shards(uint32_t n, uint64_t d, uint64_t seed, double* out) {
  for (uint32_t i = 0; i < n; ++i)
    for (uint64_t j = 0; j < d; ++j)
      out[(uint64_t)i * d + j] = gqo_rng_normal(seed, 5 /* ShardGen */, i, j, 0);
  return ST_OK;
}

/* Columns [j0, j0 + cnt) of gaussian_shards(n, d, seed) for any d > j0 + cnt
 * (verify.cpp:118-128: element (i, j) is normal(ShardGen, i, j, 0), independent
 * of d), so one 25 MiB bucket of a 340M-element gradient needs no 10 GB array.
 * Each element is a pure function of its keys, so splitting the index range
 * over threads gives the same bits as the sequential loop. */
typedef struct {
  uint64_t t0, t1, cnt, j0, seed;
  double* out;
} GaussJob;

static void* gauss_worker(void* arg) {
  const GaussJob* g = (const GaussJob*)arg;
  for (uint64_t t = g->t0; t < g->t1; ++t)
    g->out[t] = gqo_rng_normal(g->seed, 5 /* ShardGen */, t / g->cnt, g->j0 + t % g->cnt, 0);
  return NULL;
}

int gqo_gaussian_range(uint32_t n, uint64_t j0, uint64_t cnt, uint64_t seed, double* out) {
  enum { kMaxThreads = 32 };
  const uint64_t total = (uint64_t)n * cnt;
  long nt = sysconf(_SC_NPROCESSORS_ONLN);
  if (nt < 1) nt = 1;
  if (nt > kMaxThreads) nt = kMaxThreads;
  if (total < (1u << 16)) nt = 1;
  pthread_t th[kMaxThreads];
  GaussJob jobs[kMaxThreads];
  for (long i = 0; i < nt; ++i) {
    jobs[i] = (GaussJob){total * (uint64_t)i / (uint64_t)nt, total * (uint64_t)(i + 1) / (uint64_t)nt, cnt, j0,
                         seed, out};
    if (i > 0 && pthread_create(&th[i], NULL, gauss_worker, &jobs[i]) != 0) gauss_worker(&jobs[i]), th[i] = 0;
  }
  gauss_worker(&jobs[0]);
  for (long i = 1; i < nt; ++i)
    if (th[i]) pthread_join(th[i], NULL);
  return ST_OK;
}
