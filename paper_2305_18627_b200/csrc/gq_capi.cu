// extern "C" entry points of libgq_b200.so (declared in include/gq_b200.h).
// Host-side validation mirrors the reference's configuration checks and
// exception wording; kernels are launched stream-ordered with no host sync
// (except gq_check, whose job is to sync).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <cmath>
#include <algorithm>
#include <vector>

#include "gq_b200.h"
#include "gq_common.cuh"
#include "gq_internal.h"

#define GQ_EXPORT extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

int fail(int code, const char* msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e) {
  g_err = std::string("CUDA error: ") + cudaGetErrorString(e);
  return GQ_ERR_CUDA;
}

uint32_t ceil_log2_u64(uint64_t v) {
  uint32_t bits = 0;
  uint64_t p = 1;
  while (p < v) {
    p <<= 1;
    ++bits;
  }
  return bits;
}

// exp_arith.cpp:24-41. Note width_bits > 32 is refused for both kinds, so
// standard_lane_width's 64 candidate (algorithm.cpp:25) never admits and the
// reference refuses n(s+1) > 2^31; 64-bit lanes exist only as the IntSumOps
// plugin (collectives.cpp:23-27) and its payloads.
bool check_width(uint32_t kind, uint32_t s, uint32_t n, uint32_t width) {
  if (s == 0 || n == 0 || width < 2 || width > 32) return false;
  const uint64_t capacity = 1ull << (width - 1);
  if (kind == GQ_KIND_STANDARD) return static_cast<uint64_t>(n) * (s + 1ull) <= capacity;
  return s + 1ull + ceil_log2_u64(n) <= capacity;
}

bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

// lanes per 32-bit lane word (64-bit lanes: one lane per unit)
uint32_t lanes_per_word(uint32_t width) { return width >= 32 ? 1u : 32u / width; }

bool valid_norm_order(uint32_t v) { return v == 2 || v == GQ_NORM_INF; }
bool valid_q(uint32_t v) { return valid_norm_order(v) || v == GQ_NORM_L2_SEQUENTIAL; }
// norm_spec_from_string (norms.cpp:17-30) admits orders 1..16 besides inf;
// orders other than 2 / inf take a host step (norm_general below)
bool general_order(uint32_t v) { return v >= 1 && v <= 16 && v != 2; }
bool valid_q_any(uint32_t v) { return valid_q(v) || general_order(v); }
bool valid_p_any(uint32_t v) { return valid_norm_order(v) || general_order(v); }
bool device_orders(uint32_t q, uint32_t p) { return valid_q(q) && valid_norm_order(p); }

// local_norm_stat's power (norms.cpp:58-61) and, after the tree fold of the
// stats (collectives.cpp:210-233: std::max or +=), combine_norm_stats' root
// (norms.cpp:64-75) - with the same libm calls as the reference.
double host_stat(double nq, uint32_t p) {
  if (p == GQ_NORM_INF) return nq;
  if (p == 2) return nq * nq;
  return std::pow(nq, static_cast<double>(p));
}
double host_fold(std::vector<double> st, uint32_t p) {
  const uint32_t n = static_cast<uint32_t>(st.size());
  for (uint32_t span = 1; span < n; span <<= 1)
    for (uint32_t r = span; r < n; r += 2 * span)
      st[r - span] = (p == GQ_NORM_INF) ? std::max(st[r - span], st[r]) : st[r - span] + st[r];
  if (p == GQ_NORM_INF) return st[0];
  if (p == 2) return std::sqrt(st[0]);
  return std::pow(st[0], 1.0 / static_cast<double>(p));
}

// Norm orders other than 2 / inf (q or p in 1..16): the device forms each
// worker's nq (inf / 2: the usual kernels) or sum |x|^q (general q, correctly
// rounded powers, launch_norm_pow); the stream is synchronised and the root,
// power and fold run on the host. Not graph-capturable.
int norm_general(const void* const* shards, uint32_t dtype, uint32_t n, uint64_t d, uint32_t q, uint32_t p,
                 double* stats, double* norm_out, void* workspace, uint32_t* err, cudaStream_t st) {
  cudaError_t e = general_order(q)
                      ? gqb::launch_norm_pow(shards, dtype, n, d, q, stats, workspace, err, st)
                      : gqb::launch_norm(shards, dtype, n, d, q, GQ_NORM_INF, stats, nullptr, workspace, err, st);
  std::vector<double> h(n);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), stats, n * sizeof(double), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e);
  for (uint32_t w = 0; w < n; ++w) {
    const double nq = general_order(q) ? std::pow(h[w], 1.0 / static_cast<double>(q)) : h[w];  // vector_norm
    h[w] = host_stat(nq, p);
  }
  double nm = 0.0;
  if (norm_out) nm = host_fold(h, p);
  e = cudaMemcpyAsync(stats, h.data(), n * sizeof(double), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && norm_out) e = cudaMemcpyAsync(norm_out, &nm, sizeof(double), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // the host buffers go out of scope
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

int check_lane_args(uint32_t kind, uint32_t width, uint32_t s, uint32_t n) {
  if (kind != GQ_KIND_STANDARD && kind != GQ_KIND_EXPONENTIAL)
    return fail(GQ_ERR_INVALID, "aggregation requires a named level scheme");
  if (s == 0) return fail(GQ_ERR_INVALID, "level count s must be >= 1");
  if (n == 0 || n > GQ_MAX_WORKERS)
    return fail(GQ_ERR_INVALID, "worker count must be in [1, GQ_MAX_WORKERS]");
  if (width != 4 && width != 8 && width != 16 && width != 32 && !(width == 64 && kind == GQ_KIND_STANDARD)) {
    return fail(GQ_ERR_INVALID, kind == GQ_KIND_EXPONENTIAL
                                    ? "token lane width must be 4, 8, 16, or 32 bits"
                                    : "integer lane width must be 4, 8, 16, 32, or 64 bits");
  }
  if (kind == GQ_KIND_EXPONENTIAL && !check_width(kind, s, n, width))
    return fail(GQ_ERR_INVALID, "refused configuration: exponent range does not fit the lane width");
  return GQ_OK;
}

}  // namespace

GQ_EXPORT int gq_abi_version(void) { return GQ_ABI_VERSION; }

GQ_EXPORT int gq_set_option(uint32_t key, int64_t value) {
  if (key == GQ_OPT_COMM_TIMEOUT_S) {
    if (value < 1 || value > 86400) return fail(GQ_ERR_INVALID, "option value out of range");
    gqb::g_comm_timeout_s = static_cast<int>(value);
    return GQ_OK;
  }
  if (value < 0 || value > 64) return fail(GQ_ERR_INVALID, "option value out of range");
  switch (key) {
    case GQ_OPT_QUANT_CTAS_PER_SM: gqb::g_quant_ctas_per_sm = static_cast<int>(value); return GQ_OK;
    case GQ_OPT_REDUCE_CTAS_PER_SM: gqb::g_reduce_ctas_per_sm = static_cast<int>(value); return GQ_OK;
    case GQ_OPT_PDL:
      if (value > 1) return fail(GQ_ERR_INVALID, "option value out of range");
      gqb::g_pdl = static_cast<int>(value);
      return GQ_OK;
    case GQ_OPT_COMM_WAIT:
      if (value > 2) return fail(GQ_ERR_INVALID, "option value out of range");
      gqb::g_comm_wait = static_cast<int>(value);
      return GQ_OK;
    case GQ_OPT_COMM_FOLD:
      if (value > 1) return fail(GQ_ERR_INVALID, "option value out of range");
      gqb::g_comm_fold = static_cast<int>(value);
      return GQ_OK;
    case GQ_OPT_SMALL_PATH:
      if (value > 2) return fail(GQ_ERR_INVALID, "option value out of range");
      gqb::g_small_path = static_cast<int>(value);
      return GQ_OK;
    case GQ_OPT_FUSED_PATH:
      if (value > 1) return fail(GQ_ERR_INVALID, "option value out of range");
      gqb::g_fused_path = static_cast<int>(value);
      return GQ_OK;
    default: return fail(GQ_ERR_INVALID, "unknown option");
  }
}



GQ_EXPORT const char* gq_last_error(void) { return g_err.c_str(); }

GQ_EXPORT uint64_t gq_lane_bytes(uint64_t d, uint32_t width) {
  const uint64_t b = (d * width + 7) / 8;
  return (b + 15) & ~uint64_t{15};
}

// plan_path (algorithm.cpp:40-67) + standard_lane_width (algorithm.cpp:22-29)
// + ReduceContext::make (exp_arith.cpp:63-80); width 4 admitted as an
// extension when check_width holds.
GQ_EXPORT int gq_plan_path(const gq_config* cfg, gq_plan* out) {
  if (!cfg || !out) return fail(GQ_ERR_INVALID, "null argument");
  if (cfg->kind != GQ_KIND_STANDARD && cfg->kind != GQ_KIND_EXPONENTIAL)
    return fail(GQ_ERR_INVALID, "aggregation requires a named level scheme");
  if (cfg->s == 0) return fail(GQ_ERR_INVALID, "level count s must be >= 1");
  if (cfg->workers == 0) return fail(GQ_ERR_INVALID, "shard count does not match the worker count");
  if (cfg->workers > GQ_MAX_WORKERS)
    return fail(GQ_ERR_INVALID, "worker count exceeds GQ_MAX_WORKERS on one device");
  if (!valid_q_any(cfg->norm_q) || !valid_p_any(cfg->norm_p)) return fail(GQ_ERR_INVALID, "norm order out of range");
  if (cfg->topo != GQ_TOPO_TREE && cfg->topo != GQ_TOPO_RING)
    return fail(GQ_ERR_INVALID, "unknown topology");
  const uint32_t n = cfg->workers, s = cfg->s;
  gq_plan p{};
  if (cfg->kind == GQ_KIND_STANDARD) {
    uint32_t w = 0;
    if (cfg->width_bits == 4 && check_width(GQ_KIND_STANDARD, s, n, 4)) {
      w = 4;
    } else {
      for (uint32_t c : {8u, 16u, 32u, 64u}) {
        if (c >= cfg->width_bits && check_width(GQ_KIND_STANDARD, s, n, c)) {
          w = c;
          break;
        }
      }
    }
    if (w == 0)
      return fail(GQ_ERR_INVALID, "refused configuration: level sums cannot fit any integer lane");
    p.lane_width = w;
  } else {
    const uint32_t w = cfg->width_bits;
    if (w != 4 && w != 8 && w != 16 && w != 32)
      return fail(GQ_ERR_INVALID, "token lane width must be 4, 8, 16, or 32 bits");
    if (!check_width(GQ_KIND_EXPONENTIAL, s, n, w))
      return fail(GQ_ERR_INVALID, "refused configuration: exponent range does not fit the lane width");
    p.lane_width = w;
    p.m = s + 1;
    p.shift = ceil_log2_u64(2ull * n);
    p.max_e = (1u << (w - 1)) - 1;
  }
  *out = p;
  return GQ_OK;
}

GQ_EXPORT size_t gq_norm_workspace_bytes(uint32_t n, uint64_t d) {
  if (n == 0) return 256;
  return gqb::norm_workspace_bytes(n, d);
}

GQ_EXPORT int gq_norm(const void* const* shards, uint32_t dtype, uint32_t n, uint64_t d,
                      uint32_t q, uint32_t p, double* stats, double* norm_out,
                      void* workspace, uint32_t* err, void* stream) {
  if (n == 0 || n > GQ_MAX_WORKERS) return fail(GQ_ERR_INVALID, "worker count must be in [1, GQ_MAX_WORKERS]");
  if (!valid_q_any(q) || !valid_p_any(p)) return fail(GQ_ERR_INVALID, "norm order out of range");
  if (dtype != GQ_DTYPE_F32 && dtype != GQ_DTYPE_F64) return fail(GQ_ERR_INVALID, "unknown dtype");
  if (!shards || !stats || !workspace) return fail(GQ_ERR_INVALID, "null argument");
  for (uint32_t i = 0; i < n; ++i)
    if (!shards[i] || !aligned(shards[i], 16)) return fail(GQ_ERR_INVALID, "device buffers must be 16-byte aligned");
  if (!device_orders(q, p))
    return norm_general(shards, dtype, n, d, q, p, stats, norm_out, workspace, err, static_cast<cudaStream_t>(stream));
  const cudaError_t e = gqb::launch_norm(shards, dtype, n, d, q, p, stats, norm_out, workspace, err,
                                         static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

namespace {
bool kdraws_applicable(const gq_kdraws* k) {
  return k && k->kind == GQ_KIND_EXPONENTIAL && (k->width == 4 || k->width == 8) && k->topo == GQ_TOPO_TREE &&
         (k->n == 2 || k->n == 4 || k->n == 8) && k->s >= 1 && k->s + 1 <= 32 && k->lane_end > k->lane_begin &&
         k->lane_begin % (32 / k->width) == 0;
}
uint64_t kdraws_words(const gq_kdraws* k) {
  const uint64_t G = 32 / k->width;
  return (k->lane_end + G - 1) / G - k->lane_begin / G;
}
}  // namespace

GQ_EXPORT size_t gq_kdraws_bytes(const gq_kdraws* spec) {
  if (!kdraws_applicable(spec)) return 0;
  return static_cast<size_t>(kdraws_words(spec)) * (spec->n - 1) * sizeof(uint32_t);
}

GQ_EXPORT int gq_norm_kdraws(const void* const* shards, uint32_t dtype, uint32_t n, uint64_t d, uint32_t q,
                             uint32_t p, double* stats, double* norm_out, void* workspace, uint32_t* err,
                             const gq_kdraws* spec, void* stream) {
  if (!kdraws_applicable(spec)) return fail(GQ_ERR_INVALID, "k-draw precompute does not apply to this configuration");
  if (!spec->buf) return fail(GQ_ERR_INVALID, "null argument");
  if (n == 0 || n > GQ_MAX_WORKERS) return fail(GQ_ERR_INVALID, "worker count must be in [1, GQ_MAX_WORKERS]");
  if (!device_orders(q, p))
    return fail(GQ_ERR_INVALID, "norm orders other than 2 / inf take a host step: use gq_norm");
  if (dtype != GQ_DTYPE_F32 && dtype != GQ_DTYPE_F64) return fail(GQ_ERR_INVALID, "unknown dtype");
  if (!shards || !stats || !workspace) return fail(GQ_ERR_INVALID, "null argument");
  for (uint32_t i = 0; i < n; ++i)
    if (!shards[i] || !aligned(shards[i], 16)) return fail(GQ_ERR_INVALID, "device buffers must be 16-byte aligned");
  gqb::KDrawJob job{};
  job.buf = spec->buf;
  job.kwords = kdraws_words(spec);
  job.width = spec->width;
  job.m = spec->s + 1;
  // the keys of the events, with the word offset folded into the lane index:
  // kdraw_share evaluates lane (w0 + wi) * G through key ^ j only, so the
  // global word index is restored by evaluating at j0 = (w0 + wi) G.
  job.events = gqb::tree_event_keys(spec->n, spec->seed, spec->round, job.keys, gqb::kMaxKEvents);
  job.w0 = spec->lane_begin / (32 / spec->width);
  const cudaError_t e = gqb::launch_norm(shards, dtype, n, d, q, p, stats, norm_out, workspace, err,
                                         static_cast<cudaStream_t>(stream), &job);
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT int gq_norm_combine(const double* stats, uint32_t n, uint32_t q, uint32_t p,
                              double* norm_out, void* stream) {
  if (n == 0 || n > GQ_MAX_WORKERS) return fail(GQ_ERR_INVALID, "no norm statistics");
  if (!valid_q_any(q) || !valid_p_any(p) || q == GQ_NORM_L2_SEQUENTIAL)
    return fail(GQ_ERR_INVALID, "norm order out of range");
  if (general_order(p)) {  // the root on the host (combine_norm_stats, norms.cpp:64-75)
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::vector<double> h(n);
    cudaError_t e = cudaMemcpyAsync(h.data(), stats, n * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    const double nm = e == cudaSuccess ? host_fold(h, p) : 0.0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(norm_out, &nm, sizeof(double), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return e == cudaSuccess ? GQ_OK : cuda_fail(e);
  }
  const cudaError_t e = gqb::launch_norm_combine(stats, n, p, norm_out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT int gq_quantize(const void* const* shards, uint32_t dtype, uint32_t n_local,
                          const uint32_t* worker_ids, uint64_t d, const double* norm,
                          uint32_t kind, uint32_t s, uint32_t n_total, uint32_t width,
                          uint64_t seed, uint64_t round, void* const* lanes_out,
                          uint32_t* err, void* stream) {
  if (n_local == 0 || n_local > GQ_MAX_WORKERS) return fail(GQ_ERR_INVALID, "worker count must be in [1, GQ_MAX_WORKERS]");
  if (n_total < n_local) return fail(GQ_ERR_INVALID, "n_total must cover the local workers");
  if (int rc = check_lane_args(kind, width, s, n_total)) return rc;
  // (64-bit lanes: encode_dense_std with lane_width 64 holds any level value)
  if (kind == GQ_KIND_STANDARD && width != 64 && !check_width(kind, s, 1, width))
    return fail(GQ_ERR_INVALID, "level index does not fit the lane width");
  if (dtype != GQ_DTYPE_F32 && dtype != GQ_DTYPE_F64) return fail(GQ_ERR_INVALID, "unknown dtype");
  if (!shards || !worker_ids || !norm || !lanes_out) return fail(GQ_ERR_INVALID, "null argument");
  for (uint32_t i = 0; i < n_local; ++i) {
    if (!shards[i] || !lanes_out[i] || !aligned(shards[i], 16) || !aligned(lanes_out[i], 16))
      return fail(GQ_ERR_INVALID, "device buffers must be 16-byte aligned");
  }
  gqb::QuantLaunch q{shards, dtype, n_local, worker_ids, d, norm, kind, s, n_total, width,
                     seed, round, lanes_out, err};
  const cudaError_t e = gqb::launch_quantize(q, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT int gq_reduce_lanes(const void* const* worker_lanes, uint32_t n, uint64_t d,
                              uint64_t lane_begin, uint64_t lane_end, uint32_t kind,
                              uint32_t width, uint32_t s, uint32_t topo, uint64_t seed,
                              uint64_t round, const double* norm, void* out_lanes,
                              float* out_mean, float* param, float lr, uint32_t* err,
                              void* stream) {
  if (int rc = check_lane_args(kind, width, s, n)) return rc;
  if (topo != GQ_TOPO_TREE && topo != GQ_TOPO_RING) return fail(GQ_ERR_INVALID, "unknown topology");
  const uint32_t G = lanes_per_word(width);
  if (lane_end > d || lane_begin > lane_end) return fail(GQ_ERR_INVALID, "bad lane range");
  if (lane_begin % G != 0 || (lane_end % G != 0 && lane_end != d))
    return fail(GQ_ERR_INVALID, "lane range must be aligned to 32-bit lane words");
  if (!worker_lanes) return fail(GQ_ERR_INVALID, "null argument");
  for (uint32_t i = 0; i < n; ++i)
    if (!worker_lanes[i] || !aligned(worker_lanes[i], 16)) return fail(GQ_ERR_INVALID, "device buffers must be 16-byte aligned");
  if ((out_mean || param) && !norm) return fail(GQ_ERR_INVALID, "decode epilogue needs the norm");
  if ((out_lanes && !aligned(out_lanes, 16)) || (out_mean && !aligned(out_mean, 16)) ||
      (param && !aligned(param, 4)))
    return fail(GQ_ERR_INVALID, "device buffers must be 16-byte aligned");
  gqb::ReduceLaunch r{worker_lanes, n, d, lane_begin, lane_end, kind, width, s, topo, seed, round,
                      norm, out_lanes, out_mean, param, lr, err};
  const cudaError_t e = gqb::launch_reduce(r, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

// Same schedule replay on one slice of the lanes, with every pointer at the
// slice start (lane lane_begin): the form the multi-GPU exchange produces,
// where slice g of each worker arrives in its own receive buffer. Keys and
// chunk boundaries still use the global lane index and the full d.
GQ_EXPORT int gq_reduce_slice(const void* const* worker_slices, uint32_t n, uint64_t d,
                              uint64_t lane_begin, uint64_t lane_end, uint32_t kind,
                              uint32_t width, uint32_t s, uint32_t topo, uint64_t seed,
                              uint64_t round, const double* norm, void* out_slice,
                              float* out_mean_slice, float* param_slice, float lr,
                              uint32_t* err, void* stream) {
  if (width != 4 && width != 8 && width != 16 && width != 32 && !(width == 64 && kind == GQ_KIND_STANDARD))
    return fail(GQ_ERR_INVALID, "lane width must be 4, 8, 16, or 32 bits (64 for standard lanes)");
  if (n == 0 || n > GQ_MAX_WORKERS) return fail(GQ_ERR_INVALID, "worker count must be in [1, GQ_MAX_WORKERS]");
  if (!worker_slices) return fail(GQ_ERR_INVALID, "null argument");
  if ((lane_begin * width) % 128 != 0 || lane_begin % 4 != 0)
    return fail(GQ_ERR_INVALID, "slice start must be 16-byte aligned in the lane buffer");
  if (lane_end > d || lane_begin > lane_end) return fail(GQ_ERR_INVALID, "bad lane range");
  const uint64_t lane_off = lane_begin * width / 8;
  const void* base[GQ_MAX_WORKERS];
  for (uint32_t i = 0; i < n; ++i) {
    if (!worker_slices[i]) return fail(GQ_ERR_INVALID, "null argument");
    base[i] = static_cast<const uint8_t*>(worker_slices[i]) - lane_off;
  }
  void* out = out_slice ? static_cast<uint8_t*>(out_slice) - lane_off : nullptr;
  float* mean = out_mean_slice ? out_mean_slice - lane_begin : nullptr;
  float* prm = param_slice ? param_slice - lane_begin : nullptr;
  return gq_reduce_lanes(base, n, d, lane_begin, lane_end, kind, width, s, topo, seed, round, norm,
                         out, mean, prm, lr, err, stream);
}

GQ_EXPORT int gq_rng_draws(uint64_t seed, uint64_t stream_id, uint64_t a, uint64_t b, uint64_t c0, uint64_t count,
                           uint32_t m, const uint64_t* bits_in, uint64_t* bits_out, uint32_t* hi_out,
                           uint32_t* k_out, void* stream) {
  if (k_out && m == 0) return fail(GQ_ERR_INVALID, "truncation depth must be >= 1");
  const cudaError_t e = gqb::launch_rng_draws(seed, stream_id, a, b, c0, count, m, bits_in, bits_out, hi_out,
                                              k_out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

// PayloadOps::combine (collectives.hpp:39-48) for one event on device lanes:
// IntSumOps (collectives.cpp:60-81) or TokenReduceOps (collectives.cpp:125-153).
GQ_EXPORT int gq_combine_lanes(void* acc, const void* in, uint64_t lanes, uint64_t elem_offset,
                               uint32_t kind, uint32_t width, uint32_t s, uint32_t n,
                               uint64_t seed, uint64_t round, uint32_t step, uint32_t dst,
                               uint32_t* err, void* stream) {
  if (kind == GQ_KIND_STANDARD) {
    if (width != 4 && width != 8 && width != 16 && width != 32 && width != 64)
      return fail(GQ_ERR_INVALID, "integer lane width must be 4, 8, 16, 32, or 64 bits");
  } else if (int rc = check_lane_args(kind, width, s, n)) {
    return rc;
  }
  if (lanes && (!acc || !in)) return fail(GQ_ERR_INVALID, "null argument");
  if (width == 4 && elem_offset % 2 != 0)
    return fail(GQ_ERR_INVALID, "4-bit lanes combine from an even lane");
  const cudaError_t e = gqb::launch_combine(acc, in, lanes, elem_offset, kind, width, s, seed, round,
                                            step, dst, err, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT int gq_reduce_lanes_kdraws(const void* const* worker_lanes, uint32_t n, uint64_t d, uint64_t lane_begin,
                                     uint64_t lane_end, uint32_t kind, uint32_t width, uint32_t s, uint32_t topo,
                                     uint64_t seed, uint64_t round, const double* norm, void* out_lanes,
                                     float* out_mean, float* param, float lr, uint32_t* err,
                                     const gq_kdraws* spec, void* stream) {
  if (!kdraws_applicable(spec) || spec->n != n || spec->kind != kind || spec->width != width || spec->s != s ||
      spec->topo != topo || spec->seed != seed || spec->round != round || lane_begin < spec->lane_begin ||
      lane_end > spec->lane_end || !spec->buf)
    return fail(GQ_ERR_INVALID, "k-draw buffer does not match this reduce");
  if (int rc = check_lane_args(kind, width, s, n)) return rc;
  const uint32_t G = lanes_per_word(width);
  if (lane_end > d || lane_begin > lane_end) return fail(GQ_ERR_INVALID, "bad lane range");
  if (lane_begin % G != 0 || (lane_end % G != 0 && lane_end != d))
    return fail(GQ_ERR_INVALID, "lane range must be aligned to 32-bit lane words");
  if (!worker_lanes) return fail(GQ_ERR_INVALID, "null argument");
  for (uint32_t i = 0; i < n; ++i)
    if (!worker_lanes[i] || !aligned(worker_lanes[i], 16)) return fail(GQ_ERR_INVALID, "device buffers must be 16-byte aligned");
  if ((out_mean || param) && !norm) return fail(GQ_ERR_INVALID, "decode epilogue needs the norm");
  gqb::ReduceLaunch r{worker_lanes, n, d, lane_begin, lane_end, kind, width, s, topo, seed, round,
                      norm, out_lanes, out_mean, param, lr, err};
  // the consumer indexes kpre[e * kstride + global word]: rebase by the spec's first word
  r.kdraws = spec->buf - spec->lane_begin / G;
  r.kstride = kdraws_words(spec);
  const cudaError_t e = gqb::launch_reduce(r, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

// ---- peer-memory exchange (one worker per GPU, one NVSwitch node) ----
int gqb::quantize_scatter_impl(const void* const* shards, uint32_t n_local, const uint32_t* workers, uint32_t dtype,
                               uint64_t d, const double* norm, uint32_t kind, uint32_t s, uint32_t n_total,
                               uint32_t width, uint64_t seed, uint64_t round, const uint64_t* round_ptr,
                               void* const* slice_dst, uint32_t nslices, uint64_t slice_lanes, uint64_t row_bytes,
                               uint32_t* err, void* stream, const PeerSignal* signal, const PeerWait* wait,
                               const double* stats_all, uint32_t norm_p) {
  if (int rc = check_lane_args(kind, width, s, n_total)) return rc;
  if (kind == GQ_KIND_STANDARD && width != 64 && !check_width(kind, s, 1, width))
    return fail(GQ_ERR_INVALID, "level index does not fit the lane width");
  if (dtype != GQ_DTYPE_F32 && dtype != GQ_DTYPE_F64) return fail(GQ_ERR_INVALID, "unknown dtype");
  if (nslices == 0 || nslices > gqb::kMaxPeers) return fail(GQ_ERR_INVALID, "slice count must be in [1, 16]");
  // slices hold whole warp chunks (128 quads) and cover d
  if (slice_lanes == 0 || slice_lanes % 512 != 0 || slice_lanes * nslices < d)
    return fail(GQ_ERR_INVALID, "slices must be multiples of 512 lanes covering d");
  if (n_local == 0 || n_local > GQ_MAX_WORKERS || !shards || !workers || !norm || !slice_dst)
    return fail(GQ_ERR_INVALID, "null argument");
  for (uint32_t i = 0; i < n_local; ++i)
    if (!shards[i] || !aligned(shards[i], 16)) return fail(GQ_ERR_INVALID, "device buffers must be 16-byte aligned");
  for (uint32_t i = 0; i < nslices; ++i)
    if (!slice_dst[i] || !aligned(slice_dst[i], 16)) return fail(GQ_ERR_INVALID, "device buffers must be 16-byte aligned");
  if (row_bytes % 16 != 0) return fail(GQ_ERR_INVALID, "device buffers must be 16-byte aligned");
  void* lanes[GQ_MAX_WORKERS];
  for (uint32_t i = 0; i < n_local; ++i) lanes[i] = slice_dst[0];  // unused in scatter mode
  gqb::QuantLaunch q{shards, dtype, n_local, workers, d, norm, kind, s, n_total, width, seed, round, lanes, err};
  q.slice_dst = slice_dst;
  q.nslices = nslices;
  q.slice_lanes = slice_lanes;
  q.row_bytes = row_bytes;
  q.signal = signal;
  q.round_ptr = round_ptr;
  if (wait) {  // folded norm exchange: wait for every rank's stats, fold them, store the norm
    if (!stats_all) return fail(GQ_ERR_INVALID, "null argument");
    q.wait = wait;
    q.fold.stats = stats_all;
    q.fold.n = n_total;
    q.fold.p = norm_p;
    q.fold.norm_out = const_cast<double*>(norm);
  }
  const cudaError_t e = gqb::launch_quantize(q, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT int gq_quantize_scatter(const void* shard, uint32_t dtype, uint32_t worker, uint64_t d,
                                  const double* norm, uint32_t kind, uint32_t s, uint32_t n_total,
                                  uint32_t width, uint64_t seed, uint64_t round, void* const* slice_dst,
                                  uint32_t nslices, uint64_t slice_lanes, uint32_t* err, void* stream) {
  const void* shards[1] = {shard};
  const uint32_t ids[1] = {worker};
  return gqb::quantize_scatter_impl(shards, 1, ids, dtype, d, norm, kind, s, n_total, width, seed, round, nullptr,
                                    slice_dst, nslices, slice_lanes, 0, err, stream);
}

int gqb::reduce_slice_multicast_impl(const void* const* worker_slices, uint32_t n, uint64_t d, uint64_t lane_begin,
                                     uint64_t lane_end, uint32_t kind, uint32_t width, uint32_t s, uint32_t topo,
                                     uint64_t seed, uint64_t round, const uint64_t* round_ptr,
                                     const uint32_t* kdraws, uint64_t kstride, void* const* out_slices,
                                     uint32_t nout, uint32_t* err, void* stream, const PeerSignal* signal,
                                     const PeerWait* wait) {
  if (nout == 0 || nout > gqb::kMaxPeers || !out_slices) return fail(GQ_ERR_INVALID, "output count must be in [1, 16]");
  if (int rc = check_lane_args(kind, width, s, n)) return rc;
  if (topo != GQ_TOPO_TREE && topo != GQ_TOPO_RING) return fail(GQ_ERR_INVALID, "unknown topology");
  if ((lane_begin * width) % 128 != 0 || lane_begin % 4 != 0)
    return fail(GQ_ERR_INVALID, "slice start must be 16-byte aligned in the lane buffer");
  if (lane_end > d || lane_begin > lane_end) return fail(GQ_ERR_INVALID, "bad lane range");
  const uint64_t lane_off = lane_begin * width / 8;
  const void* base[GQ_MAX_WORKERS];
  void* outs[gqb::kMaxPeers];
  for (uint32_t i = 0; i < n; ++i) {
    if (!worker_slices[i] || !aligned(worker_slices[i], 16)) return fail(GQ_ERR_INVALID, "device buffers must be 16-byte aligned");
    base[i] = static_cast<const uint8_t*>(worker_slices[i]) - lane_off;
  }
  for (uint32_t i = 0; i < nout; ++i) {
    if (!out_slices[i] || !aligned(out_slices[i], 16)) return fail(GQ_ERR_INVALID, "device buffers must be 16-byte aligned");
    outs[i] = static_cast<uint8_t*>(out_slices[i]) - lane_off;
  }
  gqb::ReduceLaunch r{base, n, d, lane_begin, lane_end, kind, width, s, topo, seed, round,
                      nullptr, nullptr, nullptr, nullptr, 0.0f, err};
  r.out_peers = outs;
  r.npeers = nout;
  r.round_ptr = round_ptr;
  r.kdraws = kdraws;  // indexed by global lane word (caller rebases)
  r.kstride = kstride;
  r.signal = signal;
  r.wait = wait;
  const cudaError_t e = gqb::launch_reduce(r, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT int gq_reduce_slice_multicast(const void* const* worker_slices, uint32_t n, uint64_t d,
                                        uint64_t lane_begin, uint64_t lane_end, uint32_t kind, uint32_t width,
                                        uint32_t s, uint32_t topo, uint64_t seed, uint64_t round,
                                        void* const* out_slices, uint32_t nout, uint32_t* err, void* stream) {
  return gqb::reduce_slice_multicast_impl(worker_slices, n, d, lane_begin, lane_end, kind, width, s, topo, seed,
                                          round, nullptr, nullptr, 0, out_slices, nout, err, stream);
}

GQ_EXPORT int gq_p2p_signal(uint32_t* const* peer_slots, uint32_t n, uint32_t epoch, void* stream) {
  if (n == 0 || n > gqb::kMaxPeers || !peer_slots) return fail(GQ_ERR_INVALID, "peer count must be in [1, 16]");
  const cudaError_t e = gqb::launch_p2p_signal(peer_slots, n, epoch, nullptr, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT int gq_p2p_wait(const uint32_t* flags, uint32_t n, uint32_t epoch, uint32_t* err, void* stream) {
  if (n == 0 || n > gqb::kMaxPeers || !flags) return fail(GQ_ERR_INVALID, "peer count must be in [1, 16]");
  const cudaError_t e = gqb::launch_p2p_wait(flags, n, epoch, nullptr, err, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT size_t gq_ipc_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

GQ_EXPORT int gq_ipc_get(void* ptr, void* handle_out) {
  if (!ptr || !handle_out) return fail(GQ_ERR_INVALID, "null argument");
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, ptr);
  if (e != cudaSuccess) return cuda_fail(e);
  std::memcpy(handle_out, &h, sizeof(h));
  return GQ_OK;
}

GQ_EXPORT int gq_ipc_open(const void* handle, void** ptr_out) {
  if (!handle || !ptr_out) return fail(GQ_ERR_INVALID, "null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  const cudaError_t e = cudaIpcOpenMemHandle(ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT int gq_ipc_close(void* ptr) {
  const cudaError_t e = cudaIpcCloseMemHandle(ptr);
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT int gq_dequant(const void* lanes, uint64_t lane_begin, uint64_t lane_end,
                         const double* norm, uint32_t kind, uint32_t s, uint32_t n,
                         uint32_t width, float* out, float* param, float lr,
                         uint32_t* err, void* stream) {
  if (int rc = check_lane_args(kind, width, s, n)) return rc;
  const uint32_t G = lanes_per_word(width);
  if (lane_begin > lane_end || lane_begin % G != 0) return fail(GQ_ERR_INVALID, "bad lane range");
  if (!lanes || !norm || !aligned(lanes, 16)) return fail(GQ_ERR_INVALID, "device buffers must be 16-byte aligned");
  if ((out && !aligned(out, 16)) || (param && !aligned(param, 4)))
    return fail(GQ_ERR_INVALID, "device buffers must be 16-byte aligned");
  const cudaError_t e = gqb::launch_dequant(lanes, lane_begin, lane_end, norm, kind, s, n, width, out,
                                            param, lr, err, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

// decode_dense_std / decode_dense_exp (algorithm.cpp:84-110) into doubles,
// bit-identical to the reference's decoders (the drop-in's MeanResult).
GQ_EXPORT int gq_dequant_f64(const void* lanes, uint64_t lane_begin, uint64_t lane_end,
                             const double* norm, uint32_t kind, uint32_t s, uint32_t n,
                             uint32_t width, double* out, uint32_t* err, void* stream) {
  if (int rc = check_lane_args(kind, width, s, n)) return rc;
  if (lane_begin > lane_end) return fail(GQ_ERR_INVALID, "bad lane range");
  if (width == 4 && lane_begin % 2 != 0) return fail(GQ_ERR_INVALID, "4-bit lanes decode from an even lane");
  if (lane_end > lane_begin && (!lanes || !norm || !out)) return fail(GQ_ERR_INVALID, "null argument");
  const cudaError_t e = gqb::launch_dequant_f64(lanes, lane_begin, lane_end, norm, kind, s, n, width, out,
                                                err, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

// Device memory plumbing for callers that do not link the CUDA runtime
// (C/C++/Go/Java bindings of this ABI).
GQ_EXPORT int gq_malloc(size_t bytes, void** out) {
  if (!out) return fail(GQ_ERR_INVALID, "null argument");
  *out = nullptr;
  if (bytes == 0) return GQ_OK;
  const cudaError_t e = cudaMalloc(out, bytes);
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT int gq_malloc_host(size_t bytes, void** out) {
  if (!out) return fail(GQ_ERR_INVALID, "null argument");
  *out = nullptr;
  if (bytes == 0) return GQ_OK;
  const cudaError_t e = cudaMallocHost(out, bytes);
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT int gq_free_host(void* p) {
  const cudaError_t e = cudaFreeHost(p);
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT int gq_free(void* p) {
  const cudaError_t e = cudaFree(p);
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT int gq_memcpy(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes == 0) return GQ_OK;
  const cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT int gq_memset(void* dst, int value, size_t bytes, void* stream) {
  if (bytes == 0) return GQ_OK;
  const cudaError_t e = cudaMemsetAsync(dst, value, bytes, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT int gq_stream_sync(void* stream) {
  const cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

// ---- sparse path ----
namespace {
uint32_t prescale_shift_of(uint32_t n) { return ceil_log2_u64(2ull * n); }

int check_sparse_args(uint32_t kind, uint32_t s, uint32_t width) {
  if (kind != GQ_KIND_STANDARD && kind != GQ_KIND_EXPONENTIAL)
    return fail(GQ_ERR_INVALID, "aggregation requires a named level scheme");
  if (s == 0) return fail(GQ_ERR_INVALID, "level count s must be >= 1");
  // validate_level_width (serialize.cpp:114-122)
  if (width != 8 && width != 16 && width != 32) return fail(GQ_ERR_INVALID, "level lane width must be 8, 16, or 32 bits");
  if (width < 32 && s > ((1u << width) - 1)) return fail(GQ_ERR_INVALID, "level index does not fit the lane width");
  return GQ_OK;
}
}  // namespace

GQ_EXPORT uint64_t gq_sparse_payload_bytes(uint64_t nnz, uint32_t width) {
  return 16 + 4 * nnz + (nnz + 7) / 8 + nnz * (width / 8);
}

GQ_EXPORT size_t gq_sparse_workspace_bytes(uint64_t d) { return gqb::sparse_workspace_bytes(d); }

GQ_EXPORT int gq_sparse_encode(const void* lanes32, uint64_t d, uint32_t kind, uint32_t s, uint32_t n_total,
                               uint32_t width, const double* norm, void* payload, void* workspace,
                               uint32_t* nnz_out, void* stream) {
  if (int rc = check_sparse_args(kind, s, width)) return rc;
  if (d > 0xffffffffull) return fail(GQ_ERR_INVALID, "sparse shards index elements with u32");
  if (n_total == 0) return fail(GQ_ERR_INVALID, "worker count must be >= 1");
  if (!payload || !workspace || !nnz_out || !norm || (d && !lanes32) || !aligned(lanes32, 4))
    return fail(GQ_ERR_INVALID, "null argument");
  const cudaError_t e = gqb::launch_sparse_encode(static_cast<const uint32_t*>(lanes32), d, kind, s,
                                                  prescale_shift_of(n_total), width, norm, payload, workspace,
                                                  nnz_out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT int gq_sparse_mean_inproc(const void* const* lanes32, uint32_t n, uint64_t d, uint32_t kind, uint32_t s,
                                    uint32_t n_total, const double* norm, float* out32, double* out64,
                                    void* stream) {
  if (kind != GQ_KIND_STANDARD && kind != GQ_KIND_EXPONENTIAL)
    return fail(GQ_ERR_INVALID, "aggregation requires a named level scheme");
  if (n == 0 || n > GQ_MAX_WORKERS || n_total == 0) return fail(GQ_ERR_INVALID, "worker count must be in [1, GQ_MAX_WORKERS]");
  if (!lanes32 || !norm) return fail(GQ_ERR_INVALID, "null argument");
  const cudaError_t e = gqb::launch_sparse_mean(lanes32, n, d, kind, s, prescale_shift_of(n_total), norm, n, out32,
                                                out64, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT int gq_sparse_accumulate(const void* payload, uint64_t payload_bytes, uint32_t kind, uint32_t s,
                                   uint32_t width, uint64_t d, double* acc, uint32_t* err, void* stream) {
  if (int rc = check_sparse_args(kind, s, width)) return rc;
  if (!payload || !acc) return fail(GQ_ERR_INVALID, "null argument");
  const cudaError_t e = gqb::launch_sparse_scatter(payload, payload_bytes, kind, s, width, d, acc, err,
                                                   static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT int gq_sparse_finish(const double* acc, uint64_t d, uint32_t n, float* out32, double* out64,
                               float* param, float lr, void* stream) {
  if (n == 0) return fail(GQ_ERR_INVALID, "worker count must be >= 1");
  const cudaError_t e = gqb::launch_scale(acc, d, n, out32, out64, param, lr, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT int gq_mean_inproc(const void* const* shards, uint32_t dtype, uint64_t d,
                             const gq_config* cfg, uint64_t round, void* const* lane_bufs,
                             void* result_lanes, float* mean_out, float* param, float lr,
                             double* stats_out, double* norm_out, void* workspace,
                             uint32_t* err, void* stream) {
  gq_plan plan;
  if (int rc = gq_plan_path(cfg, &plan)) return rc;
  const uint32_t n = cfg->workers;
  if (!lane_bufs || !stats_out || !norm_out) return fail(GQ_ERR_INVALID, "null argument");
  if (gqb::small_path_applies(dtype, n, d, cfg->kind, cfg->s, plan.lane_width, cfg->topo, cfg->norm_q,
                              cfg->norm_p) &&
      shards && workspace) {  // one cooperative launch for the whole step
    for (uint32_t i = 0; i < n; ++i)
      if (!shards[i] || !aligned(shards[i], 16) || !lane_bufs[i] || !aligned(lane_bufs[i], 16))
        return fail(GQ_ERR_INVALID, "device buffers must be 16-byte aligned");
    if ((result_lanes && !aligned(result_lanes, 16)) || (mean_out && !aligned(mean_out, 16)) ||
        (param && !aligned(param, 4)))
      return fail(GQ_ERR_INVALID, "device buffers must be 16-byte aligned");
    const cudaError_t e = gqb::launch_mean_small(shards, n, d, cfg->kind, cfg->s, plan.lane_width, cfg->norm_p,
                                                 cfg->seed, round, nullptr, nullptr, lane_bufs, result_lanes,
                                                 mean_out, param, lr, stats_out, norm_out, workspace, err,
                                                 static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? GQ_OK : cuda_fail(e);
  }
  if (int rc = gq_norm(shards, dtype, n, d, cfg->norm_q, cfg->norm_p, stats_out, norm_out, workspace,
                       err, stream))
    return rc;
  if (gqb::fused_path_applies(dtype, n, d, cfg->kind, plan.lane_width, cfg->topo, false)) {
    if ((result_lanes && !aligned(result_lanes, 16)) || (mean_out && !aligned(mean_out, 16)) ||
        (param && !aligned(param, 4)))
      return fail(GQ_ERR_INVALID, "device buffers must be 16-byte aligned");
    for (uint32_t i = 0; i < n; ++i)
      if (!lane_bufs[i] || !aligned(lane_bufs[i], 16)) return fail(GQ_ERR_INVALID, "device buffers must be 16-byte aligned");
    const cudaError_t e = gqb::launch_fused_qr(shards, n, d, cfg->kind, cfg->s, plan.lane_width, cfg->seed, round,
                                               nullptr, nullptr, nullptr, lane_bufs, result_lanes, mean_out, param,
                                               lr, norm_out, nullptr, err, static_cast<cudaStream_t>(stream));
    return e == cudaSuccess ? GQ_OK : cuda_fail(e);
  }
  uint32_t ids[GQ_MAX_WORKERS];
  for (uint32_t i = 0; i < n; ++i) ids[i] = i;
  if (int rc = gq_quantize(shards, dtype, n, ids, d, norm_out, cfg->kind, cfg->s, n, plan.lane_width,
                           cfg->seed, round, lane_bufs, err, stream))
    return rc;
  return gq_reduce_lanes(lane_bufs, n, d, 0, d, cfg->kind, plan.lane_width, cfg->s, cfg->topo,
                         cfg->seed, round, norm_out, result_lanes, mean_out, param, lr, err, stream);
}

// ---- CUDA graph of the whole in-process path ----
namespace {

}  // namespace


GQ_EXPORT int gq_graph_mean_inproc(const void* const* shards, uint32_t dtype, uint64_t d, const gq_config* cfg,
                                   uint64_t* round_dev, void* const* lane_bufs, void* result_lanes, float* mean_out,
                                   float* param, float lr, double* stats_out, double* norm_out, void* workspace,
                                   uint32_t* kdraws_buf, uint32_t* err, gq_graph** out) {
  gq_plan plan;
  if (int rc = gq_plan_path(cfg, &plan)) return rc;
  if (!out || !round_dev || !lane_bufs || !stats_out || !norm_out || !workspace || !shards)
    return fail(GQ_ERR_INVALID, "null argument");
  const uint32_t n = cfg->workers;
  for (uint32_t i = 0; i < n; ++i) {
    if (!shards[i] || !aligned(shards[i], 16) || !lane_bufs[i] || !aligned(lane_bufs[i], 16))
      return fail(GQ_ERR_INVALID, "device buffers must be 16-byte aligned");
  }
  gq_kdraws spec{};
  spec.buf = kdraws_buf;
  spec.n = n;
  spec.kind = cfg->kind;
  spec.width = plan.lane_width;
  spec.s = cfg->s;
  spec.topo = cfg->topo;
  spec.lane_begin = 0;
  spec.lane_end = d;
  spec.seed = cfg->seed;
  const bool kd = kdraws_buf && kdraws_applicable(&spec) && cfg->norm_q != GQ_NORM_L2_SEQUENTIAL;

  if (!device_orders(cfg->norm_q, cfg->norm_p))
    return fail(GQ_ERR_INVALID, "norm orders other than 2 / inf take a host step and cannot be captured in a graph");
  const bool small = gqb::small_path_applies(dtype, n, d, cfg->kind, cfg->s, plan.lane_width, cfg->topo,
                                             cfg->norm_q, cfg->norm_p);
  cudaStream_t st;
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e != cudaSuccess) return cuda_fail(e);
  auto* g = new gq_graph();
  e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess && small) {  // the whole step is one cooperative kernel; it advances the round
    const cudaError_t le = gqb::launch_mean_small(shards, n, d, cfg->kind, cfg->s, plan.lane_width, cfg->norm_p,
                                                  cfg->seed, 0, round_dev, round_dev, lane_bufs, result_lanes,
                                                  mean_out, param, lr, stats_out, norm_out, workspace, err, st);
    e = cudaStreamEndCapture(st, &g->graph);
    if (le != cudaSuccess) e = le;
  } else if (e == cudaSuccess) {
    gqb::KDrawJob job{};
    if (kd) {
      job.buf = kdraws_buf;
      job.kwords = kdraws_words(&spec);
      job.width = spec.width;
      job.m = spec.s + 1;
      job.events = gqb::tree_event_keys(n, cfg->seed, 0, job.keys, gqb::kMaxKEvents);
      job.round_ptr = round_dev;
      job.seed = cfg->seed;
      job.n = n;
    }
    cudaError_t le = gqb::launch_norm(shards, dtype, n, d, cfg->norm_q, cfg->norm_p, stats_out, norm_out, workspace,
                                      err, st, kd ? &job : nullptr);
    uint32_t ids[GQ_MAX_WORKERS];
    for (uint32_t i = 0; i < n; ++i) ids[i] = i;
    const bool fused = gqb::fused_path_applies(dtype, n, d, cfg->kind, plan.lane_width, cfg->topo, kd);
    if (le == cudaSuccess && fused) {  // quantize + replay + decode per tile; it advances the round
      le = gqb::launch_fused_qr(shards, n, d, cfg->kind, cfg->s, plan.lane_width, cfg->seed, 0, round_dev, round_dev,
                                reinterpret_cast<unsigned int*>(static_cast<char*>(workspace) + gqb::kWsRoundTicket),
                                lane_bufs, result_lanes, mean_out, param, lr, norm_out, kd ? kdraws_buf : nullptr,
                                err, st);
    }
    if (le == cudaSuccess && !fused) {
      gqb::QuantLaunch q{shards, dtype, n, ids, d, norm_out, cfg->kind, cfg->s, n, plan.lane_width,
                         cfg->seed, 0, lane_bufs, err};
      q.round_ptr = round_dev;
      le = gqb::launch_quantize(q, st);
    }
    if (le == cudaSuccess && !fused) {
      gqb::ReduceLaunch r{lane_bufs, n, d, 0, d, cfg->kind, plan.lane_width, cfg->s, cfg->topo, cfg->seed, 0,
                          norm_out, result_lanes, mean_out, param, lr, err};
      r.round_ptr = round_dev;
      r.round_inc = round_dev;  // the reduce's last block advances the round (no extra launch)
      r.round_step = 1;
      r.round_ticket = reinterpret_cast<unsigned int*>(static_cast<char*>(workspace) + gqb::kWsRoundTicket);
      if (kd) {
        r.kdraws = kdraws_buf;
        r.kstride = kdraws_words(&spec);
      }
      le = gqb::launch_reduce(r, st);
    }
    if (le == cudaSuccess && d == 0) le = gqb::launch_round_inc(round_dev, 1, st);  // no reduce grid ran
    e = cudaStreamEndCapture(st, &g->graph);
    if (le != cudaSuccess) e = le;
  }
  if (e == cudaSuccess) e = cudaGraphInstantiate(&g->exec, g->graph, 0);
  cudaStreamDestroy(st);
  if (e != cudaSuccess) {
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
    return cuda_fail(e);
  }
  *out = g;
  return GQ_OK;
}

GQ_EXPORT int gq_graph_launch(gq_graph* g, void* stream) {
  if (!g) return fail(GQ_ERR_INVALID, "null argument");
  const cudaError_t e = cudaGraphLaunch(g->exec, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT int gq_graph_destroy(gq_graph* g) {
  if (!g) return GQ_OK;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  delete g;
  return GQ_OK;
}

GQ_EXPORT int gq_baseline_mean_inproc(const float* const* shards, uint32_t n, uint64_t d,
                                      uint32_t topo, float* mean_out, void* stream) {
  if (n == 0 || n > GQ_MAX_WORKERS) return fail(GQ_ERR_INVALID, "shard count does not match the worker count");
  if (topo != GQ_TOPO_TREE) return fail(GQ_ERR_INVALID, "device baseline walks the tree schedule");
  const cudaError_t e = gqb::launch_baseline_mean(shards, n, d, topo, mean_out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? GQ_OK : cuda_fail(e);
}

GQ_EXPORT int gq_check(uint32_t* err, void* stream) {
  cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e);
  if (!err) return GQ_OK;
  uint32_t flags = 0;
  e = cudaMemcpy(&flags, err, sizeof(flags), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e);
  if (flags == 0) return GQ_OK;
  const uint32_t zero = 0;
  e = cudaMemcpy(err, &zero, sizeof(zero), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e);
  return gqb::status_from_flags(flags);
}

namespace gqb {
int api_fail(int code, const char* msg) { return fail(code, msg); }
int api_cuda_fail(cudaError_t e) { return cuda_fail(e); }

int status_from_flags(uint32_t flags) {
  if (flags == 0) return GQ_OK;
  // Same precedence as the reference's control flow: the norm phase rejects
  // NaN/Inf before quantize ever looks at the scale.
  if (flags & GQ_FLAG_NONFINITE) return fail(GQ_ERR_INVALID, "gradient contains NaN or Inf");
  if (flags & GQ_FLAG_BAD_SCALE) return fail(GQ_ERR_INVALID, "scale must be finite and nonnegative");
  if (flags & GQ_FLAG_ZERO_SCALE) return fail(GQ_ERR_INVALID, "zero scale with nonzero gradient");
  if (flags & GQ_FLAG_EXCEEDS_SCALE) return fail(GQ_ERR_INVALID, "element magnitude exceeds the scale");
  if (flags & GQ_FLAG_LANE_OVERFLOW) return fail(GQ_ERR_OVERFLOW, "integer lane overflow during aggregation");
  if (flags & GQ_FLAG_TOKEN_RANGE)
    return fail(GQ_ERR_OVERFLOW, "aggregated exponent left the representable range");
  if (flags & GQ_FLAG_NEG_ZERO) return fail(GQ_ERR_DOMAIN, "negative zero token on the wire");
  if (flags & GQ_FLAG_BAD_PAYLOAD) return fail(GQ_ERR_DOMAIN, "malformed sparse payload");
  if (flags & GQ_FLAG_P2P_TIMEOUT) return fail(GQ_ERR_RUNTIME, "peer exchange timed out waiting for a rank");
  return fail(GQ_ERR_RUNTIME, "unknown device error flag");
}
}  // namespace gqb
