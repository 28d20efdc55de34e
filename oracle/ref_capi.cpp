// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It lets
// pytest (ctypes) and bench.py's cpu_baseline / --impl reference legs call
// the reference's own hot-path functions on the same inputs as the CUDA path.
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and the
// reference arm) may load the resulting library.
//
// Every wrapper forwards to the public reference API; the only logic written
// here is the lane encoding of the standard grid, because the reference keeps
// encode_dense_std / decode_dense_std file-private (algorithm.cpp:69-100); the
// restatement below follows those lines exactly.
//
// Status codes (shared with the product C-ABI, include/gq_b200.h):
//   0 ok, 1 std::invalid_argument, 2 std::overflow_error,
//   3 std::domain_error, 4 std::runtime_error, 5 other.

#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "gqsgd/algorithm.hpp"
#include "gqsgd/collectives.hpp"
#include "gqsgd/exp_arith.hpp"
#include "gqsgd/levels.hpp"
#include "gqsgd/norms.hpp"
#include "gqsgd/quantizer.hpp"
#include "gqsgd/rng.hpp"
#include "gqsgd/serialize.hpp"
#include "gqsgd/topology.hpp"
#include "gqsgd/verify.hpp"

#define GQR_API extern "C" __attribute__((visibility("default")))

using namespace gqsgd;

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return 1;
  } catch (const std::overflow_error& e) {
    g_last_error = e.what();
    return 2;
  } catch (const std::domain_error& e) {
    g_last_error = e.what();
    return 3;
  } catch (const std::runtime_error& e) {
    g_last_error = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return 5;
  }
}

LevelScheme make_scheme(std::uint32_t kind, std::uint32_t s) {
  return kind == 0 ? LevelScheme::standard(s) : LevelScheme::exponential(s);
}

GqsgdConfig make_cfg(std::uint32_t n, std::uint32_t kind, std::uint32_t s,
                     std::uint32_t q, std::uint32_t p, std::uint32_t width,
                     std::uint32_t topo, std::uint32_t transport,
                     std::uint64_t seed) {
  GqsgdConfig cfg;
  cfg.workers = n;
  cfg.scheme = kind == 0 ? LevelKind::Standard : LevelKind::Exponential;
  cfg.s = s;
  cfg.norm = NormSpec{q, p};
  cfg.sparse = false;
  cfg.width_bits = width;
  cfg.topo = topo == 0 ? TopologyKind::Tree : TopologyKind::Ring;
  cfg.transport = transport == 0 ? Transport::Inproc : Transport::Tcp;
  cfg.seed = seed;
  return cfg;
}

}  // namespace

GQR_API const char* gqr_last_error() { return g_last_error.c_str(); }

// rng.hpp:45-61
GQR_API std::uint64_t gqr_rng_bits(std::uint64_t seed, std::uint64_t stream,
                                   std::uint64_t a, std::uint64_t b,
                                   std::uint64_t c) {
  return CounterRng(seed).bits(static_cast<RngStream>(stream), a, b, c);
}

GQR_API double gqr_rng_u01(std::uint64_t seed, std::uint64_t stream,
                           std::uint64_t a, std::uint64_t b, std::uint64_t c) {
  return CounterRng(seed).u01(static_cast<RngStream>(stream), a, b, c);
}

// verify.cpp:118-128
GQR_API int gqr_gaussian_shards(std::uint32_t n, std::uint64_t d,
                                std::uint64_t seed, double* out) {
  return guarded([&] {
    const auto shards = gaussian_shards(n, d, seed);
    for (std::uint32_t r = 0; r < n; ++r) {
      std::memcpy(out + r * d, shards[r].data(), d * sizeof(double));
    }
  });
}

// Columns [j0, j0 + cnt) of gaussian_shards(n, d, seed) (verify.cpp:118-128
// draws element (i, j) as rng.normal(ShardGen, i, j, 0), independent of d).
GQR_API int gqr_gaussian_range(std::uint32_t n, std::uint64_t j0, std::uint64_t cnt,
                               std::uint64_t seed, double* out) {
  return guarded([&] {
    const CounterRng rng(seed);
    for (std::uint32_t i = 0; i < n; ++i)
      for (std::uint64_t j = 0; j < cnt; ++j)
        out[i * cnt + j] = rng.normal(RngStream::ShardGen, i, j0 + j, 0);
  });
}

// levels.cpp:31-48
GQR_API int gqr_levels(std::uint32_t kind, std::uint32_t s, double* out) {
  return guarded([&] {
    const LevelScheme sch = make_scheme(kind, s);
    std::memcpy(out, sch.levels().data(), (s + 1) * sizeof(double));
  });
}

// levels.cpp:63-76
GQR_API int gqr_bracket_index(std::uint32_t kind, std::uint32_t s, double y,
                              std::uint32_t* out) {
  return guarded([&] { *out = make_scheme(kind, s).bracket_index(y); });
}

// levels.cpp:78-84
GQR_API int gqr_random_round(std::uint32_t kind, std::uint32_t s, double y,
                             double u, std::uint32_t* out) {
  return guarded([&] { *out = make_scheme(kind, s).random_round(y, u); });
}

// norms.cpp:52-62
GQR_API int gqr_local_norm_stat(const double* x, std::uint64_t d,
                                std::uint32_t q, std::uint32_t p, double* out) {
  return guarded([&] {
    *out = local_norm_stat(std::span<const double>(x, d), NormSpec{q, p});
  });
}

// norms.cpp:64-75
GQR_API int gqr_combine_norm_stats(const double* stats, std::uint32_t n,
                                   std::uint32_t q, std::uint32_t p,
                                   double* out) {
  return guarded([&] {
    *out = combine_norm_stats(std::span<const double>(stats, n), NormSpec{q, p});
  });
}

// collectives.cpp:210-233
GQR_API int gqr_norm_allreduce_inproc(const double* stats, std::uint32_t n,
                                      std::uint32_t q, std::uint32_t p,
                                      std::uint64_t round, double* out) {
  return guarded([&] {
    std::vector<double> v(stats, stats + n);
    *out = norm_allreduce_inproc(v, NormSpec{q, p}, round).value;
  });
}

// quantizer.cpp:8-48
GQR_API int gqr_quantize_shard(const double* x, std::uint64_t d, double norm,
                               std::uint32_t kind, std::uint32_t s,
                               std::uint64_t seed, std::uint32_t worker,
                               std::uint64_t round, std::int8_t* sign,
                               std::uint32_t* level_idx) {
  return guarded([&] {
    const QuantizedShard q =
        quantize_shard(std::span<const double>(x, d), norm, make_scheme(kind, s),
                       CounterRng(seed), worker, round);
    std::memcpy(sign, q.sign.data(), d);
    std::memcpy(level_idx, q.level_idx.data(), d * sizeof(std::uint32_t));
  });
}

// exp_arith.cpp:24-41
GQR_API int gqr_check_width(std::uint32_t kind, std::uint32_t s,
                            std::uint32_t n, std::uint32_t width) {
  return check_width(kind == 0 ? LevelKind::Standard : LevelKind::Exponential, s,
                     n, width)
             ? 1
             : 0;
}

// algorithm.cpp:22-29
GQR_API std::uint32_t gqr_standard_lane_width(std::uint32_t s, std::uint32_t n,
                                              std::uint32_t at_least) {
  const auto w = standard_lane_width(s, n, at_least);
  return w ? *w : 0;
}

// exp_arith.cpp:43-50
GQR_API int gqr_sample_k(double u, std::uint32_t m, std::uint32_t* out) {
  return guarded([&] { *out = sample_k(u, m); });
}

// exp_arith.cpp:82-109. Tokens as (sign, e) pairs.
GQR_API int gqr_reduce_pair(std::int32_t sa, std::uint32_t ea, std::int32_t sb,
                            std::uint32_t eb, std::uint32_t k, std::uint32_t s,
                            std::uint32_t n, std::uint32_t width,
                            std::int32_t* so, std::uint32_t* eo) {
  return guarded([&] {
    const ReduceContext ctx = ReduceContext::make(s, n, width);
    const ExpToken r =
        reduce_pair(ExpToken{static_cast<std::int8_t>(sa), ea},
                    ExpToken{static_cast<std::int8_t>(sb), eb}, k, ctx);
    *so = r.sign;
    *eo = r.e;
  });
}

// Lane encoding of one quantized shard, written into `lanes`
// (d * width/8 bytes). Standard: restates encode_dense_std
// (algorithm.cpp:69-82), lane = sign * (s - idx), w-bit two's complement LE.
// Exponential: pack_tokens(tokens_from_shard(q, ctx), width)
// (exp_arith.cpp:126-136, 143-160).
GQR_API int gqr_encode(std::uint32_t kind, std::uint32_t s, std::uint32_t n,
                       std::uint32_t width, const std::int8_t* sign,
                       const std::uint32_t* level_idx, std::uint64_t d,
                       std::uint8_t* lanes) {
  return guarded([&] {
    const std::uint32_t lb = width / 8;
    if (kind == 0) {
      for (std::uint64_t j = 0; j < d; ++j) {
        const std::int64_t v =
            std::int64_t{sign[j]} * (std::int64_t{s} - level_idx[j]);
        const auto u = static_cast<std::uint64_t>(v);
        for (std::uint32_t i = 0; i < lb; ++i) {
          lanes[j * lb + i] = static_cast<std::uint8_t>((u >> (8 * i)) & 0xff);
        }
      }
      return;
    }
    const ReduceContext ctx = ReduceContext::make(s, n, width);
    QuantizedShard q;
    q.sign.assign(sign, sign + d);
    q.level_idx.assign(level_idx, level_idx + d);
    const Payload p = pack_tokens(tokens_from_shard(q, ctx), width);
    std::memcpy(lanes, p.data(), p.size());
  });
}

// collectives.cpp:155-190 with IntSumOps (kind 0, collectives.cpp:60-81) or
// TokenReduceOps (kind 1, collectives.cpp:125-153). `lanes` holds n payloads
// back to back (each lanes_per_worker * width/8 bytes); every worker's
// payload is overwritten with its result.
GQR_API int gqr_allreduce_inproc(std::uint8_t* lanes, std::uint32_t n,
                                 std::uint64_t lanes_per_worker,
                                 std::uint32_t kind, std::uint32_t width,
                                 std::uint32_t s, std::uint32_t topo,
                                 std::uint64_t seed, std::uint64_t round,
                                 std::uint64_t* traffic_bytes) {
  return guarded([&] {
    const std::uint64_t bytes = lanes_per_worker * (width / 8);
    std::vector<Payload> payloads(n, Payload(bytes));
    for (std::uint32_t r = 0; r < n; ++r) {
      std::memcpy(payloads[r].data(), lanes + r * bytes, bytes);
    }
    const Schedule sched =
        make_schedule(topo == 0 ? TopologyKind::Tree : TopologyKind::Ring, n);
    AllreduceResult res;
    if (kind == 0) {
      res = allreduce_inproc(std::move(payloads), sched, IntSumOps{width}, round);
    } else {
      const ReduceContext ctx = ReduceContext::make(s, n, width);
      res = allreduce_inproc(std::move(payloads), sched,
                             TokenReduceOps{ctx, CounterRng(seed)}, round);
    }
    for (std::uint32_t r = 0; r < n; ++r) {
      std::memcpy(lanes + r * bytes, res.per_worker[r].data(), bytes);
    }
    if (traffic_bytes) *traffic_bytes = res.traffic.total_bytes;
  });
}

// One PayloadOps::combine event (collectives.hpp:39-48): the reference's own
// IntSumOps / TokenReduceOps plugin applied to acc (+) in, `lanes` lanes of
// width/8 bytes starting at global lane elem_offset.
GQR_API int gqr_payload_combine(std::uint8_t* acc, const std::uint8_t* in,
                                std::uint64_t lanes, std::uint64_t elem_offset,
                                std::uint32_t kind, std::uint32_t width,
                                std::uint32_t s, std::uint32_t n,
                                std::uint64_t seed, std::uint64_t round,
                                std::uint32_t step, std::uint32_t dst) {
  return guarded([&] {
    const std::size_t bytes = lanes * (width / 8);
    std::span<std::byte> a(reinterpret_cast<std::byte*>(acc), bytes);
    std::span<const std::byte> b(reinterpret_cast<const std::byte*>(in), bytes);
    if (kind == 0) {
      IntSumOps{width}.combine(a, b, round, step, dst, elem_offset);
    } else {
      const ReduceContext ctx = ReduceContext::make(s, n, width);
      TokenReduceOps{ctx, CounterRng(seed)}.combine(a, b, round, step, dst, elem_offset);
    }
  });
}

// serialize_sparse(to_sparse(quantize_shard(...))) with validate_level_width
// (serialize.cpp:114-168, quantizer.cpp:59-71): the sparse wire payload.
GQR_API int gqr_sparse_payload(const double* x, std::uint64_t d, double norm, std::uint32_t kind,
                               std::uint32_t s, std::uint64_t seed, std::uint32_t worker,
                               std::uint64_t round, std::uint32_t width, std::uint8_t* out,
                               std::uint64_t cap, std::uint64_t* size) {
  return guarded([&] {
    const LevelScheme scheme = make_scheme(kind, s);
    const QuantizedShard q = quantize_shard(std::span<const double>(x, d), norm, scheme, CounterRng(seed),
                                            worker, round);
    const Payload p = serialize_sparse(to_sparse(q, scheme), validate_level_width(width, s));
    if (p.size() > cap) throw std::runtime_error("payload buffer too small");
    std::memcpy(out, p.data(), p.size());
    *size = p.size();
  });
}

// gqsgd_mean with cfg.sparse = true (algorithm.cpp:187-200): the allgather path.
GQR_API int gqr_gqsgd_mean_sparse(const double* shards, std::uint32_t n, std::uint64_t d,
                                  std::uint32_t kind, std::uint32_t s, std::uint32_t q,
                                  std::uint32_t p, std::uint32_t width, std::uint32_t transport,
                                  std::uint64_t seed, std::uint64_t round, double* mean_out,
                                  double* norm_out, std::uint64_t* payload_bytes_out) {
  return guarded([&] {
    std::vector<std::vector<double>> v(n);
    for (std::uint32_t r = 0; r < n; ++r) v[r].assign(shards + r * d, shards + (r + 1) * d);
    GqsgdConfig cfg = make_cfg(n, kind, s, q, p, width, 0, transport, seed);
    cfg.sparse = true;
    const MeanResult res = gqsgd_mean(v, cfg, round);
    std::memcpy(mean_out, res.mean().data(), d * sizeof(double));
    if (norm_out) *norm_out = res.norm;
    if (payload_bytes_out) *payload_bytes_out = res.payload_traffic.total_bytes;
  });
}

// Whole path, algorithm.cpp:127-228 (transport 0 = Inproc, 1 = Tcp).
// Writes worker 0's mean (all workers are bit-identical), the global norm and
// the lane width the plan used.
GQR_API int gqr_gqsgd_mean(const double* shards, std::uint32_t n,
                           std::uint64_t d, std::uint32_t kind, std::uint32_t s,
                           std::uint32_t q, std::uint32_t p, std::uint32_t width,
                           std::uint32_t topo, std::uint32_t transport,
                           std::uint64_t seed, std::uint64_t round,
                           double* mean_out, double* norm_out,
                           std::uint32_t* lane_width_out,
                           std::uint64_t* payload_bytes_out) {
  return guarded([&] {
    std::vector<std::vector<double>> v(n);
    for (std::uint32_t r = 0; r < n; ++r) v[r].assign(shards + r * d, shards + (r + 1) * d);
    const MeanResult res =
        gqsgd_mean(v, make_cfg(n, kind, s, q, p, width, topo, transport, seed), round);
    std::memcpy(mean_out, res.mean().data(), d * sizeof(double));
    if (norm_out) *norm_out = res.norm;
    if (lane_width_out) *lane_width_out = res.lane_width_used;
    if (payload_bytes_out) *payload_bytes_out = res.payload_traffic.total_bytes;
  });
}

// algorithm.cpp:303-340 (uncompressed fp32 reference path).
GQR_API int gqr_baseline_mean(const double* shards, std::uint32_t n,
                              std::uint64_t d, std::uint32_t topo,
                              std::uint32_t transport, std::uint64_t round,
                              double* mean_out) {
  return guarded([&] {
    std::vector<std::vector<double>> v(n);
    for (std::uint32_t r = 0; r < n; ++r) v[r].assign(shards + r * d, shards + (r + 1) * d);
    const BaselineResult res =
        baseline_mean(v, n, topo == 0 ? TopologyKind::Tree : TopologyKind::Ring,
                      transport == 0 ? Transport::Inproc : Transport::Tcp, round);
    std::memcpy(mean_out, res.per_worker.front().data(), d * sizeof(double));
  });
}

// Schedule event list (topology.cpp:19-72): writes up to `cap` events as
// (step, src, dst, op, chunk) quintuples; returns the event count.
GQR_API std::int64_t gqr_schedule(std::uint32_t topo, std::uint32_t n,
                                  std::uint32_t* out, std::uint64_t cap) {
  const Schedule sched =
      make_schedule(topo == 0 ? TopologyKind::Tree : TopologyKind::Ring, n);
  const std::uint64_t count = sched.events.size();
  for (std::uint64_t i = 0; i < count && i < cap; ++i) {
    const CommEvent& e = sched.events[i];
    out[5 * i + 0] = e.step;
    out[5 * i + 1] = e.src;
    out[5 * i + 2] = e.dst;
    out[5 * i + 3] = e.op == CommOp::Reduce ? 0 : 1;
    out[5 * i + 4] = e.chunk;
  }
  return static_cast<std::int64_t>(count);
}
