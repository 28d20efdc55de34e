// Drop-in check: the reference library's own API with the GPU path swapped in
// (gqsgd_b200::*) against the unmodified reference, bit for bit. Built by
// integration/Makefile against /root/reference/proj (headers + sources, read
// in place) and libgq_b200.so; run on a B200 by tests/test_gpu_dropin.py.
// Prints one PASS/FAIL line per check; exit status 0 iff all pass.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "gqsgd/algorithm.hpp"
#include "gqsgd/collectives.hpp"
#include "gqsgd/exp_arith.hpp"
#include "gqsgd/quantizer.hpp"
#include "gqsgd/topology.hpp"
#include "gqsgd/transport.hpp"
#include "gqsgd/verify.hpp"
#include "gqsgd_b200.hpp"

using namespace gqsgd;

namespace {

int g_fail = 0;

void report(bool ok, const std::string& what) {
  std::printf("%s %s\n", ok ? "PASS" : "FAIL", what.c_str());
  if (!ok) ++g_fail;
}

bool same_traffic(const TrafficReport& a, const TrafficReport& b) {
  return a.bytes_sent == b.bytes_sent && a.total_bytes == b.total_bytes && a.messages == b.messages &&
         a.steps == b.steps && a.reduce_invocations == b.reduce_invocations;
}

// encode_dense_std (algorithm.cpp:69-82) is file-private in the reference;
// restated here for building test payloads.
Payload encode_std(const QuantizedShard& q, std::uint32_t s, std::uint32_t width) {
  const std::uint32_t lb = width / 8;
  Payload out(q.size() * lb);
  for (std::size_t j = 0; j < q.size(); ++j) {
    const auto u = static_cast<std::uint64_t>(std::int64_t{q.sign[j]} * (std::int64_t{s} - q.level_idx[j]));
    for (std::uint32_t i = 0; i < lb; ++i) out[j * lb + i] = static_cast<std::byte>((u >> (8 * i)) & 0xff);
  }
  return out;
}

template <typename F>
std::string exception_class(F&& f) {
  try {
    f();
  } catch (const std::invalid_argument&) {
    return "invalid_argument";
  } catch (const std::overflow_error&) {
    return "overflow_error";
  } catch (const std::domain_error&) {
    return "domain_error";
  } catch (const std::exception&) {
    return "other";
  }
  return "none";
}

void check_payload_ops() {
  int cases = 0, ok = 0;
  const std::size_t d = 777;
  for (const TopologyKind topo : {TopologyKind::Tree, TopologyKind::Ring}) {
    for (const std::uint32_t n : {2u, 3u, 5u, 8u}) {
      for (const auto& [kind, width, s] :
           std::vector<std::tuple<LevelKind, std::uint32_t, std::uint32_t>>{
               {LevelKind::Standard, 8, 7}, {LevelKind::Standard, 16, 63}, {LevelKind::Standard, 32, 15},
               {LevelKind::Standard, 64, 1000},  // IntSumOps{64} payloads (encode_dense_std's 8-byte case)
               {LevelKind::Exponential, 8, 7}, {LevelKind::Exponential, 16, 12},
               {LevelKind::Exponential, 32, 30}}) {
        if (kind == LevelKind::Standard && width < 64 && n * (s + 1ull) > (1ull << (width - 1))) continue;
        const auto shards = gaussian_shards(n, d, 100 + n + width);
        double norm = 0.0;
        for (const auto& x : shards)
          for (double v : x) norm = std::max(norm, std::fabs(v));
        const LevelScheme scheme = kind == LevelKind::Standard ? LevelScheme::standard(s) : LevelScheme::exponential(s);
        const CounterRng rng(77 + s);
        std::vector<Payload> payloads;
        const ReduceContext ctx = kind == LevelKind::Exponential ? ReduceContext::make(s, n, width) : ReduceContext{};
        for (std::uint32_t r = 0; r < n; ++r) {
          const QuantizedShard q = gqsgd::quantize_shard(shards[r], norm, scheme, rng, r, 9);
          payloads.push_back(kind == LevelKind::Standard ? encode_std(q, s, width)
                                                         : pack_tokens(tokens_from_shard(q, ctx), width));
        }
        const Schedule sched = make_schedule(topo, n);
        AllreduceResult a, b;
        if (kind == LevelKind::Standard) {
          a = allreduce_inproc(payloads, sched, IntSumOps{width}, 9);
          b = allreduce_inproc(payloads, sched, gqsgd_b200::DeviceIntSumOps{width}, 9);
        } else {
          a = allreduce_inproc(payloads, sched, TokenReduceOps{ctx, rng}, 9);
          b = allreduce_inproc(payloads, sched, gqsgd_b200::DeviceTokenReduceOps{ctx, rng}, 9);
        }
        ++cases;
        ok += a.per_worker == b.per_worker && same_traffic(a.traffic, b.traffic);
      }
    }
  }
  report(ok == cases, "PayloadOps plugin: allreduce_inproc with Device{IntSum,TokenReduce}Ops == reference ops (" +
                          std::to_string(ok) + "/" + std::to_string(cases) + " schedules x widths)");
  // exception parity (collectives.cpp:76-78, exp_arith.cpp:103-107)
  Payload x{std::byte{0x7f}}, y{std::byte{0x01}};
  const std::string e1 = exception_class([&] { IntSumOps{8}.combine(x, y, 0, 0, 0, 0); });
  const std::string e2 = exception_class([&] { gqsgd_b200::DeviceIntSumOps{8}.combine(x, y, 0, 0, 0, 0); });
  Payload t1{std::byte{0x01}}, t2{std::byte{0x01}};
  const ReduceContext c7 = ReduceContext::make(7, 2, 8);
  const std::string e3 = exception_class([&] { TokenReduceOps{c7, CounterRng(1)}.combine(t1, t2, 0, 0, 0, 0); });
  Payload t3{std::byte{0x01}};
  const std::string e4 =
      exception_class([&] { gqsgd_b200::DeviceTokenReduceOps{c7, CounterRng(1)}.combine(t3, t2, 0, 0, 0, 0); });
  report(e1 == e2 && e1 == "overflow_error" && e3 == e4 && e3 == "overflow_error",
         "PayloadOps exceptions: lane overflow " + e1 + "/" + e2 + ", token range " + e3 + "/" + e4);
}

void check_quantize_shard() {
  int cases = 0, ok = 0;
  for (const auto& [kind, s] : std::vector<std::pair<LevelKind, std::uint32_t>>{
           {LevelKind::Standard, 1}, {LevelKind::Standard, 15}, {LevelKind::Standard, 31},
           {LevelKind::Standard, 1000}, {LevelKind::Exponential, 4}, {LevelKind::Exponential, 7},
           {LevelKind::Exponential, 30}}) {
    const LevelScheme scheme = kind == LevelKind::Standard ? LevelScheme::standard(s) : LevelScheme::exponential(s);
    const auto shards = gaussian_shards(2, 5003, 31 + s);
    double norm = 0.0;
    for (const auto& x : shards)
      for (double v : x) norm = std::max(norm, std::fabs(v));
    for (std::uint32_t r = 0; r < 2; ++r) {
      const CounterRng rng(5 + r);
      const QuantizedShard a = gqsgd::quantize_shard(shards[r], norm, scheme, rng, r, 1234567);
      const QuantizedShard b = gqsgd_b200::quantize_shard(shards[r], norm, scheme, rng, r, 1234567);
      ++cases;
      ok += a.sign == b.sign && a.level_idx == b.level_idx && a.norm == b.norm;
    }
  }
  const std::vector<double> zeros(64, 0.0);
  const QuantizedShard za = gqsgd::quantize_shard(zeros, 0.0, LevelScheme::exponential(3), CounterRng(3), 1, 9);
  const QuantizedShard zb = gqsgd_b200::quantize_shard(zeros, 0.0, LevelScheme::exponential(3), CounterRng(3), 1, 9);
  ++cases;
  ok += za.sign == zb.sign && za.level_idx == zb.level_idx;
  report(ok == cases, "quantize_shard: sign + level_idx identical (" + std::to_string(ok) + "/" +
                          std::to_string(cases) + ", f64 inputs, std s<=1000, exp s<=30, zero shard)");
  const std::vector<double> big{3.0};
  const std::string e1 = exception_class([&] { gqsgd::quantize_shard(big, 2.0, LevelScheme::standard(2), CounterRng(1), 0, 0); });
  const std::string e2 = exception_class([&] { gqsgd_b200::quantize_shard(big, 2.0, LevelScheme::standard(2), CounterRng(1), 0, 0); });
  report(e1 == e2 && e1 == "invalid_argument", "quantize_shard |x| > norm: " + e1 + "/" + e2);
}

void check_gqsgd_mean() {
  int cases = 0, ok = 0, l2 = 0, l2ok = 0;
  std::string first_bad;
  std::uint64_t r = 0;
  for (const std::uint32_t n : {1u, 2u, 3u, 4u, 5u, 8u, 9u, 16u}) {
    for (const std::size_t d : {std::size_t{1}, std::size_t{33}, std::size_t{1000}, std::size_t{4099}}) {
      for (int variant = 0; variant < 8; ++variant, ++r) {
        GqsgdConfig cfg;
        cfg.workers = n;
        cfg.scheme = variant % 2 ? LevelKind::Standard : LevelKind::Exponential;
        cfg.s = variant % 2 ? (variant == 3 ? 63 : 7) : (variant == 4 ? 4 : 7);
        cfg.topo = (variant / 2) % 2 ? TopologyKind::Ring : TopologyKind::Tree;
        cfg.width_bits = variant == 2 ? 16 : 8;
        cfg.seed = 9000 + r;
        if (variant == 5) cfg.norm = NormSpec{2, 2};
        if (variant >= 6) {  // the sparse allgather path (standard s=2 / exponential s=7)
          cfg.sparse = true;
          cfg.scheme = variant == 6 ? LevelKind::Standard : LevelKind::Exponential;
          cfg.s = variant == 6 ? 2 : 7;
          cfg.width_bits = 8;
        }
        const auto shards = gaussian_shards(n, d, 1200 + r);
        if (!gqsgd_b200::handles(cfg)) continue;
        const MeanResult a = gqsgd::gqsgd_mean(shards, cfg, r);
        const MeanResult b = gqsgd_b200::gqsgd_mean(shards, cfg, r);
        const bool meta = a.lane_width_used == b.lane_width_used && a.per_worker.size() == b.per_worker.size() &&
                          same_traffic(a.payload_traffic, b.payload_traffic) &&
                          same_traffic(a.norm_traffic, b.norm_traffic);
        // L2 too: the drop-in accumulates it in element order (GQ_NORM_L2_SEQUENTIAL)
        bool same = meta && a.norm == b.norm;
        for (std::size_t w = 0; same && w < a.per_worker.size(); ++w)
          same = std::memcmp(a.per_worker[w].data(), b.per_worker[w].data(), d * sizeof(double)) == 0;
        ++(cfg.norm.q == kNormInf ? cases : l2);
        (cfg.norm.q == kNormInf ? ok : l2ok) += same;
        if (!same && first_bad.empty())
          first_bad = " first mismatch n=" + std::to_string(n) + " d=" + std::to_string(d) + " variant " +
                      std::to_string(variant);
      }
    }
  }
  report(ok == cases, "gqsgd_mean (L-inf, dense + sparse): per-worker doubles, norm, lane width, payload + norm traffic identical (" +
                          std::to_string(ok) + "/" + std::to_string(cases) + ")" + first_bad);
  report(l2ok == l2, "gqsgd_mean (L2, sequential device sum): bit-identical as above (" + std::to_string(l2ok) + "/" +
                         std::to_string(l2) + ")");
  {  // 4-bit requests (a device-ABI extension): reference callers get the reference's behaviour
    GqsgdConfig t;
    t.workers = 2;
    t.scheme = LevelKind::Exponential;
    t.s = 3;
    t.width_bits = 4;
    const auto sh4 = gaussian_shards(2, 777, 44);
    const std::string e1 = exception_class([&] { gqsgd::gqsgd_mean(sh4, t, 3); });
    report(!gqsgd_b200::handles(t) && e1 == "invalid_argument",
           "exponential width_bits=4: not taken by the drop-in; the reference throws " + e1);
    t.scheme = LevelKind::Standard;  // standard_lane_width(3, 2, 4) = 8 (algorithm.cpp:22-29)
    const MeanResult a = gqsgd::gqsgd_mean(sh4, t, 3);
    const MeanResult b = gqsgd_b200::gqsgd_mean(sh4, t, 3);
    report(gqsgd_b200::handles(t) && a.lane_width_used == 8 && b.lane_width_used == 8 && a.norm == b.norm &&
               a.per_worker == b.per_worker && same_traffic(a.payload_traffic, b.payload_traffic),
           "standard width_bits=4: lane width 8, payload traffic and means identical to the reference");
  }
  {  // empty shards
    GqsgdConfig e;
    e.workers = 4;
    e.scheme = LevelKind::Standard;
    e.s = 15;
    const std::vector<std::vector<double>> none(4);
    const MeanResult a = gqsgd::gqsgd_mean(none, e, 1);
    const MeanResult b = gqsgd_b200::gqsgd_mean(none, e, 1);
    report(a.norm == b.norm && a.per_worker == b.per_worker && a.lane_width_used == b.lane_width_used &&
               same_traffic(a.payload_traffic, b.payload_traffic) && same_traffic(a.norm_traffic, b.norm_traffic),
           "gqsgd_mean on empty shards: identical result");
  }
  GqsgdConfig bad;
  bad.workers = 16;
  bad.scheme = LevelKind::Exponential;
  bad.s = 124;
  const auto sh = gaussian_shards(16, 8, 1);
  const std::string e1 = exception_class([&] { gqsgd::gqsgd_mean(sh, bad, 0); });
  const std::string e2 = exception_class([&] { gqsgd_b200::gqsgd_mean(sh, bad, 0); });
  report(e1 == e2 && e1 == "invalid_argument", "refused configuration: " + e1 + "/" + e2);
}

// gqsgd_mean_worker over the reference's own local mesh (run_local_mesh,
// transport.cpp:317-330: one thread per rank, TCP loopback sockets). Each rank
// runs the reference worker, then the device worker (gq_comm over peer
// memory, bootstrapped through the same sockets) on the same shard.
void check_mean_worker() {
  int cases = 0, ok = 0;
  std::string first_bad;
  std::uint64_t r = 500;
  for (const std::uint32_t n : {2u, 3u, 4u, 8u}) {
    for (const std::size_t d : {std::size_t{1}, std::size_t{1000}, std::size_t{70001}}) {
      for (int variant = 0; variant < 5; ++variant, ++r) {
        GqsgdConfig cfg;
        cfg.workers = n;
        cfg.transport = Transport::Tcp;
        cfg.scheme = variant % 2 ? LevelKind::Standard : LevelKind::Exponential;
        cfg.s = variant % 2 ? 15 : (variant == 4 ? 4 : 7);
        cfg.topo = (variant / 2) % 2 ? TopologyKind::Ring : TopologyKind::Tree;
        cfg.width_bits = 8;
        if (variant == 4) cfg.norm = NormSpec{2, kNormInf};
        cfg.seed = 7000 + r;
        if (variant == 3) cfg.norm = NormSpec{2, 2};
        if (!gqsgd_b200::handles_worker(cfg)) continue;
        const auto shards = gaussian_shards(n, d, 300 + r);
        std::vector<WorkerMeanResult> a(n), b(n);
        std::vector<std::string> errs(n);
        const auto t0 = std::chrono::steady_clock::now();
        run_local_mesh(n, [&](std::uint32_t rank, PeerSockets& peers) {
          try {
            a[rank] = gqsgd::gqsgd_mean_worker(peers, shards[rank], cfg, r);
            b[rank] = gqsgd_b200::gqsgd_mean_worker(peers, shards[rank], cfg, r);
          } catch (const std::exception& e) {
            errs[rank] = e.what();
          }
        });
        if (std::getenv("GQ_TRACE"))
          std::fprintf(stderr, "mesh case n=%u d=%zu variant %d: %.3f s\n", n, d, variant,
                       std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        bool same = true;
        for (std::uint32_t k = 0; k < n; ++k) {
          same = same && errs[k].empty() && a[k].norm == b[k].norm && a[k].lane_width_used == b[k].lane_width_used &&
                 a[k].payload_bytes_sent == b[k].payload_bytes_sent && a[k].norm_bytes_sent == b[k].norm_bytes_sent &&
                 a[k].mean.size() == b[k].mean.size() &&
                 std::memcmp(a[k].mean.data(), b[k].mean.data(), a[k].mean.size() * sizeof(double)) == 0;
        }
        ++cases;
        ok += same;
        if (!same && first_bad.empty()) {
          const WorkerMeanResult &x = a[0], &y = b[0];
          first_bad = " first mismatch n=" + std::to_string(n) + " d=" + std::to_string(d) + " variant " +
                      std::to_string(variant) + (errs[0].empty() ? "" : " (" + errs[0] + ")") + " [norm " +
                      std::to_string(x.norm == y.norm) + " width " + std::to_string(x.lane_width_used) + "/" +
                      std::to_string(y.lane_width_used) + " payload " + std::to_string(x.payload_bytes_sent) + "/" +
                      std::to_string(y.payload_bytes_sent) + " normbytes " + std::to_string(x.norm_bytes_sent) + "/" +
                      std::to_string(y.norm_bytes_sent) + " mean " +
                      std::to_string(x.mean.size() == y.mean.size() &&
                                     std::memcmp(x.mean.data(), y.mean.data(), x.mean.size() * 8) == 0) +
                      "]";
        }
      }
    }
  }
  report(ok == cases, "gqsgd_mean_worker over run_local_mesh (gq_comm peer memory): mean doubles, norm, lane width, "
                      "payload + norm bytes_sent identical on every rank (" +
                          std::to_string(ok) + "/" + std::to_string(cases) + ")" + first_bad);
  // a NaN on one rank: the reference raises invalid_argument on that worker;
  // the device path raises it on every rank (gq_sync)
  GqsgdConfig cfg;
  cfg.workers = 2;
  cfg.transport = Transport::Tcp;
  cfg.scheme = LevelKind::Standard;
  cfg.s = 15;
  auto shards = gaussian_shards(2, 100, 5);
  shards[1][7] = std::nan("");
  std::vector<std::string> cls(2);
  run_local_mesh(2, [&](std::uint32_t rank, PeerSockets& peers) {
    cls[rank] = exception_class([&] { gqsgd_b200::gqsgd_mean_worker(peers, shards[rank], cfg, 3); });
  });
  report(cls[0] == "invalid_argument" && cls[1] == "invalid_argument",
         "gqsgd_mean_worker NaN on rank 1: " + cls[0] + "/" + cls[1]);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "mesh") {  // the multi-rank section alone
    check_mean_worker();
    return g_fail ? 1 : 0;
  }
  check_payload_ops();
  check_quantize_shard();
  check_gqsgd_mean();
  check_mean_worker();
  std::printf("%s: %d failing check(s)\n", g_fail ? "FAIL" : "PASS", g_fail);
  return g_fail ? 1 : 0;
}
