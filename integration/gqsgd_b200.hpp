// Reference-side binding of the B200 path: what a maintainer of the
// reference library (arxiv 2305.18627, proj/) adds to route its compress /
// aggregate / decompress hot path through libgq_b200.so.
//
// Written against the reference's OWN headers (proj/include/gqsgd/*.hpp, on
// the include path at build time, never copied here) so the types are the
// reference's: gqsgd::PayloadOps, gqsgd::QuantizedShard, gqsgd::MeanResult.
// Calls cross into CUDA only through the C ABI of include/gq_b200.h; this
// file needs no CUDA headers. See INTEGRATION.md.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "gqsgd/algorithm.hpp"
#include "gqsgd/collectives.hpp"
#include "gqsgd/levels.hpp"
#include "gqsgd/quantizer.hpp"
#include "gqsgd/rng.hpp"
#include "gqsgd/transport.hpp"

namespace gqsgd_b200 {

// gqsgd::PayloadOps plugins (collectives.hpp:39-105) evaluated on the GPU:
// drop-in replacements for IntSumOps / TokenReduceOps in allreduce_inproc
// and the TCP worker walk (same bits, same exceptions).
class DeviceIntSumOps : public gqsgd::PayloadOps {
 public:
  explicit DeviceIntSumOps(std::uint32_t width_bits);
  std::size_t lane_bytes() const override { return width_bits_ / 8; }
  void combine(std::span<std::byte> acc, std::span<const std::byte> in, std::uint64_t round,
               std::uint32_t step, std::uint32_t dst, std::uint64_t elem_offset) const override;

 private:
  std::uint32_t width_bits_;
};

class DeviceTokenReduceOps : public gqsgd::PayloadOps {
 public:
  // Same construction as gqsgd::TokenReduceOps(ctx, rng) (collectives.hpp:94-95).
  DeviceTokenReduceOps(const gqsgd::ReduceContext& ctx, const gqsgd::CounterRng& rng);
  std::size_t lane_bytes() const override { return ctx_.width_bits / 8; }
  void combine(std::span<std::byte> acc, std::span<const std::byte> in, std::uint64_t round,
               std::uint32_t step, std::uint32_t dst, std::uint64_t elem_offset) const override;

 private:
  gqsgd::ReduceContext ctx_;
  std::uint64_t seed_;
};

// quantize_shard (quantizer.hpp:38-40) on the GPU for the named schemes.
gqsgd::QuantizedShard quantize_shard(std::span<const double> x, double norm,
                                     const gqsgd::LevelScheme& scheme, const gqsgd::CounterRng& rng,
                                     std::uint32_t worker, std::uint64_t round);

// gqsgd_mean (algorithm.hpp:56-57) with Transport::Inproc, dense and sparse:
// norm, quantize, schedule replay / sparse encode + accumulate and decode run
// on the GPU; the result (per-worker doubles, norm, lane width, traffic
// reports) is bit-identical to the reference's. Tcp configurations throw
// std::invalid_argument (route those to the reference's own gqsgd_mean).
gqsgd::MeanResult gqsgd_mean(const std::vector<std::vector<double>>& shards,
                             const gqsgd::GqsgdConfig& cfg, std::uint64_t round);

// True when gqsgd_b200::gqsgd_mean handles `cfg` (in-process; lane widths the
// device supports).
bool handles(const gqsgd::GqsgdConfig& cfg);

// gqsgd_mean_worker (algorithm.hpp:69-71) for the dense paths: this rank's
// shard on its GPU, the norm and lane exchanges over peer memory (gq_comm,
// NVLink / CUDA IPC) instead of the TCP frames. `peers` (the reference's mesh)
// only carries the one-time bootstrap (each rank's gq_comm handle, a Ctrl
// frame). Mean, norm, lane width and the bytes_sent accounting are the
// reference's bit for bit; a device error on any rank raises the same
// exception class on every rank.
gqsgd::WorkerMeanResult gqsgd_mean_worker(gqsgd::PeerSockets& peers, const std::vector<double>& shard,
                                          const gqsgd::GqsgdConfig& cfg, std::uint64_t round);
bool handles_worker(const gqsgd::GqsgdConfig& cfg);

}  // namespace gqsgd_b200
