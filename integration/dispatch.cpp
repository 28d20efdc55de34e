// The maintainer's swap, as it would sit in the reference's build: the
// public gqsgd::gqsgd_mean (algorithm.hpp:56-57) routes the dense in-process
// path to the GPU and everything else (sparse allgather, TCP transport) to the
// reference's own implementation, which this build compiles from
// src/algorithm.cpp with -Dgqsgd_mean=gqsgd_mean_reference.
#include "gqsgd/algorithm.hpp"
#include "gqsgd_b200.hpp"

namespace gqsgd {

MeanResult gqsgd_mean_reference(const std::vector<std::vector<double>>& shards, const GqsgdConfig& cfg,
                                std::uint64_t round);

MeanResult gqsgd_mean(const std::vector<std::vector<double>>& shards, const GqsgdConfig& cfg,
                      std::uint64_t round) {
  if (gqsgd_b200::handles(cfg)) return gqsgd_b200::gqsgd_mean(shards, cfg, round);
  return gqsgd_mean_reference(shards, cfg, round);
}

}  // namespace gqsgd
