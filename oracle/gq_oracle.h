/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the Global-QSGD hot path.
 *
 * A plain-C restatement of the reference's algorithm (arxiv 2305.18627,
 * /root/reference/proj). It is the CHECKER for the CUDA product path: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 * It is pinned against (a) the reference's own known-answer tests
 * (proj/tests/test_*.cpp), transcribed in tests/test_oracle_kat.py, and
 * (b) the unmodified reference compiled here (oracle/_ref, see Makefile) via
 * the committed fixtures in tests/golden/ (made by tests/golden/make_golden.py).
 *
 * Status codes match include/gq_b200.h:
 *   0 ok, 1 invalid_argument, 2 overflow_error, 3 domain_error.
 */
#ifndef GQ_ORACLE_H
#define GQ_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GQO_NORM_INF 0xffffffffu

uint64_t gqo_mix64(uint64_t z);
uint64_t gqo_rng_bits(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b,
                      uint64_t c);
double gqo_rng_u01(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b,
                   uint64_t c);
double gqo_rng_normal(uint64_t seed, uint64_t stream, uint64_t a, uint64_t b,
                      uint64_t c);

int gqo_levels(uint32_t kind, uint32_t s, double* out);
uint32_t gqo_bracket_index(const double* levels, uint32_t s, double y);
uint32_t gqo_random_round(const double* levels, uint32_t s, double y, double u);

uint32_t gqo_ceil_log2(uint64_t v);
uint32_t gqo_prescale_shift(uint32_t n);
int gqo_check_width(uint32_t kind, uint32_t s, uint32_t n, uint32_t width);
uint32_t gqo_standard_lane_width(uint32_t s, uint32_t n, uint32_t at_least);
uint32_t gqo_sample_k(double u, uint32_t m);
int gqo_reduce_pair(int32_t sa, uint32_t ea, int32_t sb, uint32_t eb,
                    uint32_t k, uint32_t max_e, int32_t* so, uint32_t* eo);

int gqo_local_norm_stat(const double* x, uint64_t d, uint32_t q, uint32_t p,
                        double* out);
int gqo_norm_tree_combine(const double* stats, uint32_t n, uint32_t q,
                          uint32_t p, double* out);

int gqo_quantize(const double* x, uint64_t d, double norm, uint32_t kind,
                 uint32_t s, uint64_t seed, uint32_t worker, uint64_t round,
                 int8_t* sign, uint32_t* level_idx);
int gqo_encode(uint32_t kind, uint32_t s, uint32_t n, uint32_t width,
               const int8_t* sign, const uint32_t* level_idx, uint64_t d,
               uint8_t* lanes);

int64_t gqo_schedule(uint32_t topo, uint32_t n, uint32_t* out, uint64_t cap);
int gqo_allreduce_inproc(uint8_t* lanes, uint32_t n, uint64_t lanes_per_worker,
                         uint32_t kind, uint32_t width, uint32_t s,
                         uint32_t topo, uint64_t seed, uint64_t round);
int gqo_decode(uint32_t kind, const uint8_t* lanes, uint64_t d, double norm,
               uint32_t s, uint32_t n, uint32_t width, double* out);

int gqo_mean(const double* shards, uint32_t n, uint64_t d, uint32_t kind,
             uint32_t s, uint32_t q, uint32_t p, uint32_t width, uint32_t topo,
             uint64_t seed, uint64_t round, const double* norm_override,
             double* mean_out, double* norm_out, uint32_t* lane_width_out,
             uint8_t* summed_lanes_out);

int gqo_gaussian_shards(uint32_t n, uint64_t d, uint64_t seed, double* out);
int gqo_gaussian_range(uint32_t n, uint64_t j0, uint64_t cnt, uint64_t seed, double* out);

#ifdef __cplusplus
}
#endif

#endif
