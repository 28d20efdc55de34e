// Internal launcher declarations shared by the .cu files and the C-ABI.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "gq_b200.h"
#include "gq_common.cuh"

namespace gqb {

constexpr uint32_t kNormTotalBlocks = 148 * 8;
constexpr uint32_t kMaxPeers = 16;  // GPUs of one NVSwitch node reachable by peer stores

// Process-wide launch options (gq_set_option): 0 = automatic.
extern int g_quant_ctas_per_sm;
extern int g_reduce_ctas_per_sm;
extern int g_comm_wait;  // GQ_OPT_COMM_WAIT: 0 auto, 1 device, 2 host
extern int g_comm_timeout_s;  // GQ_OPT_COMM_TIMEOUT_S: how long a peer wait may take
extern int g_pdl;        // GQ_OPT_PDL: programmatic dependent launch of quantize / reduce
extern int g_small_path; // GQ_OPT_SMALL_PATH: the fused small-d kernel (1 on, 0 off)
extern int g_fused_path; // GQ_OPT_FUSED_PATH: in-process quantize + replay + decode per tile (1 on, 0 off)
extern int g_comm_fold;  // GQ_OPT_COMM_FOLD: exchange steps folded into the kernels (1) or separate (0)

// Launch with programmatic stream serialization when g_pdl is set: the grid
// may be scheduled while its predecessor on the stream drains (its CTAs fill
// SMs the predecessor's CTAs leave); the kernel itself must call pdl_wait()
// before touching anything the predecessor produces.
template <typename... KArgs, typename... Args>
cudaError_t launch_maybe_pdl(void (*fn)(KArgs...), uint32_t grid, uint32_t block, size_t smem, cudaStream_t st,
                             Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, args...);
}

// Tree-order fold of per-worker norm stats + root (collectives.cpp:210-233,
// topology.cpp:19-43, norms.cpp:64-75). Single thread; s is clobbered.
__device__ __forceinline__ double tree_fold_stats(double* s, uint32_t n, uint32_t p) {
  for (uint32_t span = 1; span < n; span <<= 1) {
    for (uint32_t r = span; r < n; r += 2 * span) {
      const double a = s[r - span], b = s[r];
      if (p == GQ_NORM_INF) s[r - span] = (a < b) ? b : a;  // std::max(a, b)
      else s[r - span] = __dadd_rn(a, b);                   // a += b
    }
  }
  if (p == GQ_NORM_INF) return s[0];
  return __dsqrt_rn(s[0]);
}

uint32_t norm_blocks_per_worker(uint32_t n, uint64_t d, bool kdraws);
cudaError_t launch_norm_pow(const void* const* shards, uint32_t dtype, uint32_t n, uint64_t d, uint32_t q,
                            double* stats, void* workspace, uint32_t* err, cudaStream_t stream);
size_t norm_workspace_bytes(uint32_t n, uint64_t d);

// Norm-workspace header: the first kWsHeaderBytes of every norm workspace
// hold zero-initialised counters (each kernel that takes a ticket resets it);
// the per-block partials start right after. One slot per user, so an eager
// step and a graph replay of one communicator never share a ticket.
constexpr size_t kWsNormTicket = 0;          // norm_kernel's last-block ticket
constexpr size_t kWsRoundTicket = 128;       // gq_graph_mean_inproc: the reduce's round-advance ticket
constexpr size_t kWsFoldTicketQ = 160;       // eager comm step: quantize-scatter completion signal (phase 1)
constexpr size_t kWsFoldTicketR = 176;       // eager comm step: multicast-reduce completion signal (phase 2)
constexpr size_t kWsFoldTicketQGraph = 192;  // comm graph: phase 5
constexpr size_t kWsFoldTicketRGraph = 208;  // comm graph: phase 6
constexpr size_t kWsRoundTicketComm = 224;   // comm graph: the decode's round-advance ticket
constexpr size_t kWsSmallBar = 32;           // mean_small_kernel: grid-barrier counter
constexpr size_t kWsSmallDone = 40;          // mean_small_kernel: completion ticket
constexpr size_t kWsSmallMax = 64;           // mean_small_kernel: 16 per-worker max |x| words (64..127)
constexpr size_t kWsHeaderBytes = 256;
static_assert(kWsRoundTicket >= 64 && kWsRoundTicketComm + 4 <= kWsHeaderBytes,
              "ticket slots must sit inside the header, clear of the norm ticket");

// The k draws of every TokenReduceOps event of a tree schedule, precomputed
// into a buffer (they depend only on keys and lane indices, not on data):
// buf[e * kwords + wi] is token_kword for event e (reference tree order) and
// lane word wi. Filled by the norm launch, whose HBM-bound pass leaves the
// integer pipes idle; consumed by the reduce launch.
constexpr uint32_t kMaxKEvents = 15;  // tree events for n <= 16
struct KDrawJob {
  uint32_t* buf;
  uint64_t kwords;
  uint32_t events;
  uint32_t width;   // 4 or 8
  uint32_t m;       // s + 1
  uint32_t pad;
  uint64_t w0;      // first lane word (global index) of the buffer
  const uint64_t* round_ptr;  // non-null: keys derived on the device from (seed, n, *round_ptr)
  uint64_t seed;
  uint32_t n;
  uint32_t pad2;
  uint64_t keys[kMaxKEvents];
};

// mix64^3(seed, ReduceDraw, round) and the tree event keys from it (host and device)
__host__ __device__ __forceinline__ uint64_t reduce_round_prefix(uint64_t seed, uint64_t round) {
  uint64_t h = mix64(seed ^ 0x517cc1b727220a95ull);
  h = mix64(h ^ 2ull);
  return mix64(h ^ round);
}

struct StatsPut;
cudaError_t launch_norm(const void* const* shards, uint32_t dtype, uint32_t n,
                        uint64_t d, uint32_t q, uint32_t p, double* stats,
                        double* norm_out, void* workspace, uint32_t* err,
                        cudaStream_t stream, const KDrawJob* kjob = nullptr, const StatsPut* put = nullptr);

// Tree event keys in the reference's order (topology.cpp:28-35): step t,
// r = span, 3 span, ...; dst = r - span. Returns the event count.
uint32_t tree_event_keys(uint32_t n, uint64_t seed, uint64_t round, uint64_t* keys, uint32_t cap);
cudaError_t launch_norm_combine(const double* stats, uint32_t n, uint32_t p,
                                double* norm_out, cudaStream_t stream);

// Completion signal folded into a kernel: when the grid's last CTA has
// retired (every CTA fences its stores system-wide, then takes a ticket), it
// stores the epoch (*ep_dev when non-null) into every slot with st.release.sys
// - the peer-memory flag of gq_p2p_signal without a separate launch.
struct PeerSignal {
  uint32_t* slots[kMaxPeers];
  uint32_t n = 0;
  uint32_t epoch = 0;
  const uint32_t* ep_dev = nullptr;
  unsigned int* ticket = nullptr;  // zeroed device counter (reset by the last CTA)
};

// Folded exchange steps (device-side waits; ranks on distinct GPUs).
//  PeerWait: before touching its inputs, thread 0 of every CTA spins
//            (ld.acquire.sys) until all N flags reached the epoch (from
//            `epoch`, or *ep_dev in graph replays); a peer that never signals
//            raises GQ_FLAG_P2P_TIMEOUT after timeout_ns instead of hanging.
//  StatsPut: the norm pass's last block stores this rank's n_local stats into
//            every peer's stats row and raises the phase flag (graph replays:
//            the epoch is *ep_dev + 1, stored back).
//  StatsFold: after a PeerWait, fold all n stats in the reference's tree order
//            into the global norm (each CTA; CTA 0 also stores it to norm_out).
struct PeerWait {
  const uint32_t* flags = nullptr;
  uint32_t n = 0;
  uint32_t epoch = 0;
  const uint32_t* ep_dev = nullptr;
  uint64_t timeout_ns = 0;
};
struct StatsPut {
  double* dst[kMaxPeers];
  uint32_t* slots[kMaxPeers];
  uint32_t n = 0;
  uint32_t epoch = 0;
  uint32_t* ep_dev = nullptr;
};
struct StatsFold {
  const double* stats = nullptr;  // all n workers' stats (this rank's copy of the row)
  uint32_t n = 0;
  uint32_t p = 0;
  double* norm_out = nullptr;
};
uint64_t comm_timeout_ns();

struct QuantLaunch {
  const void* const* shards;
  uint32_t dtype;
  uint32_t n_local;
  const uint32_t* worker_ids;
  uint64_t d;
  const double* norm;
  uint32_t kind, s, n_total, width;
  uint64_t seed, round;
  void* const* lanes;
  uint32_t* err;
  const uint64_t* round_ptr = nullptr;  // device round (graph replays) overrides `round`
  void* const* slice_dst = nullptr;     // scatter mode: nslices destinations of slice_lanes lanes
  uint32_t nslices = 0;
  uint64_t slice_lanes = 0;
  uint64_t row_bytes = 0;               // scatter mode: local worker i writes at slice_dst[j] + i * row_bytes
  const PeerSignal* signal = nullptr;   // signal the peers when the grid is done
  const PeerWait* wait = nullptr;       // folded exchange: wait for the stats flags, then fold `fold`
  StatsFold fold{};
};
cudaError_t launch_quantize(const QuantLaunch& q, cudaStream_t stream);

struct ReduceLaunch {
  const void* const* worker_lanes;
  uint32_t n;
  uint64_t d, lane_begin, lane_end;
  uint32_t kind, width, s, topo;
  uint64_t seed, round;
  const double* norm;
  void* out_lanes;
  float* out_mean;
  float* param;
  float lr;
  uint32_t* err;
  const uint32_t* kdraws = nullptr;  // precomputed k words, indexed [e * kstride + global word]
  uint64_t kstride = 0;
  const uint64_t* round_ptr = nullptr;  // device round (graph replays) overrides `round`
  void* const* out_peers = nullptr;     // also store the result lanes here (rebased like out_lanes)
  uint32_t npeers = 0;
  uint64_t* round_inc = nullptr;        // graph replays: += round_step once the grid is done
  uint64_t round_step = 0;
  unsigned int* round_ticket = nullptr; // zeroed device counter for the above
  const PeerSignal* signal = nullptr;   // signal the peers when the grid is done
  const PeerWait* wait = nullptr;       // folded exchange: wait for these flags before reading the lanes
};
cudaError_t launch_reduce(const ReduceLaunch& r, cudaStream_t stream);
// The fused small-d in-process sync (one cooperative launch; gq_reduce.cu).
constexpr uint64_t kSmallPathElems = uint64_t{1} << 23;  // n * d at or below: fused (scripts/small_sweep.py)
bool small_path_applies(uint32_t dtype, uint32_t n, uint64_t d, uint32_t kind, uint32_t s, uint32_t width,
                        uint32_t topo, uint32_t q, uint32_t p);
cudaError_t launch_mean_small(const void* const* shards, uint32_t n, uint64_t d, uint32_t kind, uint32_t s,
                              uint32_t width, uint32_t p, uint64_t seed, uint64_t round, const uint64_t* round_ptr,
                              uint64_t* round_inc, void* const* lane_bufs, void* result_lanes, float* mean_out,
                              float* param, float lr, double* stats_out, double* norm_out, void* workspace,
                              uint32_t* err, cudaStream_t stream);
// The in-process quantize + schedule replay + decode, tile by tile (gq_reduce.cu).
bool fused_path_applies(uint32_t dtype, uint32_t n, uint64_t d, uint32_t kind, uint32_t width, uint32_t topo,
                        bool kdraws);
cudaError_t launch_fused_qr(const void* const* shards, uint32_t n, uint64_t d, uint32_t kind, uint32_t s,
                            uint32_t width, uint64_t seed, uint64_t round, const uint64_t* round_ptr,
                            uint64_t* round_inc, unsigned int* ticket, void* const* lane_bufs, void* result_lanes,
                            float* mean_out, float* param, float lr, const double* norm, const uint32_t* kdraws,
                            uint32_t* err, cudaStream_t stream);
// decode (+ SGD) with the folded phase wait and the graph's round advance
cudaError_t launch_dequant_ex(const void* lanes, uint64_t lane_begin, uint64_t lane_end, const double* norm,
                              uint32_t kind, uint32_t s, uint32_t n, uint32_t width, float* out, float* param,
                              float lr, uint32_t* err, cudaStream_t stream, const PeerWait* wait,
                              uint64_t* round_inc, uint64_t round_step, unsigned int* ticket);
cudaError_t launch_rng_draws(uint64_t seed, uint64_t stream_id, uint64_t a, uint64_t b, uint64_t c0, uint64_t count,
                             uint32_t m, const uint64_t* bits_in, uint64_t* bits_out, uint32_t* hi_out,
                             uint32_t* k_out, cudaStream_t st);

cudaError_t launch_p2p_signal(uint32_t* const* slots, uint32_t n, uint32_t epoch, const uint32_t* ep_dev,
                              cudaStream_t st);
// Flag epochs come from `epoch`, or from *ep_dev when non-null (graph replays:
// a device counter bumped once per step by launch_epoch_inc).
cudaError_t launch_p2p_put_signal(const void* src, uint32_t nbytes, void* const* dst, uint32_t* const* slots,
                                  uint32_t n, uint32_t epoch, const uint32_t* ep_dev, cudaStream_t st, bool bump = false);
cudaError_t launch_epoch_inc(uint32_t* ep_dev, cudaStream_t st);
cudaError_t launch_round_inc(uint64_t* round_dev, uint64_t step, cudaStream_t st);
// The exported gq_quantize_scatter / gq_reduce_slice_multicast with the round
// optionally read on the device (round_ptr non-null).
int quantize_scatter_impl(const void* const* shards, uint32_t n_local, const uint32_t* workers, uint32_t dtype,
                          uint64_t d, const double* norm, uint32_t kind, uint32_t s, uint32_t n_total, uint32_t width,
                          uint64_t seed, uint64_t round, const uint64_t* round_ptr, void* const* slice_dst,
                          uint32_t nslices, uint64_t slice_lanes, uint64_t row_bytes, uint32_t* err, void* stream,
                          const PeerSignal* signal = nullptr, const PeerWait* wait = nullptr,
                          const double* stats_all = nullptr, uint32_t norm_p = 0);
int reduce_slice_multicast_impl(const void* const* worker_slices, uint32_t n, uint64_t d, uint64_t lane_begin,
                                uint64_t lane_end, uint32_t kind, uint32_t width, uint32_t s, uint32_t topo,
                                uint64_t seed, uint64_t round, const uint64_t* round_ptr, const uint32_t* kdraws,
                                uint64_t kstride, void* const* out_slices, uint32_t nout, uint32_t* err,
                                void* stream, const PeerSignal* signal = nullptr, const PeerWait* wait = nullptr);
// C-ABI status plumbing shared by the entry-point files (gq_capi.cu)
int api_fail(int code, const char* msg);
int api_cuda_fail(cudaError_t e);
int status_from_flags(uint32_t flags);
cudaError_t launch_p2p_wait(const uint32_t* flags, uint32_t n, uint32_t epoch, const uint32_t* ep_dev, uint32_t* err,
                            cudaStream_t st, uint64_t* round_inc = nullptr,
                            uint64_t round_step = 0);

cudaError_t launch_dequant(const void* lanes, uint64_t lane_begin, uint64_t lane_end,
                           const double* norm, uint32_t kind, uint32_t s, uint32_t n,
                           uint32_t width, float* out, float* param, float lr,
                           uint32_t* err, cudaStream_t stream);

cudaError_t launch_combine(void* acc, const void* in, uint64_t lanes, uint64_t elem_offset,
                           uint32_t kind, uint32_t width, uint32_t s, uint64_t seed,
                           uint64_t round, uint32_t step, uint32_t dst, uint32_t* err,
                           cudaStream_t stream);

cudaError_t launch_dequant_f64(const void* lanes, uint64_t lane_begin, uint64_t lane_end,
                               const double* norm, uint32_t kind, uint32_t s, uint32_t n,
                               uint32_t width, double* out, uint32_t* err, cudaStream_t stream);

size_t sparse_workspace_bytes(uint64_t d);
cudaError_t launch_sparse_encode(const uint32_t* lanes, uint64_t d, uint32_t kind, uint32_t s, uint32_t shift,
                                 uint32_t width, const double* norm, void* payload, void* workspace,
                                 uint32_t* nnz_out, cudaStream_t st);
cudaError_t launch_sparse_mean(const void* const* lanes, uint32_t n, uint64_t d, uint32_t kind, uint32_t s,
                               uint32_t shift, const double* norm, uint32_t n_div, float* out32, double* out64,
                               cudaStream_t st);
cudaError_t launch_sparse_scatter(const void* payload, uint64_t bytes, uint32_t kind, uint32_t s, uint32_t width,
                                  uint64_t d, double* acc, uint32_t* err, cudaStream_t st);
cudaError_t launch_scale(const double* acc, uint64_t d, uint32_t n, float* out32, double* out64, float* param,
                         float lr, cudaStream_t st);

cudaError_t launch_baseline_mean(const float* const* shards, uint32_t n, uint64_t d,
                                 uint32_t topo, float* mean_out, cudaStream_t stream);

}  // namespace gqb

// A captured CUDA graph (gq_graph_mean_inproc, gq_comm_graph).
struct gq_graph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};
