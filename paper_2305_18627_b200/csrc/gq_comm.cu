// gq_comm: the multi-rank gradient sync over peer memory (include/gq_b200.h,
// "communicator"). Replaces the reference's TCP worker mesh (PeerSockets,
// connect_mesh, run_local_mesh: transport.hpp:38-58, transport.cpp:289-330)
// and the two exchanges of gqsgd_mean_worker (algorithm.cpp:230-301):
//
//   norm     each rank stores its n_local f64 stats into every peer's stats
//            row and signals; every rank folds all n stats in the reference's
//            tree order (gq_norm_combine) -> identical scale everywhere;
//   lanes    the quantizer stores lane slice j of each local worker straight
//            into rank j's receive row for that worker (gq_quantize_scatter);
//            after the flags, rank j replays the reference schedule on its
//            slice over all n rows and stores the result into every peer's
//            summed buffer (gq_reduce_slice_multicast); after the second flag
//            round every rank holds the full summed lanes.
//
// One symmetric cudaMalloc per rank holds everything peers touch, so one IPC
// handle maps it:  [flags 4 phases x 16][stats 2 x n f64][errs 2 x 16 u32]
//                  [recv n x slice][summed nranks x slice]
// Flags are monotonically increasing epochs per phase (system-scope
// release / acquire, gq_reduce.cu). Stats and error words alternate between
// two rows by epoch parity, so a fast rank's next put cannot overwrite a row
// a slow rank has not consumed: writing row (e & 1) at epoch e+2 needs every
// peer's signal of epoch e+1, issued after it consumed epoch e. Receive rows
// are reused every step; the step's own second flag round orders the reuse
// (a rank scatters step t+1 only after all peers signalled that their step-t
// reduce finished).
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <thread>
#include <vector>

#include "gq_b200.h"
#include "gq_internal.h"

#define GQ_EXPORT extern "C" __attribute__((visibility("default")))

namespace {

using gqb::api_cuda_fail;
using gqb::api_fail;
using gqb::kMaxPeers;

constexpr uint32_t kMagic = 0x47514331u;  // "GQC1"
// eager phases 0 stats, 1 rows delivered, 2 summed delivered, 3 error words;
// graph replays use their own phases 4-6 (device epoch) and stats row 2
constexpr uint32_t kPhases = 7;

struct Blob {
  uint32_t magic;
  uint32_t rank, nranks, workers;
  int32_t pid, device;
  uint64_t d, total, base;
  uint32_t width, kind;
  uint64_t host;  // hash of the host name: peer memory exists only within one node
  unsigned char uuid[16];
  cudaIpcMemHandle_t handle;
};

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

uint64_t host_id() {
  char name[256] = {};
  gethostname(name, sizeof(name) - 1);
  uint64_t h = 0xcbf29ce484222325ull;  // FNV-1a
  for (const char* p = name; *p; ++p) h = (h ^ static_cast<unsigned char>(*p)) * 0x100000001b3ull;
  return h;
}

}  // namespace

struct gq_comm {
  uint32_t rank = 0, N = 0, n = 0, n_local = 0, w0 = 0;
  gq_config cfg{};
  gq_plan plan{};
  uint64_t d = 0, slice_lanes = 0, slice_bytes = 0, lane_begin = 0, lane_end = 0;
  size_t off_flags = 0, off_stats = 0, off_errs = 0, off_recv = 0, off_summed = 0, total = 0;
  uint8_t* base = nullptr;
  int device = 0;
  unsigned char uuid[16] = {};
  cudaIpcMemHandle_t handle{};
  // local (not shared) buffers
  double* stats_local = nullptr;
  double* norm = nullptr;
  uint32_t* ep_dev = nullptr;  // graph replays: the step's flag epoch
  // k draws of this rank's slice, precomputed by the norm pass (exponential tree)
  uint32_t* kbuf = nullptr;
  uint64_t kwords = 0;
  bool kd_valid = false;
  uint64_t kd_round = 0;
  // gq_comm_quantize already raised the phase-1 flags (in-kernel) with this epoch
  uint32_t rows_signalled = 0;
  void* ws = nullptr;
  cudaStream_t poll = nullptr;
  // peers
  uint8_t* peer[kMaxPeers] = {};
  bool opened[kMaxPeers] = {};
  bool connected = false, host_wait = false;
  uint32_t epoch[kPhases] = {};
  std::vector<std::vector<void*>> scatter;  // [local worker][owner] receive-row pointers
  std::vector<uint32_t> worker_ids;         // w0 .. w0 + n_local - 1

  uint32_t* my_flags(uint32_t ph) const { return reinterpret_cast<uint32_t*>(base + off_flags) + ph * kMaxPeers; }
  uint32_t* slot(uint32_t p, uint32_t ph) const {
    return reinterpret_cast<uint32_t*>(peer[p] + off_flags) + ph * kMaxPeers + rank;
  }
};

namespace {

int signal(gq_comm* c, uint32_t ph, uint32_t e, cudaStream_t st) {
  uint32_t* slots[kMaxPeers];
  for (uint32_t p = 0; p < c->N; ++p) slots[p] = c->slot(p, ph);
  const cudaError_t ce = gqb::launch_p2p_signal(slots, c->N, e, nullptr, st);
  return ce == cudaSuccess ? GQ_OK : api_cuda_fail(ce);
}

// Wait until every rank signalled epoch e on phase ph. Device mode: one
// spinning thread on the stream (no host involvement). Host mode (a peer on
// this same GPU, where a spinning kernel could sit in a hardware queue ahead
// of the peer's producer): drain the stream and poll the flags from the host.
int wait(gq_comm* c, uint32_t ph, uint32_t e, uint32_t* err, cudaStream_t st) {
  if (!c->host_wait) {
    const cudaError_t ce = gqb::launch_p2p_wait(c->my_flags(ph), c->N, e, nullptr, err, st);
    return ce == cudaSuccess ? GQ_OK : api_cuda_fail(ce);
  }
  cudaError_t ce = cudaStreamSynchronize(st);
  if (ce != cudaSuccess) return api_cuda_fail(ce);
  uint32_t v[kMaxPeers];
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    ce = cudaMemcpyAsync(v, c->my_flags(ph), c->N * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->poll);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(c->poll);
    if (ce != cudaSuccess) return api_cuda_fail(ce);
    bool all = true;
    for (uint32_t p = 0; p < c->N; ++p) all = all && static_cast<int32_t>(v[p] - e) >= 0;
    if (all) return GQ_OK;
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > gqb::g_comm_timeout_s)
      return api_fail(GQ_ERR_RUNTIME, "peer exchange timed out waiting for a rank");
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

gqb::KDrawJob kjob(const gq_comm* c, uint64_t round, const uint64_t* round_ptr) {
  gqb::KDrawJob job{};
  job.buf = c->kbuf;
  job.kwords = c->kwords;
  job.width = c->plan.lane_width;
  job.m = c->cfg.s + 1;
  job.events = gqb::tree_event_keys(c->n, c->cfg.seed, round, job.keys, gqb::kMaxKEvents);
  job.w0 = c->plan.lane_width <= 8 ? c->lane_begin / (32 / c->plan.lane_width) : 0;  // k draws: 4/8-bit tokens only
  if (round_ptr) {  // keys derived on the device from *round_ptr (graph replays)
    job.round_ptr = round_ptr;
    job.seed = c->cfg.seed;
    job.n = c->n;
  }
  return job;
}

// k words indexed by global lane word, as the reduce consumes them
const uint32_t* kdraws_rebased(const gq_comm* c) {
  return c->kbuf - c->lane_begin / (32 / c->plan.lane_width);
}

// Completion signal of phase ph folded into a kernel (gqb::PeerSignal);
// tickets live in the communicator's norm-workspace header, one slot per
// phase (gq_internal.h kWsFoldTicket*).
gqb::PeerSignal fold_signal(const gq_comm* c, uint32_t ph, uint32_t epoch, const uint32_t* ep_dev) {
  gqb::PeerSignal s;
  for (uint32_t p = 0; p < c->N; ++p) s.slots[p] = c->slot(p, ph);
  s.n = c->N;
  s.epoch = epoch;
  s.ep_dev = ep_dev;
  const size_t off = ph == 1 ? gqb::kWsFoldTicketQ
                   : ph == 2 ? gqb::kWsFoldTicketR
                   : ph == 5 ? gqb::kWsFoldTicketQGraph
                             : gqb::kWsFoldTicketRGraph;
  s.ticket = reinterpret_cast<unsigned int*>(static_cast<char*>(c->ws) + off);
  return s;
}

int need_connected(const gq_comm* c) {
  if (!c) return api_fail(GQ_ERR_INVALID, "null communicator");
  if (!c->connected) return api_fail(GQ_ERR_INVALID, "communicator is not connected");
  return GQ_OK;
}

}  // namespace

GQ_EXPORT size_t gq_comm_handle_bytes(void) { return sizeof(Blob); }

GQ_EXPORT int gq_comm_init(uint32_t rank, uint32_t nranks, const gq_config* cfg, uint64_t d, gq_comm** out) {
  if (!cfg || !out) return api_fail(GQ_ERR_INVALID, "null argument");
  *out = nullptr;
  if (nranks == 0 || nranks > kMaxPeers) return api_fail(GQ_ERR_INVALID, "rank count must be in [1, 16]");
  if (rank >= nranks) return api_fail(GQ_ERR_INVALID, "rank out of range");
  if (cfg->workers % nranks != 0) return api_fail(GQ_ERR_INVALID, "worker count must be a multiple of the number of ranks");
  if (d == 0) return api_fail(GQ_ERR_INVALID, "empty gradient");
  gq_plan plan{};
  if (int rc = gq_plan_path(cfg, &plan)) return rc;
  const auto dev_order = [](uint32_t v) { return v == 2 || v == GQ_NORM_INF || v == GQ_NORM_L2_SEQUENTIAL; };
  if (!dev_order(cfg->norm_q) || (cfg->norm_p != 2 && cfg->norm_p != GQ_NORM_INF))
    return api_fail(GQ_ERR_INVALID, "the communicator folds norm stats on the device: orders 2 or inf");
  auto* c = new gq_comm();
  c->rank = rank;
  c->N = nranks;
  c->n = cfg->workers;
  c->n_local = cfg->workers / nranks;
  c->w0 = rank * c->n_local;
  c->cfg = *cfg;
  c->plan = plan;
  c->d = d;
  const uint64_t unit = 1024;  // whole 4 KiB chunks of the scatter quantizer (its 8-quads-per-lane form)
  c->slice_lanes = std::max<uint64_t>(unit, (d + nranks * unit - 1) / (nranks * unit) * unit);
  c->slice_bytes = c->slice_lanes * plan.lane_width / 8;
  c->lane_begin = std::min<uint64_t>(d, rank * c->slice_lanes);
  c->lane_end = std::min<uint64_t>(d, (rank + 1) * c->slice_lanes);
  size_t off = 0;
  c->off_flags = off;
  off = align_up(off + kPhases * kMaxPeers * 4, 256);
  c->off_stats = off;
  off = align_up(off + 3ull * c->n * 8, 256);
  c->off_errs = off;
  off = align_up(off + 2ull * kMaxPeers * 4, 256);
  c->off_recv = off;
  off = align_up(off + static_cast<size_t>(c->n) * c->slice_bytes, 256);
  c->off_summed = off;
  off = align_up(off + static_cast<size_t>(nranks) * c->slice_bytes, 256);
  c->total = off;
  cudaError_t e = cudaGetDevice(&c->device);
  cudaDeviceProp prop{};
  if (e == cudaSuccess) e = cudaGetDeviceProperties(&prop, c->device);
  if (e == cudaSuccess) std::memcpy(c->uuid, prop.uuid.bytes, 16);
  if (e == cudaSuccess) e = cudaMalloc(&c->base, c->total);
  if (e == cudaSuccess) e = cudaMemset(c->base, 0, c->total);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&c->handle, c->base);
  if (e == cudaSuccess) e = cudaMalloc(&c->stats_local, 8ull * c->n_local);
  if (e == cudaSuccess) e = cudaMalloc(&c->norm, 8);
  if (e == cudaSuccess) e = cudaMalloc(&c->ep_dev, 8);
  if (e == cudaSuccess) e = cudaMemset(c->ep_dev, 0, 8);
  const size_t wsb = gq_norm_workspace_bytes(c->n_local, d);
  if (e == cudaSuccess) e = cudaMalloc(&c->ws, wsb);
  if (e == cudaSuccess) e = cudaMemset(c->ws, 0, wsb);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->poll, cudaStreamNonBlocking);
  gq_kdraws spec{};  // the TokenReduceOps k draws of this rank's slice
  spec.n = c->n;
  spec.kind = cfg->kind;
  spec.width = plan.lane_width;
  spec.s = cfg->s;
  spec.topo = cfg->topo;
  spec.lane_begin = c->lane_begin;
  spec.lane_end = c->lane_end;
  spec.seed = cfg->seed;
  const size_t kb = gq_kdraws_bytes(&spec);
  if (e == cudaSuccess && kb) {
    e = cudaMalloc(&c->kbuf, kb);
    c->kwords = kb / sizeof(uint32_t) / (c->n - 1);
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    const int rc = api_cuda_fail(e);
    gq_comm_destroy(c);
    return rc;
  }
  *out = c;
  return GQ_OK;
}

GQ_EXPORT int gq_comm_handle(const gq_comm* c, void* handle_out) {
  if (!c || !handle_out) return api_fail(GQ_ERR_INVALID, "null argument");
  Blob b{};
  b.magic = kMagic;
  b.rank = c->rank;
  b.nranks = c->N;
  b.workers = c->n;
  b.pid = static_cast<int32_t>(getpid());
  b.device = c->device;
  b.d = c->d;
  b.total = c->total;
  b.base = reinterpret_cast<uint64_t>(c->base);
  b.width = c->plan.lane_width;
  b.kind = c->cfg.kind;
  b.host = host_id();
  std::memcpy(b.uuid, c->uuid, 16);
  b.handle = c->handle;
  std::memcpy(handle_out, &b, sizeof(b));
  return GQ_OK;
}

GQ_EXPORT int gq_comm_connect(gq_comm* c, const void* handles) {
  if (!c || !handles) return api_fail(GQ_ERR_INVALID, "null argument");
  if (c->connected) return api_fail(GQ_ERR_INVALID, "communicator is already connected");
  const int32_t pid = static_cast<int32_t>(getpid());
  const uint64_t host = host_id();
  for (uint32_t p = 0; p < c->N; ++p) {
    Blob b;
    std::memcpy(&b, static_cast<const uint8_t*>(handles) + p * sizeof(Blob), sizeof(Blob));
    if (b.magic != kMagic || b.rank != p || b.nranks != c->N || b.workers != c->n || b.d != c->d ||
        b.total != c->total || b.width != c->plan.lane_width || b.kind != c->cfg.kind)
      return api_fail(GQ_ERR_INVALID, "communicator handles do not describe the same job");
    if (b.host != host) return api_fail(GQ_ERR_RUNTIME, "peer-memory exchange needs every rank on one node");
    if (p == c->rank) {
      c->peer[p] = c->base;
      continue;
    }
    if (std::memcmp(b.uuid, c->uuid, 16) == 0) c->host_wait = true;
    if (b.pid == pid) {  // a rank of this process (thread): plain pointer, peer access if another GPU
      if (b.device != c->device) {
        int ok = 0;
        cudaDeviceCanAccessPeer(&ok, c->device, b.device);
        if (!ok) return api_fail(GQ_ERR_RUNTIME, "GPUs of this communicator cannot access each other");
        const cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return api_cuda_fail(e);
        cudaGetLastError();
      }
      c->peer[p] = reinterpret_cast<uint8_t*>(b.base);
    } else {
      void* ptr = nullptr;
      const cudaError_t e = cudaIpcOpenMemHandle(&ptr, b.handle, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) return api_cuda_fail(e);
      c->peer[p] = static_cast<uint8_t*>(ptr);
      c->opened[p] = true;
    }
  }
  if (gqb::g_comm_wait == 1) c->host_wait = false;
  if (gqb::g_comm_wait == 2) c->host_wait = true;
  c->scatter.assign(c->n_local, std::vector<void*>(c->N));
  c->worker_ids.resize(c->n_local);
  for (uint32_t i = 0; i < c->n_local; ++i) c->worker_ids[i] = c->w0 + i;
  for (uint32_t i = 0; i < c->n_local; ++i)
    for (uint32_t j = 0; j < c->N; ++j)
      c->scatter[i][j] = c->peer[j] + c->off_recv + static_cast<size_t>(c->w0 + i) * c->slice_bytes;
  c->connected = true;
  return GQ_OK;
}

GQ_EXPORT int gq_comm_info_get(const gq_comm* c, gq_comm_info* out) {
  if (!c || !out) return api_fail(GQ_ERR_INVALID, "null argument");
  out->lane_width = c->plan.lane_width;
  out->n_local = c->n_local;
  out->worker_begin = c->w0;
  out->host_wait = c->host_wait ? 1u : 0u;
  out->slice_lanes = c->slice_lanes;
  out->lane_begin = c->lane_begin;
  out->lane_end = c->lane_end;
  out->device = c->device;
  out->reserved = 0;
  return GQ_OK;
}

GQ_EXPORT int gq_comm_destroy(gq_comm* c) {
  if (!c) return GQ_OK;
  for (uint32_t p = 0; p < kMaxPeers; ++p)
    if (c->opened[p]) cudaIpcCloseMemHandle(c->peer[p]);
  if (c->base) cudaFree(c->base);
  if (c->stats_local) cudaFree(c->stats_local);
  if (c->norm) cudaFree(c->norm);
  if (c->ep_dev) cudaFree(c->ep_dev);
  if (c->kbuf) cudaFree(c->kbuf);
  if (c->ws) cudaFree(c->ws);
  if (c->poll) cudaStreamDestroy(c->poll);
  delete c;
  return GQ_OK;
}

GQ_EXPORT int gq_norm_exchange(gq_comm* c, const double* stats_local, double* norm_out, uint32_t* err,
                               void* stream) {
  if (int rc = need_connected(c)) return rc;
  if (!stats_local || !norm_out || !err) return api_fail(GQ_ERR_INVALID, "null argument");
  auto st = static_cast<cudaStream_t>(stream);
  const uint32_t e = ++c->epoch[0];
  const size_t row = (e & 1u) * c->n;
  void* dst[kMaxPeers];
  uint32_t* slots[kMaxPeers];
  for (uint32_t p = 0; p < c->N; ++p) {
    dst[p] = c->peer[p] + c->off_stats + (row + c->w0) * 8;
    slots[p] = c->slot(p, 0);
  }
  const cudaError_t ce = gqb::launch_p2p_put_signal(stats_local, 8 * c->n_local, dst, slots, c->N, e, nullptr, st);
  if (ce != cudaSuccess) return api_cuda_fail(ce);
  if (int rc = wait(c, 0, e, err, st)) return rc;
  const double* all = reinterpret_cast<const double*>(c->base + c->off_stats) + row;
  return gq_norm_combine(all, c->n, 2, c->cfg.norm_p, norm_out, stream);
}

GQ_EXPORT int gq_comm_norm(gq_comm* c, const void* const* shards, uint32_t dtype, uint64_t round,
                           double* norm_out, uint32_t* err, void* stream) {
  if (int rc = need_connected(c)) return rc;
  if (!shards || !err) return api_fail(GQ_ERR_INVALID, "null argument");
  if (dtype != GQ_DTYPE_F32 && dtype != GQ_DTYPE_F64) return api_fail(GQ_ERR_INVALID, "unknown dtype");
  for (uint32_t i = 0; i < c->n_local; ++i)
    if (!shards[i] || (reinterpret_cast<uintptr_t>(shards[i]) & 15) != 0)
      return api_fail(GQ_ERR_INVALID, "device buffers must be 16-byte aligned");
  const gqb::KDrawJob job = kjob(c, round, nullptr);
  const bool fold = gqb::g_comm_fold != 0 && c->cfg.norm_q != GQ_NORM_L2_SEQUENTIAL;
  if (!fold) {
    const cudaError_t ce = gqb::launch_norm(shards, dtype, c->n_local, c->d, c->cfg.norm_q, c->cfg.norm_p,
                                            c->stats_local, nullptr, c->ws, err, static_cast<cudaStream_t>(stream),
                                            c->kbuf ? &job : nullptr);
    if (ce != cudaSuccess) return api_cuda_fail(ce);
    c->kd_valid = c->kbuf != nullptr;
    c->kd_round = round;
    return gq_norm_exchange(c, c->stats_local, norm_out ? norm_out : c->norm, err, stream);
  }
  // the stats put rides in the norm pass's last block (StatsPut), as in the
  // graph step; the wait and the tree fold follow (the norm is this call's output)
  const uint32_t e = ++c->epoch[0];
  const size_t row = (e & 1u) * c->n;
  gqb::StatsPut put{};
  for (uint32_t p = 0; p < c->N; ++p) {
    put.dst[p] = reinterpret_cast<double*>(c->peer[p] + c->off_stats + (row + c->w0) * 8);
    put.slots[p] = c->slot(p, 0);
  }
  put.n = c->N;
  put.epoch = e;
  const cudaError_t ce = gqb::launch_norm(shards, dtype, c->n_local, c->d, c->cfg.norm_q, c->cfg.norm_p,
                                          c->stats_local, nullptr, c->ws, err, static_cast<cudaStream_t>(stream),
                                          c->kbuf ? &job : nullptr, &put);
  if (ce != cudaSuccess) {
    --c->epoch[0];
    return api_cuda_fail(ce);
  }
  c->kd_valid = c->kbuf != nullptr;
  c->kd_round = round;
  if (int rc = wait(c, 0, e, err, static_cast<cudaStream_t>(stream))) return rc;
  const double* all = reinterpret_cast<const double*>(c->base + c->off_stats) + row;
  return gq_norm_combine(all, c->n, 2, c->cfg.norm_p, norm_out ? norm_out : c->norm, stream);
}

GQ_EXPORT int gq_comm_quantize(gq_comm* c, const void* const* shards, uint32_t dtype, const double* norm,
                               uint64_t round, uint32_t* err, void* stream) {
  if (int rc = need_connected(c)) return rc;
  if (!shards) return api_fail(GQ_ERR_INVALID, "null argument");
  // all local workers in one launch: worker w0 + i writes row w0 + i of each owner;
  // the grid's last CTA raises the phase-1 flags (no separate signal kernel)
  if (gqb::g_comm_fold == 0)  // the flags are raised by gq_allreduce_lanes' signal kernel
    return gqb::quantize_scatter_impl(shards, c->n_local, c->worker_ids.data(), dtype, c->d, norm, c->cfg.kind,
                                      c->cfg.s, c->n, c->plan.lane_width, c->cfg.seed, round, nullptr,
                                      c->scatter[0].data(), c->N, c->slice_lanes, c->slice_bytes, err, stream);
  const uint32_t e1 = ++c->epoch[1];
  const gqb::PeerSignal sig = fold_signal(c, 1, e1, nullptr);
  const int rc = gqb::quantize_scatter_impl(shards, c->n_local, c->worker_ids.data(), dtype, c->d, norm, c->cfg.kind,
                                            c->cfg.s, c->n, c->plan.lane_width, c->cfg.seed, round, nullptr,
                                            c->scatter[0].data(), c->N, c->slice_lanes, c->slice_bytes, err, stream,
                                            &sig);
  if (rc) {
    --c->epoch[1];
    return rc;
  }
  c->rows_signalled = e1;
  return GQ_OK;
}

namespace {
int allreduce_lanes_impl(gq_comm* c, const void* const* lanes, uint64_t round, void* summed_out, uint32_t* err,
                         void* stream, bool final_wait);
}

GQ_EXPORT int gq_allreduce_lanes(gq_comm* c, const void* const* lanes, uint64_t round, void* summed_out,
                                 uint32_t* err, void* stream) {
  return allreduce_lanes_impl(c, lanes, round, summed_out, err, stream, true);
}

namespace {
// final_wait = false: the caller's next kernel waits for phase 2 itself
// (gq_comm_mean's decode, device waits only) and summed_out must be null.
int allreduce_lanes_impl(gq_comm* c, const void* const* lanes, uint64_t round, void* summed_out, uint32_t* err,
                         void* stream, bool final_wait) {
  if (int rc = need_connected(c)) return rc;
  if (!err) return api_fail(GQ_ERR_INVALID, "null argument");
  auto st = static_cast<cudaStream_t>(stream);
  const uint64_t lb = gq_lane_bytes(c->d, c->plan.lane_width);
  if (lanes) {  // caller-quantized lanes: copy each slice to its owner (copy engines over NVLink)
    for (uint32_t i = 0; i < c->n_local; ++i) {
      if (!lanes[i]) return api_fail(GQ_ERR_INVALID, "null argument");
      for (uint32_t j = 0; j < c->N; ++j) {
        const uint64_t off = j * c->slice_bytes;
        if (off >= lb) break;
        const uint64_t bytes = std::min<uint64_t>(c->slice_bytes, lb - off);
        const cudaError_t ce = cudaMemcpyAsync(c->scatter[i][j], static_cast<const uint8_t*>(lanes[i]) + off, bytes,
                                               cudaMemcpyDeviceToDevice, st);
        if (ce != cudaSuccess) return api_cuda_fail(ce);
      }
    }
  }
  uint32_t e1;
  if (!lanes && c->rows_signalled == c->epoch[1] && c->rows_signalled != 0) {
    e1 = c->rows_signalled;  // gq_comm_quantize's kernel raised the flags
  } else {
    e1 = ++c->epoch[1];
    if (int rc = signal(c, 1, e1, st)) return rc;
  }
  c->rows_signalled = 0;
  // device waits: the reduce's CTAs wait for phase 1 in their prologue
  const bool fold_wait = gqb::g_comm_fold != 0 && !c->host_wait && c->lane_end > c->lane_begin;
  gqb::PeerWait w1{};
  if (fold_wait) {
    w1.flags = c->my_flags(1);
    w1.n = c->N;
    w1.epoch = e1;
    w1.timeout_ns = gqb::comm_timeout_ns();
  } else if (int rc = wait(c, 1, e1, err, st)) {
    return rc;
  }
  const uint32_t e2 = ++c->epoch[2];
  bool signalled = false;
  if (c->lane_end > c->lane_begin) {
    const void* rows[GQ_MAX_WORKERS];
    void* outs[kMaxPeers];
    for (uint32_t w = 0; w < c->n; ++w) rows[w] = c->base + c->off_recv + static_cast<size_t>(w) * c->slice_bytes;
    for (uint32_t p = 0; p < c->N; ++p) outs[p] = c->peer[p] + c->off_summed + c->rank * c->slice_bytes;
    // k draws from the norm pass when it ran for this round (gq_comm_norm)
    const bool kd = c->kd_valid && c->kd_round == round;
    const bool fold = gqb::g_comm_fold != 0;
    const gqb::PeerSignal sig = fold_signal(c, 2, e2, nullptr);  // the reduce's last CTA raises phase 2
    const int rc = gqb::reduce_slice_multicast_impl(rows, c->n, c->d, c->lane_begin, c->lane_end, c->cfg.kind,
                                                    c->plan.lane_width, c->cfg.s, c->cfg.topo, c->cfg.seed, round,
                                                    nullptr, kd ? kdraws_rebased(c) : nullptr, c->kwords, outs,
                                                    c->N, err, stream, fold ? &sig : nullptr,
                                                    fold_wait ? &w1 : nullptr);
    if (rc) return rc;
    signalled = fold;
  }
  if (!signalled)
    if (int rc = signal(c, 2, e2, st)) return rc;
  if (!final_wait) return GQ_OK;
  if (int rc = wait(c, 2, e2, err, st)) return rc;
  if (summed_out) {
    const cudaError_t ce = cudaMemcpyAsync(summed_out, c->base + c->off_summed, lb, cudaMemcpyDeviceToDevice, st);
    if (ce != cudaSuccess) return api_cuda_fail(ce);
  }
  return GQ_OK;
}
}  // namespace

GQ_EXPORT const void* gq_comm_summed(const gq_comm* c) { return c ? c->base + c->off_summed : nullptr; }

GQ_EXPORT int gq_comm_mean(gq_comm* c, const void* const* shards, uint32_t dtype, uint64_t round, float* mean_out,
                           double* mean64_out, float* param, float lr, double* norm_out, uint32_t* err,
                           void* stream) {
  if (int rc = need_connected(c)) return rc;
  if (!shards || !err) return api_fail(GQ_ERR_INVALID, "null argument");
  const gq_config& k = c->cfg;
  if (int rc = gq_comm_norm(c, shards, dtype, round, c->norm, err, stream)) return rc;
  if (int rc = gq_comm_quantize(c, shards, dtype, c->norm, round, err, stream)) return rc;
  // device waits: the decode waits for the summed lanes in its prologue
  const bool fold_wait = gqb::g_comm_fold != 0 && !c->host_wait && (mean_out || param) &&
                         (reinterpret_cast<uintptr_t>(mean_out) & 15) == 0 &&
                         (reinterpret_cast<uintptr_t>(param) & 3) == 0;
  if (int rc = allreduce_lanes_impl(c, nullptr, round, nullptr, err, stream, !fold_wait)) return rc;
  const void* summed = gq_comm_summed(c);
  const uint32_t w = c->plan.lane_width;
  if (fold_wait) {
    gqb::PeerWait w2{};
    w2.flags = c->my_flags(2);
    w2.n = c->N;
    w2.epoch = c->epoch[2];
    w2.timeout_ns = gqb::comm_timeout_ns();
    const cudaError_t ce = gqb::launch_dequant_ex(summed, 0, c->d, c->norm, k.kind, k.s, c->n, w, mean_out, param,
                                                  lr, err, static_cast<cudaStream_t>(stream), &w2, nullptr, 0,
                                                  nullptr);
    if (ce != cudaSuccess) return api_cuda_fail(ce);
  } else if (mean_out || param) {
    if (int rc = gq_dequant(summed, 0, c->d, c->norm, k.kind, k.s, c->n, w, mean_out, param, lr, err, stream))
      return rc;
  }
  if (mean64_out) {
    if (int rc = gq_dequant_f64(summed, 0, c->d, c->norm, k.kind, k.s, c->n, w, mean64_out, err, stream))
      return rc;
  }
  if (norm_out) {
    const cudaError_t ce =
        cudaMemcpyAsync(norm_out, c->norm, 8, cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream));
    if (ce != cudaSuccess) return api_cuda_fail(ce);
  }
  return GQ_OK;
}

GQ_EXPORT int gq_sync(gq_comm* c, uint32_t* err, void* stream) {
  if (int rc = need_connected(c)) return rc;
  if (!err) return api_fail(GQ_ERR_INVALID, "null argument");
  auto st = static_cast<cudaStream_t>(stream);
  const uint32_t e = ++c->epoch[3];
  const size_t row = (e & 1u) * kMaxPeers;
  void* dst[kMaxPeers];
  uint32_t* slots[kMaxPeers];
  for (uint32_t p = 0; p < c->N; ++p) {
    dst[p] = c->peer[p] + c->off_errs + (row + c->rank) * 4;
    slots[p] = c->slot(p, 3);
  }
  cudaError_t ce = gqb::launch_p2p_put_signal(err, 4, dst, slots, c->N, e, nullptr, st);
  if (ce != cudaSuccess) return api_cuda_fail(ce);
  if (int rc = wait(c, 3, e, err, st)) return rc;
  ce = cudaStreamSynchronize(st);
  if (ce != cudaSuccess) return api_cuda_fail(ce);
  uint32_t words[kMaxPeers + 1] = {};
  ce = cudaMemcpyAsync(words, c->base + c->off_errs + row * 4, c->N * 4, cudaMemcpyDeviceToHost, c->poll);
  if (ce == cudaSuccess)  // own late flags (a wait timeout)
    ce = cudaMemcpyAsync(words + c->N, err, 4, cudaMemcpyDeviceToHost, c->poll);
  if (ce == cudaSuccess) ce = cudaMemsetAsync(err, 0, 4, c->poll);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(c->poll);
  if (ce != cudaSuccess) return api_cuda_fail(ce);
  uint32_t flags = 0;
  for (uint32_t p = 0; p <= c->N; ++p) flags |= words[p];
  return gqb::status_from_flags(flags);
}

// gq_comm_mean for fixed buffers captured as one CUDA graph. Replays read the
// round from *round_dev (and add round_step) and take their flag epoch from a device
// counter, so each gq_graph_launch is one step with no host work; every rank
// must replay its graph the same number of times. Waits are device kernels, so
// this needs ranks on distinct GPUs (or GQ_OPT_COMM_WAIT = 1).
GQ_EXPORT int gq_comm_graph(gq_comm* c, const void* const* shards, uint32_t dtype, float* mean_out,
                            double* mean64_out, float* param, float lr, uint64_t* round_dev,
                            uint64_t round_step, uint32_t* err, gq_graph** out) {
  if (int rc = need_connected(c)) return rc;
  if (!shards || !round_dev || !err || !out) return api_fail(GQ_ERR_INVALID, "null argument");
  if (c->host_wait)
    return api_fail(GQ_ERR_INVALID, "graph capture needs device-side waits (ranks on distinct GPUs, or GQ_OPT_COMM_WAIT=1)");
  const gq_config& k = c->cfg;
  const uint32_t w = c->plan.lane_width;
  cudaStream_t st;
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e != cudaSuccess) return api_cuda_fail(e);
  auto* g = new gq_graph();
  int rc = GQ_OK;
  e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    auto cu = [&](cudaError_t ce) {
      if (rc == GQ_OK && ce != cudaSuccess) rc = api_cuda_fail(ce);
    };
    auto api = [&](int r) {
      if (rc == GQ_OK) rc = r;
    };
    uint32_t* slots[kMaxPeers];
    void* dst[kMaxPeers];
    // Four kernels per step: every exchange step is folded into a producer's
    // last CTA (stats put in the norm pass, phase signals in quantize and
    // reduce) or a consumer's prologue (the quantize waits for the stats and
    // folds the norm, the reduce waits for the rows, the decode for the
    // summed lanes and advances the round).
    // GQ_OPT_COMM_FOLD = 0 keeps every exchange step a kernel of its own
    // (stats put, waits, signals, norm combine): the fallback should the
    // folded forms misbehave on a platform they were not verified on.
    const bool fold = gqb::g_comm_fold != 0;
    const gqb::KDrawJob job = kjob(c, 0, round_dev);
    gqb::StatsPut put{};
    for (uint32_t p = 0; p < c->N; ++p) {
      dst[p] = c->peer[p] + c->off_stats + (2ull * c->n + c->w0) * 8;
      slots[p] = c->slot(p, 4);
      put.dst[p] = static_cast<double*>(dst[p]);
      put.slots[p] = slots[p];
    }
    put.n = c->N;
    put.ep_dev = c->ep_dev;
    const bool fold_put = fold && k.norm_q != GQ_NORM_L2_SEQUENTIAL;  // the sequential L2 pass has no last block
    cu(gqb::launch_norm(shards, dtype, c->n_local, c->d, k.norm_q, k.norm_p, c->stats_local, nullptr, c->ws, err, st,
                        c->kbuf ? &job : nullptr, fold_put ? &put : nullptr));
    if (!fold_put)
      cu(gqb::launch_p2p_put_signal(c->stats_local, 8 * c->n_local, dst, slots, c->N, 0, c->ep_dev, st,
                                    /*bump=*/true));
    gqb::PeerWait w4{}, w5{}, w6{};
    w4.flags = c->my_flags(4);
    w5.flags = c->my_flags(5);
    w6.flags = c->my_flags(6);
    w4.n = w5.n = w6.n = c->N;
    w4.ep_dev = w5.ep_dev = w6.ep_dev = c->ep_dev;
    w4.timeout_ns = w5.timeout_ns = w6.timeout_ns = gqb::comm_timeout_ns();
    const gqb::PeerSignal sig5 = fold_signal(c, 5, 0, c->ep_dev);  // raised by the quantize's last CTA
    const double* stats_row = reinterpret_cast<const double*>(c->base + c->off_stats) + 2ull * c->n;
    if (!fold) {
      cu(gqb::launch_p2p_wait(c->my_flags(4), c->N, 0, c->ep_dev, err, st));
      cu(gqb::launch_norm_combine(stats_row, c->n, k.norm_p, c->norm, st));
    }
    if (rc == GQ_OK)
      api(gqb::quantize_scatter_impl(shards, c->n_local, c->worker_ids.data(), dtype, c->d, c->norm, k.kind, k.s,
                                     c->n, w, k.seed, 0, round_dev, c->scatter[0].data(), c->N, c->slice_lanes,
                                     c->slice_bytes, err, st, fold ? &sig5 : nullptr, fold ? &w4 : nullptr,
                                     fold ? stats_row : nullptr, k.norm_p));
    if (!fold) {
      for (uint32_t p = 0; p < c->N; ++p) slots[p] = c->slot(p, 5);
      cu(gqb::launch_p2p_signal(slots, c->N, 0, c->ep_dev, st));
      cu(gqb::launch_p2p_wait(c->my_flags(5), c->N, 0, c->ep_dev, err, st));
    }
    if (c->lane_end > c->lane_begin && rc == GQ_OK) {
      const void* rows[GQ_MAX_WORKERS];
      void* outs[kMaxPeers];
      for (uint32_t r = 0; r < c->n; ++r) rows[r] = c->base + c->off_recv + static_cast<size_t>(r) * c->slice_bytes;
      for (uint32_t p = 0; p < c->N; ++p) outs[p] = c->peer[p] + c->off_summed + c->rank * c->slice_bytes;
      const gqb::PeerSignal sig6 = fold_signal(c, 6, 0, c->ep_dev);  // raised by the reduce's last CTA
      api(gqb::reduce_slice_multicast_impl(rows, c->n, c->d, c->lane_begin, c->lane_end, k.kind, w, k.s, k.topo,
                                           k.seed, 0, round_dev, c->kbuf ? kdraws_rebased(c) : nullptr, c->kwords,
                                           outs, c->N, err, st, fold ? &sig6 : nullptr, fold ? &w5 : nullptr));
      if (!fold) {
        for (uint32_t p = 0; p < c->N; ++p) slots[p] = c->slot(p, 6);
        cu(gqb::launch_p2p_signal(slots, c->N, 0, c->ep_dev, st));
      }
    } else {
      if (fold) cu(gqb::launch_p2p_wait(c->my_flags(5), c->N, 0, c->ep_dev, err, st));
      for (uint32_t p = 0; p < c->N; ++p) slots[p] = c->slot(p, 6);
      cu(gqb::launch_p2p_signal(slots, c->N, 0, c->ep_dev, st));
    }
    const void* summed = c->base + c->off_summed;
    const uint64_t rstep = round_step ? round_step : 1;
    if ((mean_out || param) && rc == GQ_OK && fold) {
      // the decode waits for phase 6 and its last CTA advances the round
      cu(gqb::launch_dequant_ex(summed, 0, c->d, c->norm, k.kind, k.s, c->n, w, mean_out, param, lr, err, st, &w6,
                                  round_dev, rstep,
                                  reinterpret_cast<unsigned int*>(static_cast<char*>(c->ws) + gqb::kWsRoundTicketComm)));
    } else {
      cu(gqb::launch_p2p_wait(c->my_flags(6), c->N, 0, c->ep_dev, err, st, round_dev, rstep));
      if ((mean_out || param) && rc == GQ_OK)
        api(gq_dequant(summed, 0, c->d, c->norm, k.kind, k.s, c->n, w, mean_out, param, lr, err, st));
    }
    if (mean64_out && rc == GQ_OK) api(gq_dequant_f64(summed, 0, c->d, c->norm, k.kind, k.s, c->n, w, mean64_out, err, st));
    e = cudaStreamEndCapture(st, &g->graph);
  }
  if (rc == GQ_OK && e == cudaSuccess) e = cudaGraphInstantiate(&g->exec, g->graph, 0);
  cudaStreamDestroy(st);
  if (rc == GQ_OK && e != cudaSuccess) rc = api_cuda_fail(e);
  if (rc != GQ_OK) {
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
    return rc;
  }
  *out = g;
  return GQ_OK;
}
