// Reference-side binding of libgq_b200.so (see gqsgd_b200.hpp).
// Every per-element step runs in the sm_100a kernels behind include/gq_b200.h;
// this file only moves buffers, maps status codes to the reference's
// exception classes and fills the reference's result structs.
#include "gqsgd_b200.hpp"

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>

#include "gq_b200.h"
#include "gqsgd/exp_arith.hpp"
#include "gqsgd/serialize.hpp"
#include "gqsgd/topology.hpp"

namespace gqsgd_b200 {

namespace {

// gq_status -> the reference's exception classes (include/gq_b200.h).
[[noreturn]] void raise(int rc) {
  const std::string msg = gq_last_error();
  switch (rc) {
    case GQ_ERR_INVALID: throw std::invalid_argument(msg);
    case GQ_ERR_OVERFLOW: throw std::overflow_error(msg);
    case GQ_ERR_DOMAIN: throw std::domain_error(msg);
    default: throw std::runtime_error(msg);
  }
}

void ok(int rc) {
  if (rc != GQ_OK) raise(rc);
}

// Owning device allocation through the C ABI (no CUDA headers here).
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(std::size_t bytes) : n_(bytes) { ok(gq_malloc(bytes, &p_)); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(std::exchange(o.p_, nullptr)), n_(o.n_) {}
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      if (p_) gq_free(p_);
      p_ = std::exchange(o.p_, nullptr);
      n_ = o.n_;
    }
    return *this;
  }
  ~DevBuf() {
    if (p_) gq_free(p_);
  }
  void* get() const { return p_; }
  template <typename T>
  T* as() const { return static_cast<T*>(p_); }
  void upload(const void* src, std::size_t bytes) { ok(gq_memcpy(p_, src, bytes, nullptr)); }
  void download(void* dst, std::size_t bytes) const { ok(gq_memcpy(dst, p_, bytes, nullptr)); }
  void zero() { ok(gq_memset(p_, 0, n_, nullptr)); }

 private:
  void* p_ = nullptr;
  std::size_t n_ = 0;
};

// Owning pinned host allocation (one H2D of all shards per call).
class HostBuf {
 public:
  HostBuf() = default;
  explicit HostBuf(std::size_t bytes) { ok(gq_malloc_host(bytes, &p_)); }
  HostBuf(const HostBuf&) = delete;
  HostBuf& operator=(const HostBuf&) = delete;
  HostBuf& operator=(HostBuf&& o) noexcept {
    if (this != &o) {
      if (p_) gq_free_host(p_);
      p_ = std::exchange(o.p_, nullptr);
    }
    return *this;
  }
  ~HostBuf() {
    if (p_) gq_free_host(p_);
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p_); }

 private:
  void* p_ = nullptr;
};

// The device error word: gq_check synchronises and rethrows raised flags.
class ErrWord {
 public:
  ErrWord() : b_(sizeof(std::uint32_t)) { b_.zero(); }
  std::uint32_t* get() const { return b_.as<std::uint32_t>(); }
  void check() const { ok(gq_check(get(), nullptr)); }

 private:
  DevBuf b_;
};

// IntSumOps / TokenReduceOps::combine on host spans: stage both chunks on
// the device, one gq_combine_lanes launch, copy the result back.
void device_combine(std::span<std::byte> acc, std::span<const std::byte> in, std::uint32_t kind,
                    std::uint32_t width, std::uint32_t s, std::uint32_t n, std::uint64_t seed,
                    std::uint64_t round, std::uint32_t step, std::uint32_t dst,
                    std::uint64_t elem_offset) {
  const std::size_t lb = width / 8;
  if (acc.size() != in.size() || acc.size() % lb != 0) {
    throw std::invalid_argument("payload chunks disagree or are not lane-aligned");
  }
  if (acc.empty()) return;
  DevBuf a(acc.size()), b(in.size());
  a.upload(acc.data(), acc.size());
  b.upload(in.data(), in.size());
  ErrWord err;
  ok(gq_combine_lanes(a.get(), b.get(), acc.size() / lb, elem_offset, kind, width, s, n, seed, round,
                      step, dst, err.get(), nullptr));
  err.check();
  a.download(acc.data(), acc.size());
}

// The TrafficReport allreduce_inproc (collectives.cpp:155-190) records for a
// payload of `lanes` lanes of `lb` bytes on `sched`.
gqsgd::TrafficReport schedule_traffic(const gqsgd::Schedule& sched, std::size_t lanes, std::size_t lb) {
  gqsgd::TrafficReport t;
  t.bytes_sent.assign(sched.workers, 0);
  t.steps = sched.steps;
  for (const gqsgd::CommEvent& ev : sched.events) {
    const auto [b, e] = gqsgd::chunk_lane_range(lanes, sched.chunks, ev.chunk);
    if (ev.op == gqsgd::CommOp::Reduce) ++t.reduce_invocations;
    t.add_send(ev.src, (e - b) * lb);
  }
  return t;
}

// Per-thread device buffers reused across gqsgd_mean calls (grown on demand):
// the reference's API is called in tight loops (Monte Carlo, training steps),
// so allocation must not sit on the per-call path. One pinned staging buffer
// carries all n shards in (one H2D), and the decoded mean and the norm sit in
// one device buffer so a single D2H returns both.
struct Workspace {
  std::uint32_t n = 0, width = 0;
  std::size_t d = 0, xs = 0, ls = 0, last_payload = ~std::size_t{0};
  DevBuf xbuf, lbuf, summed, stats, out, ws;
  HostBuf stage_in, stage_out;
  ErrWord err;
  std::vector<const void*> x_ptr;
  std::vector<void*> lane_ptr;

  static Workspace& get(std::uint32_t n, std::size_t d, std::uint32_t width) {
    thread_local Workspace w;
    if (n > w.n || d > w.d || width > w.width) w.grow(std::max(n, w.n), std::max(d, w.d), std::max(width, w.width));
    w.x_ptr.resize(n);
    w.lane_ptr.resize(n);
    for (std::uint32_t r = 0; r < n; ++r) {
      w.x_ptr[r] = w.xbuf.as<char>() + r * w.xs;
      w.lane_ptr[r] = w.lbuf.as<char>() + r * w.ls;
    }
    // lanes past d are read as zero padding by the aggregation: clear them
    // whenever the payload byte count changes (quantize never writes past it)
    const std::size_t payload = (d * width + 7) / 8;
    if (payload != w.last_payload) {
      ok(gq_memset(w.lbuf.get(), 0, w.n * w.ls, nullptr));
      w.last_payload = payload;
    }
    return w;
  }

  void grow(std::uint32_t n2, std::size_t d2, std::uint32_t w2) {
    n = n2;
    d = d2;
    width = w2;
    xs = (d * sizeof(double) + 255) & ~std::size_t{255};
    ls = (gq_lane_bytes(d, width) + 255) & ~std::size_t{255};
    xbuf = DevBuf(n * xs);
    lbuf = DevBuf(n * ls);
    summed = DevBuf(ls);
    stats = DevBuf(n * sizeof(double));
    out = DevBuf((d + 2) * sizeof(double));  // mean, norm, error word
    out.zero();
    ws = DevBuf(gq_norm_workspace_bytes(n, d));
    ws.zero();
    stage_in = HostBuf(n * xs);
    stage_out = HostBuf((d + 2) * sizeof(double));
    last_payload = ~std::size_t{0};
  }

  double* mean() const { return out.as<double>(); }
  double* norm_at(std::size_t dd) const { return out.as<double>() + dd; }  // right after this call's mean
  // the device error word rides in the same D2H, right after the norm
  std::uint32_t* err_at(std::size_t dd) const { return reinterpret_cast<std::uint32_t*>(out.as<double>() + dd + 1); }
};

gq_config to_c(const gqsgd::GqsgdConfig& cfg) {
  gq_config c{};
  c.workers = cfg.workers;
  c.kind = cfg.scheme == gqsgd::LevelKind::Standard ? GQ_KIND_STANDARD : GQ_KIND_EXPONENTIAL;
  c.s = cfg.s;
  // L2 accumulated in element order: the reference's doubles bit for bit (norms.cpp:40-43)
  c.norm_q = cfg.norm.q == gqsgd::kNormInf ? GQ_NORM_INF : (cfg.norm.q == 2 ? GQ_NORM_L2_SEQUENTIAL : cfg.norm.q);
  c.norm_p = cfg.norm.p == gqsgd::kNormInf ? GQ_NORM_INF : cfg.norm.p;
  // The 4-bit lanes are a device-ABI extension: reference callers get the
  // reference's plan, so a standard request below 8 bits becomes
  // standard_lane_width's first candidate, 8 (algorithm.cpp:22-29).
  c.width_bits = (c.kind == GQ_KIND_STANDARD && cfg.width_bits < 8) ? 8 : cfg.width_bits;
  c.topo = cfg.topo == gqsgd::TopologyKind::Tree ? GQ_TOPO_TREE : GQ_TOPO_RING;
  c.seed = cfg.seed;
  return c;
}

}  // namespace

DeviceIntSumOps::DeviceIntSumOps(std::uint32_t width_bits) : width_bits_(width_bits) {
  if (width_bits != 8 && width_bits != 16 && width_bits != 32 && width_bits != 64) {  // collectives.cpp:23-27
    throw std::invalid_argument("integer lane width must be 8, 16, 32, or 64 bits");
  }
}

void DeviceIntSumOps::combine(std::span<std::byte> acc, std::span<const std::byte> in,
                              std::uint64_t round, std::uint32_t step, std::uint32_t dst,
                              std::uint64_t elem_offset) const {
  device_combine(acc, in, GQ_KIND_STANDARD, width_bits_, 1, 1, 0, round, step, dst, elem_offset);
}

DeviceTokenReduceOps::DeviceTokenReduceOps(const gqsgd::ReduceContext& ctx, const gqsgd::CounterRng& rng)
    : ctx_(ctx), seed_(rng.seed()) {}

void DeviceTokenReduceOps::combine(std::span<std::byte> acc, std::span<const std::byte> in,
                                   std::uint64_t round, std::uint32_t step, std::uint32_t dst,
                                   std::uint64_t elem_offset) const {
  device_combine(acc, in, GQ_KIND_EXPONENTIAL, ctx_.width_bits, ctx_.s, ctx_.n, seed_, round, step, dst,
                 elem_offset);
}

gqsgd::QuantizedShard quantize_shard(std::span<const double> x, double norm,
                                     const gqsgd::LevelScheme& scheme, const gqsgd::CounterRng& rng,
                                     std::uint32_t worker, std::uint64_t round) {
  if (scheme.kind() == gqsgd::LevelKind::Custom) {
    throw std::invalid_argument("the device quantizer supports the standard and exponential grids");
  }
  const std::uint32_t s = scheme.s();
  const std::uint32_t kind = scheme.kind() == gqsgd::LevelKind::Standard ? GQ_KIND_STANDARD : GQ_KIND_EXPONENTIAL;
  const std::size_t d = x.size();
  gqsgd::QuantizedShard out;
  out.norm = norm;
  out.sign.assign(d, 1);
  out.level_idx.assign(d, s);
  if (d == 0) return out;
  // 32-bit lanes, one worker (exponential lanes carry idx + prescale_shift(1) = idx + 1).
  DevBuf xd(d * sizeof(double)), lanes(gq_lane_bytes(d, 32)), nd(sizeof(double));
  xd.upload(x.data(), d * sizeof(double));
  nd.upload(&norm, sizeof(double));
  ErrWord err;
  const void* xs[1] = {xd.get()};
  void* ls[1] = {lanes.get()};
  const std::uint32_t wid[1] = {worker};
  ok(gq_quantize(xs, GQ_DTYPE_F64, 1, wid, d, nd.as<double>(), kind, s, 1, 32, rng.seed(), round, ls,
                 err.get(), nullptr));
  err.check();
  std::vector<std::int32_t> lane(d);
  lanes.download(lane.data(), d * sizeof(std::int32_t));
  for (std::size_t j = 0; j < d; ++j) {
    const std::int32_t v = lane[j];
    if (kind == GQ_KIND_STANDARD) {  // lane = sign * (s - idx)   (algorithm.cpp:69-82)
      out.sign[j] = v < 0 ? -1 : 1;
      out.level_idx[j] = s - static_cast<std::uint32_t>(v < 0 ? -v : v);
    } else {  // lane = (idx + 1) | sign bit, 0 = zero level (exp_arith.cpp:126-160)
      const std::uint32_t u = static_cast<std::uint32_t>(v);
      const std::uint32_t e = u & 0x7fffffffu;
      if (e != 0) {
        out.sign[j] = (u >> 31) ? -1 : 1;
        out.level_idx[j] = e - 1;
      }
    }
  }
  return out;
}

bool handles(const gqsgd::GqsgdConfig& cfg) {
  if (cfg.transport != gqsgd::Transport::Inproc) return false;
  if (cfg.scheme == gqsgd::LevelKind::Custom) return false;
  if (cfg.workers == 0 || cfg.workers > GQ_MAX_WORKERS) return false;
  // norm orders 2 / inf: the drop-in is bit-identical there; other orders
  // (the device's power sums agree with glibc's pow to rounding only) stay
  // on the reference
  const bool qok = cfg.norm.q == gqsgd::kNormInf || cfg.norm.q == 2;
  const bool pok = cfg.norm.p == gqsgd::kNormInf || cfg.norm.p == 2;
  if (!qok || !pok) return false;
  if (cfg.sparse) {  // validate_level_width (serialize.cpp:114-122)
    const std::uint32_t w = cfg.width_bits;
    return (w == 8 || w == 16 || w == 32) && (w == 32 || cfg.s <= (1u << w) - 1) && cfg.s > 0;
  }
  // token lanes: ReduceContext::make takes 8, 16 or 32 bits only
  // (exp_arith.cpp:63-80); anything else goes to the reference, which throws
  if (cfg.scheme == gqsgd::LevelKind::Exponential && cfg.width_bits != 8 && cfg.width_bits != 16 &&
      cfg.width_bits != 32)
    return false;
  gq_config c = to_c(cfg);
  gq_plan plan;
  return gq_plan_path(&c, &plan) == GQ_OK;
}

namespace {

// cfg.sparse (algorithm.cpp:187-200): every worker's quantized shard travels
// as serialize_sparse(to_sparse()) through allgather_inproc; each worker
// accumulates all of them in rank order and divides by n. On the device the
// n payloads are built by gq_sparse_encode (their sizes give the allgather
// traffic) and the mean comes from the rank-ordered accumulation kernel.
gqsgd::MeanResult gqsgd_mean_sparse(const std::vector<std::vector<double>>& shards,
                                    const gqsgd::GqsgdConfig& cfg, std::uint64_t round) {
  const std::uint32_t n = cfg.workers;
  const std::size_t d = shards.front().size();
  const std::uint32_t kind = cfg.scheme == gqsgd::LevelKind::Standard ? GQ_KIND_STANDARD : GQ_KIND_EXPONENTIAL;
  const std::uint32_t width = gqsgd::validate_level_width(cfg.width_bits, cfg.s);
  if (d > 0xffffffffull) throw std::invalid_argument("sparse shards index elements with u32");
  gqsgd::MeanResult res;
  res.lane_width_used = width;
  res.norm_traffic = schedule_traffic(gqsgd::tree_schedule(n), 1, 8);

  const std::size_t xs = (d * sizeof(double) + 255) & ~std::size_t{255};
  const std::size_t ls = (gq_lane_bytes(d, 32) + 255) & ~std::size_t{255};
  DevBuf x(n * xs + 16), lanes(n * ls + 16), stats(n * sizeof(double)), normd(sizeof(double)),
      ws(gq_norm_workspace_bytes(n, d)), mean((d + 1) * sizeof(double)),
      payload(gq_sparse_payload_bytes(d, width) + 16), sws(gq_sparse_workspace_bytes(d)), nnz(4 * n + 4);
  ws.zero();
  lanes.zero();
  ErrWord err;
  std::vector<const void*> xp(n);
  std::vector<void*> lp(n);
  std::vector<std::uint32_t> ids(n);
  for (std::uint32_t r = 0; r < n; ++r) {
    xp[r] = x.as<char>() + r * xs;
    lp[r] = lanes.as<char>() + r * ls;
    ids[r] = r;
    ok(gq_memcpy(const_cast<void*>(xp[r]), shards[r].data(), d * sizeof(double), nullptr));
  }
  gq_config c = to_c(cfg);
  ok(gq_norm(xp.data(), GQ_DTYPE_F64, n, d, c.norm_q, c.norm_p, stats.as<double>(), normd.as<double>(), ws.get(),
             err.get(), nullptr));
  ok(gq_quantize(xp.data(), GQ_DTYPE_F64, n, ids.data(), d, normd.as<double>(), kind, cfg.s, n, 32, cfg.seed,
                 round, lp.data(), err.get(), nullptr));
  for (std::uint32_t r = 0; r < n; ++r) {
    ok(gq_sparse_encode(lp[r], d, kind, cfg.s, n, width, normd.as<double>(), payload.get(), sws.get(),
                        nnz.as<std::uint32_t>() + r, nullptr));
  }
  ok(gq_sparse_mean_inproc(lp.data(), n, d, kind, cfg.s, n, normd.as<double>(), nullptr, mean.as<double>(),
                           nullptr));
  err.check();
  normd.download(&res.norm, sizeof(double));
  if (res.norm == 0.0) {  // algorithm.cpp:175-178
    res.per_worker.assign(n, std::vector<double>(d, 0.0));
    return res;
  }
  std::vector<double> m(d);
  mean.download(m.data(), d * sizeof(double));
  res.per_worker.assign(n, m);
  std::vector<std::uint32_t> counts(n);
  nnz.download(counts.data(), n * sizeof(std::uint32_t));
  // allgather_inproc traffic (collectives.cpp:192-208): each event forwards
  // the origin worker's payload
  const gqsgd::Schedule sched = gqsgd::allgather_schedule(n);
  res.payload_traffic.bytes_sent.assign(n, 0);
  res.payload_traffic.steps = sched.steps;
  for (const gqsgd::CommEvent& ev : sched.events) {
    res.payload_traffic.add_send(ev.src, gq_sparse_payload_bytes(counts[ev.chunk], width));
  }
  return res;
}

}  // namespace

gqsgd::MeanResult gqsgd_mean(const std::vector<std::vector<double>>& shards,
                             const gqsgd::GqsgdConfig& cfg, std::uint64_t round) {
  const std::uint32_t n = cfg.workers;
  if (shards.size() != n || n == 0) {
    throw std::invalid_argument("shard count does not match the worker count");
  }
  const std::size_t d = shards.front().size();
  for (const auto& x : shards) {
    if (x.size() != d) throw std::invalid_argument("shard dimensions disagree");
  }
  if (cfg.transport != gqsgd::Transport::Inproc) {
    throw std::invalid_argument("gqsgd_b200::gqsgd_mean covers the in-process transport");
  }
  if (d == 0) {  // nothing to quantize: the scale is 0 and every worker gets an empty mean (algorithm.cpp:175-178)
    gqsgd::MeanResult res;
    res.lane_width_used = cfg.sparse ? gqsgd::validate_level_width(cfg.width_bits, cfg.s) : 0;
    if (!cfg.sparse) {
      const gq_config c0 = to_c(cfg);
      gq_plan p0;
      ok(gq_plan_path(&c0, &p0));
      res.lane_width_used = p0.lane_width;
    }
    res.norm_traffic = schedule_traffic(gqsgd::tree_schedule(n), 1, 8);
    res.per_worker.assign(n, std::vector<double>());
    return res;
  }
  if (cfg.sparse) return gqsgd_mean_sparse(shards, cfg, round);
  const gq_config c = to_c(cfg);
  gq_plan plan;
  ok(gq_plan_path(&c, &plan));

  gqsgd::MeanResult res;
  res.lane_width_used = plan.lane_width;
  const gqsgd::Schedule norm_sched = gqsgd::tree_schedule(n);
  res.norm_traffic = schedule_traffic(norm_sched, 1, 8);  // one f64 per worker (collectives.cpp:210-233)

  // Upload the shards (f64: the reference's element type) into the calling
  // thread's cached device workspace, run the fused path (norm -> quantize ->
  // schedule replay), decode to doubles, read mean + norm back in one copy.
  Workspace& w = Workspace::get(n, d, plan.lane_width);
  for (std::uint32_t r = 0; r < n; ++r) {
    std::memcpy(w.stage_in.as<char>() + r * w.xs, shards[r].data(), d * sizeof(double));
  }
  ok(gq_memcpy(w.xbuf.get(), w.stage_in.as<char>(), n * w.xs, nullptr));
  std::uint32_t* errw = w.err_at(d);  // its slot moves with d: cleared per call (async)
  ok(gq_memset(errw, 0, sizeof(std::uint32_t), nullptr));
  ok(gq_mean_inproc(w.x_ptr.data(), GQ_DTYPE_F64, d, &c, round, w.lane_ptr.data(), w.summed.get(), nullptr,
                    nullptr, 0.0f, w.stats.as<double>(), w.norm_at(d), w.ws.get(), errw, nullptr));
  ok(gq_dequant_f64(w.summed.get(), 0, d, w.norm_at(d), c.kind, c.s, n, plan.lane_width, w.mean(), errw, nullptr));
  // one D2H brings the mean, the norm and the error word; one stream sync
  ok(gq_memcpy(w.stage_out.as<char>(), w.mean(), (d + 2) * sizeof(double), nullptr));
  ok(gq_stream_sync(nullptr));
  if (*reinterpret_cast<const std::uint32_t*>(w.stage_out.as<double>() + d + 1) != 0)
    ok(gq_check(errw, nullptr));  // maps the device flags to the reference's exception class
  const double* host = w.stage_out.as<double>();
  res.norm = host[d];
  if (res.norm == 0.0) {  // algorithm.cpp:175-178: zeros, no payload traffic
    res.per_worker.assign(n, std::vector<double>(d, 0.0));
    return res;
  }
  res.per_worker.assign(n, std::vector<double>(host, host + d));  // every worker decodes the same lanes
  res.payload_traffic = schedule_traffic(gqsgd::make_schedule(cfg.topo, n), d, plan.lane_width / 8);
  return res;
}

bool handles_worker(const gqsgd::GqsgdConfig& cfg) {
  if (cfg.sparse || cfg.workers > 16) return false;
  // the communicator folds the norm stats on the device: orders 2 / inf only
  const auto dev_order = [](std::uint32_t v) { return v == gqsgd::kNormInf || v == 2; };
  if (!dev_order(cfg.norm.q) || !dev_order(cfg.norm.p)) return false;
  gqsgd::GqsgdConfig inproc = cfg;
  inproc.transport = gqsgd::Transport::Inproc;
  return handles(inproc);
}

namespace {

// One communicator per thread (= per rank of run_local_mesh, or per process),
// rebuilt when the job changes. Bootstrap: every rank's gq_comm handle goes to
// every peer as one Ctrl frame over the reference's own mesh.
struct WorkerComm {
  gq_comm* comm = nullptr;
  const gqsgd::PeerSockets* peers = nullptr;
  std::uint32_t rank = 0;
  std::size_t d = 0;
  gq_config cfg{};
  DevBuf x, mean;  // shard in, f64 mean + norm out
  HostBuf stage;
  ErrWord err;

  ~WorkerComm() { gq_comm_destroy(comm); }

  void open(gqsgd::PeerSockets& p, const gq_config& c, std::size_t dd, std::uint64_t round) {
    const bool same = comm && peers == &p && rank == p.rank() && d == dd && std::memcmp(&cfg, &c, sizeof(c)) == 0;
    if (same) return;
    gq_comm_destroy(comm);
    comm = nullptr;
    peers = &p;
    rank = p.rank();
    d = dd;
    cfg = c;
    ok(gq_comm_init(p.rank(), p.workers(), &c, dd, &comm));
    const std::size_t hb = gq_comm_handle_bytes();
    std::vector<std::byte> all(hb * p.workers());
    ok(gq_comm_handle(comm, all.data() + hb * p.rank()));
    const std::span<const std::byte> mine(all.data() + hb * p.rank(), hb);
    const auto r32 = static_cast<std::uint32_t>(round);
    for (std::uint32_t q = 0; q < p.workers(); ++q)
      if (q != p.rank()) p.send_frame(q, gqsgd::MsgType::Ctrl, r32, mine);
    for (std::uint32_t q = 0; q < p.workers(); ++q) {
      if (q == p.rank()) continue;
      const gqsgd::Payload h = p.recv_frame(q, gqsgd::MsgType::Ctrl, r32);
      if (h.size() != hb) throw std::runtime_error("bad communicator handle frame");
      std::memcpy(all.data() + hb * q, h.data(), hb);
    }
    ok(gq_comm_connect(comm, all.data()));
    x = DevBuf(dd * sizeof(double));
    mean = DevBuf((dd + 1) * sizeof(double));
    stage = HostBuf((dd + 1) * sizeof(double));
  }
};

}  // namespace

gqsgd::WorkerMeanResult gqsgd_mean_worker(gqsgd::PeerSockets& peers, const std::vector<double>& shard,
                                          const gqsgd::GqsgdConfig& cfg, std::uint64_t round) {
  if (peers.workers() != cfg.workers) throw std::invalid_argument("mesh size does not match the worker count");
  if (!handles_worker(cfg)) throw std::invalid_argument("gqsgd_b200::gqsgd_mean_worker covers the dense paths");
  const std::size_t d = shard.size();
  if (d == 0) throw std::invalid_argument("empty shard");
  const gq_config c = to_c(cfg);
  gq_plan plan;
  ok(gq_plan_path(&c, &plan));
  thread_local WorkerComm w;
  w.open(peers, c, d, round);

  gqsgd::WorkerMeanResult out;
  out.lane_width_used = plan.lane_width;
  w.x.upload(shard.data(), d * sizeof(double));
  const void* xs[1] = {w.x.get()};
  double* m = w.mean.as<double>();
  const int rc = gq_comm_mean(w.comm, xs, GQ_DTYPE_F64, round, nullptr, m, nullptr, 0.0f, m + d, w.err.get(), nullptr);
  // every rank learns every rank's device errors (and a launch failure here
  // still lets the peers' exchange time out rather than hang)
  const int rs = gq_sync(w.comm, w.err.get(), nullptr);
  if (rc != GQ_OK) raise(rc);
  if (rs != GQ_OK) raise(rs);
  ok(gq_memcpy(w.stage.as<char>(), m, (d + 1) * sizeof(double), nullptr));
  ok(gq_stream_sync(nullptr));
  const double* host = w.stage.as<double>();
  out.norm = host[d];
  // bytes this rank sends in the reference's walks (run_allreduce_worker,
  // transport.cpp:232-287): the tree norm exchange of one f64, and the lane
  // schedule unless the scale is zero (algorithm.cpp:265-268)
  out.norm_bytes_sent = schedule_traffic(gqsgd::tree_schedule(cfg.workers), 1, 8).bytes_sent[peers.rank()];
  if (out.norm == 0.0) {
    out.mean.assign(d, 0.0);
    return out;
  }
  out.mean.assign(host, host + d);
  out.payload_bytes_sent =
      schedule_traffic(gqsgd::make_schedule(cfg.topo, cfg.workers), d, plan.lane_width / 8).bytes_sent[peers.rank()];
  return out;
}

}  // namespace gqsgd_b200
