/* gq_b200.h — C-ABI of the B200-native Global-QSGD gradient-sync hot path.
 *
 * This is the drop-in boundary. Each entry point replaces one piece of the
 * reference's compress / aggregate / decompress interface
 * (/root/reference/proj/include/gqsgd/ *.hpp); the replaced declaration is
 * cited beside it. Conventions:
 *   - plain C types only; every buffer is a DEVICE pointer owned by the
 *     caller, except arrays documented as "host array" (small per-call
 *     descriptors such as the n per-worker pointers);
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream);
 *     every call is stream-ordered and returns before the GPU finishes;
 *   - the return value is a gq_status for argument/launch errors detected on
 *     the host (the reference's std::invalid_argument cases that depend only
 *     on the configuration). Data-dependent errors (NaN/Inf, |x| > norm,
 *     lane overflow, token range, negative-zero tokens) are raised by the
 *     kernels into the caller's `err` word (GQ_FLAG_*) and surfaced by
 *     gq_check(), which maps them to the same status classes;
 *   - gq_last_error() gives the message of the last failing call on the
 *     calling thread, worded like the reference's exception text.
 * Status classes map to the reference's exceptions:
 *   GQ_ERR_INVALID  -> std::invalid_argument
 *   GQ_ERR_OVERFLOW -> std::overflow_error
 *   GQ_ERR_DOMAIN   -> std::domain_error
 *   GQ_ERR_RUNTIME  -> std::runtime_error
 */
#ifndef GQ_B200_H
#define GQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GQ_ABI_VERSION 1
#define GQ_MAX_WORKERS 128

/* status codes */
#define GQ_OK 0
#define GQ_ERR_INVALID 1
#define GQ_ERR_OVERFLOW 2
#define GQ_ERR_DOMAIN 3
#define GQ_ERR_RUNTIME 4
#define GQ_ERR_CUDA 6

/* device error flags (OR-ed into the caller's uint32 `err` word) */
#define GQ_FLAG_NONFINITE 0x1u      /* invalid_argument: NaN or Inf (norms.cpp:55-57, quantizer.cpp:35-37) */
#define GQ_FLAG_EXCEEDS_SCALE 0x2u  /* invalid_argument: |x| > norm (quantizer.cpp:39-41) */
#define GQ_FLAG_ZERO_SCALE 0x4u     /* invalid_argument: norm 0, x != 0 (quantizer.cpp:22-26) */
#define GQ_FLAG_LANE_OVERFLOW 0x8u  /* overflow_error: integer lane overflow (collectives.cpp:76-78) */
#define GQ_FLAG_TOKEN_RANGE 0x10u   /* overflow_error: token exponent range (exp_arith.cpp:103-107) */
#define GQ_FLAG_NEG_ZERO 0x20u      /* domain_error: negative zero token (exp_arith.cpp:178-179) */
#define GQ_FLAG_BAD_SCALE 0x40u     /* invalid_argument: norm not finite/negative (quantizer.cpp:11-13) */
#define GQ_FLAG_BAD_PAYLOAD 0x80u   /* domain_error: malformed sparse payload (serialize.cpp:170-190, quantizer.cpp:80-87) */
#define GQ_FLAG_P2P_TIMEOUT 0x100u  /* runtime_error: a peer never signalled (peer-memory exchange, GQ_OPT_COMM_TIMEOUT_S) */

/* enums (LevelKind levels.hpp:9, TopologyKind topology.hpp:10, NormSpec norms.hpp:12-19) */
#define GQ_KIND_STANDARD 0u
#define GQ_KIND_EXPONENTIAL 1u
#define GQ_TOPO_TREE 0u
#define GQ_TOPO_RING 1u
#define GQ_NORM_INF 0xffffffffu
/* norm_q = GQ_NORM_L2_SEQUENTIAL: the L2 sum accumulated in element order in
 * f64, bit-identical to the reference's vector_norm (norms.cpp:40-43) at the
 * cost of one sequential chain per worker (use for reference-exact results
 * at small d; the default L2 is a parallel sum within 1e-12 relative). */
#define GQ_NORM_L2_SEQUENTIAL 0x102u
#define GQ_DTYPE_F32 0u
#define GQ_DTYPE_F64 1u

/* Mirrors gqsgd::GqsgdConfig (algorithm.hpp:21-32) for the dense paths. */
typedef struct gq_config {
  uint32_t workers;    /* n */
  uint32_t kind;       /* GQ_KIND_* */
  uint32_t s;          /* level count */
  uint32_t norm_q;     /* GQ_NORM_INF, 2, GQ_NORM_L2_SEQUENTIAL, or 1..16 (host step, see gq_norm) */
  uint32_t norm_p;     /* GQ_NORM_INF, 2, or 1..16 (host step) */
  uint32_t width_bits; /* requested lane width: 4, 8, 16 or 32 */
  uint32_t topo;       /* GQ_TOPO_* */
  uint32_t reserved;
  uint64_t seed;
} gq_config;

/* Result of plan_path (algorithm.cpp:40-67). */
typedef struct gq_plan {
  uint32_t lane_width; /* width actually used (dense standard may widen) */
  uint32_t shift;      /* prescale_shift(n) (exponential) */
  uint32_t m;          /* k truncation depth s+1 (exponential) */
  uint32_t max_e;      /* largest lane exponent (exponential) */
} gq_plan;

int gq_abi_version(void);

/* Process-wide launch options. The persistent quantize / reduce kernels size
 * their grid to fill every SM (one wave of resident CTAs); capping CTAs per SM
 * leaves room for kernels on a concurrent stream (e.g. the norm pass of the
 * next bucket). value 0 = automatic. */
#define GQ_OPT_QUANT_CTAS_PER_SM 1u
#define GQ_OPT_REDUCE_CTAS_PER_SM 2u
/* How a gq_comm waits for its peers (read at gq_comm_connect): 0 automatic
 * (host waits only when a peer shares this GPU), 1 always in a device kernel,
 * 2 always on the host. */
#define GQ_OPT_COMM_WAIT 3u
/* 1: launch quantize / reduce with programmatic dependent launch (their CTAs
 * may be scheduled while the previous kernel drains). Measured neutral inside
 * CUDA graphs (profiles/r1/variants.md); default 0. */
#define GQ_OPT_PDL 4u
/* Seconds a communicator waits for a peer before raising GQ_FLAG_P2P_TIMEOUT
 * (device waits) or returning GQ_ERR_RUNTIME (host waits). Default 60. */
#define GQ_OPT_COMM_TIMEOUT_S 5u
/* 1 (default): gq_mean_inproc / gq_graph_mean_inproc run small syncs
 * (n * d <= 2^23, f32, n in {2,4,8}, 4/8-bit lanes, tree, L-inf shard norms)
 * as one cooperative kernel with grid barriers instead of three launches;
 * results are bit-identical. 0: always the three-kernel path; 2: the fused
 * kernel up to n * d <= 2^24 (measurements). */
#define GQ_OPT_SMALL_PATH 6u
/* 1 (default): a communicator step folds its exchange steps into the
 * kernels (the norm pass stores the stats into the peers, the quantize /
 * reduce / decode wait for their inputs in their prologues and their last CTAs
 * raise the flags): four kernels per graph step. 0: every exchange step is a
 * kernel of its own (the fallback; read when a step is issued or captured). */
#define GQ_OPT_COMM_FOLD 7u
/* GQ_OPT_FUSED_PATH (0 default, 1 on): in-process syncs with all workers on
 * one device (f32, tree, n in {2,4,8}, 4/8-bit lanes, d a multiple of 256
 * lane words; tokens with the k-draw buffer) quantize, replay and decode tile
 * by tile in one kernel, so the per-worker lanes never round-trip through
 * HBM. Bit-identical, but measured 15-18 % slower than the separate TMA-staged
 * quantize and vectorised reduce kernels (C2 397 vs 336 us), so off. */
#define GQ_OPT_FUSED_PATH 8
int gq_set_option(uint32_t key, int64_t value);
const char* gq_last_error(void);

/* plan_path + standard_lane_width + ReduceContext::make admission
 * (algorithm.cpp:22-29,40-67; exp_arith.cpp:24-41,63-80). Host only.
 * Extension: width 4 is admitted when check_width(kind, s, n, 4) holds. */
int gq_plan_path(const gq_config* cfg, gq_plan* out);

/* Bytes of one worker's lane buffer: ceil(d * width / 8). */
uint64_t gq_lane_bytes(uint64_t d, uint32_t width);

/* ---- norm phase: local_norm_stat + norm_allreduce_inproc ----------------
 * Replaces gqsgd::local_norm_stat (norms.hpp:27, norms.cpp:52-62) for the n
 * shards in `shards` (host array of n device pointers, each d elements of
 * dtype), writing stats[r]. When `norm_out` is non-NULL the same launch also
 * folds the stats in the reference's tree order and applies the root
 * (norm_allreduce_inproc, collectives.cpp:210-233; combine_norm_stats,
 * norms.cpp:64-75). q in {2, GQ_NORM_L2_SEQUENTIAL, GQ_NORM_INF}, p in {2, GQ_NORM_INF}
 * run entirely on the stream; other orders (q or p in 1..16, as
 * norm_spec_from_string admits, norms.cpp:17-30) sum correctly rounded |x|^q
 * on the device, then synchronise the stream and take the root, the p-th
 * power and the fold on the host with the reference's libm (stats within
 * rounding of the reference's: its element-order sum of glibc pow values;
 * not graph-capturable, not on the communicator). `workspace` must hold
 * gq_norm_workspace_bytes(n, d) bytes and be zeroed once before first use
 * (the kernel leaves it reusable). */
size_t gq_norm_workspace_bytes(uint32_t n, uint64_t d);
int gq_norm(const void* const* shards, uint32_t dtype, uint32_t n, uint64_t d,
            uint32_t q, uint32_t p, double* stats, double* norm_out,
            void* workspace, uint32_t* err, void* stream);

/* Tree-order fold of n per-worker stats already on the device (e.g. after an
 * allgather across GPUs) into the global scale (collectives.cpp:210-233). */
int gq_norm_combine(const double* stats, uint32_t n, uint32_t q, uint32_t p,
                    double* norm_out, void* stream);

/* ---- compress: quantize_shard + encode -----------------------------------
 * Replaces gqsgd::quantize_shard (quantizer.hpp:38-40, quantizer.cpp:8-48)
 * followed by encode_dense_std (algorithm.cpp:69-82) or
 * pack_tokens(tokens_from_shard()) (exp_arith.cpp:126-160): for each of the
 * n_local shards, worker id worker_ids[i] (host array), writes the lane
 * buffer lanes_out[i] (gq_lane_bytes(d, width) bytes). The dither of element
 * j is u01(Dither, worker, round, j) exactly as rng.hpp:45-61; `norm` is a
 * device scalar (the exchanged global scale). n_total is the worker count
 * of the whole job (the exponential prescale depends on it). */
int gq_quantize(const void* const* shards, uint32_t dtype, uint32_t n_local,
                const uint32_t* worker_ids, uint64_t d, const double* norm,
                uint32_t kind, uint32_t s, uint32_t n_total, uint32_t width,
                uint64_t seed, uint64_t round, void* const* lanes_out,
                uint32_t* err, void* stream);

/* ---- aggregate: allreduce_inproc with IntSumOps / TokenReduceOps ----------
 * Replaces allreduce_inproc (collectives.hpp:111-113, collectives.cpp:155-190)
 * driving the PayloadOps plugin IntSumOps (collectives.cpp:60-81, kind 0) or
 * TokenReduceOps (collectives.cpp:125-153, kind 1) over the tree or ring
 * schedule (topology.cpp:19-72). worker_lanes is a host array of n device
 * pointers (local or peer-mapped), each a full lane buffer of d lanes. The
 * call evaluates the schedule for lanes [lane_begin, lane_end) and writes the
 * result every worker would hold. k draws are keyed
 * (round, step<<32|dst, lane) as collectives.cpp:132-146.
 * Optional fused epilogues on the same lane range (NULL to skip):
 *   out_lanes: result lanes;
 *   out_mean : decoded mean as fp32 (decode_dense_std / decode_dense_exp,
 *              algorithm.cpp:84-110, computed in f64 then rounded);
 *   param    : param[j] -= lr * mean[j] (the SGD step, trainer.cpp:335).
 * lane_begin must be a multiple of 32/width. `norm` is needed only for the
 * decode epilogues. */
int gq_reduce_lanes(const void* const* worker_lanes, uint32_t n, uint64_t d,
                    uint64_t lane_begin, uint64_t lane_end, uint32_t kind,
                    uint32_t width, uint32_t s, uint32_t topo, uint64_t seed,
                    uint64_t round, const double* norm, void* out_lanes,
                    float* out_mean, float* param, float lr, uint32_t* err,
                    void* stream);

/* gq_reduce_lanes on one slice [lane_begin, lane_end) where worker_slices[i]
 * (and out_slice / out_mean_slice / param_slice) point at lane lane_begin
 * rather than lane 0: the layout the multi-GPU reduce-scatter-by-pull
 * delivers. k draws and ring chunks still use the global lane
 * index and the full d, so the result equals the same lanes of
 * allreduce_inproc (collectives.cpp:155-190). lane_begin must be a multiple
 * of 4 lanes and of 16 bytes of lanes. */
int gq_reduce_slice(const void* const* worker_slices, uint32_t n, uint64_t d,
                    uint64_t lane_begin, uint64_t lane_end, uint32_t kind,
                    uint32_t width, uint32_t s, uint32_t topo, uint64_t seed,
                    uint64_t round, const double* norm, void* out_slice,
                    float* out_mean_slice, float* param_slice, float lr,
                    uint32_t* err, void* stream);

/* The PayloadOps plugin itself (collectives.hpp:39-48): acc = acc (+) in for
 * one schedule event (step, dst) on `lanes` device lanes whose first lane has
 * global index elem_offset - IntSumOps::combine (collectives.cpp:60-81, kind
 * 0, overflow -> GQ_FLAG_LANE_OVERFLOW) or TokenReduceOps::combine
 * (collectives.cpp:125-153, kind 1, k keyed (round, step<<32|dst, lane)).
 * acc/in may start at any byte; 4-bit lanes need an even elem_offset. n is
 * the job's worker count (token admission, exp_arith.cpp:24-41). */
int gq_combine_lanes(void* acc, const void* in, uint64_t lanes, uint64_t elem_offset,
                     uint32_t kind, uint32_t width, uint32_t s, uint32_t n,
                     uint64_t seed, uint64_t round, uint32_t step, uint32_t dst,
                     uint32_t* err, void* stream);

/* Device counter RNG, for known-answer tests of the hot-loop hash forms
 * (rng.hpp:45-61, exp_arith.cpp:43-50). For i < count, c = c0 + i:
 *   bits_out[i] = bits(stream, a, b, c)   (the generic device mix64 chain);
 *   hi_out[i]   = the 32-bit word the hot loops derive from it - hi32 of the
 *                 state before mix64's last xor-shift, through the
 *                 group-shared form quantize / the token reduce use (so
 *                 bits >> 32 == hi ^ (hi >> 31), bits >> 41 == hi >> 9);
 *   k_out[i]    = sample_k(u01(stream, a, b, c), m) as the token reduce
 *                 computes it: m <= 32 through the 8-bit packed k word of the
 *                 SWAR path, m > 32 through the 64-bit sample_k_bits.
 * With bits_in non-NULL, k_out[i] = sample_k_bits(bits_in[i], m) instead (the
 * u -> k map of exp_arith.cpp:43-50 on chosen bit patterns). Any output may be
 * NULL. Test infrastructure for the device RNG; not on the sync path. */
int gq_rng_draws(uint64_t seed, uint64_t stream_id, uint64_t a, uint64_t b, uint64_t c0, uint64_t count,
                 uint32_t m, const uint64_t* bits_in, uint64_t* bits_out, uint32_t* hi_out, uint32_t* k_out,
                 void* stream);

/* ---- precomputed k draws (exponential tree path) -----------------------------
 * The TokenReduceOps k draws (collectives.cpp:132-146) depend only on (seed,
 * round, step, dst, lane), not on the data. gq_norm_kdraws runs the norm pass
 * (HBM-bound, integer pipes idle) and in the same launch fills spec->buf with
 * the packed k words of every tree event for lanes [lane_begin, lane_end);
 * gq_reduce_lanes_kdraws then reads them instead of hashing, which makes the
 * token reduce memory-bound. Applies to the exponential kind, width 4 or 8,
 * tree topology, n in {2, 4, 8}, s <= 31; gq_kdraws_bytes returns 0 otherwise
 * (callers fall back to gq_norm / gq_reduce_lanes). Results are identical. */
typedef struct gq_kdraws {
  uint32_t* buf;          /* gq_kdraws_bytes(spec) bytes of device memory */
  uint32_t n;             /* schedule workers */
  uint32_t kind, width, s, topo;
  uint32_t reserved;
  uint64_t lane_begin, lane_end;
  uint64_t seed, round;
} gq_kdraws;
size_t gq_kdraws_bytes(const gq_kdraws* spec);
int gq_norm_kdraws(const void* const* shards, uint32_t dtype, uint32_t n, uint64_t d, uint32_t q,
                   uint32_t p, double* stats, double* norm_out, void* workspace, uint32_t* err,
                   const gq_kdraws* spec, void* stream);
int gq_reduce_lanes_kdraws(const void* const* worker_lanes, uint32_t n, uint64_t d, uint64_t lane_begin,
                           uint64_t lane_end, uint32_t kind, uint32_t width, uint32_t s, uint32_t topo,
                           uint64_t seed, uint64_t round, const double* norm, void* out_lanes,
                           float* out_mean, float* param, float lr, uint32_t* err,
                           const gq_kdraws* spec, void* stream);

/* ---- peer-memory exchange (fused collectives over NVLink / NVSwitch) --------
 * One worker per GPU, N <= 16 GPUs of one node, buffers mapped into every
 * peer with gq_ipc_get / gq_ipc_open (cudaIpc*). The lane exchange of
 * DESIGN.md §5 without NCCL:
 *   gq_quantize_scatter      quantize_shard whose lane stores go straight to
 *                            the owner of each slice (slice j of this worker ->
 *                            slice_dst[j], typically peer j's receive row for
 *                            this rank): the all_to_all fused into the quantizer;
 *   gq_p2p_signal / _wait    epoch flags with system-scope release / acquire;
 *   gq_reduce_slice_multicast the schedule replay of this rank's slice
 *                            (as gq_reduce_slice) storing the summed lanes into
 *                            every peer's summed buffer: the all_gather fused
 *                            into the reduce epilogue.
 * slice_lanes must be a multiple of 512 lanes (1024 lets large launches take
 * the quantizer's 4 KiB chunks; gq_comm cuts its slices so). */
int gq_quantize_scatter(const void* shard, uint32_t dtype, uint32_t worker, uint64_t d,
                        const double* norm, uint32_t kind, uint32_t s, uint32_t n_total,
                        uint32_t width, uint64_t seed, uint64_t round, void* const* slice_dst,
                        uint32_t nslices, uint64_t slice_lanes, uint32_t* err, void* stream);
int gq_reduce_slice_multicast(const void* const* worker_slices, uint32_t n, uint64_t d,
                              uint64_t lane_begin, uint64_t lane_end, uint32_t kind, uint32_t width,
                              uint32_t s, uint32_t topo, uint64_t seed, uint64_t round,
                              void* const* out_slices, uint32_t nout, uint32_t* err, void* stream);
int gq_p2p_signal(uint32_t* const* peer_slots, uint32_t n, uint32_t epoch, void* stream);
int gq_p2p_wait(const uint32_t* flags, uint32_t n, uint32_t epoch, uint32_t* err, void* stream);
size_t gq_ipc_handle_bytes(void);
int gq_ipc_get(void* ptr, void* handle_out);
int gq_ipc_open(const void* handle, void** ptr_out);
int gq_ipc_close(void* ptr);

/* ---- communicator: the multi-rank path (one rank per process or thread) -----
 * Replaces the reference's worker mesh - PeerSockets / connect_mesh /
 * run_local_mesh (transport.hpp:38-58, transport.cpp:289-330) - and the two
 * exchanges of gqsgd_mean_worker (algorithm.cpp:230-301) with peer memory over
 * NVLink / NVSwitch (CUDA IPC), no NCCL and no host round trip on the data
 * path. A gq_comm is bound to one dense configuration and d; rank r hosts the
 * workers [r*n/nranks, (r+1)*n/nranks). Bootstrap like an NCCL unique id:
 *   gq_comm_init  -> gq_comm_handle (this rank's gq_comm_handle_bytes() blob)
 *   -> the caller all-gathers the blobs out of band (sockets, torch.distributed,
 *   MPI) -> gq_comm_connect(all blobs, rank order).
 * Ranks of one process share pointers directly; ranks on the same GPU (tests)
 * wait on the host instead of in a spinning kernel. Per step, on one stream:
 *   gq_norm (stats of the local workers) -> gq_norm_exchange -> gq_comm_quantize
 *   -> gq_allreduce_lanes -> gq_dequant(gq_comm_summed) ; or gq_comm_mean for all
 * of it. A peer that never arrives raises GQ_FLAG_P2P_TIMEOUT instead of hanging. */
typedef struct gq_comm gq_comm;
typedef struct gq_comm_info {
  uint32_t lane_width;   /* plan.lane_width */
  uint32_t n_local;      /* workers on this rank */
  uint32_t worker_begin; /* first (global) worker id of this rank */
  uint32_t host_wait;    /* 1 when some peer shares this GPU */
  uint64_t slice_lanes;  /* lanes per owner slice (multiple of 1024) */
  uint64_t lane_begin, lane_end; /* the slice this rank reduces */
  int32_t device;        /* CUDA device the communicator's buffers live on */
  uint32_t reserved;
} gq_comm_info;
size_t gq_comm_handle_bytes(void);
int gq_comm_init(uint32_t rank, uint32_t nranks, const gq_config* cfg, uint64_t d, gq_comm** out);
int gq_comm_handle(const gq_comm* c, void* handle_out);
int gq_comm_connect(gq_comm* c, const void* handles);
int gq_comm_info_get(const gq_comm* c, gq_comm_info* out);
int gq_comm_destroy(gq_comm* c);
/* norm_allreduce over the mesh (algorithm.cpp:247-263): stats_local holds the
 * n_local device stats of gq_norm; every rank gets the tree-folded global
 * scale in *norm_out (device). */
int gq_norm_exchange(gq_comm* c, const double* stats_local, double* norm_out, uint32_t* err, void* stream);
/* gq_norm of the n_local shards (host array) + gq_norm_exchange into
 * *norm_out (device; NULL = the communicator's own scalar). For exponential
 * tree configurations the same pass precomputes the TokenReduceOps k draws of
 * this rank's slice for `round`, which gq_allreduce_lanes of that round then
 * reads instead of hashing (gq_norm_kdraws). */
int gq_comm_norm(gq_comm* c, const void* const* shards, uint32_t dtype, uint64_t round, double* norm_out,
                 uint32_t* err, void* stream);
/* quantize_shard of the n_local shards (host array) with the lane slices
 * stored straight into their owners' receive rows. */
int gq_comm_quantize(gq_comm* c, const void* const* shards, uint32_t dtype, const double* norm,
                     uint64_t round, uint32_t* err, void* stream);
/* The lane allreduce (run_allreduce_worker with IntSumOps / TokenReduceOps,
 * transport.cpp:232-287): lanes = host array of n_local lane buffers to send,
 * or NULL when gq_comm_quantize already delivered them. Every rank ends with
 * the summed lanes in gq_comm_summed(c) (and in summed_out when non-NULL,
 * gq_lane_bytes(d, width) bytes). */
int gq_allreduce_lanes(gq_comm* c, const void* const* lanes, uint64_t round, void* summed_out,
                       uint32_t* err, void* stream);
const void* gq_comm_summed(const gq_comm* c);
/* gqsgd_mean_worker for this rank's workers: norm -> exchange -> quantize ->
 * allreduce -> decode into mean_out (fp32, optional) and/or mean64_out (f64,
 * the reference's doubles, optional), + param -= lr * mean when param given. */
int gq_comm_mean(gq_comm* c, const void* const* shards, uint32_t dtype, uint64_t round, float* mean_out,
                 double* mean64_out, float* param, float lr, double* norm_out, uint32_t* err, void* stream);
/* gq_comm_mean on fixed buffers captured as one CUDA graph (run it with
 * gq_graph_launch, free it with gq_graph_destroy): each replay is one step
 * with the round read from *round_dev (then += round_step, 0 meaning 1: a
 * bucketed step numbers bucket b of step t as t*buckets + b) and the flag epochs kept on
 * the device - no host work per step. Every rank replays the same number of
 * times. Needs device-side waits (ranks on distinct GPUs, or GQ_OPT_COMM_WAIT
 * = 1). gq_graph is declared with gq_graph_mean_inproc below. */
typedef struct gq_graph gq_graph;
int gq_comm_graph(gq_comm* c, const void* const* shards, uint32_t dtype, float* mean_out, double* mean64_out,
                  float* param, float lr, uint64_t* round_dev, uint64_t round_step, uint32_t* err,
                  gq_graph** out);
/* gq_check across the mesh: every rank's error word is OR-ed and mapped to
 * one status, identical on all ranks (the reference raises on every worker). */
int gq_sync(gq_comm* c, uint32_t* err, void* stream);

/* ---- decompress ------------------------------------------------------------
 * Replaces decode_dense_std / decode_dense_exp (algorithm.cpp:84-110) on
 * already-aggregated lanes [lane_begin, lane_end) of `lanes`, with the same
 * optional fused SGD step as gq_reduce_lanes. */
int gq_dequant(const void* lanes, uint64_t lane_begin, uint64_t lane_end,
               const double* norm, uint32_t kind, uint32_t s, uint32_t n,
               uint32_t width, float* out, float* param, float lr,
               uint32_t* err, void* stream);

/* decode_dense_std / decode_dense_exp (algorithm.cpp:84-110) into f64,
 * bit-identical to the reference's doubles (used by the C++ drop-in, whose
 * MeanResult carries doubles). out[0] is lane lane_begin. */
int gq_dequant_f64(const void* lanes, uint64_t lane_begin, uint64_t lane_end,
                   const double* norm, uint32_t kind, uint32_t s, uint32_t n,
                   uint32_t width, double* out, uint32_t* err, void* stream);

/* Device memory plumbing for bindings that do not link the CUDA runtime. */
int gq_malloc(size_t bytes, void** out);
int gq_free(void* p);
int gq_malloc_host(size_t bytes, void** out); /* pinned host memory */
int gq_free_host(void* p);
int gq_memcpy(void* dst, const void* src, size_t bytes, void* stream); /* any direction */
int gq_memset(void* dst, int value, size_t bytes, void* stream);
int gq_stream_sync(void* stream);

/* ---- the sparse allgather path (cfg.sparse) ---------------------------------
 * gq_sparse_encode: serialize_sparse(to_sparse(shard)) (serialize.cpp:156-168,
 * quantizer.cpp:59-71) of one worker whose quantized lanes come from
 * gq_quantize at width 32 (n_total as passed there; it fixes the exponential
 * lane offset). width is the level lane width (validate_level_width,
 * serialize.cpp:114-122). payload must hold gq_sparse_payload_bytes(d, width)
 * bytes; the actual size is 16 + 4 nnz + ceil(nnz/8) + nnz*width/8 with nnz
 * written to the device word *nnz_out. workspace: gq_sparse_workspace_bytes(d). */
uint64_t gq_sparse_payload_bytes(uint64_t nnz, uint32_t width);
size_t gq_sparse_workspace_bytes(uint64_t d);
int gq_sparse_encode(const void* lanes32, uint64_t d, uint32_t kind, uint32_t s, uint32_t n_total,
                     uint32_t width, const double* norm, void* payload, void* workspace,
                     uint32_t* nnz_out, void* stream);

/* accumulate_sparse + decode_sparse_set (quantizer.cpp:92-110,
 * algorithm.cpp:112-123) for n workers held on this device (their width-32
 * lanes): mean = (sum over workers in rank order of (norm*sign)*level) / n,
 * into out32 (fp32) and/or out64 (f64). */
int gq_sparse_mean_inproc(const void* const* lanes32, uint32_t n, uint64_t d, uint32_t kind,
                          uint32_t s, uint32_t n_total, const double* norm, float* out32,
                          double* out64, void* stream);

/* One received payload (deserialize_sparse checks, accumulate_sparse) added
 * into the f64 accumulator acc[d]; call in rank order, then gq_sparse_finish.
 * Malformed payloads raise GQ_FLAG_BAD_PAYLOAD. */
int gq_sparse_accumulate(const void* payload, uint64_t payload_bytes, uint32_t kind, uint32_t s,
                         uint32_t width, uint64_t d, double* acc, uint32_t* err, void* stream);
int gq_sparse_finish(const double* acc, uint64_t d, uint32_t n, float* out32, double* out64,
                     float* param, float lr, void* stream);  /* param -= lr * mean (optional) */

/* ---- whole path (one device, n simulated workers) ---------------------------
 * Replaces gqsgd::gqsgd_mean with Transport::Inproc (algorithm.hpp:56,
 * algorithm.cpp:127-228) for the dense paths: norm -> quantize -> schedule
 * replay -> decode (+SGD). lane_bufs: host array of cfg->workers device
 * buffers of gq_lane_bytes(d, plan.lane_width) bytes each (the per-worker
 * communication buffers). result_lanes / mean_out / param may be NULL.
 * stats_out (n doubles) and norm_out (1 double) are device outputs.
 * workspace: gq_norm_workspace_bytes(cfg->workers, d) bytes. */
int gq_mean_inproc(const void* const* shards, uint32_t dtype, uint64_t d,
                   const gq_config* cfg, uint64_t round,
                   void* const* lane_bufs, void* result_lanes, float* mean_out,
                   float* param, float lr, double* stats_out,
                   double* norm_out, void* workspace, uint32_t* err,
                   void* stream);

/* The whole in-process path captured once as a CUDA graph for fixed buffers:
 * norm (+ the k draws when gq_kdraws applies and kdraws_buf is given,
 * gq_kdraws_bytes bytes) -> quantize -> reduce/decode (+ SGD), whose last
 * block does *round_dev += 1 (three kernels per replay; the workspace header
 * holds its ticket). The kernels read the round from round_dev (a device uint64 the
 * caller initialises), so each gq_graph_launch is one gqsgd_mean call with
 * the next round at the cost of a single launch - for small d, where the
 * per-kernel launch latency would dominate. Same results as gq_mean_inproc. */
typedef struct gq_graph gq_graph;
int gq_graph_mean_inproc(const void* const* shards, uint32_t dtype, uint64_t d, const gq_config* cfg,
                         uint64_t* round_dev, void* const* lane_bufs, void* result_lanes, float* mean_out,
                         float* param, float lr, double* stats_out, double* norm_out, void* workspace,
                         uint32_t* kdraws_buf, uint32_t* err, gq_graph** out);
int gq_graph_launch(gq_graph* g, void* stream);
int gq_graph_destroy(gq_graph* g);

/* Uncompressed fp32 reference path on one device (baseline_mean,
 * algorithm.cpp:303-340): tree-order fp32 sum of n shards, then /n. */
int gq_baseline_mean_inproc(const float* const* shards, uint32_t n, uint64_t d,
                            uint32_t topo, float* mean_out, void* stream);

/* Synchronise `stream`, read and clear the device error word, and map any
 * raised flag to a status (+ gq_last_error message). */
int gq_check(uint32_t* err, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GQ_B200_H */
