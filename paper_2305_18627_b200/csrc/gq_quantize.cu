// Compress: quantize_shard + lane encoding, written straight into the
// per-worker communication buffer.
//
//   reference: quantizer.cpp:8-48 (quantize_shard), levels.cpp:63-84
//              (bracket_index / random_round), rng.hpp:45-61 (dither
//              u01(Dither, worker, round, j)), algorithm.cpp:69-82
//              (encode_dense_std: lane = sign * (s - idx)),
//              exp_arith.cpp:126-160 (tokens_from_shard + pack_tokens:
//              lane = (idx + shift) | sign bit, idx == s -> 0).
//
// Bit-exactness strategy. The reference decides each element with IEEE f64
// arithmetic: y = |x|/norm, bracket by comparison with the level table,
// p = (y - lo)/(hi - lo), round up iff u < p. Two correctly rounded f64
// divisions per element would make this kernel FP64-bound, so each element
// first takes an f32 FAST PATH that computes an approximation of the
// fractional position f ~ p with a proven error bound M:
//   standard    t = |x| * fl32(s/norm), f = t - floor(t), |f - p| < M
//               with M = (s+1) 2^-21 (f32 product error s*2^-23 dominates)
//   exponential y = |x| * fl32(1/norm), bracket from the f32 exponent,
//               f = mantissa fraction (or y 2^(s-1) in the last bracket),
//               |f - p| < M = 2^-20
// and a 23-bit truncation uf <= u < uf + 2^-23 of the dither. The element
// rounds up iff uf + M + 2^-23 <= f, down iff uf >= f + M, and any element
// within M of a bracket edge or of the decision boundary (probability
// ~4M, <1e-4) falls to the SLOW PATH, which replays the reference's f64
// sequence literally (__ddiv_rn / __dsub_rn, exact level values), so every
// decision equals the reference's.
//
// Memory: thread-per-quad (4 elements) with 128-bit streaming loads; each
// quad emits 4 lanes (2/4/8/16 bytes for w = 4/8/16/32) with one coalesced
// store. HBM bytes per element: 4 (f32 in) + w/8 (lanes out).
#include <cuda_runtime.h>

#include "gq_common.cuh"
#include "gq_internal.h"
#include "gq_quant_dev.cuh"

namespace gqb {

int g_quant_ctas_per_sm = 0;


namespace {

#ifndef GQ_QMIN_CHUNKS
#define GQ_QMIN_CHUNKS 4  // staged chunks per warp at least (small d: fewer, fuller CTAs)
#endif

// Folded norm exchange (gq_comm graphs): thread 0 of every CTA waits for all
// ranks' stats flags, then folds the n stats in the reference's tree order
// (collectives.cpp:210-233, norms.cpp:64-75) - every CTA gets the identical
// norm; CTA 0 also stores it for the decode.
__device__ __noinline__ double wait_and_fold_norm(const PeerWait& pw, const StatsFold& f, uint32_t* err) {
  __shared__ double s_st[kMaxWorkers];
  __shared__ double s_norm;
  if (threadIdx.x == 0) {
    peer_wait_flags(pw.flags, pw.n, pw.ep_dev ? *pw.ep_dev : pw.epoch, err, pw.timeout_ns);
    for (uint32_t w = 0; w < f.n; ++w) s_st[w] = __ldcv(f.stats + w);  // peers' stores, not a stale L1 line
    const double nm = tree_fold_stats(s_st, f.n, f.p);
    s_norm = nm;
    if (blockIdx.x == 0 && f.norm_out) *f.norm_out = nm;
  }
  __syncthreads();
  return s_norm;
}

#ifndef GQ_QINNER  // quads of a lane's chunk interleaved by the compiler (0: all U)
#define GQ_QINNER 0
#endif
// U: quads per lane per staged chunk, ST: stages per warp (see launch_w).
template <typename T, int KIND, int W, int U, int ST>
__global__ void __launch_bounds__(kQThreads, GQ_QMINBLOCKS)
quantize_kernel(const __grid_constant__ QuantArgs args) {
  constexpr int kWq = 32 * U;  // quads per warp chunk
  constexpr int kQInner = GQ_QINNER > 0 && GQ_QINNER < U ? GQ_QINNER : U;
  constexpr uint32_t kHiMask = static_cast<uint32_t>((1ull << 32) / (4ull * kWq)) - 1u;
  pdl_wait();     // the norm (and the previous step) are complete and visible
  pdl_trigger();  // the reduce may take SM slots as this grid's CTAs retire
  const uint64_t d = args.d;
  const uint32_t s = args.s;
  const uint32_t shift = args.shift;
  const uint32_t nl = args.n_local;
  const double norm = args.pw.n ? wait_and_fold_norm(args.pw, args.fold, args.err) : *args.norm;
  uint32_t flags = 0;
  const uint64_t nquad = d / 4;

  if (!(norm >= 0.0) || !isfinite(norm)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_flag(args.err, GQ_FLAG_BAD_SCALE);
    grid_done_signal(args.sig);  // peers must not wait for the timeout: the error travels via gq_sync
    return;
  }
  if (norm == 0.0) {
    // quantizer.cpp:21-32: every element must be zero; all idx = s (lane 0).
    const uint64_t total = nquad * nl;
    for (uint64_t g = blockIdx.x * static_cast<uint64_t>(kQThreads) + threadIdx.x; g < total;
         g += static_cast<uint64_t>(gridDim.x) * kQThreads) {
      const uint32_t r = static_cast<uint32_t>(g / nquad);
      const uint64_t q = g - r * nquad;
      T v[4];
      load_quad<T>(static_cast<const T*>(args.x[r]), q, v);
#pragma unroll
      for (int e = 0; e < 4; ++e) if (v[e] != T(0)) flags |= GQ_FLAG_ZERO_SCALE;
      const int32_t c[4] = {0, 0, 0, 0};
      store_quad<W>(lane_base_for<W>(args, r, q), q, c);
    }
    if (threadIdx.x == 0) {
      for (uint32_t r = blockIdx.x; r < nl; r += gridDim.x) {
        const T* x = static_cast<const T*>(args.x[r]);
        for (uint64_t j = nquad * 4; j < d; ++j) if (x[j] != T(0)) flags |= GQ_FLAG_ZERO_SCALE;
        uint8_t* lb = static_cast<uint8_t*>(lane_base_for<W>(args, r, nquad));
        const uint64_t b0 = nquad * 4 * W / 8, b1 = (d * W + 7) / 8;
        for (uint64_t bb = b0; bb < b1; ++bb) lb[bb] = 0;
      }
    }
    raise_flags_warp(args.err, flags);
    grid_done_signal(args.sig);
    return;
  }

  const QConst K = make_const<KIND>(norm, s, shift);
  const MulConsts MK = args.mk;
  __shared__ uint8_t s_qtab[kUseQtab<KIND, W> ? kQtabBytes<KIND> : 4];
  if constexpr (kUseQtab<KIND, W> && KIND == 1) build_exp_tab<W>(s_qtab, s, shift);
  else if constexpr (kUseQtab<KIND, W>) build_std_tab<W>(s_qtab, s, K.cm);
  // per-worker RNG prefixes mix64^4(seed, Dither, worker, round): from the
  // launch (host-computed) or, in graph replays, from the device round
  __shared__ uint64_t s_h4[kMaxWorkers];
  for (uint32_t i = threadIdx.x; i < nl; i += kQThreads)
    s_h4[i] = args.round_ptr ? hoist_prefix(args.seed, 1ull, args.wid[i], *args.round_ptr) : args.h4[i];
  __syncthreads();

  // ---- per-warp TMA bulk-copy pipelines over a global list of (worker, chunk) pairs ----
  // Warp w owns global warp-chunks [g0, g0 + cnt) (kWq quads each). Its
  // lane 0 issues one 1-D bulk copy per chunk into one of the warp's kStages
  // shared-memory stages (cp.async.bulk, completion on the stage's mbarrier);
  // the warp waits on the mbarrier, quantizes U quads per lane from
  // shared memory, stores its lanes, and lane 0 refills the stage after a
  // __syncwarp. No block-wide barrier: a warp delayed by a slow-path element
  // never stalls the others.
  extern __shared__ __align__(128) uint8_t qsmem[];
  constexpr uint32_t kChunkB = kWq * 4 * sizeof(T);
  constexpr int kStages = ST;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // all warps' stage buffers first (each 128-byte aligned), then the mbarriers
  uint8_t* wsm = qsmem + warp * (kStages * kChunkB);
  uint64_t* bars = reinterpret_cast<uint64_t*>(qsmem + (kQThreads / 32) * kStages * kChunkB) + warp * kStages;
  // Chunk cursors are 32-bit (d < 2^41) and advance incrementally: no
  // division in the loop. The chunk-shared hash constants depend only on the
  // worker's prefix and the high word of the element index, so they are
  // rebuilt when the worker changes or j crosses a multiple of 2^32.
  const uint32_t nch = static_cast<uint32_t>(nquad / kWq);
  const uint64_t gtotal = static_cast<uint64_t>(nch) * nl;
  const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * (kQThreads / 32);
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * (kQThreads / 32) + warp;
  const uint64_t per = (gtotal + nwarps - 1) / nwarps;
  const uint64_t g0 = min(gtotal, per * gw);
  const uint32_t cnt = static_cast<uint32_t>(min(gtotal, g0 + per) - g0);
  uint32_t r = nch ? static_cast<uint32_t>(g0 / nch) : 0;
  uint32_t cidx = static_cast<uint32_t>(g0 - static_cast<uint64_t>(r) * nch);
  auto chunk_src = [&](uint32_t wr, uint32_t c) -> const T* {
    return static_cast<const T*>(args.x[wr]) + static_cast<uint64_t>(c) * (kWq * 4);
  };
  uint32_t pr = r, pc = cidx;  // producer cursor (lane 0): the next chunk to load
  if (lane == 0) {
#pragma unroll
    for (int st = 0; st < kStages; ++st) mbar_init(&bars[st], 1);
    mbar_fence_init();
    for (uint32_t k = 0; k < static_cast<uint32_t>(kStages) && k < cnt; ++k) {
      mbar_expect_tx(&bars[k], kChunkB);
      bulk_g2s(wsm + k * kChunkB, chunk_src(pr, pc), kChunkB, &bars[k]);
      if (++pc == nch) { pc = 0; ++pr; }
    }
  }
  __syncwarp();
  uint64_t h4 = 0;
  void* lanes = nullptr;
  ChunkMix cm{};
  uint64_t slice_end = 0;  // scatter mode: first quad past the current slice
  uint32_t slice_j = 0;
  for (uint32_t k = 0; k < cnt; ++k) {
    const int st = static_cast<int>(k % kStages);
    const uint64_t qbase = static_cast<uint64_t>(cidx) * kWq;
    if (k == 0 || (cidx & kHiMask) == 0) {  // new worker, or a new 2^32 block of j
      h4 = s_h4[r];
      cm = chunk_mix(h4, 4 * qbase);
      if (args.nslices) {
        slice_j = static_cast<uint32_t>(min(qbase / args.slice_quads, static_cast<uint64_t>(args.nslices - 1)));
        slice_end = (slice_j + 1 == args.nslices) ? ~0ull : (slice_j + 1) * args.slice_quads;
        lanes = lane_base_for<W>(args, r, qbase);
      } else {
        lanes = args.lanes[r];
      }
    } else if (args.nslices && qbase >= slice_end) {  // chunks never straddle slices
      ++slice_j;
      slice_end = (slice_j + 1 == args.nslices) ? ~0ull : (slice_j + 1) * args.slice_quads;
      lanes = lane_base_for<W>(args, r, qbase);
    }
    mbar_wait(&bars[st], (k / kStages) & 1u);
    const T* src = reinterpret_cast<const T*>(wsm + st * kChunkB);
    if constexpr (sizeof(T) == 4) {
      bool any = !K.fast;
#pragma unroll kQInner
      for (int u = 0; u < U; ++u) {
        const int ql = u * 32 + lane;
        const float4 f = reinterpret_cast<const float4*>(src)[ql];
        const float v[4] = {f.x, f.y, f.z, f.w};
        int32_t c[4];
        fast_quad<KIND, W>(v, cm, static_cast<uint32_t>(4 * (qbase + ql)), K, MK, s, shift, s_qtab, any, c);
#ifndef GQ_QPACK_MAD  // 0: pack the table lanes with shifts / ors (ALU) instead of multiply-adds
#define GQ_QPACK_MAD 1
#endif
        if constexpr (kUseQtab<KIND, W> && GQ_QPACK_MAD) store_quad_mad<W>(lanes, qbase + ql, c, args.pk);
        else store_quad<W, KIND == 1>(lanes, qbase + ql, c);
      }
      if (__builtin_expect(any, 0)) {  // exact handling of this lane's quads, stored over the fast ones
#pragma unroll 1
        for (int u = 0; u < U; ++u) {
          const int ql = u * 32 + lane;
          const float4 f = reinterpret_cast<const float4*>(src)[ql];
          const T v[4] = {f.x, f.y, f.z, f.w};
          int32_t c[4];
          quant_quad<KIND, W, T>(v, 4, h4, cm, 4 * (qbase + ql), K, MK, s, shift, flags, c);
          store_quad<W, KIND == 1>(lanes, qbase + ql, c);
        }
      }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int ql = u * 32 + lane;
        const double2 a0 = reinterpret_cast<const double2*>(src)[2 * ql];
        const double2 a1 = reinterpret_cast<const double2*>(src)[2 * ql + 1];
        const T v[4] = {a0.x, a0.y, a1.x, a1.y};
        int32_t c[4];
        quant_quad<KIND, W, T>(v, 4, h4, cm, 4 * (qbase + ql), K, MK, s, shift, flags, c);
        store_quad<W, KIND == 1>(lanes, qbase + ql, c);
      }
    }
    __syncwarp();  // every lane is done with stage st
    if (lane == 0 && k + kStages < cnt) {
      mbar_expect_tx(&bars[st], kChunkB);
      bulk_g2s(wsm + st * kChunkB, chunk_src(pr, pc), kChunkB, &bars[st]);
      if (++pc == nch) { pc = 0; ++pr; }
    }
    if (++cidx == nch) {
      cidx = 0;
      ++r;
    }
  }

  // ---- per-worker remainder: quads past the last whole chunk + tail ----
  for (uint32_t r = blockIdx.x; r < nl; r += gridDim.x) {
    const T* x = static_cast<const T*>(args.x[r]);
    const uint64_t h4 = s_h4[r];
    for (uint64_t q = nch * kWq + threadIdx.x; q < nquad; q += kQThreads) {
      T v[4];
      load_quad<T>(x, q, v);
      int32_t c[4];
      quant_quad<KIND, W, T>(v, 4, h4, chunk_mix(h4, 4 * q), 4 * q, K, MK, s, shift, flags, c);
      store_quad<W>(lane_base_for<W>(args, r, q), q, c);
    }
    // d % 4 tail elements: one thread writes whole bytes, zero-padded
    if (threadIdx.x == 0 && nquad * 4 < d) {
      int32_t c[4] = {0, 0, 0, 0};
      T tv[4] = {T(0), T(0), T(0), T(0)};
      const int tc = static_cast<int>(d - nquad * 4);
      for (int e = 0; e < tc; ++e) tv[e] = x[nquad * 4 + e];
      quant_quad<KIND, W, T>(tv, tc, h4, chunk_mix(h4, nquad * 4), nquad * 4, K, MK, s, shift, flags, c);
      uint8_t* lb = static_cast<uint8_t*>(lane_base_for<W>(args, r, nquad));
      const uint64_t b0 = nquad * 4 * W / 8;
      const uint64_t nb = ((d - nquad * 4) * W + 7) / 8;
      uint64_t packed[2] = {0, 0};
      for (int e = 0; e < 4; ++e) {
        const uint64_t mask = (W == 64) ? ~0ull : ((1ull << W) - 1);
        const uint64_t bitpos = static_cast<uint64_t>(e) * W;
        const uint64_t val = static_cast<uint64_t>(static_cast<uint32_t>(c[e])) & mask;
        packed[bitpos / 64] |= val << (bitpos % 64);
      }
      for (uint64_t bb = 0; bb < nb; ++bb) lb[b0 + bb] = static_cast<uint8_t>(packed[bb / 8] >> (8 * (bb % 8)));
    }
  }
  raise_flags_warp(args.err, flags);
  grid_done_signal(args.sig);
}

// 64-bit standard lanes (standard_lane_width, algorithm.cpp:22-29: the
// reference moves to int64 lanes when n(s+1) > 2^31, or when 64 bits are
// asked for). Every element takes the reference's f64 decision (slow_index:
// the f32 fast path needs s < 2^14, and s may be up to 2^32 - 1 here), the
// lane is sign * (s - idx) as a little-endian int64 (encode_dense_std,
// algorithm.cpp:69-82). One quad (32 lane bytes) per thread iteration; scatter
// mode and the grid-completion signal work as in quantize_kernel.
template <typename T>
__global__ void __launch_bounds__(kQThreads)
quantize64_kernel(const __grid_constant__ QuantArgs args) {
  pdl_wait();
  pdl_trigger();
  const uint64_t d = args.d;
  const uint32_t s = args.s;
  const uint32_t nl = args.n_local;
  const double norm = *args.norm;
  uint32_t flags = 0;
  if (!(norm >= 0.0) || !isfinite(norm)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_flag(args.err, GQ_FLAG_BAD_SCALE);
    grid_done_signal(args.sig);
    return;
  }
  __shared__ uint64_t s_h4[kMaxWorkers];
  for (uint32_t i = threadIdx.x; i < nl; i += kQThreads)
    s_h4[i] = args.round_ptr ? hoist_prefix(args.seed, 1ull, args.wid[i], *args.round_ptr) : args.h4[i];
  __syncthreads();
  const uint64_t nq = (d + 3) / 4;  // quads, the last one possibly partial
  const uint64_t total = nq * nl;
  for (uint64_t g = blockIdx.x * static_cast<uint64_t>(kQThreads) + threadIdx.x; g < total;
       g += static_cast<uint64_t>(gridDim.x) * kQThreads) {
    const uint32_t r = static_cast<uint32_t>(g / nq);
    const uint64_t q = g - static_cast<uint64_t>(r) * nq;
    const T* x = static_cast<const T*>(args.x[r]);
    const uint64_t h4 = s_h4[r];
    int64_t c[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint64_t j = 4 * q + e;
      c[e] = 0;
      if (j >= d) continue;
      const T v = x[j];
      if (norm == 0.0) {  // quantizer.cpp:21-32: all idx = s (lane 0); every element must be zero
        if (v != T(0)) flags |= GQ_FLAG_ZERO_SCALE;
        continue;
      }
      const double ad = Abs<T>::dbl(v);
      if (!isfinite(ad)) {
        flags |= GQ_FLAG_NONFINITE;
        continue;
      }
      if (ad > norm) flags |= GQ_FLAG_EXCEEDS_SCALE;
      const uint32_t idx = slow_index<0>(ad, norm, mix64(h4 ^ j), s);
      const int64_t mag = static_cast<int64_t>(s) - static_cast<int64_t>(idx);
      c[e] = Abs<T>::neg(v) ? -mag : mag;
    }
    int64_t* out = static_cast<int64_t*>(lane_base_for<64>(args, r, q)) + 4 * q;
    if (4 * q + 4 <= d) {
      reinterpret_cast<longlong2*>(out)[0] = make_longlong2(c[0], c[1]);
      reinterpret_cast<longlong2*>(out)[1] = make_longlong2(c[2], c[3]);
    } else {
      for (int e = 0; 4 * q + e < d; ++e) out[e] = c[e];
    }
  }
  raise_flags_warp(args.err, flags);
  grid_done_signal(args.sig);
}

template <typename T>
cudaError_t launch_q64(const QuantArgs& a, cudaStream_t st) {
  const uint64_t units = (a.d + 3) / 4 * a.n_local;
  uint64_t blocks = (units + kQThreads - 1) / kQThreads;
  if (blocks > 148ull * 8) blocks = 148ull * 8;
  if (blocks == 0) blocks = 1;
  const cudaError_t e = launch_maybe_pdl(quantize64_kernel<T>, static_cast<uint32_t>(blocks), kQThreads, 0, st, a);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <typename T, int KIND, int W, int U, int ST>
cudaError_t launch_one(const QuantArgs& a, uint64_t work_chunks, cudaStream_t st) {
  auto* fn = quantize_kernel<T, KIND, W, U, ST>;
  const size_t smem = (kQThreads / 32) * (ST * (32 * U * 4 * sizeof(T)) + ST * sizeof(uint64_t));
  // one-time per instantiation: opt in to >48 KiB smem, read the residency
  static int blocks_per_sm = 0;
  static int sms = 0;
  if (blocks_per_sm == 0) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, fn, kQThreads, smem);
    if (e != cudaSuccess) return e;
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  // persistent grid: exactly one wave of resident blocks (never a tail wave)
  const int per_sm = (g_quant_ctas_per_sm > 0 && g_quant_ctas_per_sm < blocks_per_sm) ? g_quant_ctas_per_sm
                                                                                     : blocks_per_sm;
  uint64_t blocks = static_cast<uint64_t>(sms) * per_sm * GQ_QWAVES;
  if (blocks > work_chunks) blocks = work_chunks;
  if (blocks == 0) blocks = 1;
  const cudaError_t e = launch_maybe_pdl(fn, static_cast<uint32_t>(blocks), kQThreads, smem, st, a);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// Chunk geometry. Large launches that are alone on the GPU (a single-bucket
// step: C2's 8 x 2^24 elements) run 4 KiB chunks (8 quads per lane, 2
// stages: half the per-chunk overhead, measured 185 -> 175 us at C2); the
// default 2 KiB x 3 stages keeps the shared-memory footprint that lets a
// bucket pipeline's norm / reduce kernels co-reside (C4: the 4 KiB form was
// 8 % slower, profiles/r2/variants_unroll8.txt). In scatter mode a chunk
// must not straddle a slice: the 4 KiB form needs slices of whole 1024-lane
// units (gq_comm cuts them so).
#ifndef GQ_QBIG_QUADS  // quads (all local workers) at or above which a launch takes the 4 KiB chunks
#define GQ_QBIG_QUADS (1ull << 25)
#endif
template <typename T, int KIND, int U, int ST>
cudaError_t launch_wu(const QuantArgs& a, uint64_t work_chunks, uint32_t width, cudaStream_t st) {
  switch (width) {
    case 4: return launch_one<T, KIND, 4, U, ST>(a, work_chunks, st);
    case 8: return launch_one<T, KIND, 8, U, ST>(a, work_chunks, st);
    case 16: return launch_one<T, KIND, 16, U, ST>(a, work_chunks, st);
    case 32: return launch_one<T, KIND, 32, U, ST>(a, work_chunks, st);
    default: return cudaErrorInvalidValue;
  }
}
template <typename T, int KIND>
cudaError_t launch_w(const QuantArgs& a, uint32_t width, cudaStream_t st) {
  const uint64_t quads = a.d / 4 * a.n_local;
  // work units for the grid: whole staged chunks over all local workers
  // (at least one per worker so the remainder/tail loop has an owner)
  auto work_of = [&](uint64_t wq) {
    uint64_t w = ((a.d / 4 / wq) * a.n_local + (kQThreads / 32) * GQ_QMIN_CHUNKS - 1) /
                 ((kQThreads / 32) * GQ_QMIN_CHUNKS);
    return w < a.n_local ? static_cast<uint64_t>(a.n_local) : w;
  };
  // one worker alone (an N-rank step's quantize): 4 KiB chunks from 2^22 quads (C2 rank: 31.2 -> 29.9 us)
  const bool big = quads >= GQ_QBIG_QUADS || (a.n_local == 1 && quads >= (GQ_QBIG_QUADS >> 3));
  if (sizeof(T) == 4 && (!a.nslices || a.slice_quads % 256 == 0) && big && width <= 8)
    return launch_wu<T, KIND, 8, 2>(a, work_of(256), width, st);
  return launch_wu<T, KIND, GQ_QUNROLL, GQ_QSTAGES>(a, work_of(32 * GQ_QUNROLL), width, st);
}

}  // namespace

cudaError_t launch_quantize(const QuantLaunch& q, cudaStream_t stream) {
  QuantArgs a{};
  for (uint32_t i = 0; i < q.n_local; ++i) {
    a.x[i] = q.shards[i];
    a.lanes[i] = q.lanes[i];
    // RngStream::Dither = 1 (rng.hpp:31-37); keys (worker, round, j).
    a.h4[i] = hoist_prefix(q.seed, 1ull, q.worker_ids[i], q.round);
    a.wid[i] = q.worker_ids[i];
  }
  a.round_ptr = q.round_ptr;
  a.seed = q.seed;
  a.nslices = q.nslices;
  a.slice_quads = q.slice_lanes / 4;
  a.row_bytes = q.row_bytes;
  if (q.wait) {
    a.pw = *q.wait;
    a.fold = q.fold;
  }
  if (q.signal) {
    for (uint32_t i = 0; i < q.signal->n; ++i) a.sig.slots[i] = q.signal->slots[i];
    a.sig.n = q.signal->n;
    a.sig.epoch = q.signal->epoch;
    a.sig.ep_dev = q.signal->ep_dev;
    a.sig.ticket = q.signal->ticket;
  }
  for (uint32_t i = 0; i < q.nslices; ++i) a.sdst[i] = q.slice_dst[i];
  a.d = q.d;
  a.norm = q.norm;
  a.err = q.err;
  a.s = q.s;
  uint32_t shift = 0;
  for (uint64_t p = 1; p < 2ull * q.n_total; p <<= 1) ++shift;  // prescale_shift
  a.shift = shift;
  a.mk = GQ_MULCONSTS_INIT;
  if (q.width < 32) {
    a.pk[0] = 1u << q.width;
    a.pk[1] = 1u << (2 * q.width);
    a.pk[2] = q.width < 16 ? 1u << (3 * q.width) : 0u;
  }
  a.n_local = q.n_local;
  if (q.width == 64) {
    if (q.kind != 0 || a.pw.n) return cudaErrorInvalidValue;
    return q.dtype == GQ_DTYPE_F32 ? launch_q64<float>(a, stream) : launch_q64<double>(a, stream);
  }
  if (q.dtype == GQ_DTYPE_F32) {
    return q.kind == 0 ? launch_w<float, 0>(a, q.width, stream) : launch_w<float, 1>(a, q.width, stream);
  }
  return q.kind == 0 ? launch_w<double, 0>(a, q.width, stream) : launch_w<double, 1>(a, q.width, stream);
}

}  // namespace gqb
