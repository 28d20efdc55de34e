// Global-norm phase: local_norm_stat for every local worker, plus (optionally)
// the tree-order fold + root of norm_allreduce_inproc, in ONE launch.
//
//   reference: norms.cpp:34-75 (vector_norm / local_norm_stat /
//              combine_norm_stats), collectives.cpp:210-233 (the scalar
//              exchange always walks tree_schedule, dst op= src).
//
// Layout: grid (bx, n). Block (b, r) streams a contiguous 1/bx slice of worker
// r's shard with 128-bit loads, reducing
//   L-inf: max |x| as the max of the sign-cleared bit patterns (monotone for
//          non-NaN IEEE values; NaN/Inf show up as bits >= the Inf pattern);
//   L2:    sum of x*x in f64 (a float product is exact in f64), plus the same
//          max-bits word for the NaN/Inf check.
// Partials go to the workspace; the last block to finish (atomic ticket)
// folds them in a fixed order (deterministic for a given d), forms the
// per-worker stat exactly as norms.cpp:58-61 (sqrt then square for p = 2),
// then walks the tree schedule over the n stats.
//
// HBM roofline: 4 B (f32) read per element, nothing written per element.
#include <cuda_runtime.h>

#include "gq_common.cuh"
#include "gq_internal.h"

namespace gqb {

namespace {

#ifndef GQ_NORM_THREADS
#define GQ_NORM_THREADS 256
#endif
constexpr int kNormThreads = GQ_NORM_THREADS;
constexpr uint32_t kNormMaxSpb = 64;  // slices per block (k draws riding along)
#ifndef GQ_NORM_MEM_THREADS
#define GQ_NORM_MEM_THREADS 128  // streaming threads per block when the k draws ride along
#endif

template <typename T>
struct AbsBits;
template <>
struct AbsBits<float> {
  using U = uint32_t;
  static constexpr U kInf = 0x7f800000u;
  __device__ static U get(float v) { return __float_as_uint(v) & 0x7fffffffu; }
  __device__ static double val(U b) { return static_cast<double>(__uint_as_float(b)); }
};
template <>
struct AbsBits<double> {
  using U = unsigned long long;
  static constexpr U kInf = 0x7ff0000000000000ull;
  __device__ static U get(double v) {
    return static_cast<U>(__double_as_longlong(v)) & 0x7fffffffffffffffull;
  }
  __device__ static double val(U b) { return __longlong_as_double(static_cast<long long>(b)); }
};

#ifndef GQ_NORM_FMAX
#define GQ_NORM_FMAX 1
#endif
// |x|^q for an integer q in [3, 16], x finite: x = m 2^e with m in [1, 2),
// m^q by square-and-multiply in double-double (FMA error-free products),
// rounded once; the scale 2^(eq) is exact unless the result is subnormal.
// The result is the correctly rounded power except when m^q lies within
// ~2^-100 (relative) of a rounding midpoint. (The reference's std::pow, glibc,
// is not correctly rounded: it differs from the correctly rounded power in
// ~0.1 % of f32 inputs, tests/test_gpu_norm_orders.py, so general-order stats
// agree with the reference to rounding, not bit for bit.)
__device__ __forceinline__ double pow_int(double x, uint32_t q) {
  if (x == 0.0) return 0.0;
  int e;
  const double m = 2.0 * frexp(x, &e);
  --e;
  double rh = 1.0, rl = 0.0, bh = m, bl = 0.0;
  for (uint32_t k = q; k != 0; k >>= 1) {
    if (k & 1u) {
      const double ph = rh * bh;
      double pe = fma(rh, bh, -ph);
      pe = fma(rh, bl, pe);
      pe = fma(rl, bh, pe);
      rh = ph + pe;
      rl = pe - (rh - ph);
    }
    if (k > 1u) {
      const double ph = bh * bh;
      double pe = fma(bh, bh, -ph);
      pe = fma(2.0 * bh, bl, pe);
      bh = ph + pe;
      bl = pe - (bh - ph);
    }
  }
  return ldexp(rh, e * static_cast<int>(q));
}

template <typename T, bool kL2, bool kPow = false>
__device__ __forceinline__ void accum(T v, typename AbsBits<T>::U& mb, double& ss, uint32_t qpow = 0) {
  if constexpr (kPow) {  // general order: sum of |x|^q (the max still flags NaN / Inf)
    const auto b = AbsBits<T>::get(v);
    mb = b > mb ? b : mb;
    ss = __dadd_rn(ss, pow_int(fabs(static_cast<double>(v)), qpow));
    return;
  }
  if constexpr (GQ_NORM_FMAX && sizeof(T) == 4) {
    // max of |x| on the FP pipe (the integer pipe is the k draws'): for
    // non-NaN values the float max is the max of the sign-cleared bit
    // patterns; max.NaN makes any NaN the canonical 0x7fffffff, which sorts
    // above Inf as the integer max does (C2 norm + k draws 126 -> 119 us)
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(fabsf(static_cast<float>(v))), "f"(__uint_as_float(mb)));
    mb = __float_as_uint(r);
  } else {
    const auto b = AbsBits<T>::get(v);
    mb = b > mb ? b : mb;
  }
  if constexpr (kL2) {
    const double x = static_cast<double>(v);
    ss = __dadd_rn(ss, __dmul_rn(x, x));
  }
}

// This block's share of the precomputed k draws (KDrawJob): integer work
// overlapping the other resident blocks' HBM streaming.
template <int W>
__device__ __noinline__ void kdraw_share(const KDrawJob& job, uint64_t block, uint64_t nblocks) {
  const MulConsts MK = GQ_MULCONSTS_INIT;
  __shared__ uint64_t s_keys[kMaxKEvents];
  for (uint32_t e = threadIdx.x; e < kMaxKEvents; e += blockDim.x) s_keys[e] = job.keys[e];
  __syncthreads();
  const uint64_t total = job.kwords * job.events;
  const uint64_t per = (total + nblocks - 1) / nblocks;
  const uint64_t b0 = per * block;
  const uint64_t b1 = b0 + per < total ? b0 + per : total;
  kdraw_run<W>(job.buf, job.kwords, job.w0, job.m, s_keys, b0 + threadIdx.x, b1, blockDim.x, MK);
}

template <int W>
__global__ void __launch_bounds__(kNormThreads) kdraw_kernel(const __grid_constant__ KDrawJob job) {
  kdraw_share<W>(job, blockIdx.x, gridDim.x);
}


// KW = 0: plain norm pass. KW = 4 / 8: the block also produces its share of
// the precomputed k words (warp-specialised, see below).
//
// The stat of a worker is a function of its data and d only: its vectors are
// cut into `slices` contiguous slices (norm_slices(d)), each slice reduced by
// kNormThreads (virtual) threads in ascending order per thread, a fixed
// butterfly per warp and the warps in order; the slice partials folded in the
// last block. A launch covers `spb` consecutive slices per block. The plain
// pass (spb = 1) has one thread per virtual thread; with the k draws riding
// along only kMem threads stream, each standing in for kNormThreads / kMem
// virtual threads with its own accumulators, so the partials are bit-identical
// whether a worker is reduced alone on its GPU (an N-rank step) or beside
// n - 1 others, with or without the k draws.
#ifndef GQ_NORM_KD_THREADS
#define GQ_NORM_KD_THREADS 128  // k-draw threads per block when the k draws ride along
#endif
template <int KW>
constexpr int norm_block_threads() { return KW ? GQ_NORM_MEM_THREADS + GQ_NORM_KD_THREADS : kNormThreads; }

// The last block of a norm launch: per-worker stats from the slice partials
// (fixed order), NaN / Inf flag, the folded stats put to peers (StatsPut),
// the tree fold. Leaves the ticket at 0.
template <typename T, bool kL2, bool kPow>
__device__ __forceinline__ void norm_last_block(uint32_t n, uint32_t p, uint32_t slices,
                                                const double* partial_ss, const unsigned long long* partial_mb,
                                                unsigned int* ticket, double* stats, double* norm_out,
                                                uint32_t* err, const StatsPut& put) {
  using U = typename AbsBits<T>::U;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bx = slices;
  __shared__ double s_stats[kMaxWorkers];
  __shared__ uint32_t s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  for (uint32_t w = warp; w < n; w += blockDim.x / 32) {
    U m = 0;
    double acc = 0.0;
    // Fixed-order strided partial sums then a fixed butterfly.
    for (uint32_t b = lane; b < bx; b += 32) {
      const U pm = static_cast<U>(__ldcg(partial_mb + w * bx + b));
      m = pm > m ? pm : m;
      if constexpr (kL2 || kPow) acc = __dadd_rn(acc, __ldcg(partial_ss + w * bx + b));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const U om = __shfl_xor_sync(0xffffffffu, m, o);
      m = om > m ? om : m;
      if constexpr (kL2 || kPow) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    }
    if (lane == 0) {
      if (m >= AbsBits<T>::kInf) atomicOr(&s_bad, 1u);
      // vector_norm (norms.cpp:34-48) then local_norm_stat's power
      // (norms.cpp:58-61).
      // general order (kPow): the raw sum of |x|^q; the host takes the root
      const double nq = kPow ? acc : kL2 ? __dsqrt_rn(acc) : AbsBits<T>::val(m);
      const double st = (p == GQ_NORM_INF) ? nq : __dmul_rn(nq, nq);
      s_stats[w] = st;
      stats[w] = st;
    }
  }
  __syncthreads();
  if (put.n) {  // the stats exchange folded in (StatsPut): peers' rows, then the flag
    for (uint32_t i = threadIdx.x; i < put.n * n; i += blockDim.x) put.dst[i / n][i % n] = s_stats[i % n];
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      const uint32_t e = put.ep_dev ? *put.ep_dev + 1u : put.epoch;
      if (put.ep_dev) *put.ep_dev = e;
      for (uint32_t q2 = 0; q2 < put.n; ++q2)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(put.slots[q2]), "r"(e) : "memory");
    }
  }
  if (threadIdx.x == 0) {
    if (s_bad) raise_flag(err, GQ_FLAG_NONFINITE);
    if (norm_out) *norm_out = tree_fold_stats(s_stats, n, p);
    *ticket = 0u;  // leave the workspace reusable (graph replays)
  }
}

#ifndef GQ_NORM_TMA  // k-draw launches: the streaming warps read through TMA bulk copies into shared memory
#define GQ_NORM_TMA 0    // measured slower at C2 (125-160 vs 119 us, profiles/r2/variants_norm.txt)
#endif
#ifndef GQ_NORM_TMA_STAGES
#define GQ_NORM_TMA_STAGES 4
#endif
#ifndef GQ_NORM_TMA_ROWS  // rows of kNormThreads 16-byte vectors per stage
#define GQ_NORM_TMA_ROWS 4
#endif
constexpr uint32_t kTmaStageVec = GQ_NORM_TMA_ROWS * kNormThreads;  // vectors per stage
constexpr size_t norm_tma_smem() {
  return static_cast<size_t>(GQ_NORM_TMA_STAGES) * kTmaStageVec * 16 + GQ_NORM_TMA_STAGES * 8;
}

template <typename T, bool kL2, int KW, bool kPow = false, bool kTma = false>
__global__ void __launch_bounds__(norm_block_threads<KW>())
norm_kernel(PtrArray shards, uint64_t d, uint32_t n, uint32_t q, uint32_t p,
            double* partial_ss, unsigned long long* partial_mb,
            unsigned int* ticket, double* stats, double* norm_out,
            uint32_t* err, const __grid_constant__ KDrawJob kjob, const __grid_constant__ StatsPut put,
            uint32_t slices, uint32_t spb) {
  using U = typename AbsBits<T>::U;
  const uint32_t r = blockIdx.y;
  const T* x = static_cast<const T*>(shards.p[r]);
  constexpr int kVec = 16 / sizeof(T);
  const uint64_t nvec = d / kVec;
  const uint64_t per = (nvec + slices - 1) / slices;
  const uint4* xv = reinterpret_cast<const uint4*>(x);
  constexpr int kUnroll = 4;
  constexpr int kMem = KW ? GQ_NORM_MEM_THREADS : kNormThreads;
  constexpr int kVirt = kNormThreads / kMem;  // virtual threads per streaming thread
  static_assert(kNormThreads % kMem == 0 && kMem % 32 == 0, "streaming threads: whole warps");
  constexpr int kVW = kNormThreads / 32;      // virtual warps
  // per-slice virtual-warp results, folded once after the block's slices
  __shared__ double s_ss[kNormMaxSpb * kVW];
  __shared__ U s_mb[kNormMaxSpb * kVW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (kTma && threadIdx.x < kMem) {
    // TMA-staged streaming: thread 0 keeps GQ_NORM_TMA_STAGES bulk copies of
    // up to kTmaStageVec vectors in flight (slice by slice, rows of
    // kNormThreads vectors from the slice start), so four warps hold the
    // SM's share of the HBM stream with a few instructions per 16 bytes and
    // the k-draw warps keep the issue slots. Each thread takes the same
    // virtual threads' vectors in the same order as the register path.
    extern __shared__ __align__(128) uint8_t nsm[];
    const uint4* sbuf = reinterpret_cast<const uint4*>(nsm);
    uint64_t* bars = reinterpret_cast<uint64_t*>(nsm + static_cast<size_t>(GQ_NORM_TMA_STAGES) * kTmaStageVec * 16);
    const uint32_t s0 = blockIdx.x * spb;
    const uint32_t s1 = s0 + spb < slices ? s0 + spb : slices;
    // producer cursor (thread 0): slice ps, vector offset pa within it
    uint32_t ps = s0;
    uint64_t pa = 0;
    auto issue = [&](uint32_t st) {  // the next chunk into stage st, if any
      while (ps < s1) {
        const uint64_t v0 = per * ps;
        const uint64_t v1 = v0 + per < nvec ? v0 + per : nvec;
        if (v0 + pa < v1) {
          const uint64_t c = v1 - (v0 + pa) < kTmaStageVec ? v1 - (v0 + pa) : kTmaStageVec;
          mbar_expect_tx(&bars[st], static_cast<uint32_t>(c * 16));
          bulk_g2s(nsm + static_cast<size_t>(st) * kTmaStageVec * 16, xv + v0 + pa, static_cast<uint32_t>(c * 16),
                   &bars[st]);
          pa += c;
          return;
        }
        ++ps;
        pa = 0;
      }
      mbar_expect_tx(&bars[st], 0);  // nothing left: complete the phase empty
    };
    if (threadIdx.x == 0) {
      for (int st = 0; st < GQ_NORM_TMA_STAGES; ++st) mbar_init(&bars[st], 1);
      mbar_fence_init();
      for (int st = 0; st < GQ_NORM_TMA_STAGES; ++st) issue(st);
    }
    asm volatile("bar.sync 1, %0;" ::"r"(kMem) : "memory");
    uint32_t k = 0;  // chunk counter (stage k % S, parity (k / S) & 1)
    for (uint32_t sl = s0; sl < s1; ++sl) {
      const uint64_t v0 = per * sl;
      const uint64_t v1 = v0 + per < nvec ? v0 + per : nvec;
      U mb[kVirt];
      double ss[kVirt];
#pragma unroll
      for (int kk = 0; kk < kVirt; ++kk) {
        mb[kk] = 0;
        ss[kk] = 0.0;
      }
      for (uint64_t a = v0; a < v1; a += kTmaStageVec, ++k) {
        const uint32_t st = k % GQ_NORM_TMA_STAGES;
        mbar_wait(&bars[st], (k / GQ_NORM_TMA_STAGES) & 1u);
        const uint4* sb = sbuf + static_cast<size_t>(st) * kTmaStageVec;
        const uint32_t c = static_cast<uint32_t>(v1 - a < kTmaStageVec ? v1 - a : kTmaStageVec);
#pragma unroll
        for (int row = 0; row < GQ_NORM_TMA_ROWS; ++row) {
          uint4 w[kVirt];
#pragma unroll
          for (int kk = 0; kk < kVirt; ++kk) {
            const uint32_t o = row * kNormThreads + threadIdx.x + kk * kMem;
            w[kk] = o < c ? sb[o] : make_uint4(0u, 0u, 0u, 0u);
          }
#pragma unroll
          for (int kk = 0; kk < kVirt; ++kk) {
            if (row * kNormThreads + threadIdx.x + kk * kMem < c) {
              const T* e = reinterpret_cast<const T*>(&w[kk]);
#pragma unroll
              for (int t = 0; t < kVec; ++t) accum<T, kL2, kPow>(e[t], mb[kk], ss[kk], q);
            }
          }
        }
        asm volatile("bar.sync 1, %0;" ::"r"(kMem) : "memory");  // stage st consumed by every thread
        if (threadIdx.x == 0) issue(st);
      }
#pragma unroll
      for (int kk = 0; kk < kVirt; ++kk) {
        const uint32_t vt = threadIdx.x + kk * kMem;
        // Scalar tail (d % kVec elements) belongs to the last slice.
        if (sl == slices - 1)
          for (uint64_t j = nvec * kVec + vt; j < d; j += kNormThreads) accum<T, kL2, kPow>(x[j], mb[kk], ss[kk], q);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const U om = __shfl_xor_sync(0xffffffffu, mb[kk], o);
          mb[kk] = om > mb[kk] ? om : mb[kk];
          if constexpr (kL2 || kPow) ss[kk] = __dadd_rn(ss[kk], __shfl_xor_sync(0xffffffffu, ss[kk], o));
        }
        if (lane == 0) {
          s_ss[(sl - s0) * kVW + kk * (kMem / 32) + warp] = ss[kk];
          s_mb[(sl - s0) * kVW + kk * (kMem / 32) + warp] = mb[kk];
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(kMem) : "memory");
    if (threadIdx.x < s1 - s0) {  // one thread per slice: the warps in order
      U m = 0;
      double acc = 0.0;
      for (int w = 0; w < kVW; ++w) {
        m = s_mb[threadIdx.x * kVW + w] > m ? s_mb[threadIdx.x * kVW + w] : m;
        acc = __dadd_rn(acc, s_ss[threadIdx.x * kVW + w]);
      }
      partial_ss[r * slices + s0 + threadIdx.x] = acc;
      partial_mb[r * slices + s0 + threadIdx.x] = static_cast<unsigned long long>(m);
    }
  } else if (threadIdx.x < kMem) {
    const uint32_t s0 = blockIdx.x * spb;
    const uint32_t s1 = s0 + spb < slices ? s0 + spb : slices;
    for (uint32_t sl = s0; sl < s1; ++sl) {
      const uint64_t v0 = per * sl;
      const uint64_t v1 = v0 + per < nvec ? v0 + per : nvec;
      U mb[kVirt];
      double ss[kVirt];
#pragma unroll
      for (int k = 0; k < kVirt; ++k) {
        mb[k] = 0;
        ss[k] = 0.0;
      }
      // all virtual threads' loads of a batch in flight together; each
      // virtual thread still accumulates its own elements in ascending order
      uint64_t i = v0 + threadIdx.x;
      for (; i + (kVirt - 1) * kMem + (kUnroll - 1) * kNormThreads < v1; i += kUnroll * kNormThreads) {
        uint4 w[kUnroll][kVirt];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
#pragma unroll
          for (int k = 0; k < kVirt; ++k) w[u][k] = __ldcs(xv + i + u * kNormThreads + k * kMem);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
#pragma unroll
          for (int k = 0; k < kVirt; ++k) {
            const T* e = reinterpret_cast<const T*>(&w[u][k]);
#pragma unroll
            for (int t = 0; t < kVec; ++t) accum<T, kL2, kPow>(e[t], mb[k], ss[k], q);
          }
      }
#pragma unroll
      for (int k = 0; k < kVirt; ++k) {
        const uint32_t vt = threadIdx.x + k * kMem;
        for (uint64_t ik = i + k * kMem; ik < v1; ik += kNormThreads) {
          const uint4 w = __ldcs(xv + ik);
          const T* e = reinterpret_cast<const T*>(&w);
#pragma unroll
          for (int t = 0; t < kVec; ++t) accum<T, kL2, kPow>(e[t], mb[k], ss[k], q);
        }
        // Scalar tail (d % kVec elements) belongs to the last slice.
        if (sl == slices - 1)
          for (uint64_t j = nvec * kVec + vt; j < d; j += kNormThreads) accum<T, kL2, kPow>(x[j], mb[k], ss[k], q);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const U om = __shfl_xor_sync(0xffffffffu, mb[k], o);
          mb[k] = om > mb[k] ? om : mb[k];
          if constexpr (kL2 || kPow) ss[k] = __dadd_rn(ss[k], __shfl_xor_sync(0xffffffffu, ss[k], o));
        }
        if (lane == 0) {
          s_ss[(sl - s0) * kVW + k * (kMem / 32) + warp] = ss[k];
          s_mb[(sl - s0) * kVW + k * (kMem / 32) + warp] = mb[k];
        }
      }
    }
    // the streaming warps only (the k-draw warps never arrive here)
    asm volatile("bar.sync 1, %0;" ::"r"(kMem) : "memory");
    if (threadIdx.x < s1 - s0) {  // one thread per slice: the warps in order
      U m = 0;
      double acc = 0.0;
      for (int w = 0; w < kVW; ++w) {
        m = s_mb[threadIdx.x * kVW + w] > m ? s_mb[threadIdx.x * kVW + w] : m;
        acc = __dadd_rn(acc, s_ss[threadIdx.x * kVW + w]);
      }
      partial_ss[r * slices + s0 + threadIdx.x] = acc;
      partial_mb[r * slices + s0 + threadIdx.x] = static_cast<unsigned long long>(m);
    }
  } else if constexpr (KW != 0) {
    // the rest of the block produces this block's share of the k words, so
    // every SM always has both HBM streams and integer work in flight
    const MulConsts MK = GQ_MULCONSTS_INIT;
    // event keys (from the launch, or for graph replays from the device
    // round) in shared memory, read once per event run
    __shared__ uint64_t s_keys[kMaxKEvents];
    const uint32_t kt = threadIdx.x - kMem;
    if (kt < kMaxKEvents) {
      uint64_t key = kjob.keys[kt];
      if (kjob.round_ptr) {
        const uint64_t h = reduce_round_prefix(kjob.seed, *kjob.round_ptr);
        uint32_t e = 0;
        for (uint32_t t = 0; (1u << t) < kjob.n; ++t)
          for (uint32_t r2 = 1u << t; r2 < kjob.n && e < kMaxKEvents; r2 += 2u << t, ++e)
            if (e == kt) key = mix64(h ^ ((static_cast<uint64_t>(t) << 32) | (r2 - (1u << t))));
      }
      s_keys[kt] = key;
    }
    asm volatile("bar.sync 2, %0;" ::"r"(GQ_NORM_KD_THREADS) : "memory");
    const uint64_t total = kjob.kwords * kjob.events;
    const uint64_t nblk = static_cast<uint64_t>(gridDim.x) * gridDim.y;
    const uint64_t kper = (total + nblk - 1) / nblk;
    const uint64_t kb0 = kper * (static_cast<uint64_t>(blockIdx.y) * gridDim.x + blockIdx.x);
    const uint64_t kend = kb0 + kper < total ? kb0 + kper : total;
    kdraw_run<KW>(kjob.buf, kjob.kwords, kjob.w0, kjob.m, s_keys, kb0 + kt, kend, GQ_NORM_KD_THREADS, MK);
  }
  __syncthreads();
  __shared__ uint32_t s_last;
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned int total = gridDim.x * gridDim.y;
    const unsigned int t = atomicAdd(ticket, 1u);
    s_last = (t == total - 1) ? 1 : 0;
  }
  __syncthreads();
  if (s_last == 0) return;
  __threadfence();
  norm_last_block<T, kL2, kPow>(n, p, slices, partial_ss, partial_mb, ticket, stats, norm_out, err, put);
}

// Sequential L2 (GQ_NORM_L2_SEQUENTIAL): vector_norm's `ss += v * v` in
// element order (norms.cpp:40-43), bit for bit. One block per worker: the
// warps stage 2048-element tiles into shared memory with coalesced loads,
// thread 0 folds each tile in order. NaN/Inf are flagged as in norm_kernel.
template <typename T>
__global__ void __launch_bounds__(256)
norm_seq_kernel(PtrArray shards, uint64_t d, uint32_t p, double* stats, uint32_t* err) {
  constexpr int kTile = 2048;
  __shared__ double tile[kTile];
  const T* x = static_cast<const T*>(shards.p[blockIdx.x]);
  double ss = 0.0;
  uint32_t bad = 0;
  for (uint64_t base = 0; base < d; base += kTile) {
    const int cnt = static_cast<int>(d - base < kTile ? d - base : kTile);
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      const double v = static_cast<double>(x[base + i]);
      if (!isfinite(v)) bad = 1;
      tile[i] = __dmul_rn(v, v);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 0; i < cnt; ++i) ss = __dadd_rn(ss, tile[i]);
    }
    __syncthreads();
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) raise_flag(err, GQ_FLAG_NONFINITE);
  if (threadIdx.x == 0) {
    const double nq = __dsqrt_rn(ss);
    stats[blockIdx.x] = (p == GQ_NORM_INF) ? nq : __dmul_rn(nq, nq);
  }
}

__global__ void norm_combine_kernel(const double* stats, uint32_t n, uint32_t p,
                                    double* norm_out) {
  __shared__ double s[kMaxWorkers];
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) s[i] = stats[i];
  __syncthreads();
  if (threadIdx.x == 0) *norm_out = tree_fold_stats(s, n, p);
}

}  // namespace

// Slices per worker (the partial-sum partition) depend on d only, never on
// n or on the k draws, so a worker's stat is the same whether it is reduced
// alone on its own GPU or next to n-1 others on one device (dist.py vs
// gqsgd_mean): up to kNormTotalBlocks slices of >= 8 KiB of input.
uint32_t norm_slices(uint64_t d) {
  const uint64_t by_work = (d + 8191) / 8192;
  uint64_t sl = by_work < kNormTotalBlocks ? by_work : kNormTotalBlocks;
  return static_cast<uint32_t>(sl ? sl : 1);
}

// Blocks per worker: one per slice for the plain norm (many short blocks;
// they interleave with concurrent streams' kernels in the bucket pipeline).
// With the k draws riding along: about GQ_NORM_KD_WAVES waves over all n
// workers, each block streaming spb consecutive slices so its k-draw warps
// overlap its own loads (C2: step 0.426 -> 0.406 ms, profiles/r1/variants.md).
uint32_t norm_slices_per_block(uint32_t n, uint64_t d, bool kdraws) {
#ifndef GQ_NORM_KD_WAVES
#define GQ_NORM_KD_WAVES 2
#endif
#ifndef GQ_NORM_TMA_BPS  // TMA k-draw launches: one wave of this many blocks per SM (shared-memory bound)
#define GQ_NORM_TMA_BPS 3
#endif
  if (!kdraws) return 1;
  const uint64_t sl = norm_slices(d);
  const uint64_t total = GQ_NORM_TMA ? 148ull * GQ_NORM_TMA_BPS : GQ_NORM_KD_WAVES * kNormTotalBlocks;
  const uint64_t target = (total + n - 1) / n;  // blocks per worker
  uint64_t spb = target >= sl ? 1 : (sl + target - 1) / target;
#ifndef GQ_NORM_KD_SPB_MIN
#define GQ_NORM_KD_SPB_MIN 2  // one worker alone (an N-rank step): 25.0 -> 23.0 us at the C2 rank size
#endif
  if (spb < GQ_NORM_KD_SPB_MIN) spb = GQ_NORM_KD_SPB_MIN;
  if (spb > kNormMaxSpb) spb = kNormMaxSpb;
  return static_cast<uint32_t>(spb);
}

uint32_t norm_blocks_per_worker(uint32_t n, uint64_t d, bool kdraws) {
  const uint32_t sl = norm_slices(d), spb = norm_slices_per_block(n, d, kdraws);
  return (sl + spb - 1) / spb;
}

size_t norm_workspace_bytes(uint32_t n, uint64_t d) {
  (void)d;
  const uint64_t bx_max = kNormTotalBlocks;
  return kWsHeaderBytes + 2 * 8 * static_cast<size_t>(n) * bx_max;
}

uint32_t tree_event_keys(uint32_t n, uint64_t seed, uint64_t round, uint64_t* keys, uint32_t cap) {
  // RngStream::ReduceDraw = 2; keys (round, step<<32|dst, lane) (collectives.cpp:132-146)
  const uint64_t h = reduce_round_prefix(seed, round);
  uint32_t e = 0;
  for (uint32_t t = 0; (1u << t) < n; ++t) {
    const uint32_t span = 1u << t;
    for (uint32_t r = span; r < n; r += 2 * span) {
      if (e < cap) keys[e] = mix64(h ^ ((static_cast<uint64_t>(t) << 32) | (r - span)));
      ++e;
    }
  }
  return e;
}

// k-draw launches: the TMA-staged form needs its dynamic shared memory opted in once
template <typename T, bool L2, int KW>
cudaError_t launch_kd(dim3 grid, cudaStream_t stream, const PtrArray& a, uint64_t d, uint32_t n, uint32_t q,
                      uint32_t p, double* pss, unsigned long long* pmb, unsigned int* ticket, double* stats,
                      double* norm_out, uint32_t* err, const KDrawJob& job, const StatsPut& put, uint32_t slices,
                      uint32_t spb) {
  auto* fn = norm_kernel<T, L2, KW, false, GQ_NORM_TMA != 0>;
  const size_t smem = GQ_NORM_TMA ? norm_tma_smem() : 0;
  static bool attr = false;
  if (GQ_NORM_TMA && !attr) {
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  fn<<<grid, norm_block_threads<KW>(), smem, stream>>>(a, d, n, q, p, pss, pmb, ticket, stats, norm_out, err, job,
                                                        put, slices, spb);
  return cudaGetLastError();
}

cudaError_t launch_norm(const void* const* shards, uint32_t dtype, uint32_t n,
                        uint64_t d, uint32_t q, uint32_t p, double* stats,
                        double* norm_out, void* workspace, uint32_t* err,
                        cudaStream_t stream, const KDrawJob* kjob, const StatsPut* put_in) {
  KDrawJob job{};
  if (kjob) job = *kjob;
  StatsPut put{};
  if (put_in) put = *put_in;
  if (put.n && q == GQ_NORM_L2_SEQUENTIAL) return cudaErrorInvalidValue;  // caller puts with a kernel
  PtrArray a{};
  for (uint32_t i = 0; i < n; ++i) a.p[i] = shards[i];
  const uint32_t bx = norm_blocks_per_worker(n, d, job.buf != nullptr);
  const uint64_t bx_max = kNormTotalBlocks;
  auto* ticket = reinterpret_cast<unsigned int*>(static_cast<char*>(workspace) + kWsNormTicket);
  auto* pss = reinterpret_cast<double*>(static_cast<char*>(workspace) + kWsHeaderBytes);
  auto* pmb = reinterpret_cast<unsigned long long*>(pss + n * bx_max);
  if (q == GQ_NORM_L2_SEQUENTIAL) {
    if (dtype == GQ_DTYPE_F32) norm_seq_kernel<float><<<n, 256, 0, stream>>>(a, d, p, stats, err);
    else norm_seq_kernel<double><<<n, 256, 0, stream>>>(a, d, p, stats, err);
    if (job.buf) {
      const uint32_t g = kNormTotalBlocks;
      if (job.width == 4) kdraw_kernel<4><<<g, kNormThreads, 0, stream>>>(job);
      else kdraw_kernel<8><<<g, kNormThreads, 0, stream>>>(job);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || !norm_out) return e;
    return launch_norm_combine(stats, n, p, norm_out, stream);
  }
  const uint32_t slices = norm_slices(d), spb = norm_slices_per_block(n, d, job.buf != nullptr);
  const dim3 grid(bx, n);
  const bool l2 = (q == 2);
  cudaError_t e = cudaSuccess;
#define GQ_NORM_LAUNCH(T, L2)                                                                        \
  do {                                                                                               \
    if (!job.buf)                                                                                    \
      norm_kernel<T, L2, 0><<<grid, kNormThreads, 0, stream>>>(a, d, n, q, p, pss, pmb, ticket, stats, \
                                                              norm_out, err, job, put, slices, spb); \
    else if (job.width == 4)                                                                         \
      e = launch_kd<T, L2, 4>(grid, stream, a, d, n, q, p, pss, pmb, ticket, stats, norm_out, err, job, put, \
                              slices, spb);                                                          \
    else                                                                                             \
      e = launch_kd<T, L2, 8>(grid, stream, a, d, n, q, p, pss, pmb, ticket, stats, norm_out, err, job, put, \
                              slices, spb);                                                          \
  } while (0)
  if (dtype == GQ_DTYPE_F32) {
    if (l2) GQ_NORM_LAUNCH(float, true);
    else GQ_NORM_LAUNCH(float, false);
  } else {
    if (l2) GQ_NORM_LAUNCH(double, true);
    else GQ_NORM_LAUNCH(double, false);
  }
#undef GQ_NORM_LAUNCH
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// General norm order q (not 2 / inf): stats[w] = sum_j |x_j|^q of worker w
// over the same d-only partition as the L2 sums; the root, the p-th power and
// the fold run on the host (gq_capi.cu, the reference's std::pow).
cudaError_t launch_norm_pow(const void* const* shards, uint32_t dtype, uint32_t n, uint64_t d, uint32_t q,
                            double* stats, void* workspace, uint32_t* err, cudaStream_t stream) {
  PtrArray a{};
  for (uint32_t i = 0; i < n; ++i) a.p[i] = shards[i];
  const uint32_t slices = norm_slices(d);
  const uint64_t bx_max = kNormTotalBlocks;
  auto* ticket = reinterpret_cast<unsigned int*>(static_cast<char*>(workspace) + kWsNormTicket);
  auto* pss = reinterpret_cast<double*>(static_cast<char*>(workspace) + kWsHeaderBytes);
  auto* pmb = reinterpret_cast<unsigned long long*>(pss + n * bx_max);
  const dim3 grid(slices, n);
  const KDrawJob job{};
  const StatsPut put{};
  if (dtype == GQ_DTYPE_F32)
    norm_kernel<float, false, 0, true><<<grid, kNormThreads, 0, stream>>>(
        a, d, n, q, GQ_NORM_INF, pss, pmb, ticket, stats, nullptr, err, job, put, slices, 1);
  else
    norm_kernel<double, false, 0, true><<<grid, kNormThreads, 0, stream>>>(
        a, d, n, q, GQ_NORM_INF, pss, pmb, ticket, stats, nullptr, err, job, put, slices, 1);
  return cudaGetLastError();
}

cudaError_t launch_norm_combine(const double* stats, uint32_t n, uint32_t p,
                                double* norm_out, cudaStream_t stream) {
  norm_combine_kernel<<<1, 128, 0, stream>>>(stats, n, p, norm_out);
  return cudaGetLastError();
}

}  // namespace gqb
