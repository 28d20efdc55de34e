// The sparse allgather path (cfg.sparse): quantized shards travel as their
// nonzero entries and every worker accumulates them in rank order.
//
//   reference: to_sparse / accumulate_sparse (quantizer.cpp:59-110),
//              serialize_sparse / deserialize_sparse + validate_level_width
//              (serialize.cpp:114-192), decode_sparse_set (algorithm.cpp:112-123),
//              allgather_inproc (collectives.cpp:192-208).
//
// Input is a worker's 32-bit lane buffer from gq_quantize (standard lane
// sign*(s-idx), exponential lane (idx+shift)|sign), i.e. the same dithering
// keys as the dense paths. Encoding is a two-pass stream compaction:
//   count  : one CTA per 4096-element tile counts nonzeros;
//   scan   : one CTA per worker prefix-sums the tile counts, writes the
//            header [norm f64][dim u32][nnz u32];
//   write  : each tile re-reads its lanes, ranks its nonzeros with warp
//            ballots + a CTA scan, and writes index u32 / level lane / a
//            temporary sign byte at its global rank;
//   bitmap : one thread per bitmap byte packs 8 signs (LSB first, set = negative).
// The payload is byte-identical to serialize_sparse(to_sparse(...)).
//
// Accumulation follows accumulate_sparse exactly: acc[j] += (norm * sign) *
// level(idx) in f64, worker by worker in rank order (indices are unique within
// a worker, so each worker's scatter is race-free), then decode_sparse_set's
// acc / n. Adding the zero levels as +0.0 terms leaves every partial sum
// unchanged (an exact cancellation rounds to +0.0), so the in-process dense
// form equals the sparse accumulation bit for bit.
#include <cuda_runtime.h>

#include "gq_common.cuh"
#include "gq_internal.h"

namespace gqb {

namespace {

constexpr int kSThreads = 256;
constexpr int kTile = 4096;  // elements per count / write CTA

struct LaneView {
  uint32_t kind, s, shift;
  // nonzero, level index and sign of a 32-bit lane
  __device__ __forceinline__ bool nz(uint32_t lane) const {
    return kind == 0 ? lane != 0 : (lane & 0x7fffffffu) != 0;
  }
  __device__ __forceinline__ uint32_t idx(uint32_t lane) const {
    if (kind == 0) {
      const int32_t v = static_cast<int32_t>(lane);
      return s - static_cast<uint32_t>(v < 0 ? -v : v);
    }
    return (lane & 0x7fffffffu) - shift;
  }
  __device__ __forceinline__ bool neg(uint32_t lane) const { return (lane >> 31) != 0; }
};

// level(i) as levels.cpp:31-48 builds the table
__device__ __forceinline__ double level_value(uint32_t kind, uint32_t i, uint32_t s) {
  if (kind == 0) return __ddiv_rn(static_cast<double>(s - i), static_cast<double>(s));
  return i < s ? ldexp(1.0, -static_cast<int>(i)) : 0.0;
}

__global__ void __launch_bounds__(kSThreads) sparse_count_kernel(const uint32_t* lanes, uint64_t d, LaneView lv,
                                                                 uint32_t* counts) {
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kTile;
  uint32_t c = 0;
  for (int i = threadIdx.x; i < kTile; i += kSThreads) {
    const uint64_t j = base + i;
    if (j < d) c += lv.nz(lanes[j]) ? 1u : 0u;
  }
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ uint32_t ws[kSThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kSThreads / 32; ++w) t += ws[w];
    counts[blockIdx.x] = t;
  }
}

// one CTA: exclusive scan of the tile counts (in place), header, nnz
__global__ void __launch_bounds__(1024) sparse_scan_kernel(uint32_t* counts, uint32_t tiles, uint64_t d,
                                                           const double* norm, uint8_t* payload,
                                                           uint32_t* nnz_out) {
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < tiles; base += blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t v = i < tiles ? counts[i] : 0u;
    // block-wide inclusive scan (warp shuffles + one pass over warp totals)
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if ((threadIdx.x & 31) >= static_cast<uint32_t>(o)) x += y;
    }
    __shared__ uint32_t wsum[32];
    if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      uint32_t w = threadIdx.x < blockDim.x / 32 ? wsum[threadIdx.x] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (threadIdx.x >= static_cast<uint32_t>(o)) w += y;
      }
      wsum[threadIdx.x] = w;  // inclusive warp-total prefix
    }
    __syncthreads();
    const uint32_t warp_off = (threadIdx.x >> 5) ? wsum[(threadIdx.x >> 5) - 1] : 0u;
    if (i < tiles) counts[i] = carry + warp_off + x - v;  // exclusive
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry += warp_off + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const uint32_t nnz = carry;
    *nnz_out = nnz;
    // header: [norm f64][dim u32][nnz u32] (serialize.cpp:156-160)
    const double nv = *norm;
    const uint64_t nb = static_cast<uint64_t>(__double_as_longlong(nv));
    for (int b = 0; b < 8; ++b) payload[b] = static_cast<uint8_t>(nb >> (8 * b));
    const uint32_t dim = static_cast<uint32_t>(d);
    for (int b = 0; b < 4; ++b) payload[8 + b] = static_cast<uint8_t>(dim >> (8 * b));
    for (int b = 0; b < 4; ++b) payload[12 + b] = static_cast<uint8_t>(nnz >> (8 * b));
  }
}

__global__ void __launch_bounds__(kSThreads) sparse_write_kernel(const uint32_t* lanes, uint64_t d, LaneView lv,
                                                                 uint32_t width, const uint32_t* offsets,
                                                                 const uint32_t* nnz_p, uint8_t* payload,
                                                                 uint8_t* signs) {
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kTile;
  const uint32_t nnz = *nnz_p;
  const uint32_t lb = width / 8;
  uint8_t* idx_out = payload + 16;
  uint8_t* lvl_out = payload + 16 + 4ull * nnz + (nnz + 7) / 8;
  __shared__ uint32_t wcount[kSThreads / 32];
  __shared__ uint32_t running;
  if (threadIdx.x == 0) running = offsets[blockIdx.x];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t0 = 0; t0 < kTile; t0 += kSThreads) {
    const uint64_t j = base + t0 + threadIdx.x;
    uint32_t l = 0;
    bool z = false;
    if (j < d) {
      l = lanes[j];
      z = lv.nz(l);
    }
    const uint32_t ballot = __ballot_sync(0xffffffffu, z);
    if (lane == 0) wcount[warp] = __popc(ballot);
    __syncthreads();
    uint32_t before = running;
    for (int w = 0; w < warp; ++w) before += wcount[w];
    if (z) {
      const uint32_t k = before + __popc(ballot & ((1u << lane) - 1u));
      const uint32_t jj = static_cast<uint32_t>(j);
      uint8_t* ip = idx_out + 4ull * k;
      ip[0] = static_cast<uint8_t>(jj);
      ip[1] = static_cast<uint8_t>(jj >> 8);
      ip[2] = static_cast<uint8_t>(jj >> 16);
      ip[3] = static_cast<uint8_t>(jj >> 24);
      const uint32_t li = lv.idx(l);
      for (uint32_t b = 0; b < lb; ++b) lvl_out[static_cast<uint64_t>(k) * lb + b] = static_cast<uint8_t>(li >> (8 * b));
      signs[k] = lv.neg(l) ? 1 : 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t tot = 0;
      for (int w = 0; w < kSThreads / 32; ++w) tot += wcount[w];
      running += tot;
    }
    __syncthreads();
  }
}

__global__ void sparse_bitmap_kernel(const uint8_t* signs, const uint32_t* nnz_p, uint8_t* payload) {
  const uint32_t nnz = *nnz_p;
  uint8_t* bm = payload + 16 + 4ull * nnz;
  const uint32_t nbytes = (nnz + 7) / 8;
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nbytes; b += gridDim.x * blockDim.x) {
    uint32_t v = 0;
    for (uint32_t i = 0; i < 8 && 8 * b + i < nnz; ++i) v |= static_cast<uint32_t>(signs[8 * b + i]) << i;
    bm[b] = static_cast<uint8_t>(v);
  }
}

// In-process accumulate: mean[j] = (sum_r (norm * sign_r) * level(idx_r)) / n
// with the sum in rank order (accumulate_sparse + decode_sparse_set).
__global__ void sparse_mean_kernel(PtrArray lanes, uint32_t n, uint64_t d, LaneView lv, const double* normp,
                                   uint32_t n_div, float* out32, double* out64) {
  const double norm = *normp;
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < d;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    double acc = 0.0;
    for (uint32_t r = 0; r < n; ++r) {
      const uint32_t l = static_cast<const uint32_t*>(lanes.p[r])[j];
      if (lv.nz(l)) {
        const double sn = lv.neg(l) ? -norm : norm;
        acc = __dadd_rn(acc, __dmul_rn(sn, level_value(lv.kind, lv.idx(l), lv.s)));
      }
    }
    const double m = __ddiv_rn(acc, static_cast<double>(n_div));
    if (out32) out32[j] = __double2float_rn(m);
    if (out64) out64[j] = m;
  }
}

// One serialized payload scattered into acc (deserialize_sparse checks +
// accumulate_sparse), race-free: indices are unique within a payload.
__global__ void sparse_scatter_kernel(const uint8_t* payload, uint64_t bytes, uint32_t kind, uint32_t s,
                                      uint32_t width, uint64_t d, double* acc, uint32_t* err) {
  uint32_t flags = 0;
  auto rd32 = [&](uint64_t off) {
    return static_cast<uint32_t>(payload[off]) | (static_cast<uint32_t>(payload[off + 1]) << 8) |
           (static_cast<uint32_t>(payload[off + 2]) << 16) | (static_cast<uint32_t>(payload[off + 3]) << 24);
  };
  if (bytes < 16) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_flag(err, GQ_FLAG_BAD_PAYLOAD);
    return;
  }
  uint64_t nb = 0;
  for (int b = 0; b < 8; ++b) nb |= static_cast<uint64_t>(payload[b]) << (8 * b);
  const double norm = __longlong_as_double(static_cast<long long>(nb));
  const uint32_t dim = rd32(8), nnz = rd32(12);
  const uint32_t lb = width / 8;
  const uint64_t need = 16 + 4ull * nnz + (nnz + 7) / 8 + static_cast<uint64_t>(nnz) * lb;
  if (dim != d || nnz > dim || need != bytes) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_flag(err, GQ_FLAG_BAD_PAYLOAD);
    return;
  }
  const uint8_t* bm = payload + 16 + 4ull * nnz;
  const uint8_t* lv = bm + (nnz + 7) / 8;
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < nnz;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t j = rd32(16 + 4 * k);
    if (j >= dim || (k > 0 && j <= rd32(16 + 4 * (k - 1)))) {
      flags |= GQ_FLAG_BAD_PAYLOAD;
      continue;
    }
    uint32_t li = 0;
    for (uint32_t b = 0; b < lb; ++b) li |= static_cast<uint32_t>(lv[k * lb + b]) << (8 * b);
    if (li >= s) {  // "sparse entry carries the zero level" (quantizer.cpp:84-86)
      flags |= GQ_FLAG_BAD_PAYLOAD;
      continue;
    }
    const bool neg = (bm[k >> 3] >> (k & 7)) & 1u;
    acc[j] = __dadd_rn(acc[j], __dmul_rn(neg ? -norm : norm, level_value(kind, li, s)));
  }
  raise_flags_warp(err, flags);
}

// decode_sparse_set's acc / n (algorithm.cpp:120-121), optionally fused with
// the SGD step x -= eta * mean on fp32 parameters (trainer.cpp:335).
__global__ void scale_kernel(const double* acc, uint64_t d, uint32_t n, float* out32, double* out64,
                             float* param, float lr) {
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < d;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const double m = __ddiv_rn(acc[j], static_cast<double>(n));
    const float m32 = __double2float_rn(m);
    if (out32) out32[j] = m32;
    if (out64) out64[j] = m;
    if (param) param[j] = __fsub_rn(param[j], __fmul_rn(lr, m32));
  }
}

uint32_t grid_for(uint64_t items, uint32_t threads) {
  uint64_t g = (items + threads - 1) / threads;
  if (g > 148ull * 16) g = 148ull * 16;
  return static_cast<uint32_t>(g ? g : 1);
}

}  // namespace

size_t sparse_workspace_bytes(uint64_t d) {
  const uint64_t tiles = (d + kTile - 1) / kTile;
  return 256 + ((tiles * 4 + 255) & ~uint64_t{255}) + d;
}

cudaError_t launch_sparse_encode(const uint32_t* lanes, uint64_t d, uint32_t kind, uint32_t s, uint32_t shift,
                                 uint32_t width, const double* norm, void* payload, void* workspace,
                                 uint32_t* nnz_out, cudaStream_t st) {
  const uint64_t tiles = (d + kTile - 1) / kTile;
  auto* counts = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(workspace) + 256);
  auto* signs = static_cast<uint8_t*>(workspace) + 256 + ((tiles * 4 + 255) & ~uint64_t{255});
  const LaneView lv{kind, s, shift};
  auto* pl = static_cast<uint8_t*>(payload);
  if (tiles) sparse_count_kernel<<<static_cast<uint32_t>(tiles), kSThreads, 0, st>>>(lanes, d, lv, counts);
  sparse_scan_kernel<<<1, 1024, 0, st>>>(counts, static_cast<uint32_t>(tiles), d, norm, pl, nnz_out);
  if (tiles) {
    sparse_write_kernel<<<static_cast<uint32_t>(tiles), kSThreads, 0, st>>>(lanes, d, lv, width, counts, nnz_out,
                                                                             pl, signs);
    sparse_bitmap_kernel<<<grid_for((d + 7) / 8, 256), 256, 0, st>>>(signs, nnz_out, pl);
  }
  return cudaGetLastError();
}

cudaError_t launch_sparse_mean(const void* const* lanes, uint32_t n, uint64_t d, uint32_t kind, uint32_t s,
                               uint32_t shift, const double* norm, uint32_t n_div, float* out32, double* out64,
                               cudaStream_t st) {
  PtrArray a{};
  for (uint32_t i = 0; i < n; ++i) a.p[i] = lanes[i];
  if (d) sparse_mean_kernel<<<grid_for(d, 256), 256, 0, st>>>(a, n, d, LaneView{kind, s, shift}, norm, n_div,
                                                               out32, out64);
  return cudaGetLastError();
}

cudaError_t launch_sparse_scatter(const void* payload, uint64_t bytes, uint32_t kind, uint32_t s, uint32_t width,
                                  uint64_t d, double* acc, uint32_t* err, cudaStream_t st) {
  sparse_scatter_kernel<<<grid_for(d ? d : 1, 256), 256, 0, st>>>(static_cast<const uint8_t*>(payload), bytes,
                                                                   kind, s, width, d, acc, err);
  return cudaGetLastError();
}

cudaError_t launch_scale(const double* acc, uint64_t d, uint32_t n, float* out32, double* out64, float* param,
                         float lr, cudaStream_t st) {
  if (d) scale_kernel<<<grid_for(d, 256), 256, 0, st>>>(acc, d, n, out32, out64, param, lr);
  return cudaGetLastError();
}

}  // namespace gqb
