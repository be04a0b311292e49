// binning_fast.cu -- K2-K4 fast path: stable counting sort of the (tile, Gaussian) pairs by tile.
//
// The reference composites Gaussians in one global (depth, map index) order
// (proj/src/renderer.cpp:114-117).  After the depth sort (binning.cu), every tile's list must hold
// the Gaussians whose pixel rect overlaps the tile in exactly that order.  Instead of emitting
// (tile, index) pairs and radix-sorting them, the pairs are written straight into place.
//
// Conceptually the depth-sorted Gaussians emit a stream of P pairs (each Gaussian its tiles,
// row-major); excl[s] is where Gaussian s starts in that stream.  The stream is cut into chunks
// of kPairsPerChunk pairs (a Gaussian belongs to the chunk its first pair falls in), and each
// chunk into kWarps equal warp slices -- balanced by pairs, not by Gaussians, because the depth
// order puts the large near-camera splats (hundreds of tiles each) first.
//   1. count   : per chunk, a shared-memory histogram of its tiles -> counts[tile][chunk];
//   2. scan    : one exclusive scan over counts (tile-major) gives every (tile, chunk) its first
//                output slot -- lists are ordered by tile, then chunk (= depth order); the tile
//                ranges are read off the same scan;
//   3. scatter : each warp counts its slice per tile (warp-private u16 table), the CTA turns the
//                tables into per-warp starting offsets, then each warp walks its Gaussians in
//                depth order (lanes = the Gaussian's tiles) writing each map index once.
// Warps read their Gaussians' records with coalesced loads, 32 at a time, and broadcast them by
// shuffle, so the sequential walk never waits on dependent global loads.
// Bytes per pair: one 4 B store; plus ~12 B per (tile, chunk) cell for the tables and the scan.
// The debug export rebuilds the 64-bit (tile << 32 | f32bits(depth)) keys from the ranges,
// bit-identical to the oracle's stable sort of those keys.
#include <cub/device/device_scan.cuh>

#include <algorithm>

#include "lgs_internal.cuh"
#include "lgs_kernels.h"

namespace lgs {

constexpr int kWarps = 8;
// Warp slices are balanced by a cost that counts every Gaussian as kGaussCost pairs on top of its
// real pairs: a warp walks one Gaussian per step, so a slice of 1-tile far-away splats costs as
// many sequential steps as a slice of the same pair count in 32-tile near ones would cost in
// pairs / 32.  (Balancing by pairs alone left warps of the depth-order tail with ~1000 steps.)
constexpr int kGaussCost = 32;
constexpr int kCostPerWarp = 2048;
constexpr int kCostPerChunk = kWarps * kCostPerWarp;
constexpr int kMaxFastTiles = 8192;  // warp tables: 8 x 8192 x u16 = 128 KB shared memory

// excl[s] (in place over the gathered counts) and slice_first[w] = first sorted Gaussian whose
// cost offset excl[s] + kGaussCost * s is >= w * kCostPerWarp, for every warp slice w in
// [0, nchunks * kWarps]; culled Gaussians (count 0, sorted last) map past the last slice.
__device__ __forceinline__ int slice_of(uint32_t cnt, uint32_t excl, int64_t s, int nslices) {
  if (!cnt) return nslices;
  const uint64_t cost = (uint64_t)excl + (uint64_t)kGaussCost * (uint64_t)s;
  return (int)min((uint64_t)nslices, cost / kCostPerWarp);
}

// slice_first[w] = first sorted Gaussian with slice_of(s) >= w (slice_of is non-decreasing in s:
// culled Gaussians come last): one binary search per slice, reading the counts from incl only.
// The gathered counts are rewritten in place as exclusive offsets.
__global__ void chunk_bounds_kernel(uint32_t* __restrict__ cnt_to_excl, const uint32_t* __restrict__ incl, int64_t n,
                                    int nslices, uint32_t* __restrict__ slice_first) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= nslices) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      const uint32_t ex = mid ? incl[mid - 1] : 0u;
      if (slice_of(incl[mid] - ex, ex, mid, nslices) >= (int)i) hi = mid;
      else lo = mid + 1;
    }
    slice_first[i] = (uint32_t)lo;
  }
  if (i < n) cnt_to_excl[i] = i ? incl[i - 1] : 0u;
}

// Sorted-Gaussian range [s0, s1) of warp `warp` of chunk `c`.
__device__ __forceinline__ void warp_slice(const uint32_t* __restrict__ slice_first, int c, int warp, uint32_t& s0,
                                           uint32_t& s1) {
  const int w = c * kWarps + warp;
  s0 = __ldg(slice_first + w);
  s1 = __ldg(slice_first + w + 1);
}

// Visit the (Gaussian, tile) pairs of sorted Gaussians [s0, s1) in depth order, one Gaussian per
// warp step: lane l takes column l mod w of rows l / w, l / w + 32 / w, ... of the Gaussian's
// w x h tile rect (the lane's row / column come from one float multiply by 1/w: exact for
// lane < 32, w <= 512), so a Gaussian's lanes hit distinct tiles and f(g, tile) needs no
// atomics or ranking; __syncwarp orders consecutive Gaussians.  The warp's records are loaded
// 32 at a time (coalesced) and broadcast by shuffle.
template <typename F>
__device__ __forceinline__ void for_each_pair(const uint2* __restrict__ rect, const uint32_t* __restrict__ tiles,
                                              const uint32_t* __restrict__ idx_sorted, uint32_t s0, uint32_t s1,
                                              int lane, int tiles_x, F&& f) {
  for (uint32_t b = s0; b < s1; b += 32) {
    const uint32_t s = b + lane;
    uint32_t g = 0, base = 0, wh = 0;  // wh = w | h << 16
    float inv_w = 1.0f;
    if (s < s1) {
      g = __ldg(idx_sorted + s);
      const uint2 rc = __ldg(rect + g);
      const uint32_t tx0 = (rc.x & 0xffffu) / kTile, ty0 = (rc.y & 0xffffu) / kTile;
      const uint32_t w = (rc.x >> 16) / kTile - tx0 + 1, h = (rc.y >> 16) / kTile - ty0 + 1;
      base = ty0 * (uint32_t)tiles_x + tx0;
      wh = w | (h << 16);
      inv_w = 1.0f / (float)w;
    }
    const int nb = (int)min(32u, s1 - b);
    for (int j = 0; j < nb; ++j) {
      const uint32_t gj = __shfl_sync(0xffffffffu, g, j);
      const uint32_t bj = __shfl_sync(0xffffffffu, base, j);
      const uint32_t whj = __shfl_sync(0xffffffffu, wh, j);
      const float iw = __shfl_sync(0xffffffffu, inv_w, j);
      const uint32_t w = whj & 0xffffu, h = whj >> 16;
      if (w <= 32) {
        const uint32_t rpi = __float2uint_rz(32.5f * iw);           // rows per step = 32 / w
        const uint32_t r0 = __float2uint_rz(((float)lane + 0.5f) * iw);  // lane / w
        const uint32_t col = (uint32_t)lane - r0 * w;
        if (r0 < rpi)
          for (uint32_t ry = r0; ry < h; ry += rpi) f(gj, bj + ry * (uint32_t)tiles_x + col);
      } else {
        for (uint32_t ry = 0; ry < h; ++ry)
          for (uint32_t cx = lane; cx < w; cx += 32) f(gj, bj + ry * (uint32_t)tiles_x + cx);
      }
      __syncwarp();
    }
  }
}

__global__ void __launch_bounds__(kWarps * 32) tile_count_kernel(const uint2* __restrict__ rect,
                                                                  const uint32_t* __restrict__ tiles,
                                                                  const uint32_t* __restrict__ idx_sorted,
                                                                  const uint32_t* __restrict__ excl,
                                                                  const uint32_t* __restrict__ chunk_first, int ntiles,
                                                                  int tiles_x, int nchunks,
                                                                  uint32_t* __restrict__ counts) {
  extern __shared__ uint32_t s_hist[];
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) s_hist[t] = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t s0, s1;
  warp_slice(chunk_first, blockIdx.x, warp, s0, s1);
  __syncthreads();
  for_each_pair(rect, tiles, idx_sorted, s0, s1, lane, tiles_x, [&](uint32_t, uint32_t t) { atomicAdd(&s_hist[t], 1u); });
  __syncthreads();
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) counts[(size_t)t * nchunks + blockIdx.x] = s_hist[t];
}

// The pair count P is read on the device (the host sized the buffers from a capacity, not from P).
// P > cap: every list is emptied (the blend kernels then do nothing) and the overflow flag tells the
// host to re-run the binning with exact buffers.
__global__ void tile_ranges_kernel(const uint32_t* __restrict__ offs, int nchunks, int ntiles,
                                   const uint32_t* __restrict__ dev_pairs, uint32_t cap,
                                   uint32_t* __restrict__ overflow, uint2* __restrict__ ranges) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  const uint32_t pairs = *dev_pairs;
  if (pairs > cap) {
    ranges[t] = make_uint2(0u, 0u);
    if (t == 0) *overflow = 1u;
    return;
  }
  if (t == 0) *overflow = 0u;
  const uint32_t b = offs[(size_t)t * nchunks];
  const uint32_t e = t + 1 < ntiles ? offs[(size_t)(t + 1) * nchunks] : pairs;
  ranges[t] = make_uint2(b, e);
}

__global__ void __launch_bounds__(kWarps * 32) tile_scatter_kernel(const uint2* __restrict__ rect,
                                                                    const uint32_t* __restrict__ tiles,
                                                                    const uint32_t* __restrict__ idx_sorted,
                                                                    const uint32_t* __restrict__ excl,
                                                                    const uint32_t* __restrict__ chunk_first,
                                                                    int ntiles, int tiles_x, int nchunks,
                                                                    const uint32_t* __restrict__ offs,
                                                                    uint32_t cap, uint32_t* __restrict__ vals) {
  extern __shared__ uint32_t s_dyn[];
  uint32_t* s_coff = s_dyn;                                       // [ntiles] chunk start slot per tile
  uint16_t* s_tab = reinterpret_cast<uint16_t*>(s_dyn + ntiles);  // [kWarps][ntiles] offsets within chunk
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint16_t* my = s_tab + (size_t)warp * ntiles;
  for (int t = lane; t < ntiles; t += 32) my[t] = 0;
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) s_coff[t] = offs[(size_t)t * nchunks + blockIdx.x];
  uint32_t s0, s1;
  warp_slice(chunk_first, blockIdx.x, warp, s0, s1);
  __syncwarp();
  // pass 1: this warp's per-tile pair counts (distinct tiles per step: no atomics, u16 table)
  for_each_pair(rect, tiles, idx_sorted, s0, s1, lane, tiles_x,
                [&](uint32_t, uint32_t t) { my[t] = (uint16_t)(my[t] + 1); });
  __syncthreads();
  // per tile: offset of each warp within the chunk = counts of the earlier warps
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
    uint32_t run = 0;
#pragma unroll
    for (int q = 0; q < kWarps; ++q) {
      const uint32_t c = s_tab[(size_t)q * ntiles + t];
      s_tab[(size_t)q * ntiles + t] = (uint16_t)run;
      run += c;
    }
  }
  __syncthreads();
  // pass 2: depth-ordered writes (one Gaussian per step, consecutive steps ordered by __syncwarp)
  for_each_pair(rect, tiles, idx_sorted, s0, s1, lane, tiles_x, [&](uint32_t g, uint32_t t) {
    const uint32_t r = my[t];
    my[t] = (uint16_t)(r + 1);
    const uint32_t slot = s_coff[t] + r;
    if (slot < cap) vals[slot] = g;
  });
}

// One CTA: order tiles by decreasing list length, bucketed by floor(log2(length)) (approximate
// longest-processing-time-first order for the blend kernels' persistent scheduler; the order
// inside a bucket is arbitrary and does not affect any result).
__global__ void __launch_bounds__(1024) tile_order_kernel(const uint2* __restrict__ ranges, int ntiles,
                                                          uint32_t* __restrict__ order) {
  __shared__ uint32_t s_cnt[33];
  __shared__ uint32_t s_pos[33];
  if (threadIdx.x < 33) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
    const uint2 r = ranges[t];
    const uint32_t len = r.y - r.x;
    atomicAdd(&s_cnt[len ? 32 - __clz(len) : 0], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (int b = 32; b >= 0; --b) {  // longest bucket first
      s_pos[b] = run;
      run += s_cnt[b];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
    const uint2 r = ranges[t];
    const uint32_t len = r.y - r.x;
    order[atomicAdd(&s_pos[len ? 32 - __clz(len) : 0], 1u)] = (uint32_t)t;
  }
}

void launch_tile_order(const uint2* ranges, int ntiles, uint32_t* order, cudaStream_t s) {
  tile_order_kernel<<<1, 1024, 0, s>>>(ranges, ntiles, order);
}

bool fast_binning_supported(int ntiles) { return ntiles <= kMaxFastTiles; }

// chunks covering the largest possible total cost: P <= pairs, at most n Gaussians with pairs
static int nchunks_for(int64_t pairs, int64_t n) {
  const int64_t cost = pairs + (int64_t)kGaussCost * std::min(n, pairs);
  return (int)((cost + kCostPerChunk - 1) / kCostPerChunk);
}

size_t fast_binning_scratch_bytes(int64_t pairs, int64_t n, int ntiles) {
  const int nchunks = nchunks_for(pairs, n);
  const size_t cells = (size_t)nchunks * (size_t)ntiles;
  size_t scan = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)cells);
  return sizeof(uint32_t) * (cells * 2 + (size_t)nchunks * kWarps + 1) + scan + 256;
}

void launch_fast_binning(const ViewBufs& v, const uint32_t* idx_sorted, uint32_t* cnt_sorted, const uint32_t* incl,
                         int64_t n, int ntiles, int tiles_x, uint32_t* scratch, uint32_t* vals, uint2* ranges,
                         uint32_t cap, const uint32_t* dev_pairs, uint32_t* dev_overflow, cudaStream_t s) {
  if (n == 0 || cap == 0) {
    cudaMemsetAsync(ranges, 0, sizeof(uint2) * (size_t)ntiles, s);
    cudaMemsetAsync(dev_overflow, 0, sizeof(uint32_t), s);
    return;
  }
  const int nchunks = nchunks_for(cap, n);
  const size_t cells = (size_t)nchunks * (size_t)ntiles;
  uint32_t* counts = scratch;
  uint32_t* offs = counts + cells;
  uint32_t* chunk_first = offs + cells;
  void* temp = chunk_first + nchunks * kWarps + 1;
  size_t temp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, counts, offs, (int)cells);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(tile_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(uint32_t) * kMaxFastTiles));
    cudaFuncSetAttribute(tile_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(uint32_t) * kMaxFastTiles + sizeof(uint16_t) * kMaxFastTiles * kWarps));
    attr_set = true;
  }
  const uint32_t* excl = cnt_sorted;  // rewritten in place by chunk_bounds_kernel
  const int64_t nb_threads = std::max<int64_t>(n, (int64_t)nchunks * kWarps + 1);
  chunk_bounds_kernel<<<(unsigned)((nb_threads + 255) / 256), 256, 0, s>>>(cnt_sorted, incl, n, nchunks * kWarps,
                                                                           chunk_first);
  const int threads = kWarps * 32;
  tile_count_kernel<<<nchunks, threads, sizeof(uint32_t) * ntiles, s>>>(v.rect, v.tiles, idx_sorted, excl, chunk_first,
                                                                        ntiles, tiles_x, nchunks, counts);
  cub::DeviceScan::ExclusiveSum(temp, temp_bytes, counts, offs, (int)cells, s);
  tile_ranges_kernel<<<(ntiles + 255) / 256, 256, 0, s>>>(offs, nchunks, ntiles, dev_pairs, cap, dev_overflow, ranges);
  tile_scatter_kernel<<<nchunks, threads, sizeof(uint32_t) * ntiles + sizeof(uint16_t) * ntiles * kWarps, s>>>(
      v.rect, v.tiles, idx_sorted, excl, chunk_first, ntiles, tiles_x, nchunks, offs, cap, vals);
}

}  // namespace lgs
