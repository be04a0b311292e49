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
#include "dev_cache.h"

namespace lgs {

constexpr int kWarps = 8;
// Warp slices are balanced by a cost that counts every Gaussian as kGaussCost pairs on top of its
// real pairs: a warp walks one Gaussian per step, so a slice of 1-tile far-away splats costs as
// many sequential steps as a slice of the same pair count in 32-tile near ones would cost in
// pairs / 32.  (Balancing by pairs alone left warps of the depth-order tail with ~1000 steps.)
// The cost per warp slice adapts to the pass size (cost_per_warp below): ~4 CTAs per SM, slices of
// 128 .. 2048 cost units.
constexpr int kGaussCost = 32;
constexpr int kMinCostPerWarp = 128, kMaxCostPerWarp = 2048;
constexpr int kMaxFastTiles = 8192;  // warp tables: 8 x 8192 x u16 = 128 KB shared memory

// Inclusive pair count of depth-order Gaussian s in this pass: layer A clamps the full counts at
// its pair total (Gaussians past the cut own nothing).
__device__ __forceinline__ uint32_t pass_incl(const uint32_t* __restrict__ incl, const uint32_t* __restrict__ clamp,
                                              int64_t s) {
  const uint32_t v = __ldg(incl + s);
  return clamp ? min(v, *clamp) : v;
}

// The pass's pairs laid out on a cost axis: Gaussian s occupies [cs(s), cs(s + 1)) with
// cs(s) = excl(s) + kGaussCost * s -- kGaussCost units of per-Gaussian overhead, then one unit per
// pair.  Warp slice w owns the pairs whose cost lies in [w cpw, (w + 1) cpw): a splat covering
// the whole screen is split over several warps, and a run of 1-tile splats costs a warp as many
// units as the sequential steps it takes.  end_key(s) = cs(s + 1), or "infinite" after the last
// Gaussian owning pairs (so trailing pair-less ones are never visited).
__device__ __forceinline__ uint64_t end_key(const uint32_t* __restrict__ incl, const uint32_t* __restrict__ clamp,
                                            int64_t s, uint32_t total) {
  const uint32_t ex = s ? pass_incl(incl, clamp, s - 1) : 0u;
  if (ex >= total) return ~0ull;
  return (uint64_t)pass_incl(incl, clamp, s) + (uint64_t)kGaussCost * (uint64_t)(s + 1);
}

// slice_first[w] = first Gaussian s with end_key(s) > w * cpw (the one holding the slice's first
// cost unit): one warp per slice, a 32-ary search (4 dependent probes for 500k Gaussians).
__global__ void chunk_bounds_kernel(const uint32_t* __restrict__ incl, const uint32_t* __restrict__ clamp, int64_t n,
                                    int nslices, uint32_t cpw, uint32_t* __restrict__ slice_first) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w > nslices) return;
  const uint32_t total = pass_incl(incl, clamp, n - 1);
  const uint64_t target = (uint64_t)w * cpw;
  int64_t lo = 0, hi = n;  // answer in [lo, hi]; end_key(hi) > target or hi == n
  while (hi - lo > 32) {
    const int64_t stride = (hi - lo + 31) / 32;
    const int64_t p = min(lo + stride * (lane + 1) - 1, hi - 1);
    const unsigned hit = __ballot_sync(0xffffffffu, end_key(incl, clamp, p, total) > target);
    if (hit) {
      const int f = __ffs(hit) - 1;
      const int64_t pf = __shfl_sync(0xffffffffu, p, f);
      const int64_t pp = __shfl_sync(0xffffffffu, p, f > 0 ? f - 1 : 0);
      lo = f > 0 ? pp + 1 : lo;
      hi = pf;
    } else {
      lo = __shfl_sync(0xffffffffu, p, 31) + 1;
    }
  }
  const int64_t p = lo + lane;
  const unsigned hit = __ballot_sync(0xffffffffu, p < hi && end_key(incl, clamp, p, total) > target);
  if (lane == 0) slice_first[w] = (uint32_t)(hit ? lo + __ffs(hit) - 1 : hi);
}

// Visit the (Gaussian, tile) pairs of warp slice `wslice` in depth order: Gaussians
// slice_first[w] .. slice_first[w + 1] (both ends may be partial), each one's pair range clipped to
// the slice's cost window.  Pair k of a Gaussian is tile (k / w, k mod w) of its w x h tile rect
// (row-major, the float reciprocal of w gives the exact quotient for k, w < 2^13); the lanes of a
// step take 32 consecutive pairs of ONE Gaussian, so they hit distinct tiles and f(g, tile) needs
// no atomics or ranking, and __syncwarp orders consecutive Gaussians.  The warp's records are
// loaded 32 at a time (coalesced) and broadcast by shuffle.
template <typename F>
__device__ __forceinline__ void for_each_pair(const uint2* __restrict__ rect, const uint32_t* __restrict__ incl,
                                              const uint32_t* __restrict__ clamp,
                                              const uint32_t* __restrict__ idx_sorted,
                                              const uint32_t* __restrict__ slice_first, int wslice, uint32_t cpw,
                                              int64_t n, int lane, int tiles_x, F&& f) {
  const int64_t s0 = __ldg(slice_first + wslice);
  const int64_t s_last = min((int64_t)__ldg(slice_first + wslice + 1), n - 1);
  const int64_t c0 = (int64_t)wslice * cpw, c1 = c0 + cpw;
  for (int64_t b = s0; b <= s_last; b += 32) {
    const int64_t s = b + lane;
    uint32_t g = 0, base = 0, w = 1, kk = 0;  // kk = k0 | k1 << 16 (pair range in this slice)
    float inv_w = 1.0f;
    if (s <= s_last) {
      const uint32_t ex = s ? pass_incl(incl, clamp, s - 1) : 0u;
      const int64_t cnt = (int64_t)pass_incl(incl, clamp, s) - ex;
      const int64_t cs = (int64_t)ex + (int64_t)kGaussCost * (s + 1);  // cost of pair 0
      const int64_t k0 = max((int64_t)0, min(cnt, c0 - cs)), k1 = max((int64_t)0, min(cnt, c1 - cs));
      if (k1 > k0) {
        g = __ldg(idx_sorted + s);
        const uint2 rc = __ldg(rect + g);
        const uint32_t tx0 = (rc.x & 0xffffu) / kTile, ty0 = (rc.y & 0xffffu) / kTile;
        w = (rc.x >> 16) / kTile - tx0 + 1;
        base = ty0 * (uint32_t)tiles_x + tx0;
        inv_w = 1.0f / (float)w;
        kk = (uint32_t)k0 | ((uint32_t)k1 << 16);
      }
    }
    const int nb = (int)min((int64_t)32, s_last - b + 1);
    for (int j = 0; j < nb; ++j) {
      const uint32_t kkj = __shfl_sync(0xffffffffu, kk, j);
      if (!kkj) continue;  // warp-uniform: no pairs of this Gaussian in this slice
      const uint32_t gj = __shfl_sync(0xffffffffu, g, j);
      const uint32_t bj = __shfl_sync(0xffffffffu, base, j);
      const uint32_t wj = __shfl_sync(0xffffffffu, w, j);
      const float iw = __shfl_sync(0xffffffffu, inv_w, j);
      const uint32_t k1 = kkj >> 16;
      for (uint32_t k = (kkj & 0xffffu) + (uint32_t)lane; k < k1; k += 32) {
        const uint32_t ry = __float2uint_rz(((float)k + 0.5f) * iw);
        const uint32_t cx = k - ry * wj;
        f(gj, bj + ry * (uint32_t)tiles_x + cx);
      }
      __syncwarp();
    }
  }
}

template <bool MASKED>
__global__ void __launch_bounds__(kWarps * 32) tile_count_kernel(const uint2* __restrict__ rect,
                                                                  const uint32_t* __restrict__ incl,
                                                                  const uint32_t* __restrict__ clamp,
                                                                  const uint32_t* __restrict__ idx_sorted,
                                                                  const uint32_t* __restrict__ chunk_first,
                                                                  const uint32_t* __restrict__ mask,
                                                                  const uint32_t* __restrict__ active, int ntiles,
                                                                  int tiles_x, int nchunks, uint32_t cpw, int64_t n,
                                                                  uint32_t* __restrict__ counts) {
  if (MASKED && !*active) return;  // second layered pass with every tile saturated: nothing to bin
  extern __shared__ uint32_t s_hist[];
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) s_hist[t] = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  for_each_pair(rect, incl, clamp, idx_sorted, chunk_first, blockIdx.x * kWarps + warp, cpw, n, lane, tiles_x,
                [&](uint32_t, uint32_t t) {
    if (!MASKED || __ldg(mask + t)) atomicAdd(&s_hist[t], 1u);
  });
  __syncthreads();
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) counts[(size_t)t * nchunks + blockIdx.x] = s_hist[t];
}

// The pair count P is read on the device (the host sized the buffers from a capacity, not from P).
// P > cap: every list is emptied (the blend kernels then do nothing) and the overflow flag tells the
// host to re-run the binning with exact buffers.
// With a tile mask (the second pass of the depth-layered binning) only the masked tiles' ranges are
// (re)written, offset by `base`; P > cap empties them.
__global__ void tile_ranges_kernel(const uint32_t* __restrict__ offs, int nchunks, int ntiles,
                                   const uint32_t* __restrict__ dev_pairs, uint32_t cap, uint32_t base,
                                   const uint32_t* __restrict__ mask, uint32_t* __restrict__ overflow,
                                   uint2* __restrict__ ranges) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  const uint32_t pairs = *dev_pairs;
  if (pairs > cap) {
    if (t == 0) *overflow = 1u;
    if (!mask || mask[t]) ranges[t] = make_uint2(0u, 0u);
    return;
  }
  if (t == 0) *overflow = 0u;
  if (mask && !mask[t]) return;
  const uint32_t b = offs[(size_t)t * nchunks];
  const uint32_t e = t + 1 < ntiles ? offs[(size_t)(t + 1) * nchunks] : pairs;
  ranges[t] = make_uint2(base + b, base + e);
}

template <bool MASKED>
__global__ void __launch_bounds__(kWarps * 32) tile_scatter_kernel(const uint2* __restrict__ rect,
                                                                    const uint32_t* __restrict__ incl,
                                                                    const uint32_t* __restrict__ clamp,
                                                                    const uint32_t* __restrict__ idx_sorted,
                                                                    const uint32_t* __restrict__ chunk_first,
                                                                    const uint32_t* __restrict__ mask,
                                                                    const uint32_t* __restrict__ active,
                                                                    int ntiles, int tiles_x, int nchunks, uint32_t cpw,
                                                                    int64_t n, const uint32_t* __restrict__ offs,
                                                                    uint32_t cap, uint32_t* __restrict__ vals) {
  if (MASKED && !*active) return;
  extern __shared__ uint32_t s_dyn[];
  uint32_t* s_coff = s_dyn;                                       // [ntiles] chunk start slot per tile
  uint16_t* s_tab = reinterpret_cast<uint16_t*>(s_dyn + ntiles);  // [kWarps][ntiles] offsets within chunk
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint16_t* my = s_tab + (size_t)warp * ntiles;
  for (int t = lane; t < ntiles; t += 32) my[t] = 0;
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) s_coff[t] = offs[(size_t)t * nchunks + blockIdx.x];
  const int ws = blockIdx.x * kWarps + warp;
  __syncwarp();
  // pass 1: this warp's per-tile pair counts (distinct tiles per step: no atomics, u16 table)
  for_each_pair(rect, incl, clamp, idx_sorted, chunk_first, ws, cpw, n, lane, tiles_x, [&](uint32_t, uint32_t t) {
    if (!MASKED || __ldg(mask + t)) my[t] = (uint16_t)(my[t] + 1);
  });
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
  for_each_pair(rect, incl, clamp, idx_sorted, chunk_first, ws, cpw, n, lane, tiles_x, [&](uint32_t g, uint32_t t) {
    if (MASKED && !__ldg(mask + t)) return;
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

// Largest possible total cost: at most `pairs` pairs, owned by at most min(gauss, pairs) Gaussians.
static int64_t cost_bound(int64_t pairs, int64_t gauss) { return pairs + (int64_t)kGaussCost * (gauss + 1); }

// cost units per warp slice: ~4 CTAs of kWarps warps per SM over the bound, power of two in range
static uint32_t cost_per_warp(int64_t pairs, int64_t gauss) {
  const int64_t want = cost_bound(pairs, gauss) / (148 * 4 * kWarps);
  uint32_t c = kMinCostPerWarp;
  while (c < (uint32_t)kMaxCostPerWarp && (int64_t)c < want) c <<= 1;
  return c;
}

static int nchunks_for(int64_t pairs, int64_t gauss) {
  const int64_t per_chunk = (int64_t)kWarps * cost_per_warp(pairs, gauss);
  return (int)((cost_bound(pairs, gauss) + per_chunk - 1) / per_chunk);
}

size_t fast_binning_scratch_bytes(int64_t pairs, int64_t gauss, int ntiles) {
  const int nchunks = nchunks_for(pairs, gauss);
  const size_t cells = (size_t)nchunks * (size_t)ntiles;
  size_t scan = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)cells);
  return sizeof(uint32_t) * (cells * 2 + (size_t)nchunks * kWarps + 1) + scan + 256;
}

void launch_fast_binning(const ViewBufs& v, const uint32_t* idx_sorted, int64_t n, int ntiles, int tiles_x,
                         const BinPass& bp, uint32_t* scratch, uint32_t* vals, uint2* ranges, uint32_t* dev_overflow,
                         cudaStream_t s) {
  if (n == 0 || bp.cap == 0) {
    if (!bp.mask) cudaMemsetAsync(ranges, 0, sizeof(uint2) * (size_t)ntiles, s);
    cudaMemsetAsync(dev_overflow, 0, sizeof(uint32_t), s);
    return;
  }
  const int nchunks = nchunks_for(bp.cap, bp.gauss_cap);
  const size_t cells = (size_t)nchunks * (size_t)ntiles;
  uint32_t* counts = scratch;
  uint32_t* offs = counts + cells;
  uint32_t* chunk_first = offs + cells;
  void* temp = chunk_first + nchunks * kWarps + 1;
  size_t temp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, counts, offs, (int)cells);
  {
    const int cnt_smem = (int)(sizeof(uint32_t) * kMaxFastTiles);
    const int sct_smem = (int)(sizeof(uint32_t) * kMaxFastTiles + sizeof(uint16_t) * kMaxFastTiles * kWarps);
    ensure_dyn_smem(reinterpret_cast<const void*>(tile_count_kernel<false>), cnt_smem);
    ensure_dyn_smem(reinterpret_cast<const void*>(tile_count_kernel<true>), cnt_smem);
    ensure_dyn_smem(reinterpret_cast<const void*>(tile_scatter_kernel<false>), sct_smem);
    ensure_dyn_smem(reinterpret_cast<const void*>(tile_scatter_kernel<true>), sct_smem);
  }
  const int nslices = nchunks * kWarps;
  const uint32_t cpw = cost_per_warp(bp.cap, bp.gauss_cap);
  chunk_bounds_kernel<<<(unsigned)((32 * (int64_t)(nslices + 1) + 255) / 256), 256, 0, s>>>(bp.incl, bp.clamp, n,
                                                                                           nslices, cpw, chunk_first);
  const int threads = kWarps * 32;
  const size_t cnt_smem = sizeof(uint32_t) * ntiles;
  const size_t sct_smem = sizeof(uint32_t) * ntiles + sizeof(uint16_t) * ntiles * kWarps;
  if (bp.mask)
    tile_count_kernel<true><<<nchunks, threads, cnt_smem, s>>>(v.rect, bp.incl, bp.clamp, idx_sorted, chunk_first, bp.mask, bp.active,
                                                                ntiles, tiles_x, nchunks, cpw, n, counts);
  else
    tile_count_kernel<false><<<nchunks, threads, cnt_smem, s>>>(v.rect, bp.incl, bp.clamp, idx_sorted, chunk_first, nullptr, nullptr,
                                                                 ntiles, tiles_x, nchunks, cpw, n, counts);
  cub::DeviceScan::ExclusiveSum(temp, temp_bytes, counts, offs, (int)cells, s);
  tile_ranges_kernel<<<(ntiles + 255) / 256, 256, 0, s>>>(offs, nchunks, ntiles, bp.dev_pairs, bp.cap, bp.base,
                                                          bp.mask, dev_overflow, ranges);
  uint32_t* out = vals + bp.base;
  if (bp.mask)
    tile_scatter_kernel<true><<<nchunks, threads, sct_smem, s>>>(v.rect, bp.incl, bp.clamp, idx_sorted, chunk_first, bp.mask, bp.active,
                                                                  ntiles, tiles_x, nchunks, cpw, n, offs, bp.cap, out);
  else
    tile_scatter_kernel<false><<<nchunks, threads, sct_smem, s>>>(v.rect, bp.incl, bp.clamp, idx_sorted, chunk_first, nullptr, nullptr,
                                                                   ntiles, tiles_x, nchunks, cpw, n, offs, bp.cap, out);
}

// ------------------------------------------------------------------------------------------
// Depth-layered binning.  A pixel stops compositing once T < T_min (renderer.cpp:140), and in a
// dense map every tile saturates on its nearest few hundred splats: at the headline config all 1200
// tiles are saturated by the nearest 0.4% of the visible Gaussians, whose lists hold ~5% of the
// 7.6M pairs.  So the lists are built in two passes:
//   1. layer A = the depth-order prefix owning ~P / kLayerDiv pairs (depth_order.cu orders only
//      these and builds their per-tile lists: one warp per tile compacts the candidates in
//      order), blended for every tile; a tile whose every pixel saturates is final (its list is an
//      exact prefix of the complete list, and no later Gaussian can change any of its pixels or
//      gradients);
//   2. the complete lists of the remaining (unfinished) tiles only: the Gaussians' counts are
//      restricted to those tiles through a summed-area table of the unfinished-tile mask, binned
//      after layer A's lists, then blended again from scratch.
// Images, gradients and every list entry a kernel reads are identical to the single-pass binning.
// ------------------------------------------------------------------------------------------
size_t layer_a_cap(int64_t pairs_cap, int ntiles, uint32_t div) {
  return (size_t)std::max<int64_t>(std::min<int64_t>(pairs_cap, kLayerMinPairs), pairs_cap / div) + ntiles + 1024;
}


// Copies up to 4 device counters into page-locked host memory mapped into the device: posted PCIe
// writes from the SMs, so a tiny readback never queues behind another context's bulk copy in the
// copy engines (the host reads them once an event after this kernel has completed).
__global__ void publish_counters_kernel(CounterSrc c, uint32_t* dst) {
  if ((int)threadIdx.x < c.n) {
    reinterpret_cast<volatile uint32_t*>(dst)[threadIdx.x] = *c.src[threadIdx.x];
    __threadfence_system();
  }
}

void launch_publish_counters(const CounterSrc& c, uint32_t* dst_mapped, cudaStream_t s) {
  publish_counters_kernel<<<1, 32, 0, s>>>(c, dst_mapped);
}

// One CTA: the number of unfinished tiles, and inside a captured plan the conditional that runs the
// second pass only when there is one.
__global__ void __launch_bounds__(1024) layer_flag_kernel(const uint32_t* __restrict__ unfinished, int ntiles,
                                                          uint32_t* __restrict__ count2, uint32_t* __restrict__ total2,
                                                          cudaGraphConditionalHandle cond, int use_cond) {
  griddep_wait();
  __shared__ uint32_t s_w[32];
  uint32_t c = 0;
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) c += unfinished[t] ? 1u : 0u;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += s_w[w];
    *count2 = tot;
    *total2 = 0u;
    if (use_cond) cudaGraphSetConditional(cond, tot ? 1u : 0u);
  }
}

void launch_layer_flag(const uint32_t* unfinished, int ntiles, uint32_t* count2, uint32_t* total2,
                       const cudaGraphConditionalHandle* cond, cudaStream_t s) {
  launch_pdl(layer_flag_kernel, dim3(1), dim3(1024), 0, s, unfinished, ntiles, count2, total2,
             cond ? *cond : cudaGraphConditionalHandle{}, cond ? 1 : 0);
}

// One CTA (first kernel of the second pass): unfinished-tile summed-area table
// sat[(ty + 1) * (tiles_x + 1) + tx + 1] and the unfinished tiles in longest-list-first order.
__global__ void __launch_bounds__(1024) layer_prep_kernel(const uint32_t* __restrict__ unfinished,
                                                          const uint2* __restrict__ ranges, int tiles_x, int tiles_y,
                                                          uint32_t* __restrict__ sat, uint32_t* __restrict__ order2) {
  extern __shared__ uint32_t s_sat[];  // (tiles_y + 1) x (tiles_x + 1)
  const int ntiles = tiles_x * tiles_y;
  const int sw = tiles_x + 1, nsat = sw * (tiles_y + 1);
  __shared__ uint32_t s_cnt[33], s_pos[33];
  if (threadIdx.x < 33) s_cnt[threadIdx.x] = 0;
  for (int i = threadIdx.x; i < nsat; i += blockDim.x) {
    const int y = i / sw, x = i - y * sw;
    s_sat[i] = (x && y && unfinished[(y - 1) * tiles_x + x - 1]) ? 1u : 0u;
  }
  __syncthreads();
  for (int y = 1 + (int)threadIdx.x; y <= tiles_y; y += blockDim.x)  // prefix along x
    for (int x = 1; x <= tiles_x; ++x) s_sat[y * sw + x] += s_sat[y * sw + x - 1];
  __syncthreads();
  for (int x = 1 + (int)threadIdx.x; x <= tiles_x; x += blockDim.x)  // then along y
    for (int y = 1; y <= tiles_y; ++y) s_sat[y * sw + x] += s_sat[(y - 1) * sw + x];
  __syncthreads();
  for (int i = threadIdx.x; i < nsat; i += blockDim.x) sat[i] = s_sat[i];
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
    if (!unfinished[t]) continue;
    const uint32_t len = ranges[t].y - ranges[t].x;
    atomicAdd(&s_cnt[len ? 32 - __clz(len) : 0], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (int b = 32; b >= 0; --b) {
      s_pos[b] = run;
      run += s_cnt[b];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
    if (!unfinished[t]) continue;
    const uint32_t len = ranges[t].y - ranges[t].x;
    order2[atomicAdd(&s_pos[len ? 32 - __clz(len) : 0], 1u)] = (uint32_t)t;
  }
}

void launch_layer_prep(const uint32_t* unfinished, const uint2* ranges, int tiles_x, int tiles_y, uint32_t* sat,
                       uint32_t* order2, cudaStream_t s) {
  const size_t smem = sizeof(uint32_t) * (size_t)(tiles_x + 1) * (tiles_y + 1);
  ensure_dyn_smem(reinterpret_cast<const void*>(layer_prep_kernel), (int)(sizeof(uint32_t) * 9 * 1024 * 4));
  layer_prep_kernel<<<1, 1024, smem, s>>>(unfinished, ranges, tiles_x, tiles_y, sat, order2);
}

// Second layered pass: Gaussian s (depth order) takes part iff its tile rect holds an unfinished
// tile (summed-area table); it is then enumerated over its whole rect with the tile mask
// (cnt_enum[s] = its full tile count, else 0), and *total2 accumulates the pairs it emits.
__global__ void __launch_bounds__(256) layer_count_kernel(const uint2* __restrict__ rect,
                                                          const uint32_t* __restrict__ tiles,
                                                          const uint32_t* __restrict__ idx_sorted, int64_t n,
                                                          int tiles_x, const uint32_t* __restrict__ sat,
                                                          const uint32_t* __restrict__ count2,
                                                          uint32_t* __restrict__ cnt_enum,
                                                          uint32_t* __restrict__ total2,
                                                          uint8_t* __restrict__ active,
                                                          float* __restrict__ gacc_zero, ColorJob cj) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t c = 0, e = 0;
  if (s < n && *count2) {
    const uint32_t g = idx_sorted[s];
    const uint32_t tc = tiles[g];
    if (tc) {
      const uint2 rc = rect[g];
      const uint32_t tx0 = (rc.x & 0xffffu) / kTile, tx1 = (rc.x >> 16) / kTile + 1;
      const uint32_t ty0 = (rc.y & 0xffffu) / kTile, ty1 = (rc.y >> 16) / kTile + 1;
      const uint32_t sw = (uint32_t)tiles_x + 1;
      c = sat[ty1 * sw + tx1] - sat[ty0 * sw + tx1] - sat[ty1 * sw + tx0] + sat[ty0 * sw + tx0];
      e = c ? tc : 0u;
      if (c && cj.color && (!active || !active[g])) color_job_run(cj, g);  // first listed here
      if (c && active && !active[g]) {  // listed for an unfinished tile: may receive gradients
        active[g] = 1;
        if (gacc_zero) {  // fused step: its accumulator row is zeroed here (layer-A rows already were)
          float4* row = reinterpret_cast<float4*>(gacc_zero + (size_t)g * 32);
#pragma unroll
          for (int q = 0; q < 8; ++q) row[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    }
  }
  if (s < n) cnt_enum[s] = e;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(total2, c);
}

void launch_layer_count(const ViewBufs& v, const uint32_t* idx_sorted, int64_t n, int tiles_x, const uint32_t* sat,
                        const uint32_t* count2, uint32_t* cnt_enum, uint32_t* total2, cudaStream_t s,
                        float* gacc_zero, const ColorJob& cj) {
  if (n == 0) return;
  layer_count_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(v.rect, v.tiles, idx_sorted, n, tiles_x, sat, count2,
                                                                 cnt_enum, total2, v.active, gacc_zero, cj);
}

}  // namespace lgs
