// binning_fast.cu -- K2-K4 fast path: stable counting sort of the (tile, Gaussian) pairs by tile.
//
// The reference composites Gaussians in one global (depth, map index) order
// (proj/src/renderer.cpp:114-117).  After the depth sort (binning.cu), every tile's list must hold
// the Gaussians whose pixel rect overlaps the tile in exactly that order.  Instead of emitting
// (tile, index) pairs and radix-sorting them, the pairs are written straight into place:
//   1. count   : the depth-sorted Gaussians are cut into chunks of kChunk (one CTA); a shared-memory
//                histogram of the tiles each chunk touches is written tile-major, counts[t][c];
//   2. scan    : one exclusive scan over counts (tile-major) gives, for every (tile, chunk), the
//                global slot of that chunk's first pair in that tile -- lists are ordered by tile,
//                then chunk (= depth order); the per-tile ranges are read off the same scan;
//   3. scatter : each warp owns kWarpRun consecutive Gaussians; it counts its own pairs per tile
//                (warp-private table), the CTA turns the warp tables into starting slots, then
//                each warp walks its Gaussians in depth order (lanes = the Gaussian's tiles) and
//                writes each map index once, bumping its table.
// The per-warp Gaussian records are loaded once, coalesced, and broadcast with shuffles, so the
// sequential walks never wait on dependent global loads.  Bytes per pair: one 4 B store (plus
// the per-chunk tables, ~ntiles x V / kChunk x 12 B).  Debug exports rebuild the 64-bit
// (tile << 32 | f32bits(depth)) keys from the ranges, bit-identical to the oracle's stable sort.
#include <cub/device/device_scan.cuh>

#include "lgs_internal.cuh"
#include "lgs_kernels.h"

namespace lgs {

constexpr int kWarpRun = 128;                      // Gaussians per warp
constexpr int kChunkWarps = 4;                     // warps per CTA
constexpr int kChunk = kWarpRun * kChunkWarps;     // Gaussians per CTA chunk
constexpr int kMaxFastTiles = 12288;               // 4 warp tables x 12288 x 4 B = 192 KB shared memory
constexpr int kRegs = kWarpRun / 32;               // preloaded Gaussians per lane

struct WarpGaussians {  // lane l holds Gaussians l, l + 32, l + 64, l + 96 of the warp's run
  uint32_t g[kRegs];
  uint32_t cnt[kRegs];
  uint32_t origin[kRegs];  // tx0 | ty0 << 16
  uint32_t tw[kRegs];
};

__device__ __forceinline__ void load_warp_gaussians(WarpGaussians& w, const uint2* __restrict__ rect,
                                                    const uint32_t* __restrict__ tiles,
                                                    const uint32_t* __restrict__ idx_sorted, int64_t s0, int64_t n,
                                                    int lane) {
#pragma unroll
  for (int r = 0; r < kRegs; ++r) {
    const int64_t s = s0 + r * 32 + lane;
    w.g[r] = 0; w.cnt[r] = 0; w.origin[r] = 0; w.tw[r] = 1;
    if (s < n) {
      const uint32_t g = __ldg(idx_sorted + s);
      const uint32_t c = __ldg(tiles + g);
      w.g[r] = g;
      w.cnt[r] = c;
      if (c) {
        const uint2 rc = __ldg(rect + g);
        const uint32_t tx0 = (rc.x & 0xffffu) / kTile, ty0 = (rc.y & 0xffffu) / kTile;
        w.origin[r] = tx0 | (ty0 << 16);
        w.tw[r] = (rc.x >> 16) / kTile - tx0 + 1;
      }
    }
  }
}

// Visit every (Gaussian, tile) pair of the warp's run in depth order; f(g, tile) is called by the
// lanes of one Gaussian at a time (distinct tiles), with a __syncwarp between Gaussians.
template <typename F>
__device__ __forceinline__ void for_each_pair(const WarpGaussians& w, int lane, int tiles_x, F&& f) {
#pragma unroll
  for (int r = 0; r < kRegs; ++r) {
    for (int j = 0; j < 32; ++j) {
      const uint32_t cnt = __shfl_sync(0xffffffffu, w.cnt[r], j);
      if (cnt == 0) return;  // culled Gaussians sort last (depth key 0xffffffff)
      const uint32_t g = __shfl_sync(0xffffffffu, w.g[r], j);
      const uint32_t org = __shfl_sync(0xffffffffu, w.origin[r], j);
      const uint32_t tw = __shfl_sync(0xffffffffu, w.tw[r], j);
      for (uint32_t i = lane; i < cnt; i += 32) {
        const uint32_t ry = i / tw;
        f(g, ((org >> 16) + ry) * (uint32_t)tiles_x + (org & 0xffffu) + (i - ry * tw));
      }
      __syncwarp();
    }
  }
}

__global__ void __launch_bounds__(kChunkWarps * 32) tile_count_kernel(const uint2* __restrict__ rect,
                                                                       const uint32_t* __restrict__ tiles,
                                                                       const uint32_t* __restrict__ idx_sorted,
                                                                       int64_t n, int ntiles, int tiles_x, int nchunks,
                                                                       uint32_t* __restrict__ counts) {
  extern __shared__ uint32_t s_hist[];
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) s_hist[t] = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpGaussians w;
  load_warp_gaussians(w, rect, tiles, idx_sorted, (int64_t)blockIdx.x * kChunk + (int64_t)warp * kWarpRun, n, lane);
  __syncthreads();
  for_each_pair(w, lane, tiles_x, [&](uint32_t, uint32_t t) { atomicAdd(&s_hist[t], 1u); });
  __syncthreads();
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) counts[(size_t)t * nchunks + blockIdx.x] = s_hist[t];
}

__global__ void tile_ranges_kernel(const uint32_t* __restrict__ offs, int nchunks, int ntiles, uint32_t pairs,
                                   uint2* __restrict__ ranges) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  const uint32_t b = offs[(size_t)t * nchunks];
  const uint32_t e = t + 1 < ntiles ? offs[(size_t)(t + 1) * nchunks] : pairs;
  ranges[t] = make_uint2(b, e);
}

__global__ void __launch_bounds__(kChunkWarps * 32) tile_scatter_kernel(const uint2* __restrict__ rect,
                                                                         const uint32_t* __restrict__ tiles,
                                                                         const uint32_t* __restrict__ idx_sorted,
                                                                         int64_t n, int ntiles, int tiles_x, int nchunks,
                                                                         const uint32_t* __restrict__ offs,
                                                                         uint32_t* __restrict__ vals) {
  extern __shared__ uint32_t s_tab[];  // [kChunkWarps][ntiles]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* my = s_tab + (size_t)warp * ntiles;
  for (int t = lane; t < ntiles; t += 32) my[t] = 0;
  WarpGaussians w;
  load_warp_gaussians(w, rect, tiles, idx_sorted, (int64_t)blockIdx.x * kChunk + (int64_t)warp * kWarpRun, n, lane);
  __syncwarp();
  // pass 1: this warp's per-tile pair counts (distinct tiles per Gaussian -> no atomics)
  for_each_pair(w, lane, tiles_x, [&](uint32_t, uint32_t t) { my[t] += 1; });
  __syncthreads();
  // per tile: starting slot of each warp = chunk start + counts of the earlier warps
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
    uint32_t run = offs[(size_t)t * nchunks + blockIdx.x];
#pragma unroll
    for (int q = 0; q < kChunkWarps; ++q) {
      const uint32_t c = s_tab[(size_t)q * ntiles + t];
      s_tab[(size_t)q * ntiles + t] = run;
      run += c;
    }
  }
  __syncthreads();
  // pass 2: depth-ordered writes
  for_each_pair(w, lane, tiles_x, [&](uint32_t g, uint32_t t) {
    const uint32_t pos = my[t];
    my[t] = pos + 1;
    vals[pos] = g;
  });
}

bool fast_binning_supported(int ntiles) { return ntiles <= kMaxFastTiles; }

static int nchunks_for(int64_t n) { return (int)((n + kChunk - 1) / kChunk); }

size_t fast_binning_scratch_bytes(int64_t n, int ntiles) {
  const size_t cells = (size_t)nchunks_for(n) * (size_t)ntiles;
  size_t scan = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)cells);
  return sizeof(uint32_t) * cells * 2 + scan + 256;
}

void launch_fast_binning(const ViewBufs& v, const uint32_t* idx_sorted, int64_t n, int ntiles, int tiles_x,
                         uint32_t* scratch, uint32_t* vals, uint2* ranges, uint32_t pairs, cudaStream_t s) {
  if (n == 0 || pairs == 0) {
    cudaMemsetAsync(ranges, 0, sizeof(uint2) * (size_t)ntiles, s);
    return;
  }
  const int nchunks = nchunks_for(n);
  const size_t cells = (size_t)nchunks * (size_t)ntiles;
  uint32_t* counts = scratch;
  uint32_t* offs = scratch + cells;
  void* temp = scratch + 2 * cells;
  size_t temp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, counts, offs, (int)cells);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(tile_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(uint32_t) * kMaxFastTiles));
    cudaFuncSetAttribute(tile_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(uint32_t) * kMaxFastTiles * kChunkWarps));
    attr_set = true;
  }
  const int threads = kChunkWarps * 32;
  tile_count_kernel<<<nchunks, threads, sizeof(uint32_t) * ntiles, s>>>(v.rect, v.tiles, idx_sorted, n, ntiles,
                                                                        tiles_x, nchunks, counts);
  cub::DeviceScan::ExclusiveSum(temp, temp_bytes, counts, offs, (int)cells, s);
  tile_ranges_kernel<<<(ntiles + 255) / 256, 256, 0, s>>>(offs, nchunks, ntiles, pairs, ranges);
  tile_scatter_kernel<<<nchunks, threads, sizeof(uint32_t) * ntiles * kChunkWarps, s>>>(
      v.rect, v.tiles, idx_sorted, n, ntiles, tiles_x, nchunks, offs, vals);
}

}  // namespace lgs
