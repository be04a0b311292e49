// binning.cu -- K2 (scan + key duplication), K3 (radix sorts) and K4 (tile ranges).
//
// The reference sorts all projected Gaussians once by (depth, map index)
// (proj/src/renderer.cpp:114-117) and composites each Gaussian over its pixel rect.  The tile
// rasterizer needs, per 16x16 tile, the list of Gaussians whose pixel rect overlaps it, in that
// same (depth, index) order.  It is built in two sorts instead of one 64-bit (tile|depth) sort:
//   1. a stable radix sort of the N 32-bit depth keys (f32 bits; culled = 0xffffffff), values =
//      map index in ascending order, so ties keep index order (renderer.cpp:116);
//   2. a scan of tiles-touched in that order and the duplication of one (tile id, index) pair per
//      overlapped tile, emitted in depth order;
//   3. a stable radix sort of the pairs on the ceil(log2(tiles)) tile bits only.
// The result is exactly the stable sort of the (tile << 32 | f32bits(depth)) keys (the debug
// export rebuilds those 64-bit keys for the bit-exact test) but moves 6 B per pair per pass over
// 1-2 passes instead of 12 B over 5-6.
// Roofline: HBM-bound.  Bytes per pair: 6 (emit) + 2 x 12 (sort passes) + 2 (ranges).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>

#include "lgs_internal.cuh"
#include "lgs_kernels.h"

namespace lgs {

size_t binning_temp_bytes(int64_t n, int64_t pairs_cap, int tile_bits) {
  size_t a = 0, b = 0, c = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (uint32_t*)nullptr, (uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (int)n, 0, 32);
  cub::DeviceScan::InclusiveSum(nullptr, b, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)n);
  cub::DeviceRadixSort::SortPairs(nullptr, c, (uint16_t*)nullptr, (uint16_t*)nullptr, (uint32_t*)nullptr,
                                  (uint32_t*)nullptr, (int)pairs_cap, 0, tile_bits > 0 ? tile_bits : 1);
  size_t m = a > b ? a : b;
  return m > c ? m : c;
}

void launch_depth_sort(const ViewBufs& v, int64_t n, uint32_t* dkey_sorted, uint32_t* idx_sorted, void* temp,
                       size_t temp_bytes, cudaStream_t s) {
  if (n == 0) return;
  cub::DeviceRadixSort::SortPairs(temp, temp_bytes, v.dkey, dkey_sorted, v.iota, idx_sorted, (int)n, 0, 32, s);
}

// out[0] = sum of tiles[0..n) (the pair count P): block reduction + one atomic per block.
__global__ void __launch_bounds__(256) sum_tiles_kernel(const uint32_t* __restrict__ tiles, int64_t n,
                                                        uint32_t* __restrict__ out) {
  __shared__ uint32_t s_w[8];
  uint32_t acc = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc += tiles[i];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < 8; ++w) t += s_w[w];
    atomicAdd(out, t);
  }
}

void launch_sum_tiles(const uint32_t* tiles, int64_t n, uint32_t* out, cudaStream_t s) {
  cudaMemsetAsync(out, 0, sizeof(uint32_t), s);
  if (n == 0) return;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 8);
  sum_tiles_kernel<<<(unsigned)blocks, 256, 0, s>>>(tiles, n, out);
}

__global__ void gather_tiles_kernel(const uint32_t* __restrict__ tiles, const uint32_t* __restrict__ idx_sorted,
                                    int64_t n, uint32_t* __restrict__ out) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n) out[s] = tiles[idx_sorted[s]];
}

// incl[s] = sum_{s' <= s} tiles[idx_sorted[s']]; `scratch` (n u32) receives the gathered counts.
void launch_scan_tiles(const uint32_t* tiles, const uint32_t* idx_sorted, int64_t n, uint32_t* scratch,
                       uint32_t* incl, void* temp, size_t temp_bytes, cudaStream_t s) {
  if (n == 0) return;
  gather_tiles_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(tiles, idx_sorted, n, scratch);
  cub::DeviceScan::InclusiveSum(temp, temp_bytes, scratch, incl, (int)n, s);
}

// incl = inclusive scan of counts already in depth order (depth_order.cu gathers them).
void launch_scan_counts(const uint32_t* cnt_sorted, int64_t n, uint32_t* incl, void* temp, size_t temp_bytes,
                        cudaStream_t s) {
  if (n == 0) return;
  cub::DeviceScan::InclusiveSum(temp, temp_bytes, cnt_sorted, incl, (int)n, s);
}

// Each CTA owns 256 consecutive depth-sorted Gaussians and writes their pairs cooperatively:
// thread t handles output slots chunk_begin + t, + 256, ... and finds the owning Gaussian by a
// binary search over the chunk's inclusive offsets in shared memory, so the key/value stores of a
// warp are consecutive (coalesced) however unevenly the Gaussians' tile counts are spread.  Tile
// ids run row-major over each Gaussian's tile rect, in depth order.
constexpr int kDupChunk = 256;
constexpr int kDupRun = 8;

__global__ void __launch_bounds__(kDupChunk) duplicate_kernel(const uint2* __restrict__ rect,
                                                              const uint32_t* __restrict__ tiles,
                                                              const uint32_t* __restrict__ idx_sorted,
                                                              const uint32_t* __restrict__ incl, int64_t n,
                                                              int tiles_x, uint16_t* __restrict__ key_out,
                                                              uint32_t* __restrict__ val_out) {
  __shared__ uint32_t s_end[kDupChunk];
  __shared__ uint32_t s_g[kDupChunk];
  __shared__ uint32_t s_rect[kDupChunk];  // tx0 | ty0 << 16
  __shared__ uint32_t s_w[kDupChunk];     // tile-rect width
  const int64_t s0 = (int64_t)blockIdx.x * kDupChunk;
  const int tid = threadIdx.x;
  __shared__ uint32_t s_begin;
  const int cnt_items = (int)min((int64_t)kDupChunk, n - s0);
  if (tid < cnt_items) {
    const uint32_t g = idx_sorted[s0 + tid];
    const uint32_t c = tiles[g];
    const uint2 r = rect[g];
    const uint32_t tx0 = (r.x & 0xffffu) / kTile, tx1 = (r.x >> 16) / kTile;
    const uint32_t ty0 = (r.y & 0xffffu) / kTile;
    s_end[tid] = incl[s0 + tid];
    s_g[tid] = g;
    s_rect[tid] = tx0 | (ty0 << 16);
    s_w[tid] = c ? tx1 - tx0 + 1 : 1;
  }
  if (tid == 0) s_begin = incl[s0] - tiles[idx_sorted[s0]];
  __syncthreads();
  const uint32_t begin = s_begin;
  const uint32_t end = s_end[cnt_items - 1];
  // each thread emits kDupRun consecutive slots: one binary search per run, then an incremental
  // walk over the (row-major) tile rects -- no per-slot search or integer division
  for (uint32_t o0 = begin + (uint32_t)tid * kDupRun; o0 < end; o0 += kDupChunk * kDupRun) {
    int lo = 0, hi = cnt_items - 1;  // first j with s_end[j] > o0
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (s_end[mid] > o0) hi = mid;
      else lo = mid + 1;
    }
    uint32_t w = s_w[lo];
    uint32_t gstart = lo == 0 ? begin : s_end[lo - 1];
    uint32_t local = o0 - gstart;
    uint32_t ly = local / w, lxx = local - ly * w;
    const uint32_t o1 = min(o0 + kDupRun, end);
    for (uint32_t o = o0; o < o1; ++o) {
      if (o == s_end[lo]) {  // next Gaussian (culled ones have no slots and are skipped)
        do { ++lo; } while (s_end[lo] == o);
        w = s_w[lo];
        ly = 0;
        lxx = 0;
      }
      const uint32_t tx = (s_rect[lo] & 0xffffu) + lxx;
      const uint32_t ty = (s_rect[lo] >> 16) + ly;
      key_out[o] = (uint16_t)(ty * (uint32_t)tiles_x + tx);
      val_out[o] = s_g[lo];
      if (++lxx == w) {
        lxx = 0;
        ++ly;
      }
    }
  }
}

void launch_duplicate(const ViewBufs& v, const uint32_t* idx_sorted, const uint32_t* incl, int64_t n,
                      int tiles_x, uint16_t* key_out, uint32_t* val_out, cudaStream_t s) {
  if (n == 0) return;
  duplicate_kernel<<<(unsigned)((n + kDupChunk - 1) / kDupChunk), kDupChunk, 0, s>>>(v.rect, v.tiles, idx_sorted,
                                                                                      incl, n, tiles_x, key_out,
                                                                                      val_out);
}

void launch_tile_sort(uint16_t* keys_in, uint16_t* keys_out, uint32_t* vals_in, uint32_t* vals_out, int64_t pairs,
                      int tile_bits, void* temp, size_t temp_bytes, cudaStream_t s) {
  if (pairs == 0) return;
  cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, vals_out, (int)pairs, 0,
                                  tile_bits > 0 ? tile_bits : 1, s);
}

// ------------------------------------------------------------------------------------------
// Fallback (more tiles than the shared-memory tables hold): duplicate + radix sort + ranges.
// ------------------------------------------------------------------------------------------
__global__ void ranges_kernel(const uint16_t* __restrict__ keys, int64_t pairs, uint2* __restrict__ ranges) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= pairs) return;
  const uint32_t t = keys[i];
  if (i == 0 || keys[i - 1] != t) ranges[t].x = (uint32_t)i;
  if (i == pairs - 1 || keys[i + 1] != t) ranges[t].y = (uint32_t)(i + 1);
}

void launch_ranges(const uint16_t* keys, int64_t pairs, int ntiles, uint2* ranges, cudaStream_t s) {
  cudaMemsetAsync(ranges, 0, sizeof(uint2) * (size_t)ntiles, s);
  if (pairs == 0) return;
  const int threads = 256;
  ranges_kernel<<<(unsigned)((pairs + threads - 1) / threads), threads, 0, s>>>(keys, pairs, ranges);
}

}  // namespace lgs
