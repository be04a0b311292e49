// depth_order.cu -- the global (depth, map index) order of the projected Gaussians
// (proj/src/renderer.cpp:114-117) without a device-wide radix sort.
//
// The reference composites every Gaussian in one order: depth ascending, ties by map index.  The
// depth keys are the f32 bits of positive depths (monotone as integers), so the order is the
// lexicographic order of (key, index).  A 4-pass onesweep radix sort of 500k keys runs on ~60
// CTAs per pass and is latency-bound (~60 us at the headline config).  Here instead:
//   1. hist    : every Gaussian takes a slot in its depth bucket (key >> kDepthShift, relative to
//                the near plane; 2^18 buckets = 2^13 per octave of depth); culled Gaussians
//                (key 0xffffffff) go to one extra bucket after all visible ones;
//   2. scan    : exclusive scan of the bucket counts (bucket begin offsets; visible count V);
//   3. scatter : (key, index) to bucket begin + slot (slot order within a bucket is arbitrary);
//   4. rank    : the element's final position inside its bucket is the number of bucket members
//                that precede it in (key, index) order -- an exact, deterministic rank however
//                the slots were assigned -- and it writes the sorted index and its tile count
//                (the gather the binning's scan needs).  Buckets hold ~10 Gaussians here.
//   5. big     : buckets larger than kMaxRankBucket (e.g. thousands of splats at one identical
//                depth) are sorted by one CTA each with a bitonic network over the 64-bit
//                (key << 32 | index) composite in scratch memory; normally none, and the kernel
//                exits at once.
// Culled Gaussians follow the visible ones in arbitrary order: they own no tile pairs, so their
// order affects no output.
// Roofline: HBM/L2 latency; ~(4 + 4) B read + written per Gaussian per step, ~20 B in total.
#include <cub/device/device_scan.cuh>

#include <cstring>

#include "lgs_internal.cuh"
#include "lgs_kernels.h"

namespace lgs {

constexpr int kDepthShift = 10;
constexpr int kDepthBuckets = 1 << 18;  // visible buckets; bucket kDepthBuckets holds the culled
constexpr int kMaxRankBucket = 1024;

__device__ __forceinline__ uint32_t depth_bucket(uint32_t key, uint32_t base) {
  if (key == 0xffffffffu) return kDepthBuckets;
  const uint32_t b = key >> kDepthShift;
  return b > base ? min(b - base, (uint32_t)kDepthBuckets - 1u) : 0u;
}

// Culled Gaussians all share one bucket: their slots are handed out per CTA (shared-memory
// counter + one global atomic) instead of one global atomic each on a single address.
__global__ void __launch_bounds__(256) depth_hist_kernel(const uint32_t* __restrict__ dkey, int64_t n, uint32_t base,
                                                         uint32_t* __restrict__ hist, uint32_t* __restrict__ slot) {
  __shared__ uint32_t s_culled, s_base;
  if (threadIdx.x == 0) s_culled = 0;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t b = kDepthBuckets, local = 0;
  if (i < n) {
    b = depth_bucket(dkey[i], base);
    if (b == kDepthBuckets) local = atomicAdd(&s_culled, 1u);
    else slot[i] = atomicAdd(hist + b, 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0 && s_culled) s_base = atomicAdd(hist + kDepthBuckets, s_culled);
  __syncthreads();
  if (i < n && b == kDepthBuckets) slot[i] = s_base + local;
}

__global__ void depth_scatter_kernel(const uint32_t* __restrict__ dkey, int64_t n, uint32_t base,
                                     const uint32_t* __restrict__ off, const uint32_t* __restrict__ slot,
                                     uint2* __restrict__ tmp) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t k = dkey[i];
  tmp[off[depth_bucket(k, base)] + slot[i]] = make_uint2(k, (uint32_t)i);
}

__device__ __forceinline__ bool precedes(uint2 a, uint2 b) { return a.x < b.x || (a.x == b.x && a.y < b.y); }

// big[0] = number of big buckets, big[1 ..] their ids; big_cursor = scratch entries handed out
__global__ void depth_rank_kernel(const uint2* __restrict__ tmp, int64_t n, uint32_t base,
                                  const uint32_t* __restrict__ off, const uint32_t* __restrict__ tiles,
                                  uint32_t* __restrict__ idx_sorted, uint32_t* __restrict__ cnt_sorted,
                                  uint32_t* __restrict__ big) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint2 me = tmp[p];
  const uint32_t b = depth_bucket(me.x, base);
  if (b == kDepthBuckets) {  // culled: no pairs, any order
    idx_sorted[p] = me.y;
    cnt_sorted[p] = 0u;
    return;
  }
  const uint32_t lo = off[b], hi = off[b + 1];
  if (hi - lo > kMaxRankBucket) {
    if (p == lo) big[1 + atomicAdd(big, 1u)] = b;
    return;
  }
  uint32_t rank = 0;
  for (uint32_t q = lo; q < hi; ++q) rank += precedes(tmp[q], me) ? 1u : 0u;
  idx_sorted[lo + rank] = me.y;
  cnt_sorted[lo + rank] = tiles[me.y];
}

// One CTA per big bucket: bitonic sort of the padded composite keys in `scratch` (2 n entries:
// the padded sizes of all big buckets sum to less than twice their element count).
__global__ void __launch_bounds__(1024) depth_big_kernel(const uint2* __restrict__ tmp, const uint32_t* __restrict__ off,
                                                         const uint32_t* __restrict__ tiles,
                                                         const uint32_t* __restrict__ big,
                                                         unsigned long long* __restrict__ scratch,
                                                         uint32_t* __restrict__ cursor,
                                                         uint32_t* __restrict__ idx_sorted,
                                                         uint32_t* __restrict__ cnt_sorted) {
  const uint32_t nbig = big[0];
  __shared__ uint32_t s_base;
  for (uint32_t k = blockIdx.x; k < nbig; k += gridDim.x) {
    const uint32_t b = big[1 + k];
    const uint32_t lo = off[b], m = off[b + 1] - lo;
    uint32_t M = 1;
    while (M < m) M <<= 1;
    __syncthreads();
    if (threadIdx.x == 0) s_base = atomicAdd(cursor, M);
    __syncthreads();
    unsigned long long* a = scratch + s_base;
    for (uint32_t i = threadIdx.x; i < M; i += blockDim.x) {
      if (i < m) {
        const uint2 e = tmp[lo + i];
        a[i] = ((unsigned long long)e.x << 32) | e.y;
      } else {
        a[i] = ~0ull;
      }
    }
    __syncthreads();
    for (uint32_t kk = 2; kk <= M; kk <<= 1) {
      for (uint32_t j = kk >> 1; j > 0; j >>= 1) {
        for (uint32_t i = threadIdx.x; i < M; i += blockDim.x) {
          const uint32_t l = i ^ j;
          if (l > i) {
            const unsigned long long x = a[i], y = a[l];
            const bool up = (i & kk) == 0;
            if ((x > y) == up) {
              a[i] = y;
              a[l] = x;
            }
          }
        }
        __syncthreads();
      }
    }
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
      const uint32_t g = (uint32_t)(a[i] & 0xffffffffull);
      idx_sorted[lo + i] = g;
      cnt_sorted[lo + i] = tiles[g];
    }
  }
}

size_t depth_order_temp_bytes(int64_t n) {
  size_t scan = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan, (uint32_t*)nullptr, (uint32_t*)nullptr, kDepthBuckets + 2);
  const size_t words = 2 * (size_t)(kDepthBuckets + 2)  // hist, off
                       + (size_t)n                      // slot
                       + 2 * (size_t)n                  // tmp (uint2)
                       + 4 * (size_t)n                  // scratch (2n u64)
                       + (size_t)n / kMaxRankBucket + 2 // big list
                       + 2;                             // cursor
  return sizeof(uint32_t) * (words + 8 * 64) + scan + 1024;  // + per-region 256 B alignment
}

static uint32_t* align256(uint8_t* p) {
  return reinterpret_cast<uint32_t*>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255));
}

void launch_depth_order(const ViewBufs& v, int64_t n, float near_plane, void* temp, size_t temp_bytes,
                        uint32_t* idx_sorted, uint32_t* cnt_sorted, cudaStream_t s) {
  if (n == 0) return;
  const int nb = kDepthBuckets + 1;  // + culled bucket
  uint32_t* hist = align256(static_cast<uint8_t*>(temp));
  uint32_t* off = hist + ((nb + 1 + 63) & ~63);
  uint32_t* slot = off + ((nb + 1 + 63) & ~63);
  uint2* tmp = reinterpret_cast<uint2*>(slot + ((n + 63) & ~63ll));
  unsigned long long* scratch = reinterpret_cast<unsigned long long*>(tmp + ((n + 63) & ~63ll));
  uint32_t* big = reinterpret_cast<uint32_t*>(scratch + 2 * ((n + 63) & ~63ll));
  uint32_t* cursor = big + ((n / kMaxRankBucket + 2 + 63) & ~63ll);
  void* scan_temp = align256(reinterpret_cast<uint8_t*>(cursor + 64));
  size_t scan_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, hist, off, nb + 1);
  // near plane in key space: depths are > near, so buckets start there (2^13 per octave)
  const float nearp = near_plane > 0.f ? near_plane : 0.f;
  uint32_t nbits;
  memcpy(&nbits, &nearp, sizeof(nbits));
  const uint32_t base = nbits >> kDepthShift;
  cudaMemsetAsync(hist, 0, sizeof(uint32_t) * (nb + 1), s);
  cudaMemsetAsync(big, 0, sizeof(uint32_t), s);
  cudaMemsetAsync(cursor, 0, sizeof(uint32_t), s);
  const unsigned grid = (unsigned)((n + 255) / 256);
  depth_hist_kernel<<<grid, 256, 0, s>>>(v.dkey, n, base, hist, slot);
  cub::DeviceScan::ExclusiveSum(scan_temp, scan_bytes, hist, off, nb + 1, s);
  depth_scatter_kernel<<<grid, 256, 0, s>>>(v.dkey, n, base, off, slot, tmp);
  depth_rank_kernel<<<grid, 256, 0, s>>>(tmp, n, base, off, v.tiles, idx_sorted, cnt_sorted, big);
  depth_big_kernel<<<8, 1024, 0, s>>>(tmp, off, v.tiles, big, scratch, cursor, idx_sorted, cnt_sorted);
}

}  // namespace lgs
