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
#include <algorithm>
#include <cstring>

#include "lgs_internal.cuh"
#include "lgs_kernels.h"

namespace lgs {

constexpr int kMaxRankBucket = 1024;

__device__ __forceinline__ uint32_t depth_bucket(uint32_t key, uint32_t base) {
  if (key == 0xffffffffu) return kDepthBuckets;
  const uint32_t b = key >> kDepthShift;
  return b > base ? min(b - base, (uint32_t)kDepthBuckets - 1u) : 0u;
}

// Per bucket one u64: Gaussians << 32 | their tile pairs (the depth-layered binning cuts at a
// bucket boundary by pairs); one 64-bit atomic per Gaussian returns its slot in the high word.
// Culled Gaussians all share one bucket: their slots are handed out per CTA (shared-memory counter
// + one global atomic) instead of one global atomic each on one address.
typedef unsigned long long u64;
__device__ __forceinline__ uint32_t cnt_of(u64 v) { return (uint32_t)(v >> 32); }
__device__ __forceinline__ uint32_t prs_of(u64 v) { return (uint32_t)(v & 0xffffffffull); }

__global__ void __launch_bounds__(256) depth_hist_kernel(const uint32_t* __restrict__ dkey,
                                                         const uint32_t* __restrict__ tiles, int64_t n, uint32_t base,
                                                         u64* __restrict__ hist, uint32_t* __restrict__ slot) {
  __shared__ uint32_t s_culled, s_base;
  if (threadIdx.x == 0) s_culled = 0;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t b = kDepthBuckets, local = 0;
  if (i < n) {
    b = depth_bucket(dkey[i], base);
    if (b == kDepthBuckets) local = atomicAdd(&s_culled, 1u);
    else slot[i] = cnt_of(atomicAdd(hist + b, (1ull << 32) | tiles[i]));
  }
  __syncthreads();
  if (threadIdx.x == 0 && s_culled) s_base = cnt_of(atomicAdd(hist + kDepthBuckets, (u64)s_culled << 32));
  __syncthreads();
  if (i < n && b == kDepthBuckets) slot[i] = s_base + local;
}

// Layer A of the depth-layered binning = buckets [0, cut_end): the smallest bucket prefix whose
// pairs reach max(min(P, min_pairs), P / div), shortened to at most gauss_cap Gaussians and cap_a
// pairs.  Stored as cut = kDepthBuckets + 1 - cut_end (zero-initialized with the other scalars) and
// raised with atomicMax by the (unique) threads that find the crossing / the last feasible bucket.
__device__ __forceinline__ uint32_t cut_end_of(const uint32_t* cut) {
  return (uint32_t)kDepthBuckets + 1u - max(*cut, 1u);
}

__global__ void depth_cut_kernel(const u64* __restrict__ off, uint32_t div, uint32_t min_pairs, int64_t gauss_cap,
                                 uint32_t cap_a, uint32_t* __restrict__ cut) {
  griddep_wait();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= kDepthBuckets) return;
  const uint32_t P = prs_of(off[kDepthBuckets]);
  const uint32_t target = max(min(P, min_pairs), P / div);
  const u64 ex = off[b], in = off[b + 1];
  auto offer = [&](uint32_t end) { atomicMax(cut, (uint32_t)kDepthBuckets + 1u - end); };
  if (prs_of(in) >= target && prs_of(ex) < target) offer((uint32_t)b + 1u);
  const bool feas = (int64_t)cnt_of(in) <= gauss_cap && prs_of(in) <= cap_a;
  if (b == 0 && !feas) offer(0u);
  if (feas) {
    bool next_feas = false;
    if (b + 1 < kDepthBuckets) {
      const u64 in2 = off[b + 2];
      next_feas = (int64_t)cnt_of(in2) <= gauss_cap && prs_of(in2) <= cap_a;
    }
    if (!next_feas) offer((uint32_t)b + 1u);
  }
}

// ---- bucket offsets in one launch ---------------------------------------------------------------
// Exclusive scan of the kDepthBuckets + 2 bucket words (count << 32 | pairs) in one launch: each
// CTA takes the next 2048-word tile (dynamic tile id, so every predecessor is already running),
// stages it through shared memory (coalesced loads and stores, a blocked 4-word run per thread),
// publishes its tile aggregate with a release flag, and adds up its (at most 128) predecessors'
// aggregates in one parallel round, thread j waiting for tile j (a decoupled look-back without the
// serial chain: the aggregates all land at about the same time).  The pair total P comes from K1's
// per-CTA partial sums (read while the predecessors publish), so every thread also applies
// depth_cut_kernel's rule to its own buckets: CUB's init + scan kernels and the cut kernel become
// one launch.  Flags, aggregates and the tile counter live in the scalar block zeroed with the
// histogram.
constexpr int kScanThreads = 512, kScanItems = 4, kScanTile = kScanThreads * kScanItems;
constexpr int kScanTiles = (kDepthBuckets + 2 + kScanTile - 1) / kScanTile;
static_assert(kScanTiles <= kScanThreads, "one predecessor per thread");

struct ScanCut {
  const uint32_t* part;  // K1's per-CTA pair sums (null: offsets only, no cut)
  uint32_t nparts;
  uint32_t div, min_pairs, cap_a;
  int64_t gauss_cap;
  uint32_t* cut;
};

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ u64 warp_incl_scan(u64 v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u64 y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

__device__ __forceinline__ int scan_pad(int i) { return i + (i >> 4); }  // one spare word per 16

__global__ void __launch_bounds__(kScanThreads) bucket_scan_kernel(const u64* __restrict__ hist, u64* __restrict__ off,
                                                                   uint32_t* __restrict__ tile_ctr,
                                                                   uint32_t* __restrict__ flags, u64* __restrict__ agg,
                                                                   ScanCut sc) {
  constexpr int nitems = kDepthBuckets + 2;
  constexpr int kWarps = kScanThreads / 32;
  __shared__ u64 s_buf[kScanTile + kScanTile / 16];
  __shared__ uint32_t s_tile, s_p[kWarps];
  __shared__ u64 s_warp[kWarps], s_look[kWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  griddep_wait();
  if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const int t = (int)s_tile;
  const int base = t * kScanTile;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int i = base + k * kScanThreads + tid;
    s_buf[scan_pad(k * kScanThreads + tid)] = i < nitems ? __ldcg(hist + i) : 0ull;
  }
  __syncthreads();
  u64 v[kScanItems];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) v[k] = s_buf[scan_pad(tid * kScanItems + k)];
  u64 mine = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) mine += v[k];
  const u64 wincl = warp_incl_scan(mine, lane);
  if (lane == 31) s_warp[warp] = wincl;
  __syncthreads();
  if (warp == 0) {
    const u64 x = lane < kWarps ? s_warp[lane] : 0ull;
    const u64 xi = warp_incl_scan(x, lane);
    if (lane < kWarps) s_warp[lane] = xi - x;  // exclusive warp offsets
    if (lane == 31) {  // publish the tile aggregate
      agg[t] = xi;
      st_release_u32(flags + t, 1u);
    }
  }
  // the pair total from K1's partial sums (independent loads, issued while predecessors publish)
  uint32_t p = 0;
  if (sc.part) {
    uint32_t j = tid;
    for (; j + 3 * kScanThreads < sc.nparts; j += 4 * kScanThreads) {
      const uint32_t a0 = __ldcg(sc.part + j), a1 = __ldcg(sc.part + j + kScanThreads);
      const uint32_t a2 = __ldcg(sc.part + j + 2 * kScanThreads), a3 = __ldcg(sc.part + j + 3 * kScanThreads);
      p += (a0 + a1) + (a2 + a3);
    }
    for (; j < sc.nparts; j += kScanThreads) p += __ldcg(sc.part + j);
    p = __reduce_add_sync(0xffffffffu, p);
    if (lane == 0) s_p[warp] = p;
  }
  // prefix = the sum of every predecessor's aggregate, thread j waiting for tile j
  u64 pre = 0;
  if (tid < t) {
    while (ld_acquire_u32(flags + tid) == 0u) {
    }
    pre = __ldcg(agg + tid);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
  if (lane == 0) s_look[warp] = pre;
  __syncthreads();
  u64 ex = s_warp[warp] + (wincl - mine);
  uint32_t P = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    ex += s_look[w];
    if (sc.part) P += s_p[w];
  }
  const uint32_t target = sc.part ? max(min(P, sc.min_pairs), P / sc.div) : 0u;
  auto feas = [&](u64 in) { return (int64_t)cnt_of(in) <= sc.gauss_cap && prs_of(in) <= sc.cap_a; };
  auto offer = [&](uint32_t end) { atomicMax(sc.cut, (uint32_t)kDepthBuckets + 1u - end); };
  u64 exk[kScanItems];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int b = base + tid * kScanItems + k;
    exk[k] = ex;
    const u64 in = ex + v[k];
    if (sc.part && b < kDepthBuckets) {  // depth_cut_kernel's rule for bucket b
      if (prs_of(in) >= target && prs_of(ex) < target) offer((uint32_t)b + 1u);
      const bool f = feas(in);
      if (b == 0 && !f) offer(0u);
      if (f) {
        u64 nx;
        if (k + 1 < kScanItems) nx = v[k + 1];
        else if (tid + 1 < kScanThreads) nx = s_buf[scan_pad((tid + 1) * kScanItems)];
        else nx = __ldcg(hist + b + 1);
        if (!(b + 1 < kDepthBuckets && feas(in + nx))) offer((uint32_t)b + 1u);
      }
    }
    ex = in;
  }
  __syncthreads();  // every thread has read its neighbour's bucket: reuse the buffer for the offsets
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) s_buf[scan_pad(tid * kScanItems + k)] = exk[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int i = base + k * kScanThreads + tid;
    if (i < nitems) off[i] = s_buf[scan_pad(k * kScanThreads + tid)];
  }
}

enum { kDepthAll = 0, kDepthLayerA = 1, kDepthRest = 2 };

__device__ __forceinline__ bool bucket_selected(uint32_t b, int mode, uint32_t cut_end) {
  return mode == kDepthAll || (mode == kDepthLayerA ? b < cut_end : b >= cut_end);
}

__global__ void depth_scatter_kernel(const uint32_t* __restrict__ dkey, int64_t n, uint32_t base,
                                     const u64* __restrict__ off, const uint32_t* __restrict__ slot,
                                     const uint32_t* __restrict__ cut, int mode, uint2* __restrict__ tmp,
                                     uint32_t* __restrict__ ra_out, uint32_t* __restrict__ culled_cursor,
                                     const uint32_t* __restrict__ gate) {
  griddep_wait();
  if (gate && *gate == 0u) return;  // second layered pass with no unfinished tile (eager path)
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0 && ra_out) *ra_out = cnt_of(off[cut_end_of(cut)]);  // R_A: Gaussians in layer A
  if (i >= n) return;
  const uint32_t k = dkey[i];
  const uint32_t b = depth_bucket(k, base);
  if (!bucket_selected(b, mode, cut ? cut_end_of(cut) : 0u)) return;
  if (culled_cursor && b == kDepthBuckets) {  // slots of culled Gaussians (any order) handed out here
    const unsigned act = __activemask();
    const unsigned peers = __match_any_sync(act, 1u);
    const int leader = __ffs(peers) - 1;
    uint32_t basep = 0;
    if ((int)(threadIdx.x & 31) == leader) basep = atomicAdd(culled_cursor, (uint32_t)__popc(peers));
    basep = __shfl_sync(peers, basep, leader);
    tmp[cnt_of(off[b]) + basep + __popc(peers & ((1u << (threadIdx.x & 31)) - 1u))] = make_uint2(k, (uint32_t)i);
    return;
  }
  tmp[cnt_of(off[b]) + slot[i]] = make_uint2(k, (uint32_t)i);
}

__device__ __forceinline__ bool precedes(uint2 a, uint2 b) { return a.x < b.x || (a.x == b.x && a.y < b.y); }

// tile rect (tx0 | tx1 << 16, ty0 | ty1 << 16) of a pixel rect, for the forward's candidate scan
__device__ __forceinline__ uint2 tile_rect(uint2 rc) {
  return make_uint2(((rc.x & 0xffffu) / kTile) | (((rc.x >> 16) / kTile) << 16),
                    ((rc.y & 0xffffu) / kTile) | (((rc.y >> 16) / kTile) << 16));
}

struct DepthOut {
  uint32_t* idx_sorted;  // [n] map index in (depth, index) order (culled last, any order)
  uint32_t* cnt_sorted;  // [n] or null: tile counts in that order
  uint2* cand_rect;      // [n] or null: tile rects in that order (positions < R_A)
  uint8_t* active;       // or null: layer-A Gaussians flagged for the backward (lgs_kernels.h) ...
  float* gacc_zero;      // ... and, for the fused step, their accumulator rows (32 floats) zeroed
  ColorJob cj;           // lazy colours: computed here for the layer-A Gaussians (cj.color null: off)
  const uint32_t* gate = nullptr;  // rest pass: nothing to do when *gate == 0 (no unfinished tile)
};

__device__ __forceinline__ void depth_emit(const DepthOut& o, const uint32_t* __restrict__ tiles,
                                           const uint2* __restrict__ rect, uint32_t pos, uint32_t g,
                                           uint32_t cand_end) {
  o.idx_sorted[pos] = g;
  if (o.cnt_sorted) o.cnt_sorted[pos] = tiles[g];
  if (pos < cand_end) {
    if (o.cand_rect) o.cand_rect[pos] = tile_rect(rect[g]);
    if (o.active) o.active[g] = 1;
    if (o.cj.color) color_job_run(o.cj, g);
    if (o.gacc_zero) {
      float4* row = reinterpret_cast<float4*>(o.gacc_zero + (size_t)g * 32);
#pragma unroll
      for (int q = 0; q < 8; ++q) row[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}

// Big buckets (more than kMaxRankBucket members, e.g. splats at one identical depth): per bucket one
// bitonic sort of the padded composite keys (key << 32 | index) in `scratch` (2 n entries: the padded
// sizes of all big buckets sum to less than twice their element count), buckets k = first, first +
// stride, ... of the *big_n listed in big_ids, by the calling CTA.
__device__ void sort_big_buckets(const uint2* __restrict__ tmp, const u64* __restrict__ off,
                                 const uint32_t* __restrict__ tiles, const uint2* __restrict__ rect,
                                 const uint32_t* __restrict__ cut, uint32_t nbig, const uint32_t* __restrict__ big_ids,
                                 unsigned long long* __restrict__ scratch, uint32_t* __restrict__ cursor,
                                 const DepthOut& o, uint32_t first, uint32_t stride) {
  const uint32_t ra = cut ? cnt_of(off[cut_end_of(cut)]) : 0u;
  __shared__ uint32_t s_base;
  for (uint32_t k = first; k < nbig; k += stride) {
    const uint32_t b = big_ids[k];
    const uint32_t lo = cnt_of(off[b]), m = cnt_of(off[b + 1]) - lo;
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
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x)
      depth_emit(o, tiles, rect, lo + i, (uint32_t)(a[i] & 0xffffffffull), ra);
  }
}

// Exact in-bucket rank of every selected element.  Big buckets are listed (big_n, big_ids); with
// `done` (layer A) the last CTA to finish sorts them itself -- one launch less in the chain, the
// big-bucket case being rare -- otherwise depth_big_kernel follows.
__global__ void depth_rank_kernel(const uint2* __restrict__ tmp, int64_t n, uint32_t base,
                                  const u64* __restrict__ off, const uint32_t* __restrict__ tiles,
                                  const uint2* __restrict__ rect, const uint32_t* __restrict__ cut, int mode,
                                  DepthOut o, uint32_t* __restrict__ big_n, uint32_t* __restrict__ big_ids,
                                  uint32_t* __restrict__ done, unsigned long long* __restrict__ scratch,
                                  uint32_t* __restrict__ cursor) {
  griddep_wait();
  if (o.gate && *o.gate == 0u) return;
  // layer A (a few thousand positions on a grid sized for gauss_cap): positions interleaved
  // over the CTAs, so every SM takes a share of the latency-bound work
  const int64_t p0 = mode == kDepthLayerA ? (int64_t)threadIdx.x * gridDim.x + blockIdx.x
                                          : (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t ra = cut ? cnt_of(off[cut_end_of(cut)]) : 0u;  // Gaussians in layer A
  const int64_t p = mode == kDepthRest ? p0 + ra : p0;
  if (p < (mode == kDepthLayerA ? (int64_t)ra : n)) {
    const uint2 me = tmp[p];
    const uint32_t b = depth_bucket(me.x, base);
    if (b == kDepthBuckets) {  // culled: no pairs, any order
      o.idx_sorted[p] = me.y;
      if (o.cnt_sorted) o.cnt_sorted[p] = 0u;
    } else {
      const uint32_t lo = cnt_of(off[b]), hi = cnt_of(off[b + 1]);
      if (hi - lo > kMaxRankBucket) {
        if (p == lo) big_ids[atomicAdd(big_n, 1u)] = b;
      } else {
        uint32_t rank = 0;
#pragma unroll 4
        for (uint32_t q = lo; q < hi; ++q) rank += precedes(tmp[q], me) ? 1u : 0u;
        depth_emit(o, tiles, rect, lo + rank, me.y, ra);
      }
    }
  }
  if (!done) return;
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const uint32_t nbig = atomicAdd(big_n, 0u);
  if (nbig) sort_big_buckets(tmp, off, tiles, rect, cut, nbig, big_ids, scratch, cursor, o, 0u, 1u);
}

__global__ void __launch_bounds__(1024) depth_big_kernel(const uint2* __restrict__ tmp, const u64* __restrict__ off,
                                                         const uint32_t* __restrict__ tiles,
                                                         const uint2* __restrict__ rect,
                                                         const uint32_t* __restrict__ cut,
                                                         const uint32_t* __restrict__ big_n,
                                                         const uint32_t* __restrict__ big_ids,
                                                         unsigned long long* __restrict__ scratch,
                                                         uint32_t* __restrict__ cursor, DepthOut o) {
  griddep_wait();
  sort_big_buckets(tmp, off, tiles, rect, cut, *big_n, big_ids, scratch, cursor, o, blockIdx.x, gridDim.x);
}

// ------------------------------------------------------------------------------------------
// host side: one scratch block carved into the buffers below (DepthOrderState keeps the carving
// so the second layered pass can finish the order later)
// ------------------------------------------------------------------------------------------
static size_t align_words(size_t w) { return (w + 63) & ~size_t(63); }

// scalars (zeroed with the histogram): cut, big-bucket counts of layer A / the rest, bitonic
// scratch allocator, culled-slot allocator, rank-done counter (the first kScRerun are zeroed again
// by a re-run of layer A), bucket-scan tile counter, the pair total P (preprocess); then the bucket
// scan's flags (zeroed too), tile aggregates and inclusive prefixes
enum {
  kScCut = 0, kScBigA = 1, kScBigR = 2, kScScratch = 3, kScCulled = 4, kScRankDone = 5, kScRerun = 6,
  kScScanTile = 6
};
constexpr size_t kScFlags = 64, kScAgg = kScFlags + 256, kScWords = kScAgg + 2 * 256;
constexpr size_t kScZeroed = kScFlags + kScanTiles;  // words zeroed per render

size_t depth_order_temp_bytes(int64_t n) {
  const size_t nn = align_words((size_t)n);
  const size_t words = 2 * 2 * align_words(kDepthBuckets + 2)  // hist, off (u64)
                       + nn                                     // slot
                       + 2 * nn                                 // tmp (uint2)
                       + 4 * nn                                 // scratch (2n u64)
                       + align_words((size_t)n / kMaxRankBucket + 2) * 2  // big lists (layer A, rest)
                       + kScWords                               // scalars + bucket-scan state
                       + align_words((size_t)n / kPreThreads + 1);  // K1's per-CTA pair sums
  return sizeof(uint32_t) * words + 1024;
}


struct DepthCarve {
  unsigned long long *hist, *off;
  uint2* tmp;
  uint32_t *slot, *big_a, *big_r, *sc, *part;
  unsigned long long* scratch;
  uint32_t base;
};

static DepthCarve carve(void* temp, int64_t n, float near_plane) {
  DepthCarve c;
  uint32_t* w = reinterpret_cast<uint32_t*>((reinterpret_cast<uintptr_t>(temp) + 255) & ~uintptr_t(255));
  const size_t nn = align_words((size_t)n), nb = align_words(kDepthBuckets + 2);
  c.hist = reinterpret_cast<unsigned long long*>(w);
  w += 2 * nb;
  c.sc = w;  // right after the histogram: one memset zeroes both
  w += kScWords;
  c.off = reinterpret_cast<unsigned long long*>(w);
  w += 2 * nb;
  c.slot = w;
  w += nn;
  c.tmp = reinterpret_cast<uint2*>(w);
  w += 2 * nn;
  c.scratch = reinterpret_cast<unsigned long long*>(w);
  w += 4 * nn;
  const size_t nbig = align_words((size_t)n / kMaxRankBucket + 2);
  c.big_a = w;
  w += nbig;
  c.big_r = w;
  w += nbig;
  c.part = w;
  // near plane in key space: depths are > near, so buckets start there (2^13 per octave)
  const float nearp = near_plane > 0.f ? near_plane : 0.f;
  uint32_t nbits;
  memcpy(&nbits, &nearp, sizeof(nbits));
  c.base = nbits >> kDepthShift;
  return c;
}

static void launch_bucket_scan(const DepthCarve& c, const ScanCut& sc, cudaStream_t s) {
  launch_pdl(bucket_scan_kernel, dim3(kScanTiles), dim3(kScanThreads), 0, s, (const u64*)c.hist, c.off,
             c.sc + kScScanTile, c.sc + kScFlags, reinterpret_cast<u64*>(c.sc + kScAgg), sc);
}

static void depth_front(const ViewBufs& v, int64_t n, const DepthCarve& c, cudaStream_t s) {
  // histogram, scalars and scan flags (contiguous)
  cudaMemsetAsync(c.hist, 0, (size_t)(reinterpret_cast<char*>(c.sc + kScZeroed) - reinterpret_cast<char*>(c.hist)), s);
  depth_hist_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(v.dkey, v.tiles, n, c.base, c.hist, c.slot);
  launch_bucket_scan(c, ScanCut{}, s);
}

void launch_depth_order(const ViewBufs& v, int64_t n, float near_plane, void* temp, size_t temp_bytes,
                        uint32_t* idx_sorted, uint32_t* cnt_sorted, cudaStream_t s) {
  (void)temp_bytes;
  if (n == 0) return;
  const DepthCarve c = carve(temp, n, near_plane);
  depth_front(v, n, c, s);
  const unsigned grid = (unsigned)((n + 255) / 256);
  const DepthOut o{idx_sorted, cnt_sorted, nullptr, nullptr, nullptr};
  depth_scatter_kernel<<<grid, 256, 0, s>>>(v.dkey, n, c.base, c.off, c.slot, nullptr, kDepthAll, c.tmp, nullptr, nullptr,
                                            nullptr);
  depth_rank_kernel<<<grid, 256, 0, s>>>(c.tmp, n, c.base, c.off, v.tiles, v.rect, nullptr, kDepthAll, o,
                                         c.sc + kScBigA, c.big_a, nullptr, nullptr, nullptr);
  depth_big_kernel<<<8, 1024, 0, s>>>(c.tmp, c.off, v.tiles, v.rect, nullptr, c.sc + kScBigA, c.big_a, c.scratch,
                                      c.sc + kScScratch, o);
}

void launch_depth_prepare(int64_t n, float near_plane, void* temp, ViewBufs* v, cudaStream_t s) {
  const DepthCarve c = carve(temp, n, near_plane);
  // histogram and the scalars / scan flags behind it (layer A's cut, counts, allocators, P)
  cudaMemsetAsync(c.hist, 0, (size_t)(reinterpret_cast<char*>(c.sc + kScZeroed) - reinterpret_cast<char*>(c.hist)), s);
  v->dhist = c.hist;
  v->dslot = c.slot;
  v->dbase = c.base;
  v->dpart = c.part;
}

// After K1 filled the visible buckets (the culled ones get their slots in the rest pass): bucket
// offsets; *pairs_out = the low word of the offset past the last visible bucket = the pair total P.
void launch_depth_scan(int64_t n, float near_plane, void* temp, const LayerCut* cut, const uint32_t** pairs_out,
                       cudaStream_t s) {
  const DepthCarve c = carve(temp, n, near_plane);
  *pairs_out = reinterpret_cast<const uint32_t*>(c.off + kDepthBuckets);  // little endian: low word = pairs
  if (n == 0) {
    cudaMemsetAsync(c.off, 0, sizeof(unsigned long long) * (kDepthBuckets + 2), s);
    return;
  }
  ScanCut sc{};
  if (cut)
    sc = ScanCut{c.part, (uint32_t)((n + kPreThreads - 1) / kPreThreads), cut->div, cut->min_pairs, cut->cap_a,
                 cut->gauss_cap, c.sc + kScCut};
  launch_bucket_scan(c, sc, s);
}

void launch_depth_order_layer_a(const ViewBufs& v, int64_t n, float near_plane, void* temp, uint32_t div,
                                uint32_t min_pairs, int64_t gauss_cap, uint32_t cap_a, uint32_t* idx_sorted,
                                uint2* cand_rect, uint32_t* ra, uint8_t* active, float* gacc_zero, bool rerun,
                                bool cut_ready, const ColorJob& cj, cudaStream_t s) {
  if (n == 0) {
    cudaMemsetAsync(ra, 0, sizeof(uint32_t), s);
    return;
  }
  const DepthCarve c = carve(temp, n, near_plane);
  // (the scalars were zeroed with the histogram by launch_depth_prepare; a re-run after a pair
  // capacity overflow zeroes them again)
  if (rerun) cudaMemsetAsync(c.sc, 0, sizeof(uint32_t) * kScRerun, s);
  // (cut_ready: the bucket scan already applied the cut with these parameters)
  if (!cut_ready)
    launch_pdl(depth_cut_kernel, dim3((kDepthBuckets + 255) / 256), dim3(256), 0, s, (const u64*)c.off, div,
               min_pairs, gauss_cap, cap_a, c.sc + kScCut);
  const DepthOut o{idx_sorted, nullptr, cand_rect, active, gacc_zero, cj};
  const int64_t ga = std::min<int64_t>(n, gauss_cap);
  const uint32_t* cut = c.sc + kScCut;
  launch_pdl(depth_scatter_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, s, (const uint32_t*)v.dkey, n,
             c.base, (const u64*)c.off, (const uint32_t*)c.slot, cut, (int)kDepthLayerA, c.tmp, ra, (uint32_t*)nullptr,
             (const uint32_t*)nullptr);
  // (big buckets, if any, are sorted by the rank kernel's last CTA)
  launch_pdl(depth_rank_kernel, dim3((unsigned)((ga + 255) / 256)), dim3(256), 0, s, (const uint2*)c.tmp, n, c.base,
             (const u64*)c.off, (const uint32_t*)v.tiles, (const uint2*)v.rect, cut, (int)kDepthLayerA, o,
             c.sc + kScBigA, c.big_a, c.sc + kScRankDone, c.scratch, c.sc + kScScratch);
}

// Layer-A tile lists: one CTA per run of kSegTiles tiles of a tile row.  Its warps split the R_A
// depth-ordered candidates into contiguous segments; a lane turns its candidate's tile rect into
// a bitmask of the run's tiles it covers, and per tile one ballot counts (pass 1) or places (pass
// 2, order-preserving compaction) the warp's 32 candidates.  The run's lists are reserved with one
// atomic and laid out tile after tile; within a tile, warp segments follow each other, so every
// list is the exact depth-order prefix of the tile's complete list.  R_A is ~0.5-5% of the visible
// Gaussians (a few thousand), read twice per run from L2.
constexpr int kListWarps = 16;
constexpr int kSegTiles = 8;

__global__ void __launch_bounds__(kListWarps * 32) layer_tile_lists_kernel(
    const uint2* __restrict__ cand_rect, const uint32_t* __restrict__ cand_idx, const uint32_t* __restrict__ ra,
    int tiles_x, uint32_t* __restrict__ cursor, uint32_t* __restrict__ vals, uint2* __restrict__ ranges,
    int* __restrict__ blend_counter, double* __restrict__ loss, uint32_t* __restrict__ miss) {
  griddep_wait();
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // for the blend launched next (no memset nodes between)
    if (blend_counter) *blend_counter = 0;
    if (loss) *loss = 0.0;
    if (miss) *miss = 0u;
  }
  __shared__ uint32_t s_cnt[kListWarps][kSegTiles];
  __shared__ uint32_t s_base;
  const int nseg = (tiles_x + kSegTiles - 1) / kSegTiles;
  const uint32_t ty = blockIdx.x / nseg;
  const uint32_t tx0 = (blockIdx.x % nseg) * kSegTiles;
  const uint32_t ntl = min((uint32_t)kSegTiles, (uint32_t)tiles_x - tx0);  // tiles in this run
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t n_cand = *ra;
  const uint32_t seg = ((n_cand + kListWarps * 32 - 1) / (kListWarps * 32)) * 32;
  const uint32_t c0 = min(n_cand, warp * seg), c1 = min(n_cand, c0 + seg);
  // bit j: candidate i's tile rect holds tile (tx0 + j, ty)
  auto mask_of = [&](uint32_t i) -> uint32_t {
    if (i >= c1) return 0u;
    const uint2 tr = __ldg(cand_rect + i);
    const uint32_t y0 = tr.y & 0xffffu, y1 = tr.y >> 16;
    if (ty < y0 || ty > y1) return 0u;
    const int lo = max((int)(tr.x & 0xffffu) - (int)tx0, 0);
    const int hi = min((int)(tr.x >> 16) - (int)tx0, (int)ntl - 1);
    return lo > hi ? 0u : ((2u << hi) - 1u) & ~((1u << lo) - 1u);
  };
  uint32_t cnt[kSegTiles];
#pragma unroll
  for (int j = 0; j < kSegTiles; ++j) cnt[j] = 0;
#pragma unroll 2
  for (uint32_t i0 = c0; i0 < c1; i0 += 32) {
    const uint32_t m = mask_of(i0 + lane);
#pragma unroll
    for (int j = 0; j < kSegTiles; ++j) cnt[j] += __popc(__ballot_sync(0xffffffffu, (m >> j) & 1u));
  }
  if (lane < kSegTiles) {
    uint32_t mine = 0;
#pragma unroll
    for (int j = 0; j < kSegTiles; ++j) mine = lane == j ? cnt[j] : mine;
    s_cnt[warp][lane] = mine;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // run-level layout: tile after tile, warp segments in order within a tile
    uint32_t tot = 0;
    uint32_t start[kSegTiles];
    for (uint32_t j = 0; j < ntl; ++j) {
      start[j] = tot;
      for (int w = 0; w < kListWarps; ++w) {
        const uint32_t c = s_cnt[w][j];
        s_cnt[w][j] = tot;
        tot += c;
      }
    }
    s_base = atomicAdd(cursor, tot);
    for (uint32_t j = 0; j < ntl; ++j)
      ranges[ty * tiles_x + tx0 + j] = make_uint2(s_base + start[j], s_base + (j + 1 < ntl ? start[j + 1] : tot));
  }
  __syncthreads();
  uint32_t pos[kSegTiles];
#pragma unroll
  for (int j = 0; j < kSegTiles; ++j) pos[j] = s_base + (j < (int)ntl ? s_cnt[warp][j] : 0u);
  const unsigned lt = (1u << lane) - 1u;
  for (uint32_t i0 = c0; i0 < c1; i0 += 32) {
    const uint32_t i = i0 + lane;
    const uint32_t m = mask_of(i);
    const uint32_t g = m ? __ldg(cand_idx + i) : 0u;
#pragma unroll
    for (int j = 0; j < kSegTiles; ++j) {
      const bool hit = (m >> j) & 1u;
      const unsigned bal = __ballot_sync(0xffffffffu, hit);
      if (hit) vals[pos[j] + __popc(bal & lt)] = g;
      pos[j] += __popc(bal);
    }
  }
}

// Tiles longest layer-A list first (exact lengths, >= 1023 in one bin; arbitrary order inside a bin:
// which CTA takes which tile is racy anyway and no result depends on it).  One CTA counting sort.
// Longest-first tile order for the next replay: by list length, or (cost non-null) by the measured
// duration of each tile in the previous replay (the fused blend's per-tile clock deltas; a view is
// fixed between replays).  Keys are read once into shared memory (the blend of this replay may
// rewrite the costs meanwhile: the counting sort must see one key per tile to stay a permutation).
__global__ void __launch_bounds__(1024) tile_order_lpt_kernel(const uint2* __restrict__ ranges,
                                                              const uint32_t* __restrict__ cost, int ntiles,
                                                              uint32_t* __restrict__ order) {
  extern __shared__ uint32_t s_key[];  // [ntiles] when cost
  __shared__ uint32_t s_bin[1024];
  __shared__ uint32_t s_w[32];
  __shared__ uint32_t s_max;
  const int t0 = threadIdx.x, lane = t0 & 31, warp = t0 >> 5;
  s_bin[t0] = 0;
  if (t0 == 0) s_max = 0;
  __syncthreads();
  if (cost) {
    uint32_t mx = 0;
    for (int t = t0; t < ntiles; t += blockDim.x) {
      const uint32_t c = __ldcg(cost + t);
      s_key[t] = c;
      mx = max(mx, c);
    }
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (lane == 0) atomicMax(&s_max, mx);
    __syncthreads();
  }
  const uint32_t cmax = max(s_max, 1u);
  auto bin_of = [&](int t) -> uint32_t {  // bin 0 = longest
    if (cost) return 1023u - (uint32_t)(((uint64_t)s_key[t] * 1023u) / cmax);
    const uint2 r = ranges[t];
    return 1023u - min(r.y - r.x, 1023u);
  };
  for (int t = t0; t < ntiles; t += blockDim.x) atomicAdd(&s_bin[bin_of(t)], 1u);
  __syncthreads();
  const uint32_t v = s_bin[t0];
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = s_w[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    s_w[lane] = w;
  }
  __syncthreads();
  s_bin[t0] = x - v + (warp ? s_w[warp - 1] : 0u);
  __syncthreads();
  for (int t = t0; t < ntiles; t += blockDim.x) order[atomicAdd(&s_bin[bin_of(t)], 1u)] = (uint32_t)t;
}

void launch_tile_order_lpt(const uint2* ranges, const uint32_t* cost, int ntiles, uint32_t* order, cudaStream_t s) {
  if (ntiles > kLptCostMaxTiles) cost = nullptr;  // (48 KB of keys)
  tile_order_lpt_kernel<<<1, 1024, cost ? sizeof(uint32_t) * (size_t)ntiles : 0, s>>>(ranges, cost, ntiles, order);
}

__global__ void __launch_bounds__(1024) copy_u32_kernel(const uint32_t* __restrict__ src, int n,
                                                        uint32_t* __restrict__ dst) {
  griddep_wait();
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

void launch_copy_u32(const uint32_t* src, int n, uint32_t* dst, cudaStream_t s) {
  launch_pdl(copy_u32_kernel, dim3(1), dim3(1024), 0, s, src, n, dst);
}

void launch_layer_tile_lists(const uint2* cand_rect, const uint32_t* cand_idx, const uint32_t* n_cand, int tiles_x,
                             int ntiles, uint32_t* cursor, uint32_t* vals, uint2* ranges, int* blend_counter,
                             double* loss, uint32_t* miss, cudaStream_t s) {
  const int tiles_y = ntiles / tiles_x;
  const int runs = tiles_y * ((tiles_x + kSegTiles - 1) / kSegTiles);
  launch_pdl(layer_tile_lists_kernel, dim3(runs), dim3(kListWarps * 32), 0, s, cand_rect, cand_idx, n_cand, tiles_x,
             cursor, vals, ranges, blend_counter, loss, miss);
}

void launch_depth_order_rest(const ViewBufs& v, int64_t n, float near_plane, void* temp, uint32_t* idx_sorted,
                             const uint32_t* gate, cudaStream_t s) {
  if (n == 0) return;
  const DepthCarve c = carve(temp, n, near_plane);
  const unsigned grid = (unsigned)((n + 255) / 256);
  DepthOut o{idx_sorted, nullptr, nullptr, nullptr, nullptr};
  o.gate = gate;
  // the rest's big-bucket count, bitonic scratch allocator (layer A's sorts are done) and culled slots
  cudaMemsetAsync(c.sc + kScBigR, 0, sizeof(uint32_t) * 3, s);
  const uint32_t* cut = c.sc + kScCut;
  depth_scatter_kernel<<<grid, 256, 0, s>>>(v.dkey, n, c.base, c.off, c.slot, cut, kDepthRest, c.tmp, nullptr,
                                            c.sc + kScCulled, gate);
  depth_rank_kernel<<<grid, 256, 0, s>>>(c.tmp, n, c.base, c.off, v.tiles, v.rect, cut, kDepthRest, o,
                                         c.sc + kScBigR, c.big_r, nullptr, nullptr, nullptr);
  depth_big_kernel<<<8, 1024, 0, s>>>(c.tmp, c.off, v.tiles, v.rect, cut, c.sc + kScBigR, c.big_r, c.scratch,
                                      c.sc + kScScratch, o);
}

}  // namespace lgs
