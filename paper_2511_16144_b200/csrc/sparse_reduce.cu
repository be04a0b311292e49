// sparse_reduce.cu -- row-sparse sum of the per-Gaussian gradients over ranks (multi-view batches).
//
// With the depth-layered binning a view's gradient is nonzero only on the Gaussians its tiles
// reached before saturating (a few thousand of 500k at the headline config), yet the dense buffer
// is 500k x 75 fp32 = 150 MB: a dense NCCL all-reduce of it at 8 GPUs moves ~2 x 7/8 x 150 MB per
// rank.  The sparse exchange moves only the nonzero rows:
//   1. rows_scan  : every rank lists its rows with any nonzero component (one pass over the dense
//                   buffer, reading the reference layouts: position [N][3], rotation [N][4],
//                   log-scale [N][3], opacity [N], sh [N][K][3], feature [d][N]);
//   2. the counts are all-gathered (host reads them: the row exchange is sized by the largest);
//   3. rows_pack  : (row index, R values) records of the listed rows;
//   4. the records are all-gathered;
//   5. rows_zero + rows_add: every rank zeroes all listed rows of all ranks in its dense buffer,
//      then adds the ranks' records in rank order (one launch per rank: rows are unique within a
//      rank, so no atomics) -- the same fp32 sums in the same order on every rank, so replicated
//      maps stay bit-identical after identical optimizer steps.
// Rows nonzero on no rank stay zero, which is also the dense sum.
#include "lgs_internal.cuh"
#include "lgs_kernels.h"

namespace lgs {

struct RowLayout {
  float* ptr[6];      // position, rotation, log_scale, opacity, sh, feature (null: absent)
  int width[6];       // values per row in each attribute
  int64_t n;          // rows
  int R;              // values per row in total
};

// attribute a, component j of row i: feature is [d][N] (column-major), the others [N][width]
__device__ __forceinline__ float* row_elem(const RowLayout& L, int a, int j, int64_t i) {
  return a == 5 ? L.ptr[5] + (int64_t)j * L.n + i : L.ptr[a] + i * L.width[a] + j;
}

__global__ void rows_scan_kernel(RowLayout L, uint32_t* __restrict__ list, uint32_t* __restrict__ count) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool nz = false;
  if (i < L.n) {
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      if (!L.ptr[a]) continue;
      for (int j = 0; j < L.width[a] && !nz; ++j) nz = *row_elem(L, a, j, i) != 0.0f;
    }
  }
  const unsigned bal = __ballot_sync(0xffffffffu, nz);
  if (!bal) return;
  const int lane = threadIdx.x & 31;
  uint32_t base = 0;
  if (lane == 0) base = atomicAdd(count, (uint32_t)__popc(bal));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (nz) list[base + __popc(bal & ((1u << lane) - 1u))] = (uint32_t)i;
}

// record k: [index bits, R values]; one warp per record, lanes over the values; at most `cap`
// records (a rank with more rows overflows the exchange: see rows_apply_kernel)
__global__ void rows_pack_kernel(RowLayout L, const uint32_t* __restrict__ list, const uint32_t* __restrict__ count,
                                 int64_t cap, float* __restrict__ rec) {
  const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (k >= *count || k >= cap) return;
  const int64_t i = list[k];
  float* r = rec + k * (L.R + 1);
  if (lane == 0) r[0] = __uint_as_float((uint32_t)i);
  int off = 1;
  for (int a = 0; a < 6; ++a) {
    if (!L.ptr[a]) continue;
    for (int j = lane; j < L.width[a]; j += 32) r[off + j] = *row_elem(L, a, j, i);
    off += L.width[a];
  }
}

// zero (add = false) or add rank r's records into the dense rows; recs of all ranks back to back,
// each rank's block `stride` records long.  If any rank listed more rows than `stride` (a
// capacity-speculative exchange that overflowed) nothing is touched: every rank keeps its own
// gradient and the host re-runs the exchange with exact sizes.
__global__ void rows_apply_kernel(RowLayout L, const float* __restrict__ recs, const uint32_t* __restrict__ counts,
                                  int world, int rank_lo, int rank_hi, int64_t stride, int add) {
  for (int q = 0; q < world; ++q)
    if ((int64_t)counts[q] > stride) return;
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t per = stride;
  const int r = rank_lo + (int)(t / per);
  const int64_t k = t % per;
  if (r >= rank_hi || k >= counts[r]) return;
  const float* rr = recs + ((int64_t)r * stride + k) * (L.R + 1);
  const int64_t i = __float_as_uint(rr[0]);
  int off = 1;
  for (int a = 0; a < 6; ++a) {
    if (!L.ptr[a]) continue;
    for (int j = lane; j < L.width[a]; j += 32) {
      float* e = row_elem(L, a, j, i);
      *e = add ? *e + rr[off + j] : 0.0f;
    }
    off += L.width[a];
  }
}

static RowLayout make_layout(float* const ptr[6], const int width[6], int64_t n) {
  RowLayout L;
  L.n = n;
  L.R = 0;
  for (int a = 0; a < 6; ++a) {
    L.ptr[a] = width[a] ? ptr[a] : nullptr;
    L.width[a] = L.ptr[a] ? width[a] : 0;
    L.R += L.width[a];
  }
  return L;
}

void launch_rows_scan(float* const ptr[6], const int width[6], int64_t n, uint32_t* list, uint32_t* count,
                      cudaStream_t s) {
  cudaMemsetAsync(count, 0, sizeof(uint32_t), s);
  if (n == 0) return;
  rows_scan_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(make_layout(ptr, width, n), list, count);
}

int rows_values(const int width[6], float* const ptr[6]) {
  int R = 0;
  for (int a = 0; a < 6; ++a) R += ptr[a] ? width[a] : 0;
  return R;
}

void launch_rows_pack(float* const ptr[6], const int width[6], int64_t n, const uint32_t* list, const uint32_t* count,
                      int64_t max_rows, float* rec, cudaStream_t s) {
  if (max_rows == 0) return;
  rows_pack_kernel<<<(unsigned)((max_rows * 32 + 255) / 256), 256, 0, s>>>(make_layout(ptr, width, n), list, count,
                                                                           max_rows, rec);
}

// out[0] = 1 if some rank's count exceeds cap, out[1] = the largest count
__global__ void rows_overflow_kernel(const uint32_t* __restrict__ counts, int world, int64_t cap, uint32_t* out) {
  if (threadIdx.x != 0) return;
  uint32_t mx = 0;
  for (int q = 0; q < world; ++q) mx = max(mx, counts[q]);
  out[0] = (int64_t)mx > cap ? 1u : 0u;
  out[1] = mx;
}

void launch_rows_overflow(const uint32_t* counts, int world, int64_t cap, uint32_t* out, cudaStream_t s) {
  rows_overflow_kernel<<<1, 32, 0, s>>>(counts, world, cap, out);
}

void launch_rows_apply(float* const ptr[6], const int width[6], int64_t n, const float* recs, const uint32_t* counts,
                       int world, int64_t stride, cudaStream_t s) {
  if (stride == 0) return;
  const RowLayout L = make_layout(ptr, width, n);
  const int64_t all = (int64_t)world * stride * 32;
  rows_apply_kernel<<<(unsigned)((all + 255) / 256), 256, 0, s>>>(L, recs, counts, world, 0, world, stride, 0);
  for (int r = 0; r < world; ++r)  // rank order: identical sums on every rank
    rows_apply_kernel<<<(unsigned)((stride * 32 + 255) / 256), 256, 0, s>>>(L, recs, counts, world, r, r + 1, stride,
                                                                          1);
}

}  // namespace lgs
