// mma_tf32.cuh -- warp-level TF32 tensor-core MMA (m16n8k8, fp32 accumulate) with the 3-term
// hi/lo split ("3xTF32": a*b ~= a_hi b_hi + a_hi b_lo + a_lo b_hi) that keeps products at ~fp32
// accuracy, which the 1e-3 gradient parity bound needs.
//
// Fragment layouts of mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 (gid = lane / 4,
// tig = lane % 4), pinned on hardware by lgs_debug_mma_selftest (tests/test_gpu_mma.py):
//   A (16 x 8, row-major): a0 = A[gid][tig], a1 = A[gid + 8][tig], a2 = A[gid][tig + 4], a3 = A[gid + 8][tig + 4]
//   B (8 x 8):             b0 = B[tig][gid], b1 = B[tig + 4][gid]
//   C/D (16 x 8):          c0 = C[gid][2 tig], c1 = C[gid][2 tig + 1], c2 = C[gid + 8][2 tig], c3 = C[gid + 8][2 tig + 1]
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace lgs {

__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
  hi = to_tf32(x);
  lo = to_tf32(x - __uint_as_float(hi));
}

__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// d += A * B with both operands split (3 MMAs, small terms first)
__device__ __forceinline__ void mma_3xtf32(float (&d)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4],
                                           const uint32_t (&bh)[2], const uint32_t (&bl)[2]) {
  mma_tf32(d, al, bh);
  mma_tf32(d, ah, bl);
  mma_tf32(d, ah, bh);
}

// d += A * B with B exact in TF32 (2 MMAs)
__device__ __forceinline__ void mma_2xtf32(float (&d)[4], const uint32_t (&ah)[4], const uint32_t (&al)[4],
                                           const uint32_t (&b)[2]) {
  mma_tf32(d, al, b);
  mma_tf32(d, ah, b);
}

}  // namespace lgs
