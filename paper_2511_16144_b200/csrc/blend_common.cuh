// blend_common.cuh -- per-(pixel, Gaussian) arithmetic and tile scheduling shared by the forward and
// backward blend kernels.  The alpha is written with explicit _rn intrinsics so both kernels
// evaluate bit-identical alphas (the backward re-derives the forward's contributor set from them;
// a contraction difference between the two kernels could otherwise flip the alpha-skip test).
#pragma once

#include "lgs_internal.cuh"
#include "lgs_kernels.h"

namespace lgs {

// Conic pre-scaled for exp2: power = -q/2 * log2(e), q = A dx^2 + 2B dx dy + C dy^2.
struct ScaledConic {
  float a, b2, c;
};

__device__ __forceinline__ ScaledConic scale_conic(float A, float B, float C) {
  return ScaledConic{__fmul_rn(A, kNegHalfLog2e), __fmul_rn(B, 2.0f * kNegHalfLog2e), __fmul_rn(C, kNegHalfLog2e)};
}

// alpha = opacity * exp(-q/2) (renderer.cpp:143-146); also returns G = exp(-q/2) for the backward's
// clamp test (renderer.cpp:273-274) and dx, dy (pixel centres at integer coordinates, :141-142).
__device__ __forceinline__ float splat_alpha(float u, float v, ScaledConic k, float opacity, float px, float py,
                                             float& dx, float& dy, float& G) {
  dx = __fsub_rn(px, u);
  dy = __fsub_rn(py, v);
  const float p = __fmaf_rn(dx, __fmaf_rn(k.a, dx, __fmul_rn(k.b2, dy)), __fmul_rn(__fmul_rn(k.c, dy), dy));
  G = fast_exp2(p);
  return __fmul_rn(opacity, G);
}

// inclusive pixel rect test (renderer.cpp:131-136, intersected with the alpha box, preprocess.cu)
__device__ __forceinline__ bool in_rect(uint2 r, int px, int py) {
  return px >= (int)(r.x & 0xffffu) && px <= (int)(r.x >> 16) && py >= (int)(r.y & 0xffffu) &&
         py <= (int)(r.y >> 16);
}

// Pixels of thread `tid` inside the 16x16 tile when each thread owns PPT vertically stacked pixels:
// column lx, rows ly0 .. ly0 + PPT - 1.  A warp covers a compact 8-column block (8 x 4 PPT pixels)
// rather than a 16-wide strip, so a small splat's footprint fills more of the warp's lanes.
template <int PPT>
__device__ __forceinline__ void thread_pixels(int tid, int& lx, int& ly0) {
  const int warp = tid >> 5, lane = tid & 31;
  lx = (warp & 1) * 8 + (lane & 7);
  ly0 = (warp >> 1) * (4 * PPT) + (lane >> 3) * PPT;
}

// Persistent-CTA tile scheduler: CTAs pull tile slots from a global counter; slot i is the i-th
// longest tile list (TileLists::order), so the long tiles start first and the tail is short.
// With tl.count the order holds only *tl.count tiles (second pass of the layered binning).
__device__ __forceinline__ int next_tile(const TileLists& tl, int ntiles, int* s_slot) {
  __syncthreads();
  if (threadIdx.x == 0) *s_slot = atomicAdd(tl.counter, 1);
  __syncthreads();
  const int slot = *s_slot;
  const int active = tl.count ? (int)*tl.count : ntiles;
  return slot < active ? (tl.order ? (int)tl.order[slot] : slot) : -1;
}

}  // namespace lgs
