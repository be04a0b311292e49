// blend_common.cuh -- per-(pixel, Gaussian) arithmetic shared by the forward and backward blend
// kernels.  Written with explicit _rn intrinsics so both kernels evaluate bit-identical alphas
// (the backward re-derives the forward's contributor set from them; a contraction difference
// between the two kernels could otherwise flip the alpha-skip test on a pixel).
#pragma once

#include "lgs_internal.cuh"

namespace lgs {

// alpha = opacity * exp(-q/2), q = A dx^2 + 2B dx dy + C dy^2 (renderer.cpp:143-146).
// Also returns G = exp(-q/2) for the backward's clamp test (renderer.cpp:273-274).
__device__ __forceinline__ float splat_alpha(float u, float v, float A, float B, float C, float opacity,
                                             float px, float py, float& dx, float& dy, float& G) {
  dx = __fsub_rn(px, u);
  dy = __fsub_rn(py, v);
  float q = __fmul_rn(__fmul_rn(C, dy), dy);
  q = __fmaf_rn(__fmul_rn(__fmul_rn(2.0f, B), dx), dy, q);
  q = __fmaf_rn(__fmul_rn(A, dx), dx, q);
  G = fast_exp2(__fmul_rn(q, kNegHalfLog2e));
  return __fmul_rn(opacity, G);
}

// inclusive pixel rect test (renderer.cpp:131-136)
__device__ __forceinline__ bool in_rect(uint2 r, int px, int py) {
  return px >= (int)(r.x & 0xffffu) && px <= (int)(r.x >> 16) && py >= (int)(r.y & 0xffffu) &&
         py <= (int)(r.y >> 16);
}

}  // namespace lgs
