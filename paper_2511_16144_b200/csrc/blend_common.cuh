// blend_common.cuh -- per-(pixel, Gaussian) arithmetic and tile scheduling shared by the forward and
// backward blend kernels.  The alpha is written with explicit _rn intrinsics so both kernels
// evaluate bit-identical alphas (the backward re-derives the forward's contributor set from them;
// a contraction difference between the two kernels could otherwise flip the alpha-skip test).
#pragma once

#include "lgs_internal.cuh"
#include "lgs_kernels.h"

namespace lgs {

// ---- the quadratic form of a splat at a pixel ------------------------------------------------
//
// alpha = opacity * exp(-q/2), q = A dx^2 + 2B dx dy + C dy^2 (renderer.cpp:143-146), dx = px - u.
// Written term by term in fp32, q cancels catastrophically for an elongated conic (a needle, or a
// splat at the near plane seen almost edge-on, centred far outside the image): A dx^2 and C dy^2
// reach 1e10 while q is O(1).  So each staged list entry carries its conic as an orthonormal frame,
// computed ONCE per (tile, entry) in fp64 from the fp32 record and re-centred at the tile centre
// (xc, yc):
//   q = lam1 s^2 + lam2 t^2,  s = e1 . (p - mu),  t = e2 . (p - mu),  e2 = (-e1.y, e1.x),
// scaled by k = log2(e)/2 so that the exp2 power is -(S^2 + T^2) with S = sqrt(k lam1) s and
// T = sqrt(k lam2) t, both affine in the pixel offset (ex, ey) = p - (xc, yc):
//   S = S0 + ux ex + uy ey,  T = T0 + wx ex + wy ey.
// The large offsets live in S0 / T0 (fp64, then rounded), the per-pixel increments are over at most
// 7.5 px, and the sum S^2 + T^2 has no cancellation: the per-pixel error is a few fp32 ulps of the
// power whatever the conic's condition (5 FFMA + 1 FMUL per pixel, as many as the direct form).
// staged: fa = (S0, T0, ux, uy), fb = (wx, wy, dxc, dyc) with (dxc, dyc) = (xc, yc) - mu.
// Every op of the fp64 part is an explicit _rn intrinsic: oracle/lgs_oracle.c restates it bit for
// bit (the kernels' alpha decisions are what the parity tests flag).
constexpr double kHalfLog2eD = 0.72134752044448170368;  // log2(e) / 2
constexpr float kTwoOverHalfLog2e = 2.7725887222397812f;   // 2 / (log2(e) / 2) = 4 ln 2

struct ConicFrame {
  float4 a, b;
};

__device__ __forceinline__ ConicFrame stage_frame(float u, float v, float A, float B, float C, float xc, float yc) {
  const double a = A, b = B, c = C;
  const double h = __dmul_rn(0.5, __dsub_rn(a, c));
  const double r = __dsqrt_rn(__fma_rn(h, h, __dmul_rn(b, b)));
  const double l1 = __dadd_rn(__dmul_rn(0.5, __dadd_rn(a, c)), r);
  double l2 = __ddiv_rn(__fma_rn(a, c, -__dmul_rn(b, b)), l1);
  if (!(l2 > 0.0)) l2 = 0.0;  // a record conic that is not positive definite (cond > ~1e7)
  // eigenvector of lam1: (lam1 - C, B) or (B, lam1 - A), whichever has no cancellation
  double ex, ey;
  if (h >= 0.0) {
    ex = __dadd_rn(h, r);
    ey = b;
  } else {
    ex = b;
    ey = __dsub_rn(r, h);
  }
  const double nrm = __dsqrt_rn(__fma_rn(ex, ex, __dmul_rn(ey, ey)));
  double cx = 1.0, cy = 0.0;
  if (nrm > 0.0) {
    cx = __ddiv_rn(ex, nrm);
    cy = __ddiv_rn(ey, nrm);
  }
  const double a1 = __dsqrt_rn(__dmul_rn(kHalfLog2eD, l1)), a2 = __dsqrt_rn(__dmul_rn(kHalfLog2eD, l2));
  const double dxc = __dsub_rn((double)xc, (double)u), dyc = __dsub_rn((double)yc, (double)v);
  const double s0 = __dmul_rn(a1, __fma_rn(cx, dxc, __dmul_rn(cy, dyc)));
  const double t0 = __dmul_rn(a2, __fma_rn(cx, dyc, -__dmul_rn(cy, dxc)));
  ConicFrame f;
  f.a = make_float4(__double2float_rn(s0), __double2float_rn(t0), __double2float_rn(__dmul_rn(a1, cx)),
                    __double2float_rn(__dmul_rn(a1, cy)));
  f.b = make_float4(__double2float_rn(-__dmul_rn(a2, cy)), __double2float_rn(__dmul_rn(a2, cx)),
                    __double2float_rn(dxc), __double2float_rn(dyc));
  return f;
}

// S, T and the exp2 power -(S^2 + T^2) at pixel offset (ex, ey) from the tile centre
__device__ __forceinline__ float frame_power(const float4& fa, const float4& fb, float ex, float ey, float& S,
                                             float& T) {
  S = __fmaf_rn(fa.z, ex, __fmaf_rn(fa.w, ey, fa.x));
  T = __fmaf_rn(fb.x, ex, __fmaf_rn(fb.y, ey, fa.y));
  return -__fmaf_rn(S, S, __fmul_rn(T, T));
}

// alpha = opacity * exp(-q/2); G = exp(-q/2) for the backward's clamp test (renderer.cpp:273-274)
__device__ __forceinline__ float frame_alpha(const float4& fa, const float4& fb, float opacity, float ex, float ey,
                                             float& S, float& T, float& G) {
  G = fast_exp2(frame_power(fa, fb, ex, ey, S, T));
  return __fmul_rn(opacity, G);
}

// dq/d(dx), dq/d(dy) (renderer.cpp:279-282): grad q = (2/k) (S u + T w)
__device__ __forceinline__ void frame_dq(const float4& fa, const float4& fb, float S, float T, float& dq_ddx,
                                         float& dq_ddy) {
  dq_ddx = kTwoOverHalfLog2e * fmaf(S, fa.z, T * fb.x);
  dq_ddy = kTwoOverHalfLog2e * fmaf(S, fa.w, T * fb.y);
}

// ---- paired FP32 (sm_100 FFMA2 / FMUL2 / FADD2: two lanes of IEEE fp32 per instruction) ---------
// A thread's two vertically stacked pixels (PPT = 2) are evaluated as one float2; every paired
// operation is the per-lane IEEE operation of the scalar code, so the results are bit-identical.
__device__ __forceinline__ float2 bc2(float x) { return make_float2(x, x); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }

// frame_alpha for the pixel pair (ex, ey.x) and (ex, ey.y)
__device__ __forceinline__ float2 frame_alpha2(const float4& fa, const float4& fb, float opacity, float2 ex2,
                                               float2 ey2, float2& S, float2& T, float2& G) {
  S = fma2(ex2, bc2(fa.z), fma2(ey2, bc2(fa.w), bc2(fa.x)));
  T = fma2(ex2, bc2(fb.x), fma2(ey2, bc2(fb.y), bc2(fa.y)));
  const float2 p = fma2(S, S, mul2(T, T));
  G = make_float2(fast_exp2(-p.x), fast_exp2(-p.y));
  return mul2(bc2(opacity), G);
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
