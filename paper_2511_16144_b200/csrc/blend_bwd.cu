// blend_bwd.cu -- K6: per-tile reverse traversal producing per-Gaussian screen-space gradients.
//
// Restates the per-pixel reverse pass of proj/src/renderer.cpp:198-291 with the forward's tape
// instead of per-pixel contributor vectors:
//   - the contributor set of a pixel is re-derived from the tile list up to the pixel's
//     n_contrib (bit-identical alphas, blend_common.cuh), T is recovered back to front from the
//     forward's final T by T_r = T_{r+1} / (1 - alpha_r);
//   - g_draw = g_d / max(acc, 1e-6), g_acc = acc > 1e-6 ? -g_d depth / m : 0 (:204-212);
//   - dL/dw_r = g_draw z + g_acc + g_rgb.c + g_feat.f (:233-246);
//   - dL/dalpha_r = T_r dL/dw_r - (sum_{i>r} dL/dw_i w_i) / (1 - alpha_r) (:256-257);
//   - colour / feature / depth grads for every contributor (:259-265); opacity, mean and conic
//     grads only when opacity * G <= clamp (:274-288), both conic off-diagonals (:285-288).
// Per-Gaussian reduction: the up to 32 gradient values of one Gaussian are reduced across the warp
// by a transposed butterfly (31 SHFL instead of 5 per value) after which lane l holds slot l; one
// warp-wide RED then adds the warp's partial sums into that Gaussian's 128-byte accumulator line.
// Warps where no lane contributed skip both (__any_sync).
// Roofline: FP32/SFU + L2-atomic bound (~110 FLOP per contribution; 1 RED line per warp-Gaussian).
#include "blend_common.cuh"
#include "lgs_kernels.h"

namespace lgs {

template <int SLOTS>
__device__ __forceinline__ void warp_transpose_reduce(float (&v)[SLOTS], int lane) {
#pragma unroll
  for (int step = 0; step < 5; ++step) {
    const int k = 16 >> step;
    const int half = SLOTS >> (step + 1);
    const bool upper = (lane & k) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float send = upper ? v[i] : v[i + half];
      const float keep = upper ? v[i + half] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, k);
    }
  }
}

template <int DP>
struct BwdSmem {
  float4 r0[kBlock];  // u, v, depth, opacity
  float4 r1[kBlock];  // A, B, C, -
  uint2 rect[kBlock];
  float4 col[kBlock];
  uint32_t gid[kBlock];
  float4 feat[kBlock][DP > 0 ? DP / 4 : 1];
};

template <int DP, int SLOTS>
__global__ void __launch_bounds__(kBlock) blend_bwd_kernel(DevMap m, DevCam c, ViewBufs v, TileLists tl,
                                                             PixelState ps, BwdIn in, float* __restrict__ gacc) {
  __shared__ BwdSmem<DP> sm;
  __shared__ uint32_t s_max;
  const int tile = blockIdx.x;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int tx = tile % c.tiles_x, ty = tile / c.tiles_x;
  const int px = tx * kTile + (tid & (kTile - 1));
  const int py = ty * kTile + (tid >> 4);
  const bool inside = px < c.W && py < c.H;
  const float fpx = (float)px, fpy = (float)py;
  const uint2 range = tl.ranges[tile];

  float T = 1.f;
  uint32_t last = 0;
  float g_rgb[3] = {0.f, 0.f, 0.f};
  float g_f[DP > 0 ? DP : 1];
#pragma unroll
  for (int k = 0; k < (DP > 0 ? DP : 1); ++k) g_f[k] = 0.f;
  float g_draw = 0.f, g_acc = 0.f;
  if (inside) {
    const size_t pix = (size_t)py * c.W + px;
    T = ps.final_t[pix];
    last = ps.n_contrib[pix];
    float g_d = 0.f;
    if (in.cot_stride) {
      const float4* cp = reinterpret_cast<const float4*>(in.g_rgb + pix * in.cot_stride);
      const float4 c0 = cp[0];
      g_rgb[0] = c0.x; g_rgb[1] = c0.y; g_rgb[2] = c0.z; g_d = c0.w;
#pragma unroll
      for (int q = 0; q < DP / 4; ++q) {
        const float4 fv = cp[1 + q];
        g_f[q * 4 + 0] = fv.x; g_f[q * 4 + 1] = fv.y; g_f[q * 4 + 2] = fv.z; g_f[q * 4 + 3] = fv.w;
      }
    } else {
      if (in.g_rgb) {
        g_rgb[0] = in.g_rgb[pix * 3 + 0];
        g_rgb[1] = in.g_rgb[pix * 3 + 1];
        g_rgb[2] = in.g_rgb[pix * 3 + 2];
      }
      if (in.g_depth) g_d = in.g_depth[pix];
      if (DP > 0 && in.g_feat) {
#pragma unroll
        for (int k = 0; k < DP; ++k) g_f[k] = k < m.d ? in.g_feat[pix * m.d + k] : 0.f;
      }
    }
    const float acc = ps.acc[pix];
    const float mm = fmaxf(acc, 1e-6f);
    g_draw = g_d / mm;
    g_acc = acc > 1e-6f ? -g_d * ps.depth[pix] / mm : 0.f;
  }
  if (tid == 0) s_max = 0;
  __syncthreads();
  if (last) atomicMax(&s_max, last);
  __syncthreads();
  const uint32_t end = range.x + s_max;

  float accum = 0.f;
  for (int64_t bend = end; bend > (int64_t)range.x; bend -= kBlock) {
    const uint32_t bstart = (uint32_t)max((int64_t)range.x, bend - kBlock);
    const int cnt = (int)(bend - bstart);
    __syncthreads();
    if (tid < cnt) {
      const uint32_t g = __ldg(tl.vals + bstart + tid);
      sm.gid[tid] = g;
      sm.r0[tid] = __ldg(v.rec0 + g);
      sm.r1[tid] = __ldg(v.rec1 + g);
      sm.rect[tid] = __ldg(v.rect + g);
      sm.col[tid] = __ldg(v.color + g);
      if (DP > 0) {
        const float4* fg = reinterpret_cast<const float4*>(m.feat) + (size_t)g * (DP / 4);
#pragma unroll
        for (int k = 0; k < DP / 4; ++k) sm.feat[tid][k] = __ldg(fg + k);
      }
    }
    __syncthreads();
    for (int k = cnt - 1; k >= 0; --k) {
      const uint32_t jrel = bstart + (uint32_t)k - range.x;
      bool contrib = inside && jrel < last && in_rect(sm.rect[k], px, py);
      float vals[SLOTS];
#pragma unroll
      for (int q = 0; q < SLOTS; ++q) vals[q] = 0.f;
      if (contrib) {
        const float4 r0 = sm.r0[k];
        const float4 r1 = sm.r1[k];
        float dx, dy, G;
        const float alpha = splat_alpha(r0.x, r0.y, r1.x, r1.y, r1.z, r0.w, fpx, fpy, dx, dy, G);
        contrib = alpha >= c.alpha_skip;
        if (contrib) {
          const float a = fminf(alpha, c.alpha_clamp);
          const float inv1ma = 1.0f / (1.0f - a);
          T = T * inv1ma;  // transmittance before this contributor
          const float w = a * T;
          const float4 col = sm.col[k];
          float dldw = fmaf(g_draw, r0.z, g_acc);
          dldw = fmaf(g_rgb[0], col.x, dldw);
          dldw = fmaf(g_rgb[1], col.y, dldw);
          dldw = fmaf(g_rgb[2], col.z, dldw);
          if (DP > 0) {
#pragma unroll
            for (int q = 0; q < DP / 4; ++q) {
              const float4 fv = sm.feat[k][q];
              dldw = fmaf(g_f[q * 4 + 0], fv.x, dldw);
              dldw = fmaf(g_f[q * 4 + 1], fv.y, dldw);
              dldw = fmaf(g_f[q * 4 + 2], fv.z, dldw);
              dldw = fmaf(g_f[q * 4 + 3], fv.w, dldw);
            }
          }
          const float dl_da = T * dldw - accum * inv1ma;
          accum = fmaf(dldw, w, accum);
          vals[kSlotColor + 0] = g_rgb[0] * w;
          vals[kSlotColor + 1] = g_rgb[1] * w;
          vals[kSlotColor + 2] = g_rgb[2] * w;
#pragma unroll
          for (int q = 0; q < DP; ++q) vals[kSlotFeat + q] = g_f[q] * w;
          vals[kSlotZ] = g_draw * w;
          if (!(alpha > c.alpha_clamp)) {
            const float o = r0.w;
            vals[kSlotOpac] = dl_da * G * o * (1.0f - o);
            const float cf = dl_da * o * (-0.5f * G);  // dl_dg * dg_dq
            const float twoB = 2.0f * r1.y;
            const float dq_ddx = 2.0f * r1.x * dx + twoB * dy;
            const float dq_ddy = 2.0f * r1.z * dy + twoB * dx;
            vals[kSlotMuX] = -cf * dq_ddx;
            vals[kSlotMuY] = -cf * dq_ddy;
            vals[kSlotConA] = cf * dx * dx;
            vals[kSlotConB] = cf * dx * dy;
            vals[kSlotConC] = cf * dy * dy;
          }
        }
      }
      if (__any_sync(0xffffffffu, contrib)) {
        warp_transpose_reduce<SLOTS>(vals, lane);
        float* dst = gacc + (size_t)sm.gid[k] * SLOTS + lane * (SLOTS / 32);
#pragma unroll
        for (int q = 0; q < SLOTS / 32; ++q)
          if (vals[q] != 0.f) atomicAdd(dst + q, vals[q]);
      }
    }
  }
}

template <int DP>
static void launch_bwd_dp(const DevMap& m, const DevCam& c, const ViewBufs& v, const TileLists& tl,
                          const PixelState& ps, const BwdIn& in, float* gacc, cudaStream_t s) {
  const unsigned tiles = (unsigned)(c.tiles_x * c.tiles_y);
  constexpr int SLOTS = slots_for(DP);
  blend_bwd_kernel<DP, SLOTS><<<tiles, kBlock, 0, s>>>(m, c, v, tl, ps, in, gacc);
}

void launch_blend_bwd(const DevMap& m, const DevCam& c, const ViewBufs& v, const TileLists& tl,
                      const PixelState& ps, const BwdIn& in, float* gacc, int slots, cudaStream_t s) {
  (void)slots;
  switch (m.dp) {
    case 0: launch_bwd_dp<0>(m, c, v, tl, ps, in, gacc, s); break;
    case 4: launch_bwd_dp<4>(m, c, v, tl, ps, in, gacc, s); break;
    case 8: launch_bwd_dp<8>(m, c, v, tl, ps, in, gacc, s); break;
    case 16: launch_bwd_dp<16>(m, c, v, tl, ps, in, gacc, s); break;
    default: launch_bwd_dp<32>(m, c, v, tl, ps, in, gacc, s); break;
  }
}

}  // namespace lgs
