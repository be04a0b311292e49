// blend_fwd.cu -- K5: per-tile front-to-back alpha blending (RGB + depth + d-dim feature + acc).
//
// Restates the compositing loop of proj/src/renderer.cpp:125-165 tile by tile: one 256-thread CTA
// per 16x16 tile, one pixel per thread, Gaussians of the tile's (depth, index)-sorted list staged
// 256 at a time in shared memory.  Reference semantics kept exactly:
//   - pixel centres at integer coordinates (dx = x - u, :141-142);
//   - a Gaussian only touches pixels inside its inclusive pixel rect (:131-136);
//   - the transmittance test precedes evaluation, so the Gaussian that pushes T below T_min is
//     still composited and the pixel stops afterwards (:140, :158);
//   - skip when !(alpha >= 1/255) (NaN-safe, :147), then clamp alpha to 0.99 (:148);
//   - the same weight w = alpha T accumulates colour, feature, depth and acc (:150-156);
//   - depth is normalized by max(acc, 1e-6) (:163-165).
// The per-pixel feature accumulators (DP fp32) stay in registers.  A CTA leaves its list as soon as
// every pixel of the tile is done (__syncthreads_count), the tile-level early exit.
// Roofline: FP32/SFU-bound; ~30 FLOP + 1 EX2 per evaluated (pixel, Gaussian), +45 per contribution.
#include "blend_common.cuh"
#include "lgs_kernels.h"

namespace lgs {

template <int DP>
struct FwdSmem {
  float4 r0[kBlock];    // u, v, depth, opacity
  float4 r1[kBlock];    // A, B, C, -
  uint2 rect[kBlock];
  float4 col[kBlock];
  float4 feat[kBlock][DP > 0 ? DP / 4 : 1];
};

template <int DP, bool L1>
__global__ void __launch_bounds__(kBlock) blend_fwd_kernel(DevMap m, DevCam c, ViewBufs v, TileLists tl,
                                                             PixelState ps, FwdOut o) {
  __shared__ FwdSmem<DP> sm;
  __shared__ float s_loss[kBlock / 32];
  const int tile = blockIdx.x;
  const int tid = threadIdx.x;
  const int tx = tile % c.tiles_x, ty = tile / c.tiles_x;
  const int px = tx * kTile + (tid & (kTile - 1));
  const int py = ty * kTile + (tid >> 4);
  const bool inside = px < c.W && py < c.H;
  const float fpx = (float)px, fpy = (float)py;
  const uint2 range = tl.ranges[tile];

  float T = 1.0f;
  float cr = 0.f, cg = 0.f, cb = 0.f, draw = 0.f, acc = 0.f;
  float f[DP > 0 ? DP : 1];
#pragma unroll
  for (int k = 0; k < (DP > 0 ? DP : 1); ++k) f[k] = 0.f;
  uint32_t last = 0;
  uint32_t n_eval = 0, n_contrib = 0;
  bool done = !inside || !(1.0f >= c.t_min);

  for (uint32_t base = range.x; base < range.y; base += kBlock) {
    if (__syncthreads_count(done) == kBlock) break;
    const uint32_t j = base + tid;
    if (j < range.y) {
      const uint32_t g = __ldg(tl.vals + j);
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
    const int cnt = (int)min((uint32_t)kBlock, range.y - base);
    for (int k = 0; k < cnt && !done; ++k) {
      if (!in_rect(sm.rect[k], px, py)) continue;
      const float4 r0 = sm.r0[k];
      const float4 r1 = sm.r1[k];
      float dx, dy, G;
      float alpha = splat_alpha(r0.x, r0.y, r1.x, r1.y, r1.z, r0.w, fpx, fpy, dx, dy, G);
      ++n_eval;
      if (!(alpha >= c.alpha_skip)) continue;
      ++n_contrib;
      alpha = fminf(alpha, c.alpha_clamp);
      const float w = __fmul_rn(alpha, T);
      const float4 col = sm.col[k];
      cr = fmaf(w, col.x, cr);
      cg = fmaf(w, col.y, cg);
      cb = fmaf(w, col.z, cb);
      draw = fmaf(w, r0.z, draw);
      acc += w;
      if (DP > 0) {
#pragma unroll
        for (int q = 0; q < DP / 4; ++q) {
          const float4 fv = sm.feat[k][q];
          f[q * 4 + 0] = fmaf(w, fv.x, f[q * 4 + 0]);
          f[q * 4 + 1] = fmaf(w, fv.y, f[q * 4 + 1]);
          f[q * 4 + 2] = fmaf(w, fv.z, f[q * 4 + 2]);
          f[q * 4 + 3] = fmaf(w, fv.w, f[q * 4 + 3]);
        }
      }
      T = __fmul_rn(T, __fsub_rn(1.0f, alpha));
      last = base + k + 1 - range.x;
      if (T < c.t_min) done = true;
    }
  }

  float loss = 0.f;
  if (inside) {
    const size_t pix = (size_t)py * c.W + px;
    const float dnorm = draw / fmaxf(acc, 1e-6f);
    ps.final_t[pix] = T;
    ps.n_contrib[pix] = last;
    ps.depth[pix] = dnorm;
    ps.acc[pix] = acc;
    ps.work[pix] = make_uint2(n_eval, n_contrib);
    if (o.rgb) {
      o.rgb[pix * 3 + 0] = cr;
      o.rgb[pix * 3 + 1] = cg;
      o.rgb[pix * 3 + 2] = cb;
    }
    if (o.depth) o.depth[pix] = dnorm;
    if (o.acc) o.acc[pix] = acc;
    if (DP > 0 && o.feat) {
      float* fo = o.feat + pix * m.d;
      if (m.d == DP) {
#pragma unroll
        for (int q = 0; q < DP / 4; ++q)
          reinterpret_cast<float4*>(fo)[q] = make_float4(f[q * 4], f[q * 4 + 1], f[q * 4 + 2], f[q * 4 + 3]);
      } else {
#pragma unroll
        for (int k = 0; k < DP; ++k)
          if (k < m.d) fo[k] = f[k];
      }
    }
    if (L1) {
      // L = mean|rgb - T| + mean|depth - T| + mean|feat - T|; cotangent sign(diff) / count
      const float npx = (float)c.W * (float)c.H;
      const float inv_rgb = 1.0f / (3.0f * npx), inv_d = 1.0f / npx, inv_f = m.d > 0 ? 1.0f / ((float)m.d * npx) : 0.f;
      float* cot = o.cot + pix * (4 + DP);
      const float vals[3] = {cr, cg, cb};
      float lr = 0.f, lf = 0.f;
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        const float df = vals[ch] - o.t_rgb[pix * 3 + ch];
        cot[ch] = df > 0.f ? inv_rgb : (df < 0.f ? -inv_rgb : 0.f);
        lr += fabsf(df);
      }
      const float dd = dnorm - o.t_depth[pix];
      cot[3] = dd > 0.f ? inv_d : (dd < 0.f ? -inv_d : 0.f);
#pragma unroll
      for (int k = 0; k < DP; ++k) {
        float gk = 0.f;
        if (k < m.d) {
          const float df = f[k] - o.t_feat[pix * m.d + k];
          gk = df > 0.f ? inv_f : (df < 0.f ? -inv_f : 0.f);
          lf += fabsf(df);
        }
        cot[4 + k] = gk;
      }
      loss = lr * inv_rgb + fabsf(dd) * inv_d + lf * inv_f;
    }
  }
  if (L1) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) loss += __shfl_xor_sync(0xffffffffu, loss, off);
    if ((tid & 31) == 0) s_loss[tid >> 5] = loss;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < kBlock / 32; ++w) s += s_loss[w];
      atomicAdd(o.loss, s);
    }
  }
}

template <int DP>
static void launch_fwd_dp(const DevMap& m, const DevCam& c, const ViewBufs& v, const TileLists& tl,
                          const PixelState& ps, const FwdOut& o, cudaStream_t s) {
  const unsigned tiles = (unsigned)(c.tiles_x * c.tiles_y);
  if (o.cot) blend_fwd_kernel<DP, true><<<tiles, kBlock, 0, s>>>(m, c, v, tl, ps, o);
  else blend_fwd_kernel<DP, false><<<tiles, kBlock, 0, s>>>(m, c, v, tl, ps, o);
}

void launch_blend_fwd(const DevMap& m, const DevCam& c, const ViewBufs& v, const TileLists& tl,
                      const PixelState& ps, const FwdOut& o, cudaStream_t s) {
  switch (m.dp) {
    case 0: launch_fwd_dp<0>(m, c, v, tl, ps, o, s); break;
    case 4: launch_fwd_dp<4>(m, c, v, tl, ps, o, s); break;
    case 8: launch_fwd_dp<8>(m, c, v, tl, ps, o, s); break;
    case 16: launch_fwd_dp<16>(m, c, v, tl, ps, o, s); break;
    default: launch_fwd_dp<32>(m, c, v, tl, ps, o, s); break;
  }
}

}  // namespace lgs
