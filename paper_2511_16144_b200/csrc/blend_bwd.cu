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
//
// B200 structure: persistent CTAs pull tiles longest-first (blend_common.cuh).  Each thread owns
// PPT vertically adjacent pixels of one column.  Per staged Gaussian a warp first evaluates its
// pixels' alphas (cheap) and skips the Gaussian unless some pixel contributes; then each thread
// sums the up to 28 gradient values over its PPT pixels in registers, the warp reduces them with a
// transposed butterfly (31 SHFL for 32 values instead of 5 per value) after which lane l holds
// slot l, and one warp-wide RED adds the partial sums into that Gaussian's 128-byte accumulator
// line.  The per-pixel feature cotangents live in shared memory ([DP/4][256] float4, conflict-free),
// the other per-pixel state in registers.
// Roofline: FP32/SHFL; ~13 FLOP per evaluated (pixel, Gaussian) + ~100 per contribution.
#include <cstdlib>

#include "blend_common.cuh"
#include "dev_cache.h"

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

// list entries staged per shared-memory batch (static shared memory stays under 48 KB)
template <int DP>
constexpr int bwd_batch() { return DP > 16 ? 64 : 128; }

template <int DP>
struct BwdSmem {
  float4 r0[bwd_batch<DP>()];  // u, v, depth, opacity
  float4 fa[bwd_batch<DP>()];  // conic frame S0, T0, ux, uy (blend_common.cuh stage_frame)
  float4 fb[bwd_batch<DP>()];  // conic frame wx, wy, dxc, dyc
  uint2 rect[bwd_batch<DP>()];
  float4 col[bwd_batch<DP>()];
  uint32_t gid[bwd_batch<DP>()];
  float4 feat[bwd_batch<DP>()][DP > 0 ? DP / 4 : 1];
  float4 gfeat[DP > 0 ? DP / 4 : 1][kBlock];  // per-pixel feature cotangents
};

template <int DP, int SLOTS, int PPT>
__global__ void __launch_bounds__(kBlock / PPT) blend_bwd_kernel(DevMap m, DevCam c, ViewBufs v, TileLists tl,
                                                                   PixelState ps, BwdIn in, float* __restrict__ gacc) {
  constexpr int NT = kBlock / PPT;
  constexpr int DQ = DP > 0 ? DP / 4 : 1;
  constexpr int NB = bwd_batch<DP>();
  // two pixels per thread, one gradient value per lane: paired FP32 (FFMA2) arithmetic, the
  // fused kernel's backward step (blend_fused.cu) on the tape's per-pixel state
#ifdef LGS_BWD_SCALAR
  constexpr bool kPaired = false;
#else
  constexpr bool kPaired = PPT == 2 && SLOTS == 32 && DP <= 16;
#endif
  __shared__ BwdSmem<DP> sm;
  __shared__ uint32_t s_max;
  __shared__ int s_slot;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  int lx, ly0;  // this thread's column and first row in the tile
  thread_pixels<PPT>(tid, lx, ly0);
  const int ntiles = c.tiles_x * c.tiles_y;

  for (int tile = next_tile(tl, ntiles, &s_slot); tile >= 0; tile = next_tile(tl, ntiles, &s_slot)) {
    const int tx = tile % c.tiles_x, ty = tile / c.tiles_x;
    const int px = tx * kTile + lx;
    const int py0 = ty * kTile + ly0;
    // pixel offsets from the tile centre (the conic frames' origin)
    const float xc = (float)(tx * kTile) + 7.5f, yc = (float)(ty * kTile) + 7.5f;
    const float ex = (float)lx - 7.5f;
    float ey[PPT];
#pragma unroll
    for (int k = 0; k < PPT; ++k) ey[k] = (float)(ly0 + k) - 7.5f;
    const uint2 range = tl.ranges[tile];

    float T[PPT], accum[PPT], g_rgb[PPT][3], g_draw[PPT], g_acc[PPT];
    uint32_t last[PPT];
    uint32_t my_max = 0;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const int py = py0 + k;
      const int lp = (ly0 + k) * kTile + lx;  // pixel index within the tile
      T[k] = 1.f; accum[k] = 0.f; last[k] = 0; g_draw[k] = 0.f; g_acc[k] = 0.f;
      g_rgb[k][0] = g_rgb[k][1] = g_rgb[k][2] = 0.f;
      float gf[DP > 0 ? DP : 1];
#pragma unroll
      for (int q = 0; q < (DP > 0 ? DP : 1); ++q) gf[q] = 0.f;
      if (px < c.W && py < c.H) {
        const size_t pix = (size_t)py * c.W + px;
        T[k] = ps.final_t[pix];
        last[k] = ps.n_contrib[pix];
        float g_d = 0.f;
        if (in.cot_stride) {
          const float4* cp = reinterpret_cast<const float4*>(in.g_rgb + pix * in.cot_stride);
          const float4 c0 = cp[0];
          g_rgb[k][0] = c0.x; g_rgb[k][1] = c0.y; g_rgb[k][2] = c0.z; g_d = c0.w;
#pragma unroll
          for (int q = 0; q < DP / 4; ++q) {
            const float4 fv = cp[1 + q];
            gf[q * 4 + 0] = fv.x; gf[q * 4 + 1] = fv.y; gf[q * 4 + 2] = fv.z; gf[q * 4 + 3] = fv.w;
          }
        } else {
          if (in.g_rgb) {
            g_rgb[k][0] = in.g_rgb[pix * 3 + 0];
            g_rgb[k][1] = in.g_rgb[pix * 3 + 1];
            g_rgb[k][2] = in.g_rgb[pix * 3 + 2];
          }
          if (in.g_depth) g_d = in.g_depth[pix];
          if (DP > 0 && in.g_feat) {
#pragma unroll
            for (int q = 0; q < DP; ++q) gf[q] = q < m.d ? in.g_feat[pix * m.d + q] : 0.f;
          }
        }
        const float acc = ps.acc[pix];
        const float mm = fmaxf(acc, 1e-6f);
        g_draw[k] = g_d / mm;
        g_acc[k] = acc > 1e-6f ? -g_d * ps.depth[pix] / mm : 0.f;
      }
      if constexpr (kPaired) {
        // paired path: channel pairs of the thread's two pixels, (p0 c, p1 c, p0 c+1, p1 c+1) at
        // [pair][thread] -- the pixels are the two lanes of every FFMA2 (blend_fused.cu layout)
        float* g = reinterpret_cast<float*>(&sm.gfeat[0][0]);
#pragma unroll
        for (int j = 0; j < DP / 2; ++j) {
          g[((size_t)j * NT + tid) * 4 + k] = gf[2 * j];
          g[((size_t)j * NT + tid) * 4 + 2 + k] = gf[2 * j + 1];
        }
      } else if (DP > 0) {
#pragma unroll
        for (int q = 0; q < DP / 4; ++q)
          sm.gfeat[q][lp] = make_float4(gf[q * 4], gf[q * 4 + 1], gf[q * 4 + 2], gf[q * 4 + 3]);
      }
      my_max = max(my_max, last[k]);
    }
    if (tid == 0) s_max = 0;
    __syncthreads();
    // this warp's traversal length: entries past every one of its pixels' last contributor are
    // skipped without evaluation (warp-uniform)
    const uint32_t warp_last = __reduce_max_sync(0xffffffffu, my_max);
    if (lane == 0 && warp_last) atomicMax(&s_max, warp_last);
    __syncthreads();
    const uint32_t end = range.x + s_max;

    for (int64_t bend = end; bend > (int64_t)range.x; bend -= NB) {
      const uint32_t bstart = (uint32_t)max((int64_t)range.x, bend - NB);
      const int cnt = (int)(bend - bstart);
      __syncthreads();
      for (int e = tid; e < cnt; e += NT) {
        const uint32_t g = __ldg(tl.vals + bstart + e);
        sm.gid[e] = g;
        const float4 r0 = __ldg(v.rec0 + g);
        sm.r0[e] = r0;
        const float4 r1 = __ldg(v.rec1 + g);
        const ConicFrame f = stage_frame(r0.x, r0.y, r1.x, r1.y, r1.z, xc, yc);
        sm.fa[e] = f.a;
        sm.fb[e] = f.b;
        sm.rect[e] = __ldg(v.rect + g);
        sm.col[e] = __ldg(v.color + g);
        if (DP > 0) {
          const float4* fg = reinterpret_cast<const float4*>(m.feat) + (size_t)g * DQ;
#pragma unroll
          for (int q = 0; q < DQ; ++q) sm.feat[e][q] = __ldg(fg + q);
        }
      }
      __syncthreads();
      const int e_top = (int)min((int64_t)cnt - 1, (int64_t)range.x + (int64_t)warp_last - 1 - (int64_t)bstart);
      for (int e = e_top; e >= 0; --e) {
        const uint32_t jrel = bstart + (uint32_t)e - range.x;
        const uint2 rc = sm.rect[e];
        const int ry0 = (int)(rc.y & 0xffffu), ry1 = (int)(rc.y >> 16);
        const bool col_in =
            px >= (int)(rc.x & 0xffffu) && px <= (int)(rc.x >> 16) && py0 <= ry1 && py0 + PPT - 1 >= ry0;
        if (!__any_sync(0xffffffffu, col_in)) continue;  // no pixel of this warp inside the Gaussian's rect
        if constexpr (kPaired) {
          const float4 r0 = sm.r0[e];
          const float4 fa = sm.fa[e], fb = sm.fb[e];
          const float2 ex2 = bc2(ex), ey2 = make_float2(ey[0], ey[PPT - 1]);
          float2 S, Tt, G;
          const float2 al = frame_alpha2(fa, fb, r0.w, ex2, ey2, S, Tt, G);
          const bool ok0 = col_in && jrel < last[0] && py0 >= ry0 && py0 <= ry1 && al.x >= c.alpha_skip;
          const bool ok1 = col_in && jrel < last[PPT - 1] && py0 + 1 >= ry0 && py0 + 1 <= ry1 && al.y >= c.alpha_skip;
          if (!__any_sync(0xffffffffu, ok0 || ok1)) continue;
          const float2 alpha = make_float2(ok0 ? al.x : 0.f, ok1 ? al.y : 0.f);
          float vals[SLOTS];
#pragma unroll
          for (int q = 0; q < SLOTS; ++q) vals[q] = 0.f;
          const float4 col = sm.col[e];
          const float op = r0.w;
          const float do_dlogit = op * (1.0f - op);
          const float2 a = make_float2(fminf(alpha.x, c.alpha_clamp), fminf(alpha.y, c.alpha_clamp));
          const float2 inv1ma = make_float2(fast_rcp(1.0f - a.x), fast_rcp(1.0f - a.y));
          float2 Tp = make_float2(T[0], T[PPT - 1]);
          Tp = mul2(Tp, inv1ma);  // transmittance before this contributor (unchanged when a = 0)
          T[0] = Tp.x;
          T[PPT - 1] = Tp.y;
          const float2 w = mul2(a, Tp);
          const float2 g_draw2 = make_float2(g_draw[0], g_draw[PPT - 1]);
          const float2 g_r = make_float2(g_rgb[0][0], g_rgb[PPT - 1][0]);
          const float2 g_g = make_float2(g_rgb[0][1], g_rgb[PPT - 1][1]);
          const float2 g_b = make_float2(g_rgb[0][2], g_rgb[PPT - 1][2]);
          float2 dl = fma2(g_draw2, bc2(r0.z), make_float2(g_acc[0], g_acc[PPT - 1]));
          dl = fma2(g_r, bc2(col.x), dl);
          dl = fma2(g_g, bc2(col.y), dl);
          dl = fma2(g_b, bc2(col.z), dl);
          if (DP > 0) {
            const float4* gp = reinterpret_cast<const float4*>(&sm.gfeat[0][0]);
#pragma unroll
            for (int q = 0; q < DQ; ++q) {
              const float4 fv = sm.feat[e][q];
              const float4 g01 = gp[(size_t)(2 * q) * NT + tid];      // channels 4q, 4q+1 of both pixels
              const float4 g23 = gp[(size_t)(2 * q + 1) * NT + tid];  // channels 4q+2, 4q+3
              dl = fma2(make_float2(g01.x, g01.y), bc2(fv.x), dl);
              dl = fma2(make_float2(g01.z, g01.w), bc2(fv.y), dl);
              dl = fma2(make_float2(g23.x, g23.y), bc2(fv.z), dl);
              dl = fma2(make_float2(g23.z, g23.w), bc2(fv.w), dl);
              float* vf = vals + kSlotFeat + q * 4;
              vf[0] = fmaf(g01.y, w.y, g01.x * w.x);
              vf[1] = fmaf(g01.w, w.y, g01.z * w.x);
              vf[2] = fmaf(g23.y, w.y, g23.x * w.x);
              vf[3] = fmaf(g23.w, w.y, g23.z * w.x);
            }
          }
          float2 acc2 = make_float2(accum[0], accum[PPT - 1]);
          const float2 dla = fma2(make_float2(-acc2.x, -acc2.y), inv1ma, mul2(Tp, dl));
          const float2 dl_da = make_float2((alpha.x != 0.f && !(alpha.x > c.alpha_clamp)) ? dla.x : 0.f,
                                           (alpha.y != 0.f && !(alpha.y > c.alpha_clamp)) ? dla.y : 0.f);
          acc2 = fma2(dl, w, acc2);
          accum[0] = acc2.x;
          accum[PPT - 1] = acc2.y;
          vals[kSlotColor + 0] = fmaf(g_r.y, w.y, g_r.x * w.x);
          vals[kSlotColor + 1] = fmaf(g_g.y, w.y, g_g.x * w.x);
          vals[kSlotColor + 2] = fmaf(g_b.y, w.y, g_b.x * w.x);
          vals[kSlotZ] = fmaf(g_draw2.y, w.y, g_draw2.x * w.x);
          const float2 dlg = mul2(dl_da, G);
          vals[kSlotOpac] = (dlg.x + dlg.y) * do_dlogit;
          const float2 cf = mul2(mul2(dl_da, bc2(op)), mul2(bc2(-0.5f), G));  // dl_dg * dg_dq
          const float2 dqx = mul2(bc2(kTwoOverHalfLog2e), fma2(S, bc2(fa.z), mul2(Tt, bc2(fb.x))));
          const float2 dqy = mul2(bc2(kTwoOverHalfLog2e), fma2(S, bc2(fa.w), mul2(Tt, bc2(fb.y))));
          const float2 dx = add2(bc2(fb.z), ex2), dy = add2(bc2(fb.w), ey2);
          const float2 mx = mul2(cf, dqx), my = mul2(cf, dqy);
          vals[kSlotMuX] = -(mx.x + mx.y);
          vals[kSlotMuY] = -(my.x + my.y);
          const float2 cdx = mul2(cf, dx), cdy = mul2(cf, dy);
          const float2 ca = mul2(cdx, dx), cb2_ = mul2(cdx, dy), cc = mul2(cdy, dy);
          vals[kSlotConA] = ca.x + ca.y;
          vals[kSlotConB] = cb2_.x + cb2_.y;
          vals[kSlotConC] = cc.x + cc.y;
          warp_transpose_reduce<SLOTS>(vals, lane);
          gacc_add(gacc + (size_t)sm.gid[e] * SLOTS, lane, vals[0]);
          continue;
        }
        // phase 1: alphas of this thread's pixels (cheap); most rect hits fail the alpha test
        const float4 r0 = sm.r0[e];
        const float4 fa = sm.fa[e], fb = sm.fb[e];
        // Branch-free over the PPT pixels: independent chains the scheduler can interleave.  A
        // pixel that does not contribute gets alpha = 0 (T / accum / colour / feature terms add
        // exactly +0) and a zero dL/dalpha mask for the opacity, mean and conic terms.
        float alphas[PPT], Gs[PPT], Ss[PPT], Ts[PPT];
#pragma unroll
        for (int k = 0; k < PPT; ++k) alphas[k] = frame_alpha(fa, fb, r0.w, ex, ey[k], Ss[k], Ts[k], Gs[k]);
        bool any = false;
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          const int py = py0 + k;
          const float al = alphas[k];
          const bool ok = col_in && jrel < last[k] && py >= ry0 && py <= ry1 && al >= c.alpha_skip;
          alphas[k] = ok ? al : 0.f;
          any = any || ok;
        }
        if (!__any_sync(0xffffffffu, any)) continue;
        // phase 2: contributions, summed over this thread's pixels, then one warp reduction
        float vals[SLOTS];
#pragma unroll
        for (int q = 0; q < SLOTS; ++q) vals[q] = 0.f;
        const float4 col = sm.col[e];
        const float o = r0.w;
        const float do_dlogit = o * (1.0f - o);
        float w[PPT], dldw[PPT], inv1ma[PPT];
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          const float a = fminf(alphas[k], c.alpha_clamp);
          inv1ma[k] = fast_rcp(1.0f - a);
          T[k] = T[k] * inv1ma[k];  // transmittance before this contributor (unchanged when a = 0)
          w[k] = a * T[k];
          float dl = fmaf(g_draw[k], r0.z, g_acc[k]);
          dl = fmaf(g_rgb[k][0], col.x, dl);
          dl = fmaf(g_rgb[k][1], col.y, dl);
          dl = fmaf(g_rgb[k][2], col.z, dl);
          dldw[k] = dl;
        }
        if (DP > 0) {
#pragma unroll
          for (int q = 0; q < DQ; ++q) {
            const float4 fv = sm.feat[e][q];
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
              const int lp = (ly0 + k) * kTile + lx;
              const float4 gv = sm.gfeat[q][lp];
              dldw[k] = fmaf(gv.x, fv.x, dldw[k]);
              dldw[k] = fmaf(gv.y, fv.y, dldw[k]);
              dldw[k] = fmaf(gv.z, fv.z, dldw[k]);
              dldw[k] = fmaf(gv.w, fv.w, dldw[k]);
              vals[kSlotFeat + q * 4 + 0] = fmaf(gv.x, w[k], vals[kSlotFeat + q * 4 + 0]);
              vals[kSlotFeat + q * 4 + 1] = fmaf(gv.y, w[k], vals[kSlotFeat + q * 4 + 1]);
              vals[kSlotFeat + q * 4 + 2] = fmaf(gv.z, w[k], vals[kSlotFeat + q * 4 + 2]);
              vals[kSlotFeat + q * 4 + 3] = fmaf(gv.w, w[k], vals[kSlotFeat + q * 4 + 3]);
            }
          }
        }
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          const float alpha = alphas[k];
          const float G = Gs[k];
          const float dx = fb.z + ex, dy = fb.w + ey[k];  // pixel - mean (renderer.cpp:141-142)
          float dq_ddx, dq_ddy;
          frame_dq(fa, fb, Ss[k], Ts[k], dq_ddx, dq_ddy);
          // the clamped contributor (and a non-contributing pixel) gets no opacity/mean/conic grad
          const float dl_da = (alpha != 0.f && !(alpha > c.alpha_clamp)) ? T[k] * dldw[k] - accum[k] * inv1ma[k] : 0.f;
          accum[k] = fmaf(dldw[k], w[k], accum[k]);
          vals[kSlotColor + 0] = fmaf(g_rgb[k][0], w[k], vals[kSlotColor + 0]);
          vals[kSlotColor + 1] = fmaf(g_rgb[k][1], w[k], vals[kSlotColor + 1]);
          vals[kSlotColor + 2] = fmaf(g_rgb[k][2], w[k], vals[kSlotColor + 2]);
          vals[kSlotZ] = fmaf(g_draw[k], w[k], vals[kSlotZ]);
          vals[kSlotOpac] = fmaf(dl_da * G, do_dlogit, vals[kSlotOpac]);
          const float cf = dl_da * o * (-0.5f * G);  // dl_dg * dg_dq
          vals[kSlotMuX] = fmaf(-cf, dq_ddx, vals[kSlotMuX]);
          vals[kSlotMuY] = fmaf(-cf, dq_ddy, vals[kSlotMuY]);
          const float cdx = cf * dx;
          vals[kSlotConA] = fmaf(cdx, dx, vals[kSlotConA]);
          vals[kSlotConB] = fmaf(cdx, dy, vals[kSlotConB]);
          vals[kSlotConC] = fmaf(cf * dy, dy, vals[kSlotConC]);
        }
        warp_transpose_reduce<SLOTS>(vals, lane);
        float* row = gacc + (size_t)sm.gid[e] * SLOTS;
#pragma unroll
        for (int q = 0; q < SLOTS / 32; ++q) gacc_add(row, lane * (SLOTS / 32) + q, vals[q]);
      }
    }
  }
}

template <int DP, int SLOTS, int PPT>
static void launch_bwd_cfg(const DevMap& m, const DevCam& c, const ViewBufs& v, const TileLists& tl,
                           const PixelState& ps, const BwdIn& in, float* gacc, cudaStream_t s) {
  const int ctas_per_sm = kernel_ctas_per_sm(reinterpret_cast<const void*>(blend_bwd_kernel<DP, SLOTS, PPT>), kBlock / PPT, 0);
  const int sms = device_sm_count();
  const int ntiles = c.tiles_x * c.tiles_y;
  const int grid = min(ntiles, ctas_per_sm * sms);
  cudaMemsetAsync(tl.counter, 0, sizeof(int), s);
  blend_bwd_kernel<DP, SLOTS, PPT><<<grid, kBlock / PPT, 0, s>>>(m, c, v, tl, ps, in, gacc);
}

template <int DP>
static void launch_bwd_dp(const DevMap& m, const DevCam& c, const ViewBufs& v, const TileLists& tl,
                          const PixelState& ps, const BwdIn& in, float* gacc, cudaStream_t s) {
  // 2 pixels per thread (1 and 4 measured slower: DESIGN.md section 5)
  launch_bwd_cfg<DP, slots_for(DP), 2>(m, c, v, tl, ps, in, gacc, s);
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
