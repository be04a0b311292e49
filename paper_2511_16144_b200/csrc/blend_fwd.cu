// blend_fwd.cu -- K5: per-tile front-to-back alpha blending (RGB + depth + d-dim feature + acc).
//
// Restates the compositing loop of proj/src/renderer.cpp:125-165 tile by tile.  Reference
// semantics kept exactly:
//   - pixel centres at integer coordinates (dx = x - u, :141-142);
//   - a Gaussian only touches pixels inside its inclusive pixel rect (:131-136);
//   - the transmittance test precedes evaluation, so the Gaussian that pushes T below T_min is
//     still composited and the pixel stops afterwards (:140, :158);
//   - skip when !(alpha >= 1/255) (NaN-safe, :147), then clamp alpha to 0.99 (:148);
//   - the same weight w = alpha T accumulates colour, feature, depth and acc (:150-156);
//   - depth is normalized by max(acc, 1e-6) (:163-165).
//
// B200 structure: persistent CTAs (a few per SM) pull 16x16 tiles longest-list-first from a
// global counter, so the 1200-tile grid of the headline config does not end in a partial wave.
// Each thread owns PPT vertically adjacent pixels of one column (shared dx, shared column rect
// test, one shared-memory read of each staged Gaussian per PPT pixels).  Gaussians of the tile's
// (depth, index)-sorted list are staged 256 at a time in shared memory (record + 16-D feature);
// the per-pixel feature accumulators (DP fp32 each) stay in registers; the CTA leaves the list as
// soon as every pixel is done (__syncthreads_count).  The optional fused L1 loss writes the
// cotangents the backward reads and one loss partial per CTA.
// Roofline: FP32/SFU; ~13 FLOP + 1 EX2 per evaluated (pixel, Gaussian), +45 per contribution.
#include "blend_common.cuh"
#include "dev_cache.h"

namespace lgs {

template <int DP, int NB>
struct FwdSmem {
  float4 r0[NB];  // u, v, depth, opacity
  float4 fa[NB];  // conic frame S0, T0, ux, uy (blend_common.cuh stage_frame)
  float4 fb[NB];  // conic frame wx, wy, dxc, dyc
  uint2 rect[NB];
  float4 col[NB];
  float4 feat[NB][DP > 0 ? DP / 4 : 1];
};

// NB: list entries staged per shared-memory batch; MINB: launch-bounds residency hint (0: none)
// WORK: count evaluated / contributing (pixel, Gaussian) pairs per pixel (profiling only)
template <int DP, bool L1, int PPT, int NB, int MINB, bool WORK>
__global__ void __launch_bounds__(kBlock / PPT, MINB) blend_fwd_kernel(DevMap m, DevCam c, ViewBufs v, TileLists tl,
                                                                         PixelState ps, FwdOut o) {
  constexpr int NT = kBlock / PPT;
  constexpr int DQ = DP > 0 ? DP / 4 : 1;
  constexpr int FD = DP > 0 ? DP : 1;
  __shared__ FwdSmem<DP, NB> sm;
  __shared__ float s_loss[NT / 32];
  __shared__ int s_slot;
  const int tid = threadIdx.x;
  int lx, ly0;  // this thread's column and first row in the tile
  thread_pixels<PPT>(tid, lx, ly0);
  const int ntiles = c.tiles_x * c.tiles_y;
  float loss = 0.f;

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

    float T[PPT], cr[PPT], cg[PPT], cb[PPT], draw[PPT], acc[PPT];
    float f[PPT][FD];
    uint32_t last[PPT], n_eval[PPT], n_contrib[PPT];
    bool done[PPT];
    bool all_done = true;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      T[k] = 1.f; cr[k] = cg[k] = cb[k] = draw[k] = acc[k] = 0.f;
#pragma unroll
      for (int q = 0; q < FD; ++q) f[k][q] = 0.f;
      last[k] = n_eval[k] = n_contrib[k] = 0;
      done[k] = !(px < c.W && py0 + k < c.H) || !(1.0f >= c.t_min);
      all_done = all_done && done[k];
    }

    for (uint32_t base = range.x; base < range.y; base += NB) {
      if (__syncthreads_count(all_done) == NT) break;
      for (int e = tid; e < NB; e += NT) {
        const uint32_t j = base + e;
        if (j < range.y) {
          const uint32_t g = __ldg(tl.vals + j);
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
      }
      __syncthreads();
      const int cnt = (int)min((uint32_t)NB, range.y - base);
      // Composite one staged entry given its pixels' alphas (evaluated earlier): a pixel that does
      // not contribute gets alpha = 0, which leaves T, the accumulators and the counters exactly
      // unchanged (w = +0).
      auto composite = [&](int e, const float (&al)[PPT], const bool (&in)[PPT], float depth_z) {
        float a[PPT];
        bool ok[PPT];
        bool any = false;
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          const bool live = in[k] && !done[k];
          ok[k] = live && al[k] >= c.alpha_skip;
          if (WORK) {
            n_eval[k] += live ? 1u : 0u;
            n_contrib[k] += ok[k] ? 1u : 0u;
          }
          a[k] = ok[k] ? fminf(al[k], c.alpha_clamp) : 0.f;
          any = any || ok[k];
        }
        if (!any) return;
        const float4 col = sm.col[e];
        float w[PPT];
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          w[k] = __fmul_rn(a[k], T[k]);
          cr[k] = fmaf(w[k], col.x, cr[k]);
          cg[k] = fmaf(w[k], col.y, cg[k]);
          cb[k] = fmaf(w[k], col.z, cb[k]);
          draw[k] = fmaf(w[k], depth_z, draw[k]);
          acc[k] += w[k];
        }
        if (DP > 0) {
#pragma unroll
          for (int q = 0; q < DQ; ++q) {
            const float4 fv = sm.feat[e][q];
#pragma unroll
            for (int k = 0; k < PPT; ++k) {
              f[k][q * 4 + 0] = fmaf(w[k], fv.x, f[k][q * 4 + 0]);
              f[k][q * 4 + 1] = fmaf(w[k], fv.y, f[k][q * 4 + 1]);
              f[k][q * 4 + 2] = fmaf(w[k], fv.z, f[k][q * 4 + 2]);
              f[k][q * 4 + 3] = fmaf(w[k], fv.w, f[k][q * 4 + 3]);
            }
          }
        }
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          T[k] = __fmul_rn(T[k], __fsub_rn(1.0f, a[k]));
          if (ok[k]) last[k] = base + e + 1 - range.x;
          done[k] = done[k] || T[k] < c.t_min;
        }
      };
      // Two entries per step: both entries' alphas are evaluated first (independent chains the
      // scheduler interleaves), then they are composited in list order.
      for (int e = 0; e < cnt && !all_done; e += 2) {
        const bool has1 = e + 1 < cnt;
        const uint2 rc0 = sm.rect[e];
        const uint2 rc1 = has1 ? sm.rect[e + 1] : make_uint2(0xffffu, 0xffffu);  // empty rect
        const bool hit0 = px >= (int)(rc0.x & 0xffffu) && px <= (int)(rc0.x >> 16) &&
                          py0 <= (int)(rc0.y >> 16) && py0 + PPT - 1 >= (int)(rc0.y & 0xffffu);
        const bool hit1 = px >= (int)(rc1.x & 0xffffu) && px <= (int)(rc1.x >> 16) &&
                          py0 <= (int)(rc1.y >> 16) && py0 + PPT - 1 >= (int)(rc1.y & 0xffffu);
        if (!hit0 && !hit1) continue;
        const float4 r00 = sm.r0[e], fa0 = sm.fa[e], fb0 = sm.fb[e];
        const float4 r01 = has1 ? sm.r0[e + 1] : r00, fa1 = has1 ? sm.fa[e + 1] : fa0, fb1 = has1 ? sm.fb[e + 1] : fb0;
        float al0[PPT], al1[PPT];
        bool in0[PPT], in1[PPT];
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          float S, T, G;
          al0[k] = frame_alpha(fa0, fb0, r00.w, ex, ey[k], S, T, G);
          al1[k] = frame_alpha(fa1, fb1, r01.w, ex, ey[k], S, T, G);
        }
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          const int py = py0 + k;
          in0[k] = hit0 && py >= (int)(rc0.y & 0xffffu) && py <= (int)(rc0.y >> 16);
          in1[k] = hit1 && py >= (int)(rc1.y & 0xffffu) && py <= (int)(rc1.y >> 16);
        }
        if (hit0) composite(e, al0, in0, r00.z);
        if (hit1) composite(e + 1, al1, in1, r01.z);
        all_done = true;
#pragma unroll
        for (int k = 0; k < PPT; ++k) all_done = all_done && done[k];
      }
    }

    // layered first pass: a tile with an unsaturated pixel is rendered again on its complete list
    const bool tile_done = o.unfinished ? __syncthreads_and(all_done) != 0 : true;
    if (!tile_done && tid == 0) {
      o.unfinished[tile] = 1u;
      if (o.unfinished_any) {
        *reinterpret_cast<volatile uint32_t*>(o.unfinished_any) = 1u;
        *o.miss = 1u;
      }
    }
    if (o.consumed && tile_done) {  // list length this warp consumed (layer-A size policy)
      uint32_t mx = 0;
#pragma unroll
      for (int k = 0; k < PPT; ++k) mx = max(mx, last[k]);
      mx = __reduce_max_sync(0xffffffffu, mx);
      if ((tid & 31) == 0 && mx) atomicAdd(o.consumed, mx);
    }
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const int py = py0 + k;
      if (!(px < c.W && py < c.H)) continue;
      const size_t pix = (size_t)py * c.W + px;
      const float dnorm = draw[k] / fmaxf(acc[k], 1e-6f);
      ps.final_t[pix] = T[k];
      ps.n_contrib[pix] = last[k];
      ps.depth[pix] = dnorm;
      ps.acc[pix] = acc[k];
      if (WORK) ps.work[pix] = make_uint2(n_eval[k], n_contrib[k]);
      if (o.rgb) {
        o.rgb[pix * 3 + 0] = cr[k];
        o.rgb[pix * 3 + 1] = cg[k];
        o.rgb[pix * 3 + 2] = cb[k];
      }
      if (o.depth) o.depth[pix] = dnorm;
      if (o.acc) o.acc[pix] = acc[k];
      if (DP > 0 && o.feat) {
        float* fo = o.feat + pix * m.d;
        if (m.d == DP) {
#pragma unroll
          for (int q = 0; q < DQ; ++q)
            reinterpret_cast<float4*>(fo)[q] = make_float4(f[k][q * 4], f[k][q * 4 + 1], f[k][q * 4 + 2], f[k][q * 4 + 3]);
        } else {
#pragma unroll
          for (int q = 0; q < FD; ++q)
            if (q < m.d) fo[q] = f[k][q];
        }
      }
      if (L1 && tile_done) {
        // L = mean|rgb - T| + mean|depth - T| + mean|feat - T|; cotangent sign(diff) / count
        const float npx = (float)c.W * (float)c.H;
        const float inv_rgb = 1.0f / (3.0f * npx), inv_d = 1.0f / npx;
        const float inv_f = m.d > 0 ? 1.0f / ((float)m.d * npx) : 0.f;
        float* cot = o.cot + pix * (4 + DP);
        const float vals[3] = {cr[k], cg[k], cb[k]};
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
        for (int q = 0; q < DP; ++q) {
          float gk = 0.f;
          if (q < m.d) {
            const float df = f[k][q] - o.t_feat[pix * m.d + q];
            gk = df > 0.f ? inv_f : (df < 0.f ? -inv_f : 0.f);
            lf += fabsf(df);
          }
          cot[4 + q] = gk;
        }
        loss += lr * inv_rgb + fabsf(dd) * inv_d + lf * inv_f;
      }
    }
  }

  if (L1) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) loss += __shfl_xor_sync(0xffffffffu, loss, off);
    if ((tid & 31) == 0) s_loss[tid >> 5] = loss;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < NT / 32; ++w) s += s_loss[w];
      atomicAdd(o.loss, s);
    }
  }
}

template <int DP, bool L1, int PPT, int NB, int MINB, bool WORK>
static void launch_fwd_work(const DevMap& m, const DevCam& c, const ViewBufs& v, const TileLists& tl,
                            const PixelState& ps, const FwdOut& o, cudaStream_t s) {
  const int ctas_per_sm = kernel_ctas_per_sm(reinterpret_cast<const void*>(blend_fwd_kernel<DP, L1, PPT, NB, MINB, WORK>), kBlock / PPT, 0);
  const int sms = device_sm_count();
  const int ntiles = c.tiles_x * c.tiles_y;
  const int grid = min(ntiles, ctas_per_sm * sms);
  cudaMemsetAsync(tl.counter, 0, sizeof(int), s);
  blend_fwd_kernel<DP, L1, PPT, NB, MINB, WORK><<<grid, kBlock / PPT, 0, s>>>(m, c, v, tl, ps, o);
}

template <int DP, bool L1, int PPT, int NB, int MINB>
static void launch_fwd_cfg(const DevMap& m, const DevCam& c, const ViewBufs& v, const TileLists& tl,
                           const PixelState& ps, const FwdOut& o, cudaStream_t s) {
  if (ps.work) launch_fwd_work<DP, L1, PPT, NB, MINB, true>(m, c, v, tl, ps, o, s);
  else launch_fwd_work<DP, L1, PPT, NB, MINB, false>(m, c, v, tl, ps, o, s);
}

template <int DP>
static void launch_fwd_dp(const DevMap& m, const DevCam& c, const ViewBufs& v, const TileLists& tl,
                          const PixelState& ps, const FwdOut& o, cudaStream_t s) {
  constexpr int NB = DP > 16 ? 128 : 256;  // static shared memory stays under 48 KB
  if (o.cot) launch_fwd_cfg<DP, true, 2, NB, 0>(m, c, v, tl, ps, o, s);
  else launch_fwd_cfg<DP, false, 2, NB, 0>(m, c, v, tl, ps, o, s);
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
