// blend_fused.cu -- K5 + K6 in one kernel for the fused-L1 captured step (lgs_plan).
//
// With the L1 loss of SURVEY.md §8d the cotangents of a pixel depend on that pixel's outputs only,
// so a tile can run its backward (renderer.cpp:198-291) right after its forward (:125-165):
//   - the forward part is blend_fwd.cu's compositing loop (same arithmetic, bit-identical images);
//   - its epilogue writes the images and the loss partial and keeps the cotangents, the final
//     transmittance, the last contributor, acc and depth of each pixel in registers (the feature
//     cotangents in shared memory) instead of the per-pixel tape;
//   - the backward part is blend_bwd.cu's reverse traversal, reading the records the forward
//     staged: with the depth-layered lists a tile's traversal fits one staged batch, so the
//     backward normally reloads nothing (other batches are restaged as blend_bwd does).
// Saves the backward's record staging, the tape round trip (~104 B per pixel) and a kernel
// boundary, and keeps both phases' latency in one CTA.  The first layered pass leaves unsaturated
// tiles (flagged) without backward; the second pass renders them here on their complete lists.
#include "blend_common.cuh"
#include "dev_cache.h"

namespace lgs {

template <int DP>
struct FusedSmem {
  static constexpr int NB = 192;  // list entries per staged batch (static shared memory < 48 KB)
  float4 r0[NB];                  // u, v, depth, opacity
  float4 fa[NB];                  // conic frame S0, T0, ux, uy (blend_common.cuh stage_frame)
  float4 fb[NB];                  // conic frame wx, wy, dxc, dyc
  uint2 rect[NB];
  float4 col[NB];
  uint32_t gid[NB];
  float4 feat[NB][DP > 0 ? DP / 4 : 1];
  float4 gfeat[DP > 0 ? DP / 4 : 1][kBlock];  // per-pixel feature cotangents
};

template <int SLOTS>
__device__ __forceinline__ void fused_transpose_reduce(float (&v)[SLOTS], int lane) {
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
__global__ void __launch_bounds__(kBlock / 2) blend_fused_l1_kernel(DevMap m, DevCam c, ViewBufs v, TileLists tl,
                                                                      FwdOut o, float* __restrict__ gacc) {
  griddep_wait();
  constexpr int PPT = 2;
  constexpr int NT = kBlock / PPT;
  constexpr int DQ = DP > 0 ? DP / 4 : 1;
  constexpr int FD = DP > 0 ? DP : 1;
  constexpr int SLOTS = 32;
  using Smem = FusedSmem<DP>;
  constexpr int NB = Smem::NB;
  __shared__ Smem sm;
  __shared__ float s_loss[NT / 32];
  __shared__ uint32_t s_max;
  __shared__ int s_slot;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  int lx, ly0;
  thread_pixels<PPT>(tid, lx, ly0);
  const int ntiles = c.tiles_x * c.tiles_y;
  float loss = 0.f;
  const float npx = (float)c.W * (float)c.H;
  const float inv_rgb = 1.0f / (3.0f * npx), inv_d = 1.0f / npx;
  const float inv_f = m.d > 0 ? 1.0f / ((float)m.d * npx) : 0.f;

  // stage list entries [b0, b0 + cnt) of the tile's list (range.x-relative positions); (xc, yc) =
  // the tile centre the conic frames are centred on
  auto stage = [&](uint32_t list0, int cnt, float xc, float yc) {
    for (int e = tid; e < cnt; e += NT) {
      const uint32_t g = __ldg(tl.vals + list0 + e);
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
  };

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
    const uint32_t len = range.y - range.x;

    // ---------------- forward (blend_fwd.cu) ----------------
    float T[PPT], cr[PPT], cg[PPT], cb[PPT], draw[PPT], acc[PPT];
    float f[PPT][FD];
    uint32_t last[PPT];
    bool done[PPT];
    bool all_done = true;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      T[k] = 1.f; cr[k] = cg[k] = cb[k] = draw[k] = acc[k] = 0.f;
#pragma unroll
      for (int q = 0; q < FD; ++q) f[k][q] = 0.f;
      last[k] = 0;
      done[k] = !(px < c.W && py0 + k < c.H) || !(1.0f >= c.t_min);
      all_done = all_done && done[k];
    }
    int res_batch = -1;  // batch index resident in shared memory
    for (uint32_t pos = 0; pos < len; pos += NB) {
      if (__syncthreads_count(all_done) == NT) break;
      const int cnt = (int)min((uint32_t)NB, len - pos);
      stage(range.x + pos, cnt, xc, yc);
      res_batch = (int)(pos / NB);
      __syncthreads();
      auto composite = [&](int e, const float (&al)[PPT], const bool (&in)[PPT], float depth_z) {
        float a[PPT];
        bool ok[PPT];
        bool any = false;
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          const bool live = in[k] && !done[k];
          ok[k] = live && al[k] >= c.alpha_skip;
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
          if (ok[k]) last[k] = pos + e + 1;
          done[k] = done[k] || T[k] < c.t_min;
        }
      };
      for (int e = 0; e < cnt && !all_done; e += 2) {
        const bool has1 = e + 1 < cnt;
        const uint2 rc0 = sm.rect[e];
        const uint2 rc1 = has1 ? sm.rect[e + 1] : make_uint2(0xffffu, 0xffffu);
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

    // ---------------- epilogue: images, loss, cotangents kept on chip ----------------
    const bool tile_done = o.unfinished ? __syncthreads_and(all_done) != 0 : true;
    if (!tile_done && tid == 0) o.unfinished[tile] = 1u;
    float g_rgb[PPT][3], g_draw[PPT], g_acc[PPT];
    uint32_t my_max = 0;
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const int py = py0 + k;
      const int lp = (ly0 + k) * kTile + lx;
      g_rgb[k][0] = g_rgb[k][1] = g_rgb[k][2] = 0.f;
      g_draw[k] = g_acc[k] = 0.f;
      float gf[FD];
#pragma unroll
      for (int q = 0; q < FD; ++q) gf[q] = 0.f;
      if (px < c.W && py < c.H) {
        const size_t pix = (size_t)py * c.W + px;
        const float dnorm = draw[k] / fmaxf(acc[k], 1e-6f);
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
              reinterpret_cast<float4*>(fo)[q] = make_float4(f[k][q * 4], f[k][q * 4 + 1], f[k][q * 4 + 2],
                                                             f[k][q * 4 + 3]);
          } else {
#pragma unroll
            for (int q = 0; q < FD; ++q)
              if (q < m.d) fo[q] = f[k][q];
          }
        }
        if (tile_done) {  // L1 (blend_fwd.cu): cotangent sign(diff) / count, loss partial
          const float vals[3] = {cr[k], cg[k], cb[k]};
          float lr = 0.f, lf = 0.f;
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            const float df = vals[ch] - o.t_rgb[pix * 3 + ch];
            g_rgb[k][ch] = df > 0.f ? inv_rgb : (df < 0.f ? -inv_rgb : 0.f);
            lr += fabsf(df);
          }
          const float dd = dnorm - o.t_depth[pix];
          const float g_d = dd > 0.f ? inv_d : (dd < 0.f ? -inv_d : 0.f);
#pragma unroll
          for (int q = 0; q < DP; ++q) {
            if (q < m.d) {
              const float df = f[k][q] - o.t_feat[pix * m.d + q];
              gf[q] = df > 0.f ? inv_f : (df < 0.f ? -inv_f : 0.f);
              lf += fabsf(df);
            }
          }
          loss += lr * inv_rgb + fabsf(dd) * inv_d + lf * inv_f;
          // backward per-pixel constants (renderer.cpp:204-212)
          const float mm = fmaxf(acc[k], 1e-6f);
          g_draw[k] = g_d / mm;
          g_acc[k] = acc[k] > 1e-6f ? -g_d * dnorm / mm : 0.f;
        }
      }
      if (DP > 0) {
#pragma unroll
        for (int q = 0; q < DP / 4; ++q)
          sm.gfeat[q][lp] = make_float4(gf[q * 4], gf[q * 4 + 1], gf[q * 4 + 2], gf[q * 4 + 3]);
      }
      if (!tile_done) last[k] = 0;  // rendered again by the second pass
      my_max = max(my_max, last[k]);
    }

    // ---------------- backward (blend_bwd.cu) ----------------
    if (tid == 0) s_max = 0;
    __syncthreads();
    const uint32_t warp_last = __reduce_max_sync(0xffffffffu, my_max);
    if (lane == 0 && warp_last) atomicMax(&s_max, warp_last);
    __syncthreads();
    float accum[PPT] = {};
    for (int b = s_max ? (int)((s_max - 1) / NB) : -1; b >= 0; --b) {
      const uint32_t bpos = (uint32_t)b * NB;
      const int cnt = (int)min((uint32_t)NB, len - bpos);
      if (b != res_batch) {  // restage (long traversals only); the resident batch is reused
        __syncthreads();
        stage(range.x + bpos, cnt, xc, yc);
        res_batch = b;
        __syncthreads();
      }
      const int e_top = (int)min((int64_t)cnt - 1, (int64_t)warp_last - 1 - (int64_t)bpos);
      for (int e = e_top; e >= 0; --e) {
        const uint32_t jrel = bpos + (uint32_t)e;
        const uint2 rc = sm.rect[e];
        const int ry0 = (int)(rc.y & 0xffffu), ry1 = (int)(rc.y >> 16);
        const bool col_in =
            px >= (int)(rc.x & 0xffffu) && px <= (int)(rc.x >> 16) && py0 <= ry1 && py0 + PPT - 1 >= ry0;
        if (!__any_sync(0xffffffffu, col_in)) continue;
        const float4 r0 = sm.r0[e];
        const float4 fa = sm.fa[e], fb = sm.fb[e];
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
        float vals[SLOTS];
#pragma unroll
        for (int q = 0; q < SLOTS; ++q) vals[q] = 0.f;
        const float4 col = sm.col[e];
        const float op = r0.w;
        const float do_dlogit = op * (1.0f - op);
        float w[PPT], dldw[PPT], inv1ma[PPT];
#pragma unroll
        for (int k = 0; k < PPT; ++k) {
          const float a = fminf(alphas[k], c.alpha_clamp);
          inv1ma[k] = fast_rcp(1.0f - a);
          T[k] = T[k] * inv1ma[k];
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
          const float dl_da = (alpha != 0.f && !(alpha > c.alpha_clamp)) ? T[k] * dldw[k] - accum[k] * inv1ma[k] : 0.f;
          accum[k] = fmaf(dldw[k], w[k], accum[k]);
          vals[kSlotColor + 0] = fmaf(g_rgb[k][0], w[k], vals[kSlotColor + 0]);
          vals[kSlotColor + 1] = fmaf(g_rgb[k][1], w[k], vals[kSlotColor + 1]);
          vals[kSlotColor + 2] = fmaf(g_rgb[k][2], w[k], vals[kSlotColor + 2]);
          vals[kSlotZ] = fmaf(g_draw[k], w[k], vals[kSlotZ]);
          vals[kSlotOpac] = fmaf(dl_da * G, do_dlogit, vals[kSlotOpac]);
          const float cf = dl_da * op * (-0.5f * G);
          vals[kSlotMuX] = fmaf(-cf, dq_ddx, vals[kSlotMuX]);
          vals[kSlotMuY] = fmaf(-cf, dq_ddy, vals[kSlotMuY]);
          const float cdx = cf * dx;
          vals[kSlotConA] = fmaf(cdx, dx, vals[kSlotConA]);
          vals[kSlotConB] = fmaf(cdx, dy, vals[kSlotConB]);
          vals[kSlotConC] = fmaf(cf * dy, dy, vals[kSlotConC]);
        }
        fused_transpose_reduce<SLOTS>(vals, lane);
        gacc_add(gacc + (size_t)sm.gid[e] * SLOTS, lane, vals[0]);
      }
    }
  }

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

bool blend_fused_supported(int dp) { return dp == 16 || dp == 8 || dp == 4 || dp == 0; }

template <int DP>
static void launch_fused_dp(const DevMap& m, const DevCam& c, const ViewBufs& v, const TileLists& tl, const FwdOut& o,
                            float* gacc, cudaStream_t s, bool counter_zeroed) {
  const int ctas_per_sm = kernel_ctas_per_sm(reinterpret_cast<const void*>(blend_fused_l1_kernel<DP>), kBlock / 2, 0);
  const int sms = device_sm_count();
  const int ntiles = c.tiles_x * c.tiles_y;
  const int grid = min(ntiles, ctas_per_sm * sms);
  if (!counter_zeroed) cudaMemsetAsync(tl.counter, 0, sizeof(int), s);
  launch_pdl(blend_fused_l1_kernel<DP>, dim3(grid), dim3(kBlock / 2), 0, s, m, c, v, tl, o, gacc);
}

void launch_blend_fused_l1(const DevMap& m, const DevCam& c, const ViewBufs& v, const TileLists& tl, const FwdOut& o,
                           float* gacc, cudaStream_t s, bool counter_zeroed) {
  switch (m.dp) {
    case 0: launch_fused_dp<0>(m, c, v, tl, o, gacc, s, counter_zeroed); break;
    case 4: launch_fused_dp<4>(m, c, v, tl, o, gacc, s, counter_zeroed); break;
    case 8: launch_fused_dp<8>(m, c, v, tl, o, gacc, s, counter_zeroed); break;
    default: launch_fused_dp<16>(m, c, v, tl, o, gacc, s, counter_zeroed); break;
  }
}

}  // namespace lgs
