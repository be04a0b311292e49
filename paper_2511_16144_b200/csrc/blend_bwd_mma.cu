// blend_bwd_mma.cu -- K6 on tensor cores: the backward blend restructured around three small GEMMs.
//
// Same semantics as blend_bwd.cu (proj/src/renderer.cpp:198-291; see that file's header), different
// arithmetic organization.  Per tile, with the pixels' cotangent rows
//   X[p] = [g_feat(p) (DP), g_rgb(p) (3), g_draw(p), 0 ...]                       (NCOL columns)
// and, per staged Gaussian e, Y[e] = [f_e (DP), c_e (3), z_e, 0 ...], the reference's per-pixel
// reverse pass (renderer.cpp:233-289) only needs, per (pixel p, Gaussian e):
//   dL/dw_pe   = X[p].Y[e] + g_acc(p)                                              (:236-245)
//   w_pe, dL/dalpha_pe from the transmittance recurrence                           (:253-257)
// and the per-Gaussian gradients are sums over the tile's pixels that factor into GEMMs:
//   colour / feature / depth grads (:259-265)        = sum_p w_pe X[p]             = (W^T X)[e]
//   mean, conic, opacity grads (:276-288)            = sum_p c_pe poly(dx, dy)      from
//     the moments (C^T Phi)[e], Phi[p] = [1, x, y, x^2, xy, y^2] of tile-centred pixel
//     coordinates, with c_pe = dL/dalpha o (-G/2) (0 when clamped, :274), converted back to
//     sums of dx = x - u, dy = y - v exactly (binomial shift).
// So one CTA per tile runs, for each 16-Gaussian sub-batch (in reverse list order):
//   1. D = X Y^T on tensor cores (mma.sync m16n8k8 TF32, 3xTF32 split for ~fp32 accuracy);
//   2. the per-pixel scalar recurrence (one pixel per thread, no shuffles, no reductions);
//   3. W^T X and C^T Phi on tensor cores, each warp over its own 32 pixels, summed across the
//      8 warps in shared memory, and one RED per (Gaussian, gradient value) per tile.
// This replaces the per-(warp, Gaussian) 28-value shuffle reductions and the 16-wide feature
// FMAs of the SIMT kernel.  Persistent CTAs pull tiles longest-first (blend_common.cuh).
#include <cstdlib>

#include "blend_common.cuh"
#include "mma_tf32.cuh"

namespace lgs {

namespace {

constexpr int kNT = 256;       // threads per CTA (one pixel each)
constexpr int kRec = 64;       // Gaussians staged per record batch
constexpr int kSub = 16;       // Gaussians per MMA sub-batch
constexpr int kWS = kSub + 1;  // row stride of the W / C buffers (odd: spread banks)

template <int DP>
struct MmaCfg {
  static constexpr int NCOL = ((DP + 4) + 7) / 8 * 8;  // X / Y columns (padded to the MMA k/n step)
  static constexpr int XS = NCOL;                        // X row stride
  static constexpr int YS = NCOL + 4;                    // Y row stride (conflict-free B fragments)
  static constexpr int RS = NCOL + 8 + 1;                // reduction row: NCOL linear + 8 moments
  static constexpr size_t smem_bytes() {
    return sizeof(float) * ((size_t)kNT * XS + 2 * (size_t)kNT * kWS + (size_t)kRec * YS + (size_t)kSub * RS) +
           sizeof(float4) * 3 * kRec + sizeof(uint2) * kRec + sizeof(uint32_t) * kRec + 64;
  }
};

template <int DP>
__global__ void __launch_bounds__(kNT) blend_bwd_mma_kernel(DevMap m, DevCam c, ViewBufs v, TileLists tl,
                                                          PixelState ps, BwdIn in, float* __restrict__ gacc) {
  using Cfg = MmaCfg<DP>;
  constexpr int NCOL = Cfg::NCOL, XS = Cfg::XS, YS = Cfg::YS, RS = Cfg::RS;
  constexpr int KT1 = NCOL / 8;  // k-steps of step 1 (= n-tiles of the linear part of step 3)
  extern __shared__ float4 smem4[];
  float* Xs = reinterpret_cast<float*>(smem4);             // [256][XS]
  float* Ws = Xs + kNT * XS;                               // [256][kWS]: dL/dw base, then w
  float* Cs = Ws + kNT * kWS;                              // [256][kWS]: c = dL/dalpha o (-G/2)
  float* Ys = Cs + kNT * kWS;                              // [kRec][YS]
  float* red = Ys + kRec * YS;                             // [kSub][RS]
  float4* s_r0 = reinterpret_cast<float4*>(red + kSub * RS + ((kSub * RS) & 3 ? 4 - ((kSub * RS) & 3) : 0));
  float4* s_sc = s_r0 + kRec;
  float4* s_r1 = s_sc + kRec;
  uint2* s_rect = reinterpret_cast<uint2*>(s_r1 + kRec);
  uint32_t* s_gid = reinterpret_cast<uint32_t*>(s_rect + kRec);
  __shared__ uint32_t s_max;
  __shared__ int s_slot;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid4 = lane >> 2, tig = lane & 3;
  int lx, ly;
  thread_pixels<1>(tid, lx, ly);
  const int ntiles = c.tiles_x * c.tiles_y;
  // tile-centred coordinates of the pixels of MMA rows p = tid (for Phi in step 3)
  const float cx_ = (float)lx - 7.5f, cy_ = (float)ly - 7.5f;

  for (int i = tid; i < kSub * RS; i += kNT) red[i] = 0.f;
  // B fragments of Phi (step 3), the same for every tile: Phi[p][j] for p = 32 warp + 8 kt + tig
  // (+4), j = gid4: 1, x, y, x^2, xy, y^2, 0, 0 of the pixel's tile-centred coordinates (exact in TF32)
  uint32_t phi[4][2];
#pragma unroll
  for (int kt = 0; kt < 4; ++kt)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int pl = kt * 8 + tig + 4 * h;  // lane of the pixel row within this warp
      const float px_ = __shfl_sync(0xffffffffu, cx_, pl);
      const float py_ = __shfl_sync(0xffffffffu, cy_, pl);
      const float vals[8] = {1.f, px_, py_, px_ * px_, px_ * py_, py_ * py_, 0.f, 0.f};
      float sel = vals[0];
#pragma unroll
      for (int q = 1; q < 8; ++q) sel = gid4 == q ? vals[q] : sel;
      phi[kt][h] = __float_as_uint(sel);
    }

  for (int tile = next_tile(tl, ntiles, &s_slot); tile >= 0; tile = next_tile(tl, ntiles, &s_slot)) {
    const int tx = tile % c.tiles_x, ty = tile / c.tiles_x;
    const int px = tx * kTile + lx, py = ty * kTile + ly;
    const float fpx = (float)px, fpy = (float)py;
    const float ox = (float)(tx * kTile) + 7.5f, oy = (float)(ty * kTile) + 7.5f;  // tile centre
    const uint2 range = tl.ranges[tile];

    // ---- per-pixel state and cotangent row ------------------------------------------------
    float T = 1.f, accum = 0.f, g_acc = 0.f;
    uint32_t last = 0;
    {
      float xrow[NCOL];
#pragma unroll
      for (int k = 0; k < NCOL; ++k) xrow[k] = 0.f;
      if (px < c.W && py < c.H) {
        const size_t pix = (size_t)py * c.W + px;
        T = ps.final_t[pix];
        last = ps.n_contrib[pix];
        float g_d = 0.f;
        if (in.cot_stride) {
          const float4* cp = reinterpret_cast<const float4*>(in.g_rgb + pix * in.cot_stride);
          const float4 c0 = cp[0];
          xrow[DP + 0] = c0.x; xrow[DP + 1] = c0.y; xrow[DP + 2] = c0.z; g_d = c0.w;
#pragma unroll
          for (int q = 0; q < DP / 4; ++q) {
            const float4 fv = cp[1 + q];
            xrow[q * 4 + 0] = fv.x; xrow[q * 4 + 1] = fv.y; xrow[q * 4 + 2] = fv.z; xrow[q * 4 + 3] = fv.w;
          }
        } else {
          if (in.g_rgb) {
            xrow[DP + 0] = in.g_rgb[pix * 3 + 0];
            xrow[DP + 1] = in.g_rgb[pix * 3 + 1];
            xrow[DP + 2] = in.g_rgb[pix * 3 + 2];
          }
          if (in.g_depth) g_d = in.g_depth[pix];
          if (DP > 0 && in.g_feat) {
#pragma unroll
            for (int q = 0; q < DP; ++q) xrow[q] = q < m.d ? in.g_feat[pix * m.d + q] : 0.f;
          }
        }
        const float acc = ps.acc[pix];
        const float mm = fmaxf(acc, 1e-6f);
        xrow[DP + 3] = g_d / mm;  // g_draw (renderer.cpp:211)
        g_acc = acc > 1e-6f ? -g_d * ps.depth[pix] / mm : 0.f;
      }
#pragma unroll
      for (int k = 0; k < NCOL; ++k) Xs[tid * XS + k] = xrow[k];
    }
    if (tid == 0) s_max = 0;
    __syncthreads();
    if (last) atomicMax(&s_max, last);
    __syncthreads();
    const uint32_t end = range.x + s_max;

    for (int64_t bend = end; bend > (int64_t)range.x; bend -= kRec) {
      const uint32_t bstart = (uint32_t)max((int64_t)range.x, bend - kRec);
      const int cnt = (int)(bend - bstart);
      __syncthreads();  // previous records / Y no longer in use
      for (int e = tid; e < kRec; e += kNT) {
        float yrow[NCOL];
#pragma unroll
        for (int k = 0; k < NCOL; ++k) yrow[k] = 0.f;
        if (e < cnt) {
          const uint32_t g = __ldg(tl.vals + bstart + e);
          s_gid[e] = g;
          const float4 r0 = __ldg(v.rec0 + g);
          const float4 r1 = __ldg(v.rec1 + g);
          s_r0[e] = r0;
          s_r1[e] = r1;
          const ScaledConic s = scale_conic(r1.x, r1.y, r1.z);
          s_sc[e] = make_float4(s.a, s.b2, s.c, 0.f);
          s_rect[e] = __ldg(v.rect + g);
          const float4 col = __ldg(v.color + g);
          if (DP > 0) {
            const float4* fg = reinterpret_cast<const float4*>(m.feat) + (size_t)g * (DP / 4);
#pragma unroll
            for (int q = 0; q < DP / 4; ++q) {
              const float4 fv = __ldg(fg + q);
              yrow[q * 4 + 0] = fv.x; yrow[q * 4 + 1] = fv.y; yrow[q * 4 + 2] = fv.z; yrow[q * 4 + 3] = fv.w;
            }
          }
          yrow[DP + 0] = col.x; yrow[DP + 1] = col.y; yrow[DP + 2] = col.z; yrow[DP + 3] = r0.z;
        } else {
          s_rect[e] = make_uint2(0xffffu, 0xffffu);  // empty rect: no pixel inside
          s_gid[e] = 0;
        }
#pragma unroll
        for (int k = 0; k < NCOL; ++k) Ys[e * YS + k] = yrow[k];
      }
      __syncthreads();

      const int nsub = (cnt + kSub - 1) / kSub;
      for (int sb = nsub - 1; sb >= 0; --sb) {
        const int e0 = sb * kSub;  // record-batch index of the sub-batch's first Gaussian
        // ---- step 1: base dL/dw = X Y^T for this warp's 32 pixel rows x 16 Gaussians ---------
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const int r0w = warp * 32 + mt * 16;
          float d[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
          for (int kt = 0; kt < KT1; ++kt) {
            const int k0 = kt * 8;
            uint32_t ah[4], al[4];
            split_tf32(Xs[(r0w + gid4) * XS + k0 + tig], ah[0], al[0]);
            split_tf32(Xs[(r0w + gid4 + 8) * XS + k0 + tig], ah[1], al[1]);
            split_tf32(Xs[(r0w + gid4) * XS + k0 + tig + 4], ah[2], al[2]);
            split_tf32(Xs[(r0w + gid4 + 8) * XS + k0 + tig + 4], ah[3], al[3]);
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
              const int e = e0 + nt * 8 + gid4;
              uint32_t bh[2], bl[2];
              split_tf32(Ys[e * YS + k0 + tig], bh[0], bl[0]);
              split_tf32(Ys[e * YS + k0 + tig + 4], bh[1], bl[1]);
              mma_3xtf32(d[nt], ah, al, bh, bl);
            }
          }
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            Ws[(r0w + gid4) * kWS + nt * 8 + 2 * tig] = d[nt][0];
            Ws[(r0w + gid4) * kWS + nt * 8 + 2 * tig + 1] = d[nt][1];
            Ws[(r0w + gid4 + 8) * kWS + nt * 8 + 2 * tig] = d[nt][2];
            Ws[(r0w + gid4 + 8) * kWS + nt * 8 + 2 * tig + 1] = d[nt][3];
          }
        }
        __syncwarp();
        // ---- step 2: per-pixel reverse recurrence (renderer.cpp:248-288) -----------------------
        // C starts zeroed; W entries are overwritten only where the pixel contributes, so rows are
        // zeroed where it does not; Gaussians whose rect misses the whole warp are skipped.
        float wrow[kSub];
#pragma unroll
        for (int el = 0; el < kSub; ++el) {
          wrow[el] = 0.f;
          Cs[tid * kWS + el] = 0.f;
        }
#pragma unroll
        for (int el = kSub - 1; el >= 0; --el) {
          const int e = e0 + el;
          const uint32_t jrel = bstart + (uint32_t)e - range.x;
          const bool cand = e < cnt && jrel < last && in_rect(s_rect[e], px, py);
          if (!__any_sync(0xffffffffu, cand)) continue;
          if (!cand) continue;
          const float4 r0 = s_r0[e];
          const float4 s4 = s_sc[e];
          float dx, dy, G;
          const float alpha = splat_alpha(r0.x, r0.y, ScaledConic{s4.x, s4.y, s4.z}, r0.w, fpx, fpy, dx, dy, G);
          if (!(alpha >= c.alpha_skip)) continue;
          const float a = fminf(alpha, c.alpha_clamp);
          const float inv1ma = __frcp_rn(1.0f - a);
          T = T * inv1ma;  // transmittance before this contributor
          const float w = a * T;
          const float dldw = Ws[tid * kWS + el] + g_acc;
          const float dl_da = T * dldw - accum * inv1ma;
          accum = fmaf(dldw, w, accum);
          wrow[el] = w;
          if (!(alpha > c.alpha_clamp)) Cs[tid * kWS + el] = dl_da * r0.w * (-0.5f * G);
        }
#pragma unroll
        for (int el = 0; el < kSub; ++el) Ws[tid * kWS + el] = wrow[el];
        __syncwarp();
        // ---- step 3: W^T X (linear grads) and C^T Phi (moments) over this warp's pixels -------
        float o[KT1 + 1][4];
#pragma unroll
        for (int nt = 0; nt <= KT1; ++nt) o[nt][0] = o[nt][1] = o[nt][2] = o[nt][3] = 0.f;
#pragma unroll
        for (int kt = 0; kt < 4; ++kt) {
          const int p0 = warp * 32 + kt * 8;  // pixel rows of this k-step
          uint32_t wh[4], wl[4], ch[4], cl[4];
          split_tf32(Ws[(p0 + tig) * kWS + gid4], wh[0], wl[0]);
          split_tf32(Ws[(p0 + tig) * kWS + gid4 + 8], wh[1], wl[1]);
          split_tf32(Ws[(p0 + tig + 4) * kWS + gid4], wh[2], wl[2]);
          split_tf32(Ws[(p0 + tig + 4) * kWS + gid4 + 8], wh[3], wl[3]);
          split_tf32(Cs[(p0 + tig) * kWS + gid4], ch[0], cl[0]);
          split_tf32(Cs[(p0 + tig) * kWS + gid4 + 8], ch[1], cl[1]);
          split_tf32(Cs[(p0 + tig + 4) * kWS + gid4], ch[2], cl[2]);
          split_tf32(Cs[(p0 + tig + 4) * kWS + gid4 + 8], ch[3], cl[3]);
#pragma unroll
          for (int nt = 0; nt < KT1; ++nt) {
            uint32_t bh[2], bl[2];
            split_tf32(Xs[(p0 + tig) * XS + nt * 8 + gid4], bh[0], bl[0]);
            split_tf32(Xs[(p0 + tig + 4) * XS + nt * 8 + gid4], bh[1], bl[1]);
            mma_3xtf32(o[nt], wh, wl, bh, bl);
          }
          const uint32_t b[2] = {phi[kt][0], phi[kt][1]};
          mma_2xtf32(o[KT1], ch, cl, b);
        }
        // sum the 8 warps' partial sums (rows = Gaussians of the sub-batch)
#pragma unroll
        for (int nt = 0; nt <= KT1; ++nt) {
          atomicAdd(&red[gid4 * RS + nt * 8 + 2 * tig], o[nt][0]);
          atomicAdd(&red[gid4 * RS + nt * 8 + 2 * tig + 1], o[nt][1]);
          atomicAdd(&red[(gid4 + 8) * RS + nt * 8 + 2 * tig], o[nt][2]);
          atomicAdd(&red[(gid4 + 8) * RS + nt * 8 + 2 * tig + 1], o[nt][3]);
        }
        __syncthreads();
        // ---- emit: one RED per (Gaussian, gradient slot) of the tile -------------------------
        constexpr int NV = DP + 4 + 6;  // feat, rgb, z | mu 2, conic 3, opacity
        for (int i = tid; i < kSub * NV; i += kNT) {
          const int el = i / NV, sidx = i - el * NV;
          const int e = e0 + el;
          if (e >= cnt) continue;
          const float* rr = red + el * RS;
          float val;
          int slot;
          if (sidx < DP) { val = rr[sidx]; slot = kSlotFeat + sidx; }
          else if (sidx < DP + 3) { val = rr[sidx]; slot = kSlotColor + (sidx - DP); }
          else if (sidx == DP + 3) { val = rr[DP + 3]; slot = kSlotZ; }
          else {
            // moments -> sums over dx = x - u, dy = y - v (x, y tile-centred)
            const float* mo = rr + NCOL;
            const float4 r0 = s_r0[e];
            const float4 r1 = s_r1[e];
            const float ub = r0.x - ox, vb = r0.y - oy;
            const float S0 = mo[0];
            const float Sx = mo[1] - ub * S0, Sy = mo[2] - vb * S0;
            const int gq = sidx - (DP + 4);
            if (gq == 0) { val = -(2.0f * r1.x * Sx + 2.0f * r1.y * Sy); slot = kSlotMuX; }
            else if (gq == 1) { val = -(2.0f * r1.z * Sy + 2.0f * r1.y * Sx); slot = kSlotMuY; }
            else if (gq == 2) { val = mo[3] - 2.0f * ub * mo[1] + ub * ub * S0; slot = kSlotConA; }
            else if (gq == 3) { val = mo[4] - ub * mo[2] - vb * mo[1] + ub * vb * S0; slot = kSlotConB; }
            else if (gq == 4) { val = mo[5] - 2.0f * vb * mo[2] + vb * vb * S0; slot = kSlotConC; }
            else { val = -2.0f * (1.0f - r0.w) * S0; slot = kSlotOpac; }
          }
          gacc_add(gacc + (size_t)s_gid[e] * 32, slot, val);
        }
        __syncthreads();
        for (int i = tid; i < kSub * RS; i += kNT) red[i] = 0.f;
        // (the next sub-batch's first red write follows at least one __syncthreads-free step 1-3;
        //  its atomics are ordered after this zeroing by the __syncthreads below)
        __syncthreads();
      }
    }
  }
}

}  // namespace

bool blend_bwd_mma_supported(int dp) { return dp == 16; }

void launch_blend_bwd_mma(const DevMap& m, const DevCam& c, const ViewBufs& v, const TileLists& tl,
                          const PixelState& ps, const BwdIn& in, float* gacc, cudaStream_t s) {
  using Cfg = MmaCfg<16>;
  static int ctas_per_sm = 0, sms = 0;
  const size_t smem = Cfg::smem_bytes();
  if (!ctas_per_sm) {
    cudaFuncSetAttribute(blend_bwd_mma_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm, blend_bwd_mma_kernel<16>, kNT, smem);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (ctas_per_sm < 1) ctas_per_sm = 1;
  }
  const int ntiles = c.tiles_x * c.tiles_y;
  const int grid = min(ntiles, ctas_per_sm * sms);
  cudaMemsetAsync(tl.counter, 0, sizeof(int), s);
  blend_bwd_mma_kernel<16><<<grid, kNT, smem, s>>>(m, c, v, tl, ps, in, gacc);
}

}  // namespace lgs
