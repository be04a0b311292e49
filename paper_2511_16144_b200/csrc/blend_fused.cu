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
#ifndef LGS_FUSED_NB
#define LGS_FUSED_NB 192
#endif
#ifndef LGS_FUSED_DYN_PAD
#define LGS_FUSED_DYN_PAD 0  // experiment builds only: unused dynamic shared memory (occupancy studies)
#endif
  static constexpr int NB = LGS_FUSED_NB;  // list entries per staged batch (static shared memory < 48 KB)
  float4 r0[NB];                  // u, v, depth, opacity
  float4 fa[NB];                  // conic frame S0, T0, ux, uy (blend_common.cuh stage_frame)
  float4 fb[NB];                  // conic frame wx, wy, dxc, dyc
  uint2 rect[NB];
  float4 col[NB];
  uint32_t gid[NB];
  float4 feat[NB][DP > 0 ? DP / 4 : 1];
  float4 gfeat[DP > 0 ? DP / 2 : 1][kBlock / 2];  // feature cotangents: [channel pair][thread] =
                                                  // (pixel 0 c, pixel 1 c, pixel 0 c+1, pixel 1 c+1)
};


#ifdef LGS_FUSED_BULK
// Experiment: the colour and feature rows of a staged batch are copied by the bulk-copy
// (TMA) engine, cp.async.bulk global -> shared completing on an mbarrier, instead of LDG -> STS.
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
}
#endif

// two independent reductions, step by step (their shuffles and adds interleave)
template <int SLOTS>
__device__ __forceinline__ void fused_transpose_reduce2(float (&v)[SLOTS], float (&u)[SLOTS], int lane) {
#pragma unroll
  for (int step = 0; step < 5; ++step) {
    const int k = 16 >> step;
    const int half = SLOTS >> (step + 1);
    const bool upper = (lane & k) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float sv = upper ? v[i] : v[i + half], kv = upper ? v[i + half] : v[i];
      const float su = upper ? u[i] : u[i + half], ku = upper ? u[i + half] : u[i];
      v[i] = kv + __shfl_xor_sync(0xffffffffu, sv, k);
      u[i] = ku + __shfl_xor_sync(0xffffffffu, su, k);
    }
  }
}

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

// ILPF: list entries whose alphas the forward evaluates per step before compositing them in order.
// 2 for the first layered pass (many tiles, 4 CTAs/SM at 128 registers); 4 for the second pass,
// whose few unsaturated tiles walk long complete lists with ~1 CTA per SM (latency bound: more
// independent work per warp, up to 255 registers).
template <int DP, int ILPF>
__device__ __forceinline__ void blend_fused_l1_body(const DevMap& m, const DevCam& c, const ViewBufs& v,
                                                    const TileLists& tl, const FwdOut& o, float* __restrict__ gacc) {
  constexpr int PPT = 2;  // the thread's two pixels are the two lanes of every paired (FFMA2) op
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
  __shared__ long long s_t0;  // tile_cost: clock at the current tile's start (thread 0)
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  int lx, ly0;
  thread_pixels<PPT>(tid, lx, ly0);
  const int ntiles = c.tiles_x * c.tiles_y;
  float loss = 0.f;
  const float npx = (float)c.W * (float)c.H;
  const float inv_rgb = 1.0f / (3.0f * npx), inv_d = 1.0f / npx;
  const float inv_f = m.d > 0 ? 1.0f / ((float)m.d * npx) : 0.f;
  // pixel offsets from the tile centre (the conic frames' origin), as lane pairs
  const float2 ex2 = bc2((float)lx - 7.5f);
  const float2 ey2 = make_float2((float)ly0 - 7.5f, (float)(ly0 + 1) - 7.5f);

  // stage list entries [b0, b0 + cnt) of the tile's list (range.x-relative positions); (xc, yc) =
  // the tile centre the conic frames are centred on
#ifdef LGS_FUSED_BULK
  __shared__ alignas(8) uint64_t s_bar;
  uint32_t bar_parity = 0;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&s_bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
#endif
  auto stage = [&](uint32_t list0, int cnt, float xc, float yc) {
#ifdef LGS_FUSED_BULK
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads before async writes
#endif
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
#ifdef LGS_FUSED_BULK
      bar_expect_tx(&s_bar, 16u * (1u + (DP > 0 ? DQ : 0)));
      bulk_g2s(&sm.col[e], v.color + g, 16u, &s_bar);
      if (DP > 0) bulk_g2s(&sm.feat[e][0], reinterpret_cast<const float4*>(m.feat) + (size_t)g * DQ, 16u * DQ, &s_bar);
#else
      sm.col[e] = __ldg(v.color + g);
      if (DP > 0) {
        const float4* fg = reinterpret_cast<const float4*>(m.feat) + (size_t)g * DQ;
#pragma unroll
        for (int q = 0; q < DQ; ++q) sm.feat[e][q] = __ldg(fg + q);
      }
#endif
    }
  };
  // after stage() and the __syncthreads that follows it: the bulk copies have landed
  auto staged = [&]() {
#ifdef LGS_FUSED_BULK
    if (tid == 0) bar_arrive(&s_bar);
    bar_wait(&s_bar, bar_parity);
    bar_parity ^= 1u;
#endif
  };

  int prev_tile = -1;  // tile_cost: thread 0 closes the previous tile's interval (every warp is past
                      // next_tile's barrier, so the whole tile is done)
  for (int tile = next_tile(tl, ntiles, &s_slot);; tile = next_tile(tl, ntiles, &s_slot)) {
    if (o.tile_cost && tid == 0) {
      const long long now = clock64();
      if (prev_tile >= 0) o.tile_cost[prev_tile] = (uint32_t)min((now - s_t0) >> 4, 0xffffffffll);
      s_t0 = now;
    }
    if (tile < 0) break;
    prev_tile = tile;
    const int tx = tile % c.tiles_x, ty = tile / c.tiles_x;
    const int px = tx * kTile + lx;
    const int py0 = ty * kTile + ly0;
    const float xc = (float)(tx * kTile) + 7.5f, yc = (float)(ty * kTile) + 7.5f;
    const uint2 range = tl.ranges[tile];
    const uint32_t len = range.y - range.x;

    // ---------------- forward (blend_fwd.cu arithmetic, lane-paired) ----------------
    float2 T = bc2(1.f), cr = bc2(0.f), cg = bc2(0.f), cb = bc2(0.f), draw = bc2(0.f), acc = bc2(0.f);
    float2 f[FD];
#pragma unroll
    for (int q = 0; q < FD; ++q) f[q] = bc2(0.f);
    uint32_t last0 = 0, last1 = 0;
    bool done0 = !(px < c.W && py0 < c.H) || !(1.0f >= c.t_min);
    bool done1 = !(px < c.W && py0 + 1 < c.H) || !(1.0f >= c.t_min);
    bool all_done = done0 && done1;
    int res_batch = -1;  // batch index resident in shared memory
    for (uint32_t pos = 0; pos < len; pos += NB) {
      if (__syncthreads_count(all_done) == NT) break;
      const int cnt = (int)min((uint32_t)NB, len - pos);
      stage(range.x + pos, cnt, xc, yc);
      res_batch = (int)(pos / NB);
      __syncthreads();
      staged();
      // composite one staged entry given its pixels' alphas; a pixel that does not contribute gets
      // alpha = 0, which leaves T and the accumulators exactly unchanged (w = +0)
      auto composite = [&](int e, float2 al, bool in0, bool in1, float depth_z) {
        const bool ok0 = in0 && !done0 && al.x >= c.alpha_skip;
        const bool ok1 = in1 && !done1 && al.y >= c.alpha_skip;
        if (!ok0 && !ok1) return;
        const float2 a = make_float2(ok0 ? fminf(al.x, c.alpha_clamp) : 0.f, ok1 ? fminf(al.y, c.alpha_clamp) : 0.f);
        const float4 col = sm.col[e];
        const float2 w = mul2(a, T);
        cr = fma2(w, bc2(col.x), cr);
        cg = fma2(w, bc2(col.y), cg);
        cb = fma2(w, bc2(col.z), cb);
        draw = fma2(w, bc2(depth_z), draw);
        acc = add2(acc, w);
        if (DP > 0) {
#pragma unroll
          for (int q = 0; q < DQ; ++q) {
            const float4 fv = sm.feat[e][q];
            f[q * 4 + 0] = fma2(w, bc2(fv.x), f[q * 4 + 0]);
            f[q * 4 + 1] = fma2(w, bc2(fv.y), f[q * 4 + 1]);
            f[q * 4 + 2] = fma2(w, bc2(fv.z), f[q * 4 + 2]);
            f[q * 4 + 3] = fma2(w, bc2(fv.w), f[q * 4 + 3]);
          }
        }
        T = mul2(T, make_float2(__fsub_rn(1.0f, a.x), __fsub_rn(1.0f, a.y)));
        if (ok0) last0 = pos + e + 1;
        if (ok1) last1 = pos + e + 1;
        done0 = done0 || T.x < c.t_min;
        done1 = done1 || T.y < c.t_min;
      };
      if constexpr (ILPF == 2) {  // (hand-paired: the generic form below costs 18 registers more)
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
        float2 S, Tt, G;
        const float2 al0 = frame_alpha2(fa0, fb0, r00.w, ex2, ey2, S, Tt, G);
        const float2 al1 = frame_alpha2(fa1, fb1, r01.w, ex2, ey2, S, Tt, G);
        const int ya0 = (int)(rc0.y & 0xffffu), yb0 = (int)(rc0.y >> 16);
        const int ya1 = (int)(rc1.y & 0xffffu), yb1 = (int)(rc1.y >> 16);
        if (hit0) composite(e, al0, py0 >= ya0 && py0 <= yb0, py0 + 1 >= ya0 && py0 + 1 <= yb0, r00.z);
        if (hit1) composite(e + 1, al1, py0 >= ya1 && py0 <= yb1, py0 + 1 >= ya1 && py0 + 1 <= yb1, r01.z);
        all_done = done0 && done1;
      }
      } else {
      for (int e = 0; e < cnt && !all_done; e += ILPF) {
        uint2 rc[ILPF];
        bool hit[ILPF];
        bool any_hit = false;
#pragma unroll
        for (int j = 0; j < ILPF; ++j) {
          rc[j] = e + j < cnt ? sm.rect[e + j] : make_uint2(0xffffu, 0xffffu);
          hit[j] = px >= (int)(rc[j].x & 0xffffu) && px <= (int)(rc[j].x >> 16) && py0 <= (int)(rc[j].y >> 16) &&
                   py0 + PPT - 1 >= (int)(rc[j].y & 0xffffu);
          any_hit = any_hit || hit[j];
        }
        if (!any_hit) continue;
        float2 al[ILPF];
        float zj[ILPF];
#pragma unroll
        for (int j = 0; j < ILPF; ++j) {
          const int ej = e + j < cnt ? e + j : e;
          const float4 r0 = sm.r0[ej], fa = sm.fa[ej], fb = sm.fb[ej];
          float2 S, Tt, G;
          al[j] = frame_alpha2(fa, fb, r0.w, ex2, ey2, S, Tt, G);
          zj[j] = r0.z;
        }
#pragma unroll
        for (int j = 0; j < ILPF; ++j) {
          const int ya = (int)(rc[j].y & 0xffffu), yb = (int)(rc[j].y >> 16);
          if (hit[j]) composite(e + j, al[j], py0 >= ya && py0 <= yb, py0 + 1 >= ya && py0 + 1 <= yb, zj[j]);
        }
        all_done = done0 && done1;
      }
      }
    }

    // ---------------- epilogue: images, loss, cotangents kept on chip ----------------
    const bool tile_done = o.unfinished ? __syncthreads_and(all_done) != 0 : true;
    if (!tile_done && tid == 0) {
      o.unfinished[tile] = 1u;
      if (o.unfinished_any) {
        *reinterpret_cast<volatile uint32_t*>(o.unfinished_any) = 1u;
        *o.miss = 1u;
      }
    }
    float2 g_r = bc2(0.f), g_g = bc2(0.f), g_b = bc2(0.f), g_draw = bc2(0.f), g_acc = bc2(0.f);
    float gf[PPT][FD];
    const float crv[PPT] = {cr.x, cr.y}, cgv[PPT] = {cg.x, cg.y}, cbv[PPT] = {cb.x, cb.y};
    const float drv[PPT] = {draw.x, draw.y}, acv[PPT] = {acc.x, acc.y};
#pragma unroll
    for (int k = 0; k < PPT; ++k) {
      const int py = py0 + k;
#pragma unroll
      for (int q = 0; q < FD; ++q) gf[k][q] = 0.f;
      float grgb[3] = {0.f, 0.f, 0.f}, gdr = 0.f, gac = 0.f;
      if (px < c.W && py < c.H) {
        const size_t pix = (size_t)py * c.W + px;
        const float dnorm = drv[k] / fmaxf(acv[k], 1e-6f);
        if (o.rgb) {
          o.rgb[pix * 3 + 0] = crv[k];
          o.rgb[pix * 3 + 1] = cgv[k];
          o.rgb[pix * 3 + 2] = cbv[k];
        }
        if (o.depth) o.depth[pix] = dnorm;
        if (o.acc) o.acc[pix] = acv[k];
        if (DP > 0 && o.feat) {
          float* fo = o.feat + pix * m.d;
          if (m.d == DP) {
#pragma unroll
            for (int q = 0; q < DQ; ++q)
              reinterpret_cast<float4*>(fo)[q] =
                  k == 0 ? make_float4(f[q * 4].x, f[q * 4 + 1].x, f[q * 4 + 2].x, f[q * 4 + 3].x)
                         : make_float4(f[q * 4].y, f[q * 4 + 1].y, f[q * 4 + 2].y, f[q * 4 + 3].y);
          } else {
#pragma unroll
            for (int q = 0; q < FD; ++q)
              if (q < m.d) fo[q] = k == 0 ? f[q].x : f[q].y;
          }
        }
        if (tile_done) {  // L1 (blend_fwd.cu): cotangent sign(diff) / count, loss partial
          const float vals[3] = {crv[k], cgv[k], cbv[k]};
          float lr = 0.f, lf = 0.f;
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            const float df = vals[ch] - o.t_rgb[pix * 3 + ch];
            grgb[ch] = df > 0.f ? inv_rgb : (df < 0.f ? -inv_rgb : 0.f);
            lr += fabsf(df);
          }
          const float dd = dnorm - o.t_depth[pix];
          const float g_d = dd > 0.f ? inv_d : (dd < 0.f ? -inv_d : 0.f);
#pragma unroll
          for (int q = 0; q < DP; ++q) {
            if (q < m.d) {
              const float fq = k == 0 ? f[q].x : f[q].y;
              const float df = fq - o.t_feat[pix * m.d + q];
              gf[k][q] = df > 0.f ? inv_f : (df < 0.f ? -inv_f : 0.f);
              lf += fabsf(df);
            }
          }
          loss += lr * inv_rgb + fabsf(dd) * inv_d + lf * inv_f;
          // backward per-pixel constants (renderer.cpp:204-212)
          const float mm = fmaxf(acv[k], 1e-6f);
          gdr = g_d / mm;
          gac = acv[k] > 1e-6f ? -g_d * dnorm / mm : 0.f;
        }
      }
      if (k == 0) {
        g_r.x = grgb[0]; g_g.x = grgb[1]; g_b.x = grgb[2]; g_draw.x = gdr; g_acc.x = gac;
      } else {
        g_r.y = grgb[0]; g_g.y = grgb[1]; g_b.y = grgb[2]; g_draw.y = gdr; g_acc.y = gac;
      }
    }
    // feature cotangents, channel pairs of both pixels interleaved: (p0 c, p1 c, p0 c+1, p1 c+1)
    if (DP > 0) {
#pragma unroll
      for (int j = 0; j < DP / 2; ++j)
        sm.gfeat[j][tid] = make_float4(gf[0][2 * j], gf[1][2 * j], gf[0][2 * j + 1], gf[1][2 * j + 1]);
    }
    if (!tile_done) last0 = last1 = 0;  // rendered again by the second pass
    const uint32_t my_max = max(last0, last1);

    // ---------------- backward (blend_bwd.cu arithmetic, lane-paired) ----------------
    if (tid == 0) s_max = 0;
    __syncthreads();
    const uint32_t warp_last = __reduce_max_sync(0xffffffffu, my_max);
    if (lane == 0 && warp_last) atomicMax(&s_max, warp_last);
    if (lane == 0 && warp_last && o.consumed) atomicAdd(o.consumed, warp_last);
    __syncthreads();
    float2 accum = bc2(0.f);
    for (int b = s_max ? (int)((s_max - 1) / NB) : -1; b >= 0; --b) {
      const uint32_t bpos = (uint32_t)b * NB;
      const int cnt = (int)min((uint32_t)NB, len - bpos);
      if (b != res_batch) {  // restage (long traversals only); the resident batch is reused
        __syncthreads();
        stage(range.x + bpos, cnt, xc, yc);
        res_batch = b;
        __syncthreads();
        staged();
      }
      const int e_top = (int)min((int64_t)cnt - 1, (int64_t)warp_last - 1 - (int64_t)bpos);
      if constexpr (ILPF == 4) {
        // two entries per step (e, then e - 1): their alphas, dl and gradient values are
        // independent; only T and accum carry from one to the next, so the two transposed
        // reductions interleave.  Same per-entry arithmetic and order as the loop below.
        for (int e = e_top; e >= 0; e -= 2) {
          bool col_in[2], okp[2][2];
          float2 al[2], S2[2], T2[2], G2[2];
          bool any[2];
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int ej = e - j >= 0 ? e - j : e;
            const uint2 rc = sm.rect[ej];
            const int ry0 = (int)(rc.y & 0xffffu), ry1 = (int)(rc.y >> 16);
            col_in[j] = e - j >= 0 && px >= (int)(rc.x & 0xffffu) && px <= (int)(rc.x >> 16) && py0 <= ry1 &&
                        py0 + PPT - 1 >= ry0;
            const float4 r0 = sm.r0[ej];
            al[j] = frame_alpha2(sm.fa[ej], sm.fb[ej], r0.w, ex2, ey2, S2[j], T2[j], G2[j]);
            const uint32_t jrel = bpos + (uint32_t)(e - j);
            okp[j][0] = col_in[j] && jrel < last0 && py0 >= ry0 && py0 <= ry1 && al[j].x >= c.alpha_skip;
            okp[j][1] = col_in[j] && jrel < last1 && py0 + 1 >= ry0 && py0 + 1 <= ry1 && al[j].y >= c.alpha_skip;
            any[j] = __any_sync(0xffffffffu, okp[j][0] || okp[j][1]);
          }
          if (!any[0] && !any[1]) continue;
          float vals[2][SLOTS];
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            if (!any[j]) continue;
            const int ej = e - j;
#pragma unroll
            for (int q = 0; q < SLOTS; ++q) vals[j][q] = 0.f;
            const float2 alpha = make_float2(okp[j][0] ? al[j].x : 0.f, okp[j][1] ? al[j].y : 0.f);
            const float4 r0 = sm.r0[ej];
            const float4 col = sm.col[ej];
            const float4 fa = sm.fa[ej], fb = sm.fb[ej];
            const float op = r0.w;
            const float do_dlogit = op * (1.0f - op);
            const float2 a = make_float2(fminf(alpha.x, c.alpha_clamp), fminf(alpha.y, c.alpha_clamp));
            const float2 inv1ma = make_float2(fast_rcp(1.0f - a.x), fast_rcp(1.0f - a.y));
            T = mul2(T, inv1ma);
            const float2 w = mul2(a, T);
            float2 dl = fma2(g_draw, bc2(r0.z), g_acc);
            dl = fma2(g_r, bc2(col.x), dl);
            dl = fma2(g_g, bc2(col.y), dl);
            dl = fma2(g_b, bc2(col.z), dl);
            if (DP > 0) {
#pragma unroll
              for (int q = 0; q < DQ; ++q) {
                const float4 fv = sm.feat[ej][q];
                const float4 g01 = sm.gfeat[2 * q][tid];
                const float4 g23 = sm.gfeat[2 * q + 1][tid];
                dl = fma2(make_float2(g01.x, g01.y), bc2(fv.x), dl);
                dl = fma2(make_float2(g01.z, g01.w), bc2(fv.y), dl);
                dl = fma2(make_float2(g23.x, g23.y), bc2(fv.z), dl);
                dl = fma2(make_float2(g23.z, g23.w), bc2(fv.w), dl);
                float* vf = vals[j] + kSlotFeat + q * 4;
                vf[0] = fmaf(g01.y, w.y, g01.x * w.x);
                vf[1] = fmaf(g01.w, w.y, g01.z * w.x);
                vf[2] = fmaf(g23.y, w.y, g23.x * w.x);
                vf[3] = fmaf(g23.w, w.y, g23.z * w.x);
              }
            }
            const float2 dla = fma2(make_float2(-accum.x, -accum.y), inv1ma, mul2(T, dl));
            const float2 dl_da = make_float2((alpha.x != 0.f && !(alpha.x > c.alpha_clamp)) ? dla.x : 0.f,
                                             (alpha.y != 0.f && !(alpha.y > c.alpha_clamp)) ? dla.y : 0.f);
            accum = fma2(dl, w, accum);
            vals[j][kSlotColor + 0] = fmaf(g_r.y, w.y, g_r.x * w.x);
            vals[j][kSlotColor + 1] = fmaf(g_g.y, w.y, g_g.x * w.x);
            vals[j][kSlotColor + 2] = fmaf(g_b.y, w.y, g_b.x * w.x);
            vals[j][kSlotZ] = fmaf(g_draw.y, w.y, g_draw.x * w.x);
            const float2 G = G2[j], S = S2[j], Tt = T2[j];
            const float2 dlg = mul2(dl_da, G);
            vals[j][kSlotOpac] = (dlg.x + dlg.y) * do_dlogit;
            const float2 cf = mul2(mul2(dl_da, bc2(op)), mul2(bc2(-0.5f), G));
            const float2 dqx = mul2(bc2(kTwoOverHalfLog2e), fma2(S, bc2(fa.z), mul2(Tt, bc2(fb.x))));
            const float2 dqy = mul2(bc2(kTwoOverHalfLog2e), fma2(S, bc2(fa.w), mul2(Tt, bc2(fb.y))));
            const float2 dx = add2(bc2(fb.z), ex2), dy = add2(bc2(fb.w), ey2);
            const float2 mx = mul2(cf, dqx), my = mul2(cf, dqy);
            vals[j][kSlotMuX] = -(mx.x + mx.y);
            vals[j][kSlotMuY] = -(my.x + my.y);
            const float2 cdx = mul2(cf, dx), cdy = mul2(cf, dy);
            const float2 ca = mul2(cdx, dx), cb2_ = mul2(cdx, dy), cc = mul2(cdy, dy);
            vals[j][kSlotConA] = ca.x + ca.y;
            vals[j][kSlotConB] = cb2_.x + cb2_.y;
            vals[j][kSlotConC] = cc.x + cc.y;
          }
          if (any[0] && any[1]) {
            fused_transpose_reduce2<SLOTS>(vals[0], vals[1], lane);
            gacc_add(gacc + (size_t)sm.gid[e] * SLOTS, lane, vals[0][0]);
            gacc_add(gacc + (size_t)sm.gid[e - 1] * SLOTS, lane, vals[1][0]);
          } else if (any[0]) {
            fused_transpose_reduce<SLOTS>(vals[0], lane);
            gacc_add(gacc + (size_t)sm.gid[e] * SLOTS, lane, vals[0][0]);
          } else {
            fused_transpose_reduce<SLOTS>(vals[1], lane);
            gacc_add(gacc + (size_t)sm.gid[e - 1] * SLOTS, lane, vals[1][0]);
          }
        }
      } else {
      for (int e = e_top; e >= 0; --e) {
        const uint32_t jrel = bpos + (uint32_t)e;
        const uint2 rc = sm.rect[e];
        const int ry0 = (int)(rc.y & 0xffffu), ry1 = (int)(rc.y >> 16);
        const bool col_in =
            px >= (int)(rc.x & 0xffffu) && px <= (int)(rc.x >> 16) && py0 <= ry1 && py0 + PPT - 1 >= ry0;
        if (!__any_sync(0xffffffffu, col_in)) continue;
        const float4 r0 = sm.r0[e];
        const float4 fa = sm.fa[e], fb = sm.fb[e];
        float2 S, Tt, G;
        const float2 al = frame_alpha2(fa, fb, r0.w, ex2, ey2, S, Tt, G);
        const bool ok0 = col_in && jrel < last0 && py0 >= ry0 && py0 <= ry1 && al.x >= c.alpha_skip;
        const bool ok1 = col_in && jrel < last1 && py0 + 1 >= ry0 && py0 + 1 <= ry1 && al.y >= c.alpha_skip;
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
        T = mul2(T, inv1ma);  // transmittance before this contributor (unchanged when a = 0)
        const float2 w = mul2(a, T);
        float2 dl = fma2(g_draw, bc2(r0.z), g_acc);
        dl = fma2(g_r, bc2(col.x), dl);
        dl = fma2(g_g, bc2(col.y), dl);
        dl = fma2(g_b, bc2(col.z), dl);
        if (DP > 0) {
#pragma unroll
          for (int q = 0; q < DQ; ++q) {
            const float4 fv = sm.feat[e][q];
            const float4 g01 = sm.gfeat[2 * q][tid];      // channels 4q, 4q+1 of both pixels
            const float4 g23 = sm.gfeat[2 * q + 1][tid];  // channels 4q+2, 4q+3
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
        // dL/dalpha (renderer.cpp:256-257); the clamped contributor (and a non-contributing pixel)
        // gets no opacity / mean / conic gradient (renderer.cpp:273-274)
        const float2 dla = fma2(make_float2(-accum.x, -accum.y), inv1ma, mul2(T, dl));
        const float2 dl_da = make_float2((alpha.x != 0.f && !(alpha.x > c.alpha_clamp)) ? dla.x : 0.f,
                                         (alpha.y != 0.f && !(alpha.y > c.alpha_clamp)) ? dla.y : 0.f);
        accum = fma2(dl, w, accum);
        vals[kSlotColor + 0] = fmaf(g_r.y, w.y, g_r.x * w.x);
        vals[kSlotColor + 1] = fmaf(g_g.y, w.y, g_g.x * w.x);
        vals[kSlotColor + 2] = fmaf(g_b.y, w.y, g_b.x * w.x);
        vals[kSlotZ] = fmaf(g_draw.y, w.y, g_draw.x * w.x);
        const float2 dlg = mul2(dl_da, G);
        vals[kSlotOpac] = (dlg.x + dlg.y) * do_dlogit;
        const float2 cf = mul2(mul2(dl_da, bc2(op)), mul2(bc2(-0.5f), G));  // dl_dg * dg_dq
        // grad q = (2/k) (S u + T w) (blend_common.cuh frame_dq), pixel - mean = frame offset + (ex, ey)
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
        fused_transpose_reduce<SLOTS>(vals, lane);
        gacc_add(gacc + (size_t)sm.gid[e] * SLOTS, lane, vals[0]);
      }
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

// Two entry points: the first pass (4 CTAs/SM at 128 registers; an explicit minimum-blocks bound
// changes its code generation, so none is given) and the second pass's latency-bound variant
// (register file free: ~1 CTA per SM).
template <int DP>
__global__ void __launch_bounds__(kBlock / 2) blend_fused_l1_kernel(DevMap m, DevCam c, ViewBufs v, TileLists tl,
                                                                      FwdOut o, float* __restrict__ gacc) {
  griddep_wait();
  blend_fused_l1_body<DP, 2>(m, c, v, tl, o, gacc);
}
template <int DP>
__global__ void __launch_bounds__(kBlock / 2, 1) blend_fused_l1_long_kernel(DevMap m, DevCam c, ViewBufs v,
                                                                              TileLists tl, FwdOut o,
                                                                              float* __restrict__ gacc) {
  griddep_wait();
  blend_fused_l1_body<DP, 4>(m, c, v, tl, o, gacc);
}

bool blend_fused_supported(int dp) { return dp == 16 || dp == 8 || dp == 4 || dp == 0; }

template <int DP, int ILPF>
static void launch_fused_dp(const DevMap& m, const DevCam& c, const ViewBufs& v, const TileLists& tl, const FwdOut& o,
                            float* gacc, cudaStream_t s, bool counter_zeroed) {
  auto kernel = ILPF == 2 ? blend_fused_l1_kernel<DP> : blend_fused_l1_long_kernel<DP>;
  const void* kfn = reinterpret_cast<const void*>(kernel);
  if (LGS_FUSED_DYN_PAD > 0) ensure_dyn_smem(kfn, LGS_FUSED_DYN_PAD);
  const int ctas_per_sm = kernel_ctas_per_sm(kfn, kBlock / 2, LGS_FUSED_DYN_PAD);
  const int sms = device_sm_count();
  const int ntiles = c.tiles_x * c.tiles_y;
  const int grid = min(ntiles, ctas_per_sm * sms);
  if (!counter_zeroed) cudaMemsetAsync(tl.counter, 0, sizeof(int), s);
  launch_pdl(kernel, dim3(grid), dim3(kBlock / 2), LGS_FUSED_DYN_PAD, s, m, c, v, tl, o, gacc);
}

template <int ILPF>
static void launch_fused_ilp(const DevMap& m, const DevCam& c, const ViewBufs& v, const TileLists& tl, const FwdOut& o,
                             float* gacc, cudaStream_t s, bool counter_zeroed) {
  switch (m.dp) {
    case 0: launch_fused_dp<0, ILPF>(m, c, v, tl, o, gacc, s, counter_zeroed); break;
    case 4: launch_fused_dp<4, ILPF>(m, c, v, tl, o, gacc, s, counter_zeroed); break;
    case 8: launch_fused_dp<8, ILPF>(m, c, v, tl, o, gacc, s, counter_zeroed); break;
    default: launch_fused_dp<16, ILPF>(m, c, v, tl, o, gacc, s, counter_zeroed); break;
  }
}

void launch_blend_fused_l1(const DevMap& m, const DevCam& c, const ViewBufs& v, const TileLists& tl, const FwdOut& o,
                           float* gacc, cudaStream_t s, bool counter_zeroed, bool long_lists) {
#ifndef LGS_PASS2_ILP
#define LGS_PASS2_ILP 4
#endif
  if (long_lists && LGS_PASS2_ILP == 4)
    launch_fused_ilp<4>(m, c, v, tl, o, gacc, s, counter_zeroed);
  else
    launch_fused_ilp<2>(m, c, v, tl, o, gacc, s, counter_zeroed);
}

}  // namespace lgs
