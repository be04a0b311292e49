// optim.cu -- K9b/K10: the per-attribute Adam step on the resident map and the map unpack.
//
// SURVEY.md §8f row 2 (SPEC.md:430 mapping_round: "apply one Adam step per attribute group (lr:
// position 1.6e-4, rotation 1e-3, log-scale 5e-3, opacity-logit 5e-2, color 2.5e-3, feature
// 2.5e-3)").  The reference leaves mapping.cpp unimplemented; the Adam form is the standard one
// (bias-corrected first and second moments), defaults beta1 0.9, beta2 0.999, eps 1e-8; SH bands
// above the DC term use colour lr / 20 (the usual splatting convention; SH0 == the reference colour).
//
// One thread per Gaussian over a range [g0, g1) (the whole map, or this rank's shard after a
// reduce-scatter).  Parameters and both moments live in the map's packed layout (float4 position
// + opacity logit, float4 rotation x,y,z,w, float4 log-scale, SH [N][K][3], feature [N][DP]); the
// gradients arrive in the reference layouts (renderer.hpp:59-68: rotation w,x,y,z, feature
// [d][N]).  Bytes per Gaussian: parameters + two moments read and written (6 x 304 B at SH3,
// d = 16) + gradients read (300 B) -- HBM-bound.
#include <cmath>
#include <cstdint>

#include "lgs_internal.cuh"
#include "lgs_kernels.h"

namespace lgs {

namespace {

struct AdamF {
  float b1, b2, eps, c1, c2;  // c1 = 1 / (1 - b1^t), c2 = 1 / (1 - b2^t)
};

__device__ __forceinline__ float adam1(float& p, float& m, float& v, float g, float lr, const AdamF& a) {
  m = fmaf(a.b1, m, (1.f - a.b1) * g);
  v = fmaf(a.b2, v, (1.f - a.b2) * g * g);
  const float mh = m * a.c1, vh = v * a.c2;
  p -= lr * mh / (sqrtf(vh) + a.eps);
  return p;
}

__device__ __forceinline__ void adam4(float4& p, float4& m, float4& v, const float (&g)[4], int nc, float lr,
                                      const AdamF& a) {
  float* pp = reinterpret_cast<float*>(&p);
  float* mm = reinterpret_cast<float*>(&m);
  float* vv = reinterpret_cast<float*>(&v);
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (k < nc) adam1(pp[k], mm[k], vv[k], g[k], lr, a);
}

__global__ void adam_kernel(MapParams p, MapParams m, MapParams v, GradIn g, int64_t g0, int64_t g1, AdamLr lr,
                            AdamF a) {
  const int64_t i = g0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g1) return;
  const int64_t n = p.n;
  // position xyz + opacity logit (float4)
  {
    float4 pp = p.pos_opa[i], mm = m.pos_opa[i], vv = v.pos_opa[i];
    const float gp[4] = {g.position[i * 3 + 0], g.position[i * 3 + 1], g.position[i * 3 + 2], 0.f};
    adam4(pp, mm, vv, gp, 3, lr.position, a);
    adam1(pp.w, mm.w, vv.w, g.opacity[i], lr.opacity, a);
    p.pos_opa[i] = pp; m.pos_opa[i] = mm; v.pos_opa[i] = vv;
  }
  // rotation: stored x,y,z,w; gradient ordered w,x,y,z (renderer.hpp:61)
  {
    float4 pp = p.rot[i], mm = m.rot[i], vv = v.rot[i];
    // caller-owned gradient buffers: one float4 load only where the row is 16-byte aligned (a flat
    // MapGradients buffer puts rotation at float offset 3n)
    float gq[4];
    if ((reinterpret_cast<uintptr_t>(g.rotation) & 15) == 0) {
      const float4 gr = reinterpret_cast<const float4*>(g.rotation)[i];
      gq[0] = gr.y; gq[1] = gr.z; gq[2] = gr.w; gq[3] = gr.x;
    } else {
      const float* gr = g.rotation + i * 4;
      gq[0] = gr[1]; gq[1] = gr[2]; gq[2] = gr[3]; gq[3] = gr[0];
    }
    adam4(pp, mm, vv, gq, 4, lr.rotation, a);
    p.rot[i] = pp; m.rot[i] = mm; v.rot[i] = vv;
  }
  {
    float4 pp = p.scale[i], mm = m.scale[i], vv = v.scale[i];
    const float gs[4] = {g.log_scale[i * 3 + 0], g.log_scale[i * 3 + 1], g.log_scale[i * 3 + 2], 0.f};
    adam4(pp, mm, vv, gs, 3, lr.log_scale, a);
    p.scale[i] = pp; m.scale[i] = mm; v.scale[i] = vv;
  }
  // SH [K][3]: parameters, moments and gradients share one layout -> adam_sh_kernel (flat, float4)
  // feature: packed [N][DP] (zero padding untouched), gradient [d][N]
  if (p.d > 0) {
    float4* pf = reinterpret_cast<float4*>(p.feat + i * p.dp);
    float4* mf = reinterpret_cast<float4*>(m.feat + i * p.dp);
    float4* vf = reinterpret_cast<float4*>(v.feat + i * p.dp);
    for (int c4 = 0; c4 < p.dp / 4; ++c4) {
      float gv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = c4 * 4 + k;
        gv[k] = c < p.d ? g.feature[(int64_t)c * n + i] : 0.f;
      }
      float4 pp = pf[c4], mm = mf[c4], vv = vf[c4];
      adam4(pp, mm, vv, gv, min(4, p.d - c4 * 4), lr.feature, a);
      pf[c4] = pp; mf[c4] = mm; vf[c4] = vv;
    }
  }
}

__global__ void adam_sh_kernel(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                               const float* __restrict__ g, int64_t e0, int64_t e1, int ks, float lr_dc,
                               float lr_rest, bool vec, AdamF a) {
  const int64_t q = e0 / 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // float4 index
  const int64_t e = q * 4;
  if (e >= e1) return;
  if (vec && e + 4 <= e1 && (e0 & 3) == 0) {  // vec: all four arrays 16-byte aligned
    float4 pp = reinterpret_cast<float4*>(p)[q], mm = reinterpret_cast<float4*>(m)[q],
           vv = reinterpret_cast<float4*>(v)[q];
    const float4 gg = reinterpret_cast<const float4*>(g)[q];
    const float gv[4] = {gg.x, gg.y, gg.z, gg.w};
    float* pa = reinterpret_cast<float*>(&pp);
    float* ma = reinterpret_cast<float*>(&mm);
    float* va = reinterpret_cast<float*>(&vv);
#pragma unroll
    for (int k = 0; k < 4; ++k) adam1(pa[k], ma[k], va[k], gv[k], (int)((e + k) % ks) < 3 ? lr_dc : lr_rest, a);
    reinterpret_cast<float4*>(p)[q] = pp;
    reinterpret_cast<float4*>(m)[q] = mm;
    reinterpret_cast<float4*>(v)[q] = vv;
  } else {
    for (int64_t j = max(e, e0); j < min(e + 4, e1); ++j) {
      float pk = p[j], mk = m[j], vk = v[j];
      adam1(pk, mk, vk, g[j], (int)(j % ks) < 3 ? lr_dc : lr_rest, a);
      p[j] = pk; m[j] = mk; v[j] = vk;
    }
  }
}

__global__ void unpack_map_kernel(MapParams p, float* __restrict__ pos, float* __restrict__ rot,
                                  float* __restrict__ log_s, float* __restrict__ opac, float* __restrict__ sh,
                                  float* __restrict__ feat_dn) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.n) return;
  const float4 po = p.pos_opa[i], r = p.rot[i], s = p.scale[i];
  if (pos) { pos[i * 3 + 0] = po.x; pos[i * 3 + 1] = po.y; pos[i * 3 + 2] = po.z; }
  if (opac) opac[i] = po.w;
  if (rot) {  // x,y,z,w storage order (gaussian_map.hpp); caller buffers may be only 4-byte aligned
    if ((reinterpret_cast<uintptr_t>(rot) & 15) == 0) {
      reinterpret_cast<float4*>(rot)[i] = r;
    } else {
      rot[i * 4 + 0] = r.x; rot[i * 4 + 1] = r.y; rot[i * 4 + 2] = r.z; rot[i * 4 + 3] = r.w;
    }
  }
  if (log_s) { log_s[i * 3 + 0] = s.x; log_s[i * 3 + 1] = s.y; log_s[i * 3 + 2] = s.z; }
  if (sh) {
    const int ks = 3 * p.K;
    for (int k = 0; k < ks; ++k) sh[i * ks + k] = p.sh[i * ks + k];
  }
  if (feat_dn)
    for (int c = 0; c < p.d; ++c) feat_dn[(int64_t)c * p.n + i] = p.feat[i * p.dp + c];
}

}  // namespace

void launch_adam(const MapParams& p, const MapParams& m, const MapParams& v, const GradIn& g, int64_t g0, int64_t g1,
                 const AdamLr& lr, double beta1, double beta2, double eps, int64_t step, cudaStream_t s) {
  if (g1 <= g0) return;
  AdamF a;
  a.b1 = (float)beta1;
  a.b2 = (float)beta2;
  a.eps = (float)eps;
  a.c1 = (float)(1.0 / (1.0 - std::pow(beta1, (double)step)));
  a.c2 = (float)(1.0 / (1.0 - std::pow(beta2, (double)step)));
  const int threads = 256;
  adam_kernel<<<(unsigned)((g1 - g0 + threads - 1) / threads), threads, 0, s>>>(p, m, v, g, g0, g1, lr, a);
  const int ks = 3 * p.K;
  const int64_t e0 = g0 * ks, e1 = g1 * ks;
  const int64_t nq = (e1 + 3) / 4 - e0 / 4;
  const bool vec = ((reinterpret_cast<uintptr_t>(p.sh) | reinterpret_cast<uintptr_t>(m.sh) |
                    reinterpret_cast<uintptr_t>(v.sh) | reinterpret_cast<uintptr_t>(g.sh)) & 15) == 0;
  adam_sh_kernel<<<(unsigned)((nq + threads - 1) / threads), threads, 0, s>>>(p.sh, m.sh, v.sh, g.sh, e0, e1, ks,
                                                                           lr.sh_dc, lr.sh_rest, vec, a);
}

void launch_unpack_map(const MapParams& p, float* pos, float* rot, float* log_s, float* opac, float* sh, float* feat_dn,
                       cudaStream_t s) {
  if (p.n == 0) return;
  const int threads = 256;
  unpack_map_kernel<<<(unsigned)((p.n + threads - 1) / threads), threads, 0, s>>>(p, pos, rot, log_s, opac, sh,
                                                                                   feat_dn);
}

}  // namespace lgs
