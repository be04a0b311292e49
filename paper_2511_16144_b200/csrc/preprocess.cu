// preprocess.cu -- K9 map pack and K1 preprocess (EWA projection, SH colour, tile rect).
//
// Compiled with -fmad=false: the only fused multiply-adds are the explicit fmaf() calls, so
// the result is bit-identical to the fp32 twin in oracle/lgs_oracle.c (orc32_project), which
// the key-list / sort-order / range parity tests rely on.
//
// K1 restates project_gaussian (proj/src/renderer.cpp:53-92) in fp32:
//   t = w2c(p) (:59), near cull (:60), Sigma3 = R diag(e^{2s}) R^T (:63-65),
//   Sigma_c = R_cw Sigma3 R_cw^T (:66), cov2d = J Sigma_c J^T + dilation I (:68-71),
//   lambda_max (:74-76), u, v, depth (:79-81), radius (:83), bbox cull (:86-89),
//   conic (:90), pixel rect (:131-134), opacity sigmoid (:127), colour (:128, + SH).
// Sigma_c is formed as M M^T with M = R_cw R diag(s) (same matrix, fewer flops).
// Roofline: HBM-bound, 64 B map read + 92 B record write per Gaussian (+SH: 4*3*K B).
#include "lgs_internal.cuh"
#include "lgs_kernels.h"

namespace lgs {

__global__ void pack_map_kernel(const float* __restrict__ pos, const float* __restrict__ rot,
                                const float* __restrict__ log_s, const float* __restrict__ opac,
                                const float* __restrict__ feat_dn, int64_t n, int d, int dp,
                                float4* __restrict__ pos_opa, float4* __restrict__ rot4,
                                float4* __restrict__ scale4, float* __restrict__ feat_nd) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  pos_opa[i] = make_float4(pos[i * 3 + 0], pos[i * 3 + 1], pos[i * 3 + 2], opac[i]);
  rot4[i] = make_float4(rot[i * 4 + 0], rot[i * 4 + 1], rot[i * 4 + 2], rot[i * 4 + 3]);
  scale4[i] = make_float4(log_s[i * 3 + 0], log_s[i * 3 + 1], log_s[i * 3 + 2], 0.0f);
  if (feat_dn) gather_features(feat_dn, feat_nd, n, d, dp, i);  // null: host-mapped, gathered lazily
}

__global__ void gather_features_kernel(const float* __restrict__ src, float* __restrict__ dst, int64_t n, int d,
                                       int dp) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) gather_features(src, dst, n, d, dp, i);
}

void launch_gather_features(const float* src, float* dst, int64_t n, int d, int dp, cudaStream_t s) {
  if (n == 0 || dp == 0) return;
  gather_features_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(src, dst, n, d, dp);
}

void launch_pack_map(const float* pos, const float* rot, const float* log_s, const float* opac,
                     const float* feat_dn, int64_t n, int d, int dp, float4* pos_opa, float4* rot4,
                     float4* scale4, float* feat_nd, cudaStream_t s) {
  if (n == 0) return;
  const int threads = 256;
  const unsigned blocks = (unsigned)((n + threads - 1) / threads);
  pack_map_kernel<<<blocks, threads, 0, s>>>(pos, rot, log_s, opac, feat_dn, n, d, dp, pos_opa, rot4, scale4,
                                             feat_nd);
}

// ------------------------------------------------------------------------------------------
// K1
// ------------------------------------------------------------------------------------------
// COLOR = false (depth-layered binning): no SH read here; the colours of the Gaussians that get
// listed are computed where they are first listed (ColorJob, lgs_internal.cuh)
// one Gaussian; returns the tiles it touches (0: culled)
template <int DEG, bool COLOR>
__device__ __forceinline__ uint32_t preprocess_one(const DevMap& m, const DevCam& c, const ViewBufs& v, int64_t i) {
  v.iota[i] = (uint32_t)i;
  const float4 po = m.pos_opa[i];
  const float P0 = po.x, P1 = po.y, P2 = po.z;
  const float* R = c.rcw;
  const float t0 = fmaf(R[0], P0, fmaf(R[1], P1, fmaf(R[2], P2, c.tcw[0])));
  const float t1 = fmaf(R[3], P0, fmaf(R[4], P1, fmaf(R[5], P2, c.tcw[1])));
  const float t2 = fmaf(R[6], P0, fmaf(R[7], P1, fmaf(R[8], P2, c.tcw[2])));
  bool ok = t2 > c.near_plane;  // renderer.cpp:60 (NaN -> culled)

  const float4 q = m.rot[i];  // x, y, z, w
  const float n2 = fmaf(q.w, q.w, fmaf(q.x, q.x, fmaf(q.y, q.y, q.z * q.z)));
  const float nrm = sqrtf(n2);
  const float qw = q.w / nrm, qx = q.x / nrm, qy = q.y / nrm, qz = q.z / nrm;
  const float tx = 2.0f * qx, ty = 2.0f * qy, tz = 2.0f * qz;
  const float twx = tx * qw, twy = ty * qw, twz = tz * qw;
  const float txx = tx * qx, txy = ty * qx, txz = tz * qx;
  const float tyy = ty * qy, tyz = tz * qy, tzz = tz * qz;
  const float G[9] = {1.0f - (tyy + tzz), txy - twz,          txz + twy,
                      txy + twz,          1.0f - (txx + tzz), tyz - twx,
                      txz - twy,          tyz + twx,          1.0f - (txx + tyy)};
  const float4 ls = m.scale[i];
  const float s[3] = {lgs_expf(ls.x), lgs_expf(ls.y), lgs_expf(ls.z)};
  float M[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      M[r * 3 + k] =
          fmaf(R[r * 3 + 0], G[0 * 3 + k], fmaf(R[r * 3 + 1], G[1 * 3 + k], R[r * 3 + 2] * G[2 * 3 + k])) * s[k];
  const float iz = 1.0f / t2;
  const float xz = t0 * iz, yz = t1 * iz;
  const float jx = c.fx * iz, jy = c.fy * iz;
  float T0[3], T1[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    T0[k] = jx * fmaf(-xz, M[6 + k], M[0 + k]);
    T1[k] = jy * fmaf(-yz, M[6 + k], M[3 + k]);
  }
  const float ca = fmaf(T0[0], T0[0], fmaf(T0[1], T0[1], T0[2] * T0[2])) + c.dilation;
  const float cb = fmaf(T0[0], T1[0], fmaf(T0[1], T1[1], T0[2] * T1[2]));
  const float cc = fmaf(T1[0], T1[0], fmaf(T1[1], T1[1], T1[2] * T1[2])) + c.dilation;
  const float det = fmaf(ca, cc, -(cb * cb));
  const float mid = 0.5f * (ca + cc);
  const float disc = fmaxf(fmaf(mid, mid, -det), 0.0f);
  const float lam = mid + sqrtf(disc);
  const float radius = c.radius_sigma * sqrtf(lam);
  const float u = fmaf(c.fx, xz, c.cx);
  const float vv = fmaf(c.fy, yz, c.cy);
  const float Wf = (float)c.W, Hf = (float)c.H;
  ok = ok && (u + radius >= -0.5f && u - radius <= Wf - 0.5f && vv + radius >= -0.5f && vv - radius <= Hf - 0.5f);
  ok = ok && det > 0.0f;
  const float opacity = 1.0f / (1.0f + lgs_expf(-po.w));
  // A pixel can only contribute if alpha = o exp(-q/2) >= alpha_skip, i.e. q <= Q = 2 ln(o / skip)
  // (renderer.cpp:146-147).  The ellipse q <= Q lies inside |dx| <= sqrt(Q cov_xx),
  // |dy| <= sqrt(Q cov_yy); with a safety margin for fp32 rounding this box is intersected with
  // the reference pixel rect.  Pixels cut away have alpha < skip in exact arithmetic and in both
  // implementations, so tile lists shrink and images / gradients are unchanged.
  ok = ok && !(c.alpha_skip > 0.0f && !(opacity >= c.alpha_skip));
  float ex = 3.0e38f, ey = 3.0e38f;
  if (c.alpha_skip > 0.0f) {
    const float Q = 2.0f * lgs_logf(opacity / c.alpha_skip);
    const float Qm = fmaf(Q, 1.001f, 0.01f);
    ex = sqrtf(Qm * ca) + 0.01f;
    ey = sqrtf(Qm * cc) + 0.01f;
  }
  int x0 = 0, x1 = 0, y0 = 0, y1 = 0;
  if (ok) {
    x0 = (int)fmaxf(fmaxf(0.0f, floorf(u - radius)), floorf(u - ex));
    x1 = (int)fminf(fminf(Wf - 1.0f, ceilf(u + radius)), ceilf(u + ex));
    y0 = (int)fmaxf(fmaxf(0.0f, floorf(vv - radius)), floorf(vv - ey));
    y1 = (int)fminf(fminf(Hf - 1.0f, ceilf(vv + radius)), ceilf(vv + ey));
    ok = x0 <= x1 && y0 <= y1;
  }
  if (!ok) {  // culled: no tiles, sorts last; its records are never read (left unwritten)
    v.tiles[i] = 0;
    v.dkey[i] = 0xffffffffu;
    return 0u;
  }
  v.rec0[i] = make_float4(u, vv, t2, opacity);
  v.rec1[i] = make_float4(cc / det, -cb / det, ca / det, radius);
  v.rect[i] = make_uint2((uint32_t)x0 | ((uint32_t)x1 << 16), (uint32_t)y0 | ((uint32_t)y1 << 16));
  const uint32_t ntl = (uint32_t)((x1 / kTile - x0 / kTile + 1) * (y1 / kTile - y0 / kTile + 1));
  v.tiles[i] = ntl;
  v.dkey[i] = __float_as_uint(t2);
  if (v.dhist) {  // depth bucket histogram of the layered binning (depth_order.cu depth_bucket)
    const uint32_t b = __float_as_uint(t2) >> kDepthShift;
    const uint32_t bk = b > v.dbase ? min(b - v.dbase, (uint32_t)kDepthBuckets - 1u) : 0u;
    v.dslot[i] = (uint32_t)(atomicAdd(v.dhist + bk, (1ull << 32) | ntl) >> 32);
  }

  // colour (renderer.cpp:128; SH extension)
  if (COLOR) v.color[i] = gaussian_color<DEG>(m.sh, po, c.cc, i);
  return ntl;
}

template <int DEG, bool COLOR>
__global__ void __launch_bounds__(kPreThreads) preprocess_kernel(DevMap m, DevCam c, ViewBufs v) {
  const int64_t i = (int64_t)blockIdx.x * kPreThreads + threadIdx.x;
  const uint32_t ntl = i < m.n ? preprocess_one<DEG, COLOR>(m, c, v, i) : 0u;
  if (!v.dpart) return;
  // this CTA's pair sum (plain store: the bucket scan adds them up for the layer-A cut)
  __shared__ uint32_t s_sum[kPreThreads / 32];
  const uint32_t w = __reduce_add_sync(0xffffffffu, ntl);
  if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = w;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
#pragma unroll
    for (int k = 0; k < kPreThreads / 32; ++k) t += s_sum[k];
    v.dpart[blockIdx.x] = t;
  }
}

// colours of every visible Gaussian (debug exports of a layered render)
template <int DEG>
__global__ void colors_kernel(DevMap m, DevCam c, ViewBufs v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m.n || v.tiles[i] == 0) return;
  v.color[i] = gaussian_color<DEG>(m.sh, m.pos_opa[i], c.cc, i);
}

void launch_colors(const DevMap& m, const DevCam& c, const ViewBufs& v, cudaStream_t s) {
  if (m.n == 0) return;
  const unsigned blocks = (unsigned)((m.n + 255) / 256);
  switch (m.deg) {
    case 0: colors_kernel<0><<<blocks, 256, 0, s>>>(m, c, v); break;
    case 1: colors_kernel<1><<<blocks, 256, 0, s>>>(m, c, v); break;
    case 2: colors_kernel<2><<<blocks, 256, 0, s>>>(m, c, v); break;
    default: colors_kernel<3><<<blocks, 256, 0, s>>>(m, c, v); break;
  }
}

template <int DEG>
static void launch_pre(const DevMap& m, const DevCam& c, const ViewBufs& v, bool color, unsigned blocks,
                       cudaStream_t s) {
  if (color) preprocess_kernel<DEG, true><<<blocks, kPreThreads, 0, s>>>(m, c, v);
  else preprocess_kernel<DEG, false><<<blocks, kPreThreads, 0, s>>>(m, c, v);
}

void launch_preprocess(const DevMap& m, const DevCam& c, const ViewBufs& v, bool color, cudaStream_t s) {
  if (m.n == 0) return;
  const unsigned blocks = (unsigned)((m.n + kPreThreads - 1) / kPreThreads);
  switch (m.deg) {
    case 0: launch_pre<0>(m, c, v, color, blocks, s); break;
    case 1: launch_pre<1>(m, c, v, color, blocks, s); break;
    case 2: launch_pre<2>(m, c, v, color, blocks, s); break;
    default: launch_pre<3>(m, c, v, color, blocks, s); break;
  }
}

}  // namespace lgs
