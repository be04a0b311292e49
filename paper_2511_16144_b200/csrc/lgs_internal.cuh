// lgs_internal.cuh -- device-side types and math shared by the rasterizer kernels.
//
// Data layout in HBM:
//   map (resident, lgs_map)       pos_opa float4[N] (x,y,z,opacity_logit)  rot float4[N] (x,y,z,w raw)
//                                 scale float4[N] (log_s xyz, 0)            sh float[N][K][3]
//                                 feat float[N][DP] (DP = d padded to 4/8/16/32, zero tail)
//   per view (lgs_saved)          rec0 float4[N] (u, v, depth, opacity)     rec1 float4[N] (A, B, C, radius)
//                                 rect uint2[N] (x0 | x1<<16, y0 | y1<<16)  color float4[N]
//                                 tile list vals u32[P], ranges uint2[tiles], per-pixel T / n_contrib
//   backward accumulator          gacc float[N][SLOTS] (one 128 B line per Gaussian for SLOTS = 32)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

namespace lgs {

// depth buckets of the bucketed depth order (depth_order.cu): key >> kDepthShift relative to the
// near plane, 2^13 buckets per octave of depth; bucket kDepthBuckets holds the culled Gaussians
constexpr int kDepthShift = 10;
constexpr int kDepthBuckets = 1 << 18;
constexpr int kPreThreads = 128;  // K1 (preprocess) CTA size: one pair partial sum per CTA

constexpr int kTile = 16;
constexpr int kBlock = kTile * kTile;

// Backward accumulator slots (per Gaussian, one 128-byte line for SLOTS = 32).  Slot order is
// shared by the blend kernels and preprocess_bwd.cu.  The geometric slots 0-5 accumulate as
// DOUBLES in the first 48 bytes of the row (float slots 0-11): the mean, conic and opacity
// gradients sum many pixel terms with heavy cancellation on near-camera splats, and fp32 atomics
// made them depend on the accumulation order at the 1e-3 level; the rest accumulate as floats.
enum : int {
  kSlotMuX = 0,    // doubles (index into the row viewed as double[])
  kSlotMuY = 1,
  kSlotConA = 2,   // dL/dconic(0,0)
  kSlotConB = 3,   // dL/dconic(0,1) == dL/dconic(1,0) (renderer.cpp:286-287)
  kSlotConC = 4,   // dL/dconic(1,1)
  kSlotOpac = 5,   // dL/d opacity_logit
  kSlotGeo = 6,    // number of double slots (floats 0 .. 2 kSlotGeo - 1)
  kSlotZ = 12,     // floats: dL/d depth via the depth image (renderer.cpp:265)
  kSlotColor = 13, // 3 slots
  kSlotFeat = 16   // DP slots
};

__host__ __device__ constexpr int slots_for(int dp) { return (kSlotFeat + dp) <= 32 ? 32 : 64; }

// add one reduced slot value into a Gaussian's accumulator row (doubles for the geometric slots)
__device__ __forceinline__ void gacc_add(float* row, int slot, float v) {
  if (v == 0.f) return;
  if (slot < kSlotGeo) atomicAdd(reinterpret_cast<double*>(row) + slot, (double)v);
  else atomicAdd(row + slot, v);
}

struct DevCam {
  float rcw[9];  // world -> camera rotation (row-major)
  float tcw[3];
  float cc[3];   // camera centre in world (cam_pose translation)
  float fx, fy, cx, cy;
  int W, H, tiles_x, tiles_y;
  float near_plane, dilation, radius_sigma, alpha_clamp, alpha_skip, t_min;
  // fp64 copies for the backward's 2D -> 3D chain (preprocess_bwd.cu), which runs in fp64
  double rcw_d[9], tcw_d[3], cc_d[3], fx_d, fy_d;
};

struct DevMap {
  int64_t n;
  int d, dp, deg, K;
  const float4* pos_opa;
  const float4* rot;
  const float4* scale;
  const float* sh;
  const float* feat;
};

// ------------------------------------------------------------------------------------------
// Deterministic fp32 exp: range reduction + degree-7 Taylor, explicit fma, exact scaling.
// Identical code in oracle/lgs_oracle.c (orc_expf) so preprocess is bit-exact CPU vs GPU.
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ float lgs_expf(float x) {
  if (x != x) return x;
  if (x > 88.72f) return __int_as_float(0x7f800000);
  if (x < -103.97f) return 0.0f;
  const float k = rintf(x * 1.44269504088896341f);
  float r = fmaf(k, -0.693145751953125f, x);
  r = fmaf(k, -1.428606765330187045e-06f, r);
  float p = 1.98412698412698413e-04f;
  p = fmaf(p, r, 1.38888888888888889e-03f);
  p = fmaf(p, r, 8.33333333333333333e-03f);
  p = fmaf(p, r, 4.16666666666666667e-02f);
  p = fmaf(p, r, 1.66666666666666667e-01f);
  p = fmaf(p, r, 0.5f);
  p = fmaf(p, r, 1.0f);
  p = fmaf(p, r, 1.0f);
  const int ki = (int)k;
  const int k1 = ki / 2, k2 = ki - k1;
  const float s1 = __int_as_float((k1 + 127) << 23);
  const float s2 = __int_as_float((k2 + 127) << 23);
  return (p * s1) * s2;
}

// Deterministic fp32 natural log for x >= 1 (finite): x = m 2^e with m in [sqrt(1/2), sqrt(2)),
// log m = 2 atanh((m-1)/(m+1)) by its odd series.  Identical code in oracle/lgs_oracle.c (orc_logf).
__device__ __forceinline__ float lgs_logf(float x) {
  const uint32_t bits = __float_as_uint(x);
  int e = (int)((bits >> 23) & 0xffu) - 127;
  float m = __uint_as_float((bits & 0x7fffffu) | 0x3f800000u);
  if (m > 1.41421356f) {
    m = m * 0.5f;
    e = e + 1;
  }
  const float s = (m - 1.0f) / (m + 1.0f);
  const float s2 = s * s;
  float p = fmaf(s2, 0.0909090909f, 0.111111111f);
  p = fmaf(s2, p, 0.142857143f);
  p = fmaf(s2, p, 0.2f);
  p = fmaf(s2, p, 0.333333333f);
  p = fmaf(s2, p, 1.0f);
  return fmaf((float)e, 0.693147181f, (2.0f * s) * p);
}

// Real SH basis up to degree 3 (standard constants).  Colour convention: DC is used directly
// (no C0, no +0.5, no clamp), so SH degree 0 is exactly the reference colour (renderer.cpp:128).
constexpr float kShC1 = 0.4886025119029199f;
__device__ __constant__ static const float kShC2[5] = {1.0925484305920792f, -1.0925484305920792f,
                                                       0.31539156525252005f, -1.0925484305920792f,
                                                       0.5462742152960396f};
__device__ __constant__ static const float kShC3[7] = {-0.5900435899266435f, 2.890611442640554f,
                                                       -0.4570457994644658f, 0.3731763325901154f,
                                                       -0.4570457994644658f, 1.445305721320277f,
                                                       -0.5900435899266435f};

// basis values b[0..K) for a unit direction; same op order as oracle orc32_sh_color
__device__ __forceinline__ void sh_basis_f32(int deg, float x, float y, float z, float b[16]) {
  b[0] = 1.0f;
  if (deg >= 1) {
    b[1] = -kShC1 * y;
    b[2] = kShC1 * z;
    b[3] = -kShC1 * x;
  }
  if (deg >= 2) {
    const float xx = x * x, yy = y * y, zz = z * z;
    b[4] = kShC2[0] * (x * y);
    b[5] = kShC2[1] * (y * z);
    b[6] = kShC2[2] * ((zz + zz) - xx - yy);
    b[7] = kShC2[3] * (x * z);
    b[8] = kShC2[4] * (xx - yy);
    if (deg >= 3) {
      b[9] = kShC3[0] * y * (3.0f * xx - yy);
      b[10] = kShC3[1] * (x * y) * z;
      b[11] = kShC3[2] * y * (4.0f * zz - xx - yy);
      b[12] = kShC3[3] * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
      b[13] = kShC3[4] * x * (4.0f * zz - xx - yy);
      b[14] = kShC3[5] * z * (xx - yy);
      b[15] = kShC3[6] * x * (xx - 3.0f * yy);
    }
  }
}

// The colour of Gaussian i (renderer.cpp:128; SH extension), with every operation explicitly
// rounded (__fmul_rn / __fadd_rn / __fsub_rn are never contracted into FMAs): bit-identical in
// every translation unit whatever its -fmad setting, and equal to the -fmad=false K1 arithmetic
// that oracle B restates (orc32_sh_color).  Used by K1 and, with the depth-layered binning, for
// just the Gaussians that get listed (ColorJob).
__device__ __forceinline__ void sh_basis_rn(int deg, float x, float y, float z, float b[16]) {
  b[0] = 1.0f;
  if (deg >= 1) {
    b[1] = __fmul_rn(-kShC1, y);
    b[2] = __fmul_rn(kShC1, z);
    b[3] = __fmul_rn(-kShC1, x);
  }
  if (deg >= 2) {
    const float xx = __fmul_rn(x, x), yy = __fmul_rn(y, y), zz = __fmul_rn(z, z);
    b[4] = __fmul_rn(kShC2[0], __fmul_rn(x, y));
    b[5] = __fmul_rn(kShC2[1], __fmul_rn(y, z));
    b[6] = __fmul_rn(kShC2[2], __fsub_rn(__fsub_rn(__fadd_rn(zz, zz), xx), yy));
    b[7] = __fmul_rn(kShC2[3], __fmul_rn(x, z));
    b[8] = __fmul_rn(kShC2[4], __fsub_rn(xx, yy));
    if (deg >= 3) {
      b[9] = __fmul_rn(__fmul_rn(kShC3[0], y), __fsub_rn(__fmul_rn(3.0f, xx), yy));
      b[10] = __fmul_rn(__fmul_rn(kShC3[1], __fmul_rn(x, y)), z);
      b[11] = __fmul_rn(__fmul_rn(kShC3[2], y), __fsub_rn(__fsub_rn(__fmul_rn(4.0f, zz), xx), yy));
      b[12] = __fmul_rn(__fmul_rn(kShC3[3], z),
                        __fsub_rn(__fsub_rn(__fmul_rn(2.0f, zz), __fmul_rn(3.0f, xx)), __fmul_rn(3.0f, yy)));
      b[13] = __fmul_rn(__fmul_rn(kShC3[4], x), __fsub_rn(__fsub_rn(__fmul_rn(4.0f, zz), xx), yy));
      b[14] = __fmul_rn(__fmul_rn(kShC3[5], z), __fsub_rn(xx, yy));
      b[15] = __fmul_rn(__fmul_rn(kShC3[6], x), __fsub_rn(xx, __fmul_rn(3.0f, yy)));
    }
  }
}

template <int DEG>
__device__ __forceinline__ float4 gaussian_color(const float* __restrict__ sh_all, float4 po, const float cc[3],
                                                 int64_t i) {
  constexpr int K = (DEG + 1) * (DEG + 1);
  constexpr int KS = 3 * K;
  const float* sh = sh_all + i * KS;
  if (DEG == 0) return make_float4(__ldg(sh), __ldg(sh + 1), __ldg(sh + 2), 0.0f);
  float dx = __fsub_rn(po.x, cc[0]), dy = __fsub_rn(po.y, cc[1]), dz = __fsub_rn(po.z, cc[2]);
  const float dn = sqrtf(fmaf(dx, dx, fmaf(dy, dy, __fmul_rn(dz, dz))));
  const float idn = __fdiv_rn(1.0f, dn);
  dx = __fmul_rn(dx, idn); dy = __fmul_rn(dy, idn); dz = __fmul_rn(dz, idn);
  float b[16];
  sh_basis_rn(DEG, dx, dy, dz, b);
  float e[KS];
  if (KS % 4 == 0) {
    const float4* row = reinterpret_cast<const float4*>(sh);
#pragma unroll
    for (int q = 0; q < KS / 4; ++q) {
      const float4 v4 = __ldg(row + q);
      e[4 * q] = v4.x; e[4 * q + 1] = v4.y; e[4 * q + 2] = v4.z; e[4 * q + 3] = v4.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < KS; ++j) e[j] = __ldg(sh + j);
  }
  float col[3] = {e[0], e[1], e[2]};  // each channel accumulates in k order
#pragma unroll
  for (int k = 1; k < K; ++k)
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) col[ch] = fmaf(b[k], e[3 * k + ch], col[ch]);
  return make_float4(col[0], col[1], col[2], 0.0f);
}

// Lazy colours of the depth-layered binning: K1 skips the SH evaluation and the kernels that
// first list a Gaussian (layer-A depth order, second-pass counting) compute its colour.
struct ColorJob {
  const float* sh = nullptr;
  const float4* pos_opa = nullptr;
  float cc[3] = {0.f, 0.f, 0.f};
  int deg = 0;
  float4* color = nullptr;  // null: colours were written by K1
  // host-mapped map (LGS_MEM_HOST_MAPPED): the listed Gaussian's features are gathered from the
  // page-locked [d][N] source into the packed [N][dp] array (feat_src null: packed at upload)
  const float* feat_src = nullptr;
  float* feat_dst = nullptr;
  int64_t n = 0;
  int d = 0, dp = 0;
  uint32_t* listed = nullptr;  // host-mapped maps: Gaussians listed by this render (lgs_capi.cu policy)
};

__device__ __forceinline__ void gather_features(const float* __restrict__ src, float* __restrict__ dst, int64_t n,
                                                int d, int dp, int64_t g) {
  float4* fo = reinterpret_cast<float4*>(dst + g * dp);
  for (int c4 = 0; c4 < dp / 4; ++c4) {
    float v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = c4 * 4 + k;
      v[k] = c < d ? src[(int64_t)c * n + g] : 0.0f;
    }
    fo[c4] = make_float4(v[0], v[1], v[2], v[3]);
  }
}

__device__ __forceinline__ void color_job_run(const ColorJob& j, uint32_t g) {
  if (j.listed) atomicAdd(j.listed, 1u);
  if (j.feat_src) gather_features(j.feat_src, j.feat_dst, j.n, j.d, j.dp, g);
  const float4 po = j.pos_opa[g];
  float4 col;
  switch (j.deg) {
    case 0: col = gaussian_color<0>(j.sh, po, j.cc, g); break;
    case 1: col = gaussian_color<1>(j.sh, po, j.cc, g); break;
    case 2: col = gaussian_color<2>(j.sh, po, j.cc, g); break;
    default: col = gaussian_color<3>(j.sh, po, j.cc, g); break;
  }
  j.color[g] = col;
}

// d b_k / d(x, y, z) (unnormalized direction components treated as independent)
__device__ __forceinline__ void sh_basis_grad_f32(int deg, float x, float y, float z, float db[16][3]) {
#pragma unroll
  for (int k = 0; k < 16; ++k) db[k][0] = db[k][1] = db[k][2] = 0.0f;
  if (deg < 1) return;
  db[1][1] = -kShC1;
  db[2][2] = kShC1;
  db[3][0] = -kShC1;
  if (deg < 2) return;
  const float xx = x * x, yy = y * y, zz = z * z;
  db[4][0] = kShC2[0] * y; db[4][1] = kShC2[0] * x;
  db[5][1] = kShC2[1] * z; db[5][2] = kShC2[1] * y;
  db[6][0] = -2.0f * kShC2[2] * x; db[6][1] = -2.0f * kShC2[2] * y; db[6][2] = 4.0f * kShC2[2] * z;
  db[7][0] = kShC2[3] * z; db[7][2] = kShC2[3] * x;
  db[8][0] = 2.0f * kShC2[4] * x; db[8][1] = -2.0f * kShC2[4] * y;
  if (deg < 3) return;
  db[9][0] = kShC3[0] * 6.0f * x * y; db[9][1] = kShC3[0] * (3.0f * xx - 3.0f * yy);
  db[10][0] = kShC3[1] * y * z; db[10][1] = kShC3[1] * x * z; db[10][2] = kShC3[1] * x * y;
  db[11][0] = kShC3[2] * (-2.0f * x * y); db[11][1] = kShC3[2] * (4.0f * zz - xx - 3.0f * yy);
  db[11][2] = kShC3[2] * 8.0f * y * z;
  db[12][0] = kShC3[3] * (-6.0f * x * z); db[12][1] = kShC3[3] * (-6.0f * y * z);
  db[12][2] = kShC3[3] * (6.0f * zz - 3.0f * xx - 3.0f * yy);
  db[13][0] = kShC3[4] * (4.0f * zz - 3.0f * xx - yy); db[13][1] = kShC3[4] * (-2.0f * x * y);
  db[13][2] = kShC3[4] * 8.0f * x * z;
  db[14][0] = kShC3[5] * 2.0f * x * z; db[14][1] = kShC3[5] * (-2.0f * y * z); db[14][2] = kShC3[5] * (xx - yy);
  db[15][0] = kShC3[6] * (3.0f * xx - 3.0f * yy); db[15][1] = kShC3[6] * (-6.0f * x * y);
}

// fp64 basis values and their gradient (the backward's fp64 chain, preprocess_bwd.cu)
constexpr double kShC1d = 0.4886025119029199;
__device__ __constant__ static const double kShC2d[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                              0.5462742152960396};
__device__ __constant__ static const double kShC3d[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
                              -0.4570457994644658, 1.445305721320277, -0.5900435899266435};

__device__ __forceinline__ void sh_basis_f64(int deg, double x, double y, double z, double b[16]) {
  b[0] = 1.0;
  if (deg >= 1) {
    b[1] = -kShC1d * y;
    b[2] = kShC1d * z;
    b[3] = -kShC1d * x;
  }
  if (deg >= 2) {
    const double xx = x * x, yy = y * y, zz = z * z;
    b[4] = kShC2d[0] * (x * y);
    b[5] = kShC2d[1] * (y * z);
    b[6] = kShC2d[2] * ((zz + zz) - xx - yy);
    b[7] = kShC2d[3] * (x * z);
    b[8] = kShC2d[4] * (xx - yy);
    if (deg >= 3) {
      b[9] = kShC3d[0] * y * (3.0 * xx - yy);
      b[10] = kShC3d[1] * (x * y) * z;
      b[11] = kShC3d[2] * y * (4.0 * zz - xx - yy);
      b[12] = kShC3d[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
      b[13] = kShC3d[4] * x * (4.0 * zz - xx - yy);
      b[14] = kShC3d[5] * z * (xx - yy);
      b[15] = kShC3d[6] * x * (xx - 3.0 * yy);
    }
  }
}

__device__ __forceinline__ void sh_basis_grad_f64(int deg, double x, double y, double z, double db[16][3]) {
#pragma unroll
  for (int k = 0; k < 16; ++k) db[k][0] = db[k][1] = db[k][2] = 0.0;
  if (deg < 1) return;
  db[1][1] = -kShC1d;
  db[2][2] = kShC1d;
  db[3][0] = -kShC1d;
  if (deg < 2) return;
  const double xx = x * x, yy = y * y, zz = z * z;
  db[4][0] = kShC2d[0] * y; db[4][1] = kShC2d[0] * x;
  db[5][1] = kShC2d[1] * z; db[5][2] = kShC2d[1] * y;
  db[6][0] = -2.0 * kShC2d[2] * x; db[6][1] = -2.0 * kShC2d[2] * y; db[6][2] = 4.0 * kShC2d[2] * z;
  db[7][0] = kShC2d[3] * z; db[7][2] = kShC2d[3] * x;
  db[8][0] = 2.0 * kShC2d[4] * x; db[8][1] = -2.0 * kShC2d[4] * y;
  if (deg < 3) return;
  db[9][0] = kShC3d[0] * 6.0 * x * y; db[9][1] = kShC3d[0] * (3.0 * xx - 3.0 * yy);
  db[10][0] = kShC3d[1] * y * z; db[10][1] = kShC3d[1] * x * z; db[10][2] = kShC3d[1] * x * y;
  db[11][0] = kShC3d[2] * (-2.0 * x * y); db[11][1] = kShC3d[2] * (4.0 * zz - xx - 3.0 * yy);
  db[11][2] = kShC3d[2] * 8.0 * y * z;
  db[12][0] = kShC3d[3] * (-6.0 * x * z); db[12][1] = kShC3d[3] * (-6.0 * y * z);
  db[12][2] = kShC3d[3] * (6.0 * zz - 3.0 * xx - 3.0 * yy);
  db[13][0] = kShC3d[4] * (4.0 * zz - 3.0 * xx - yy); db[13][1] = kShC3d[4] * (-2.0 * x * y);
  db[13][2] = kShC3d[4] * 8.0 * x * z;
  db[14][0] = kShC3d[5] * 2.0 * x * z; db[14][1] = kShC3d[5] * (-2.0 * y * z); db[14][2] = kShC3d[5] * (xx - yy);
  db[15][0] = kShC3d[6] * (3.0 * xx - 3.0 * yy); db[15][1] = kShC3d[6] * (-6.0 * x * y);
}

// Block-staged AoS transfers: a CTA's contiguous [nloc][W] float block (16-byte aligned base) moves
// between global memory (float4 accesses, coalesced) and per-thread shared-memory rows of stride S
// (odd S keeps each thread's row in distinct banks).
template <int W, int S, int NT>
__device__ __forceinline__ void stage_rows_in(float* __restrict__ s, const float* __restrict__ src, int nloc) {
  const int total = nloc * W;
  const int n4 = total >> 2;
  const float4* src4 = reinterpret_cast<const float4*>(src);
#pragma unroll 4
  for (int j4 = threadIdx.x; j4 < n4; j4 += NT) {
    const float4 v = __ldg(src4 + j4);
    const int j = j4 * 4;
    s[((j + 0) / W) * S + (j + 0) % W] = v.x;
    s[((j + 1) / W) * S + (j + 1) % W] = v.y;
    s[((j + 2) / W) * S + (j + 2) % W] = v.z;
    s[((j + 3) / W) * S + (j + 3) % W] = v.w;
  }
  for (int j = n4 * 4 + threadIdx.x; j < total; j += NT) s[(j / W) * S + j % W] = __ldg(src + j);
}

template <int W, int S, int NT>
__device__ __forceinline__ void stage_rows_out(const float* __restrict__ s, float* __restrict__ dst, int nloc,
                                               bool accum) {
  const int total = nloc * W;
  const int n4 = total >> 2;
  float4* dst4 = reinterpret_cast<float4*>(dst);
  const bool aligned = (reinterpret_cast<uintptr_t>(dst) & 15u) == 0;
  if (aligned) {
#pragma unroll 4
    for (int j4 = threadIdx.x; j4 < n4; j4 += NT) {
      const int j = j4 * 4;
      float4 v = make_float4(s[((j + 0) / W) * S + (j + 0) % W], s[((j + 1) / W) * S + (j + 1) % W],
                             s[((j + 2) / W) * S + (j + 2) % W], s[((j + 3) / W) * S + (j + 3) % W]);
      if (accum) {
        const float4 o = dst4[j4];
        v = make_float4(o.x + v.x, o.y + v.y, o.z + v.z, o.w + v.w);
      }
      dst4[j4] = v;
    }
  }
  for (int j = (aligned ? n4 * 4 : 0) + threadIdx.x; j < total; j += NT) {
    const float v = s[(j / W) * S + j % W];
    if (accum) dst[j] += v;
    else dst[j] = v;
  }
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 1/x to ~1 ulp (MUFU.RCP, no IEEE slow path): used where the result feeds only gradients
// (toleranced), never a threshold test that decides the contributor set.
// Programmatic dependent launch (sm_90+): kernels launched with launch_pdl may start while the
// previous kernel of the stream / graph drains; griddep_wait() (first statement of every such
// kernel) blocks until that kernel's memory operations are visible.  A no-op otherwise.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... P, typename... A>
inline cudaError_t launch_pdl(void (*kernel)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...);
}

__device__ __forceinline__ float fast_rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

constexpr float kNegHalfLog2e = -0.72134752044448170368f;  // -0.5 * log2(e)
constexpr double kNegHalfLog2eD = -0.72134752044448170368;

}  // namespace lgs
