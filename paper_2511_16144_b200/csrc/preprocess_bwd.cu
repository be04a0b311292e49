// preprocess_bwd.cu -- K7: chain per-Gaussian screen-space gradients to the map attributes.
//
// Restates proj/src/renderer.cpp:293-354 (+ rotation_derivatives :28-40) per Gaussian, in fp32:
//   g_Sigma2 = -C gC C (:315); g_Sigma_c = J^T g_Sigma2 J (:316); g_J = (g_Sigma2 + g_Sigma2^T)
//   J Sigma_c (:317-318); g_t incl. dJ/dt and the depth term (:320-327); g_p = R_cw^T g_t (:329);
//   g_Sigma3 = R_cw^T g_Sigma_c R_cw (:331); log-scale (:335-338); rotation -> unit quaternion
//   (:340-345) -> raw quaternion through the normalization (:347-353).
// Extensions (parity unpinned by the reference; pinned by finite differences in tests/):
//   - SH degree 1..3: colour -> SH coefficients and the view-direction term of the position grad;
//   - the 6-DoF pose gradient dL/dxi for cam_pose <- compose(se3_exp(xi), cam_pose).
// Outputs are written densely in the reference layouts (zeros for culled Gaussians unless
// accumulating).  One thread per Gaussian; HBM-bound (gacc line + map read + grads write).
#include "lgs_internal.cuh"
#include "lgs_kernels.h"

namespace lgs {

constexpr int kPbThreads = 128;

// Shared-memory row stride (floats) of the per-Gaussian SH block: odd, so thread t's row starts in
// bank t * stride mod 32 and the 32 lanes of a warp hit 32 different banks.
template <int DEG>
constexpr int sh_stride() { return 3 * (DEG + 1) * (DEG + 1) + 1 - (3 * (DEG + 1) * (DEG + 1)) % 2; }


// The chain for one live Gaussian i (its accumulator row is read; culled / unlisted Gaussians
// never get here).  my_sh holds its SH coefficients on entry (DEG > 0) and their gradients on exit;
// features are stored (or added) straight into g.feature; pose accumulates the pose gradient.
template <int DEG, int DP, int SLOTS>
__device__ __forceinline__ void gaussian_bwd(const DevMap& m, const DevCam& c, const ViewBufs& v,
                                             const float* __restrict__ gacc, const GradOut& g, int64_t i,
                                             bool accum, float* my_sh, float (&o_pos)[3], float (&o_rot)[4],
                                             float (&o_ls)[3], float& o_op, double (&pose)[6]) {
  constexpr int K = (DEG + 1) * (DEG + 1);
  constexpr int KS = 3 * K;
  const int64_t n = m.n;
  auto store = [accum](float* p, int64_t idx, float val) {
    if (accum) p[idx] += val;
    else p[idx] = val;
  };
  const float* ga = gacc + (size_t)i * SLOTS;
  // geometric slots: doubles (lgs_internal.cuh); z, colour and features: floats
  const double2 d01 = *reinterpret_cast<const double2*>(ga + 0);  // muX muY
  const double2 d23 = *reinterpret_cast<const double2*>(ga + 4);  // conA conB
  const double2 d45 = *reinterpret_cast<const double2*>(ga + 8);  // conC opac
  const float4 zc = *reinterpret_cast<const float4*>(ga + kSlotZ);  // z r g b
  // the chain runs in fp64 (near-plane / needle splats: J ~ f/z, conic ~ 1/det, cancellations)
  if (DP > 0 && g.feature) {  // renderer.cpp:262-264, written as [d][N]
#pragma unroll
    for (int q = 0; q < DP / 4; ++q) {
      const float4 fv = *reinterpret_cast<const float4*>(ga + kSlotFeat + q * 4);
      const float f4[4] = {fv.x, fv.y, fv.z, fv.w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (q * 4 + e < m.d) store(g.feature, (int64_t)(q * 4 + e) * n + i, f4[e]);
    }
  }
  o_op = (float)d45.y;
  const float4 po = m.pos_opa[i];
  const double P[3] = {po.x, po.y, po.z};
  double gpos[3] = {0.0, 0.0, 0.0};

  // ---- colour -> SH (renderer.cpp:259-261 for K = 1) ------------------------------------
  const double gc[3] = {zc.y, zc.z, zc.w};
  if (DEG == 0 || (gc[0] == 0.0 && gc[1] == 0.0 && gc[2] == 0.0)) {
    my_sh[0] = (float)gc[0];
    my_sh[1] = (float)gc[1];
    my_sh[2] = (float)gc[2];
#pragma unroll
    for (int k = 3; k < KS; ++k) my_sh[k] = 0.0;
  } else {
    const double dr[3] = {P[0] - c.cc_d[0], P[1] - c.cc_d[1], P[2] - c.cc_d[2]};
    const double nr = sqrt(dr[0] * dr[0] + dr[1] * dr[1] + dr[2] * dr[2]);
    const double inr = 1.0 / nr;
    const double dn[3] = {dr[0] * inr, dr[1] * inr, dr[2] * inr};
    double b[16];
    double db[16][3];
    sh_basis_f64(DEG, dn[0], dn[1], dn[2], b);
    sh_basis_grad_f64(DEG, dn[0], dn[1], dn[2], db);
    double gdn[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double s = 0.0;
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        s = fma(my_sh[k * 3 + ch], gc[ch], s);  // coefficient (staged), then overwritten by its grad
        my_sh[k * 3 + ch] = (float)(b[k] * gc[ch]);
      }
      gdn[0] = fma(db[k][0], s, gdn[0]);
      gdn[1] = fma(db[k][1], s, gdn[1]);
      gdn[2] = fma(db[k][2], s, gdn[2]);
    }
    const double dd = dn[0] * gdn[0] + dn[1] * gdn[1] + dn[2] * gdn[2];
    double gdir[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      gdir[a] = (gdn[a] - dn[a] * dd) * inr;
      gpos[a] += gdir[a];
    }
    if (g.pose) {  // dir = p - c with c' = c + omega x c + nu
      pose[0] += gdir[1] * c.cc_d[2] - gdir[2] * c.cc_d[1];
      pose[1] += gdir[2] * c.cc_d[0] - gdir[0] * c.cc_d[2];
      pose[2] += gdir[0] * c.cc_d[1] - gdir[1] * c.cc_d[0];
      pose[3] -= gdir[0];
      pose[4] -= gdir[1];
      pose[5] -= gdir[2];
    }
  }

  // ---- screen-space -> 3D (renderer.cpp:297-354) ----------------------------------------
  const double gmu0 = d01.x, gmu1 = d01.y, gA = d23.x, gB = d23.y, gC = d45.x, gz = zc.x;
  if (gmu0 != 0.0 || gmu1 != 0.0 || gA != 0.0 || gB != 0.0 || gC != 0.0 || gz != 0.0) {
    const double* R = c.rcw_d;
    double t[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) t[r] = R[r * 3 + 0] * P[0] + R[r * 3 + 1] * P[1] + R[r * 3 + 2] * P[2] + c.tcw_d[r];
    const double z = t[2];
    const float4 qr = m.rot[i];  // x,y,z,w
    const double qv[4] = {qr.w, qr.x, qr.y, qr.z};
    const double norm = sqrt(qv[0] * qv[0] + qv[1] * qv[1] + qv[2] * qv[2] + qv[3] * qv[3]);
    const double inorm = 1.0 / norm;
    const double qh[4] = {qv[0] * inorm, qv[1] * inorm, qv[2] * inorm, qv[3] * inorm};
    const double w = qh[0], x = qh[1], y = qh[2], zq = qh[3];
    double W[9];  // R_g (rotation of the Gaussian)
    {
      const double tx = 2 * x, ty = 2 * y, tz = 2 * zq;
      const double twx = tx * w, twy = ty * w, twz = tz * w, txx = tx * x, txy = ty * x, txz = tz * x;
      const double tyy = ty * y, tyz = tz * y, tzz = tz * zq;
      W[0] = 1 - (tyy + tzz); W[1] = txy - twz;       W[2] = txz + twy;
      W[3] = txy + twz;       W[4] = 1 - (txx + tzz); W[5] = tyz - twx;
      W[6] = txz - twy;       W[7] = tyz + twx;       W[8] = 1 - (txx + tyy);
    }
    const float4 ls = m.scale[i];
    const double s2[3] = {exp(2.0 * (double)ls.x), exp(2.0 * ls.y), exp(2.0 * ls.z)};
    // Sigma3 = W S^2 W^T, Sigma_c = R Sigma3 R^T
    double S3[9], RS[9], Sc[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int cc = 0; cc < 3; ++cc)
        S3[r * 3 + cc] = W[r * 3 + 0] * s2[0] * W[cc * 3 + 0] + W[r * 3 + 1] * s2[1] * W[cc * 3 + 1] +
                         W[r * 3 + 2] * s2[2] * W[cc * 3 + 2];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int cc = 0; cc < 3; ++cc)
        RS[r * 3 + cc] = R[r * 3 + 0] * S3[0 * 3 + cc] + R[r * 3 + 1] * S3[1 * 3 + cc] + R[r * 3 + 2] * S3[2 * 3 + cc];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int cc = 0; cc < 3; ++cc)
        Sc[r * 3 + cc] = RS[r * 3 + 0] * R[cc * 3 + 0] + RS[r * 3 + 1] * R[cc * 3 + 1] + RS[r * 3 + 2] * R[cc * 3 + 2];
    const double iz = 1.0 / z;
    const double J[6] = {c.fx_d * iz, 0.0, -c.fx_d * t[0] * iz * iz, 0.0, c.fy_d * iz, -c.fy_d * t[1] * iz * iz};

    // g_Sigma2 = -C gC C, C = conic (symmetric), gC = [[gA, gB], [gB, gC]]
    const float4 r1 = v.rec1[i];
    const double C0 = r1.x, C1 = r1.y, C3 = r1.z;
    const double cg00 = C0 * gA + C1 * gB, cg01 = C0 * gB + C1 * gC;
    const double cg10 = C1 * gA + C3 * gB, cg11 = C1 * gB + C3 * gC;
    const double gs[4] = {-(cg00 * C0 + cg01 * C1), -(cg00 * C1 + cg01 * C3), -(cg10 * C0 + cg11 * C1),
                         -(cg10 * C1 + cg11 * C3)};
    // g_Sigma_c = J^T gs J
    double gSc[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int cc = 0; cc < 3; ++cc)
        gSc[r * 3 + cc] = J[0 * 3 + r] * (gs[0] * J[0 * 3 + cc] + gs[1] * J[1 * 3 + cc]) +
                          J[1 * 3 + r] * (gs[2] * J[0 * 3 + cc] + gs[3] * J[1 * 3 + cc]);
    // g_J = (gs + gs^T) J Sigma_c
    const double sy[4] = {2.0 * gs[0], gs[1] + gs[2], gs[2] + gs[1], 2.0 * gs[3]};
    double JS[6], gJ[6];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int cc = 0; cc < 3; ++cc)
        JS[r * 3 + cc] = J[r * 3 + 0] * Sc[0 * 3 + cc] + J[r * 3 + 1] * Sc[1 * 3 + cc] + J[r * 3 + 2] * Sc[2 * 3 + cc];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int cc = 0; cc < 3; ++cc) gJ[r * 3 + cc] = sy[r * 2 + 0] * JS[0 * 3 + cc] + sy[r * 2 + 1] * JS[1 * 3 + cc];
    // g_t (renderer.cpp:320-327)
    double gt[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) gt[a] = J[0 * 3 + a] * gmu0 + J[1 * 3 + a] * gmu1;
    const double iz2 = iz * iz, iz3 = iz2 * iz;
    gt[0] += gJ[2] * (-c.fx_d * iz2);
    gt[1] += gJ[5] * (-c.fy_d * iz2);
    gt[2] += gJ[0] * (-c.fx_d * iz2) + gJ[2] * (2.0 * c.fx_d * t[0] * iz3) + gJ[4] * (-c.fy_d * iz2) +
             gJ[5] * (2.0 * c.fy_d * t[1] * iz3);
    gt[2] += gz;
    // g_p = R^T g_t (renderer.cpp:329)
    double gw[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      gw[a] = R[0 * 3 + a] * gt[0] + R[1 * 3 + a] * gt[1] + R[2 * 3 + a] * gt[2];
      gpos[a] += gw[a];
    }
    // G3 = R^T gSc R (symmetric)
    double tmp[9], G3[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int cc = 0; cc < 3; ++cc)
        tmp[r * 3 + cc] = R[0 * 3 + r] * gSc[0 * 3 + cc] + R[1 * 3 + r] * gSc[1 * 3 + cc] + R[2 * 3 + r] * gSc[2 * 3 + cc];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int cc = 0; cc < 3; ++cc)
        G3[r * 3 + cc] = tmp[r * 3 + 0] * R[0 * 3 + cc] + tmp[r * 3 + 1] * R[1 * 3 + cc] + tmp[r * 3 + 2] * R[2 * 3 + cc];
    // Y = G3 W; g_logs_a = (W^T G3 W)_aa 2 s2_a; g_rot = (G3 + G3^T) W S^2
    double Y[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int cc = 0; cc < 3; ++cc)
        Y[r * 3 + cc] = G3[r * 3 + 0] * W[0 * 3 + cc] + G3[r * 3 + 1] * W[1 * 3 + cc] + G3[r * 3 + 2] * W[2 * 3 + cc];
    double grot[9];
    // (G3 + G3^T) = 2 G3 only if symmetric; use the explicit sum for fidelity
    double Yt[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int cc = 0; cc < 3; ++cc)
        Yt[r * 3 + cc] = G3[0 * 3 + r] * W[0 * 3 + cc] + G3[1 * 3 + r] * W[1 * 3 + cc] + G3[2 * 3 + r] * W[2 * 3 + cc];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      o_ls[a] = (float)((W[0 * 3 + a] * Y[0 * 3 + a] + W[1 * 3 + a] * Y[1 * 3 + a] + W[2 * 3 + a] * Y[2 * 3 + a]) * 2.0 * s2[a]);
#pragma unroll
      for (int r = 0; r < 3; ++r) grot[r * 3 + a] = (Y[r * 3 + a] + Yt[r * 3 + a]) * s2[a];
    }
    // rotation_derivatives (renderer.cpp:28-40), all scaled by 2
    const double dw[9] = {0, -zq, y, zq, 0, -x, -y, x, 0};
    const double dxm[9] = {0, y, zq, y, -2 * x, -w, zq, w, -2 * x};
    const double dym[9] = {-2 * y, x, w, x, 0, zq, -w, zq, -2 * y};
    const double dzm[9] = {-2 * zq, -w, x, w, -2 * zq, y, x, y, 0};
    double gq[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int e = 0; e < 9; ++e) {
      gq[0] = fma(grot[e], dw[e], gq[0]);
      gq[1] = fma(grot[e], dxm[e], gq[1]);
      gq[2] = fma(grot[e], dym[e], gq[2]);
      gq[3] = fma(grot[e], dzm[e], gq[3]);
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) gq[a] *= 2.0;
    const double dot = qh[0] * gq[0] + qh[1] * gq[1] + qh[2] * gq[2] + qh[3] * gq[3];
#pragma unroll
    for (int a = 0; a < 4; ++a) o_rot[a] = (float)((gq[a] - qh[a] * dot) * inorm);

    if (g.pose) {
      // t' = R_cw (p - omega x p - nu) + t_cw: g_omega += g_w x p, g_nu -= g_w
      pose[0] += gw[1] * P[2] - gw[2] * P[1];
      pose[1] += gw[2] * P[0] - gw[0] * P[2];
      pose[2] += gw[0] * P[1] - gw[1] * P[0];
      pose[3] -= gw[0];
      pose[4] -= gw[1];
      pose[5] -= gw[2];
      // Sigma3' = (I - [omega]x) Sigma3 (I + [omega]x): A = Sigma3 G3 - G3 Sigma3, vee(A - A^T)
      double A1[9], A2[9];
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
          A1[r * 3 + cc] = S3[r * 3 + 0] * G3[0 * 3 + cc] + S3[r * 3 + 1] * G3[1 * 3 + cc] + S3[r * 3 + 2] * G3[2 * 3 + cc];
          A2[r * 3 + cc] = G3[r * 3 + 0] * S3[0 * 3 + cc] + G3[r * 3 + 1] * S3[1 * 3 + cc] + G3[r * 3 + 2] * S3[2 * 3 + cc];
        }
      pose[0] += (A1[7] - A2[7]) - (A1[5] - A2[5]);
      pose[1] += (A1[2] - A2[2]) - (A1[6] - A2[6]);
      pose[2] += (A1[3] - A2[3]) - (A1[1] - A2[1]);
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) o_pos[a] = (float)gpos[a];
}

template <int DEG, int DP, int SLOTS>
__global__ void __launch_bounds__(kPbThreads) preprocess_bwd_kernel(DevMap m, DevCam c, ViewBufs v,
                                                                      const float* __restrict__ gacc, GradOut g) {
  if (g.skip && *g.skip) return;
  constexpr int K = (DEG + 1) * (DEG + 1);
  constexpr int KS = 3 * K;
  constexpr int SS = sh_stride<DEG>();
  __shared__ float s_sh[kPbThreads * SS];  // SH coefficients in, SH gradients out (in place)
  __shared__ float s_pos[kPbThreads * 3];
  __shared__ float s_ls[kPbThreads * 3];
  const int tid = threadIdx.x;
  const int64_t i0 = (int64_t)blockIdx.x * kPbThreads;
  const int64_t i = i0 + tid;
  const int64_t n = m.n;
  const int nloc = (int)min((int64_t)kPbThreads, n - i0);
  const bool live = i < n && (v.active ? v.active[i] != 0 : v.tiles[i] != 0);
  const bool accum = g.accumulate != 0;
  // A block without a live Gaussian (most of them with the depth-layered binning) has an all-zero
  // gradient: nothing to add when accumulating, else streaming zero stores of its output rows.
  if (!__syncthreads_or(live)) {
    if (accum) return;
    auto zero_rows = [&](float* base, int64_t count) {
      if (!base) return;
      if ((reinterpret_cast<uintptr_t>(base) & 15u) == 0) {
        float4* b4 = reinterpret_cast<float4*>(base);
        const int64_t n4 = count >> 2;
        for (int64_t j = tid; j < n4; j += kPbThreads) b4[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int64_t j = n4 * 4 + tid; j < count; j += kPbThreads) base[j] = 0.f;
      } else {
        for (int64_t j = tid; j < count; j += kPbThreads) base[j] = 0.f;
      }
    };
    zero_rows(g.position ? g.position + i0 * 3 : nullptr, (int64_t)nloc * 3);
    zero_rows(g.rotation ? g.rotation + i0 * 4 : nullptr, (int64_t)nloc * 4);
    zero_rows(g.log_scale ? g.log_scale + i0 * 3 : nullptr, (int64_t)nloc * 3);
    zero_rows(g.opacity_logit ? g.opacity_logit + i0 : nullptr, nloc);
    zero_rows(g.sh ? g.sh + i0 * KS : nullptr, (int64_t)nloc * KS);
    if (DP > 0 && g.feature)
      for (int k = 0; k < m.d; ++k) zero_rows(g.feature + (int64_t)k * n + i0, nloc);
    return;
  }
  if (DEG > 0) stage_rows_in<KS, SS, kPbThreads>(s_sh, m.sh + i0 * KS, nloc);
  __syncthreads();
  float* my_sh = s_sh + tid * SS;
  double pose[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  if (i < n) {
    float o_pos[3] = {0.f, 0.f, 0.f}, o_rot[4] = {0.f, 0.f, 0.f, 0.f}, o_ls[3] = {0.f, 0.f, 0.f};
    float o_op = 0.f;
    auto store = [accum](float* p, int64_t idx, float val) {
      if (accum) p[idx] += val;
      else p[idx] = val;
    };
    // zero gradient unless the Gaussian sits in a traversed tile list (its accumulator row is then
    // exactly zero: every term below vanishes)
    const bool visible = live;
    if (!visible) {
#pragma unroll
      for (int k = 0; k < KS; ++k) my_sh[k] = 0.f;
      if (DP > 0 && g.feature && !accum)
        for (int k = 0; k < m.d; ++k) g.feature[(int64_t)k * n + i] = 0.f;
    } else {
      gaussian_bwd<DEG, DP, SLOTS>(m, c, v, gacc, g, i, accum, my_sh, o_pos, o_rot, o_ls, o_op, pose);
    }

    // ---- dense writes in the reference layouts (zeros for culled Gaussians) -------------------
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      s_pos[tid * 3 + a] = o_pos[a];
      s_ls[tid * 3 + a] = o_ls[a];
    }
    if (g.rotation) {  // (w,x,y,z): one 16-byte store when the buffer is 16-byte aligned
      if ((reinterpret_cast<uintptr_t>(g.rotation) & 15u) == 0) {
        float4* rp = reinterpret_cast<float4*>(g.rotation) + i;
        float4 r4 = make_float4(o_rot[0], o_rot[1], o_rot[2], o_rot[3]);
        if (accum) {
          const float4 old = *rp;
          r4 = make_float4(old.x + r4.x, old.y + r4.y, old.z + r4.z, old.w + r4.w);
        }
        *rp = r4;
      } else {
#pragma unroll
        for (int a = 0; a < 4; ++a) store(g.rotation, i * 4 + a, o_rot[a]);
      }
    }
    if (g.opacity_logit) store(g.opacity_logit, i, o_op);
  }
  __syncthreads();
  // [N][3] and [N][K][3] blocks of this CTA's Gaussians leave through shared memory, coalesced
  if (g.position) stage_rows_out<3, 3, kPbThreads>(s_pos, g.position + i0 * 3, nloc, accum);
  if (g.log_scale) stage_rows_out<3, 3, kPbThreads>(s_ls, g.log_scale + i0 * 3, nloc, accum);
  if (g.sh) stage_rows_out<KS, SS, kPbThreads>(s_sh, g.sh + i0 * KS, nloc, accum);

  if (g.pose) {  // block reduction of the pose gradient, one double atomic per value per block
    __shared__ double s_pose[kPbThreads / 32][6];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      double p = pose[a];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) p += __shfl_xor_sync(0xffffffffu, p, off);
      if (lane == 0) s_pose[wid][a] = p;
    }
    __syncthreads();
    if (threadIdx.x < 6) {
      double s = 0.0;
      for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) s += s_pose[w2][threadIdx.x];
      if (s != 0.0) atomicAdd(g.pose + threadIdx.x, s);
    }
  }
}

// ---- sparse variant (depth-layered binning): only the active Gaussians have nonzero gradients --
// With the layered lists ~15k of 500k Gaussians are active (the layer-A candidates + the second
// pass's), spread over nearly every 128-row block of the dense kernel, which then pays its full
// staging and divergent compute for a few live rows per warp.  Instead: (1) a streaming kernel
// writes the zero rows of every Gaussian (nothing when accumulating) -- inside a captured plan it
// runs on a side branch forked after the preprocess, off the critical path (lgs_capi.cu); (2) a
// kernel whose blocks each compact the active rows of a contiguous range into a shared queue and
// run the chain one queue entry per thread, storing (or adding) each active row.  Same values as
// the dense kernel per row.
struct ZeroSegs {
  float* ptr[6];  // position, rotation, log-scale, opacity, SH, feature ([d][N]: one contiguous block)
  int64_t count[6];
};

// grid-stride 16-byte streaming stores over each contiguous attribute block (scalar head / tail).
// A small grid (2 CTAs per SM): stores are fire-and-forget, so a few warps per SM saturate HBM
// writes while leaving the SMs to the kernels it runs beside (a side branch of the plan).
__global__ void __launch_bounds__(256) grad_zero_kernel(ZeroSegs z) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
#pragma unroll
  for (int a = 0; a < 6; ++a) {
    float* p = z.ptr[a];
    if (!p) continue;
    const int64_t cnt = z.count[a];
    const int64_t head = min(cnt, (int64_t)(((16u - (reinterpret_cast<uintptr_t>(p) & 15u)) & 15u) >> 2));
    if (t < head) p[t] = 0.f;
    float4* p4 = reinterpret_cast<float4*>(p + head);
    const int64_t n4 = (cnt - head) >> 2;
    for (int64_t j = t; j < n4; j += stride) __stcs(p4 + j, make_float4(0.f, 0.f, 0.f, 0.f));
    const int64_t tail = head + n4 * 4 + t;
    if (tail < cnt) p[tail] = 0.f;
  }
}

void launch_grad_zero(const GradOut& g, int64_t n, int K, int d, cudaStream_t s) {
  if (n == 0 || g.accumulate) return;
  const ZeroSegs z{{g.position, g.rotation, g.log_scale, g.opacity_logit, g.sh, d > 0 ? g.feature : nullptr},
                   {n * 3, n * 4, n * 3, n, n * 3 * K, n * d}};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  grad_zero_kernel<<<(unsigned)(sms * 2), 256, 0, s>>>(z);
}

constexpr int kActFlags = 16;                         // active flags per thread (one 16-byte load)
constexpr int kActRange = kPbThreads * kActFlags;       // rows per block

template <int DEG, int DP, int SLOTS>
__global__ void __launch_bounds__(kPbThreads) preprocess_bwd_active_kernel(DevMap m, DevCam c, ViewBufs v,
                                                                             const float* __restrict__ gacc, GradOut g) {
  if (g.skip && *g.skip) return;
  constexpr int K = (DEG + 1) * (DEG + 1);
  constexpr int KS = 3 * K;
  constexpr int SS = sh_stride<DEG>();
  __shared__ float s_sh[kPbThreads * SS];
  __shared__ uint32_t s_q[kActRange];
  __shared__ int s_wsum[kPbThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  float* my_sh = s_sh + tid * SS;
  const bool accum = g.accumulate != 0;
  double pose[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};

  // compact this block's active rows into s_q (ascending), one 16-byte flag load per thread
  const int64_t f0 = (int64_t)blockIdx.x * kActRange + (int64_t)tid * kActFlags;
  uint32_t bits = 0;
  if (f0 + kActFlags <= m.n && (reinterpret_cast<uintptr_t>(v.active + f0) & 15u) == 0) {
    const uint4 w = *reinterpret_cast<const uint4*>(v.active + f0);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int b = 0; b < 4; ++b) bits |= (((ws[k] >> (8 * b)) & 0xffu) != 0u) << (k * 4 + b);
  } else {
    for (int k = 0; k < kActFlags && f0 + k < m.n; ++k) bits |= (v.active[f0 + k] != 0) << k;
  }
  const int cnt = __popc(bits);
  int incl = cnt;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += y;
  }
  if (lane == 31) s_wsum[wid] = incl;
  __syncthreads();
  int base = incl - cnt, total = 0;
#pragma unroll
  for (int w2 = 0; w2 < kPbThreads / 32; ++w2) {
    base += w2 < wid ? s_wsum[w2] : 0;
    total += s_wsum[w2];
  }
  for (uint32_t b2 = bits; b2; b2 &= b2 - 1) s_q[base++] = (uint32_t)(f0 + __ffs(b2) - 1);
  __syncthreads();

  for (int q0 = 0; q0 < total; q0 += kPbThreads) {  // the chain, one active row per thread
    if (q0 + tid >= total) break;
    const int64_t i = s_q[q0 + tid];
    if (DEG > 0) {
      const float* src = m.sh + i * KS;
#pragma unroll
      for (int q = 0; q < KS; ++q) my_sh[q] = __ldg(src + q);
    }
    float o_pos[3] = {0.f, 0.f, 0.f}, o_rot[4] = {0.f, 0.f, 0.f, 0.f}, o_ls[3] = {0.f, 0.f, 0.f};
    float o_op = 0.f;
    gaussian_bwd<DEG, DP, SLOTS>(m, c, v, gacc, g, i, accum, my_sh, o_pos, o_rot, o_ls, o_op, pose);
    auto put = [accum](float* p, int64_t idx, float val) {
      if (accum) p[idx] += val;
      else p[idx] = val;
    };
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (g.position) put(g.position, i * 3 + a, o_pos[a]);
      if (g.log_scale) put(g.log_scale, i * 3 + a, o_ls[a]);
    }
    if (g.rotation)
#pragma unroll
      for (int a = 0; a < 4; ++a) put(g.rotation, i * 4 + a, o_rot[a]);
    if (g.opacity_logit) put(g.opacity_logit, i, o_op);
    if (g.sh)
#pragma unroll
      for (int q = 0; q < KS; ++q) put(g.sh, i * KS + q, my_sh[q]);
  }
  if (g.pose) {  // block reduction of the pose gradient, one double atomic per value per block
    __shared__ double s_pose[kPbThreads / 32][6];
#pragma unroll
    for (int a = 0; a < 6; ++a) {
      double p = pose[a];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) p += __shfl_xor_sync(0xffffffffu, p, off);
      if (lane == 0) s_pose[wid][a] = p;
    }
    __syncthreads();
    if (threadIdx.x < 6) {
      double s = 0.0;
      for (int w2 = 0; w2 < kPbThreads / 32; ++w2) s += s_pose[w2][threadIdx.x];
      if (s != 0.0) atomicAdd(g.pose + threadIdx.x, s);
    }
  }
  if (g.done) {  // the last CTA: pose as float, the next tile order (GradOut)
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(g.done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (g.pose_out && threadIdx.x < 6) g.pose_out[threadIdx.x] = (float)__ldcg(g.pose + threadIdx.x);
    for (int i = threadIdx.x; i < g.copy_n; i += blockDim.x) g.copy_dst[i] = __ldcg(g.copy_src + i);
  }
}

template <int DEG, int DP>
static void launch_pb(const DevMap& m, const DevCam& c, const ViewBufs& v, const float* gacc, const GradOut& g,
                      bool zeroed, cudaStream_t s) {
  if (v.active) {
    if (!zeroed) launch_grad_zero(g, m.n, m.K, DP > 0 ? m.d : 0, s);
    preprocess_bwd_active_kernel<DEG, DP, slots_for(DP)>
        <<<(unsigned)((m.n + kActRange - 1) / kActRange), kPbThreads, 0, s>>>(m, c, v, gacc, g);
    return;
  }
  const unsigned blocks = (unsigned)((m.n + kPbThreads - 1) / kPbThreads);
  preprocess_bwd_kernel<DEG, DP, slots_for(DP)><<<blocks, kPbThreads, 0, s>>>(m, c, v, gacc, g);
}

template <int DEG>
static void launch_pb_deg(const DevMap& m, const DevCam& c, const ViewBufs& v, const float* gacc, const GradOut& g,
                          bool zeroed, cudaStream_t s) {
  switch (m.dp) {
    case 0: launch_pb<DEG, 0>(m, c, v, gacc, g, zeroed, s); break;
    case 4: launch_pb<DEG, 4>(m, c, v, gacc, g, zeroed, s); break;
    case 8: launch_pb<DEG, 8>(m, c, v, gacc, g, zeroed, s); break;
    case 16: launch_pb<DEG, 16>(m, c, v, gacc, g, zeroed, s); break;
    default: launch_pb<DEG, 32>(m, c, v, gacc, g, zeroed, s); break;
  }
}

void launch_preprocess_bwd(const DevMap& m, const DevCam& c, const ViewBufs& v, const float* gacc, int slots,
                           const GradOut& g, bool zeroed, cudaStream_t s) {
  (void)slots;
  if (m.n == 0) return;
  switch (m.deg) {
    case 0: launch_pb_deg<0>(m, c, v, gacc, g, zeroed, s); break;
    case 1: launch_pb_deg<1>(m, c, v, gacc, g, zeroed, s); break;
    case 2: launch_pb_deg<2>(m, c, v, gacc, g, zeroed, s); break;
    default: launch_pb_deg<3>(m, c, v, gacc, g, zeroed, s); break;
  }
}

// one warp per 32 rows: lanes clear the rows of live Gaussians, float4 at a time
__global__ void zero_active_rows_kernel(const uint8_t* __restrict__ active, const uint32_t* __restrict__ tiles,
                                        int64_t n, float4* __restrict__ gacc, int q_per_row) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (!(active ? active[i] != 0 : tiles[i] != 0)) return;
  float4* row = gacc + i * q_per_row;
  for (int q = 0; q < q_per_row; ++q) row[q] = make_float4(0.f, 0.f, 0.f, 0.f);
}

void launch_zero_active_rows(const ViewBufs& v, int64_t n, float* gacc, int slots, cudaStream_t s) {
  if (n == 0) return;
  zero_active_rows_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(v.active, v.tiles, n,
                                                                      reinterpret_cast<float4*>(gacc), slots / 4);
}

// fp64 pose accumulator [6] -> float [6] in place (the floats overwrite the first 24 bytes).
__global__ void pose_to_float_kernel(double* __restrict__ pose) {
  if (threadIdx.x == 0) {
    float f[6];
    for (int a = 0; a < 6; ++a) f[a] = (float)pose[a];
    float* out = reinterpret_cast<float*>(pose);
    for (int a = 0; a < 6; ++a) out[a] = f[a];
  }
}

void launch_pose_to_float(double* pose, float* /*same storage*/, cudaStream_t s) {
  pose_to_float_kernel<<<1, 32, 0, s>>>(pose);
}

}  // namespace lgs
