// loss.cu -- K8: the mapping losses and the decoder chain that produce the rasterizer's cotangents
// (SPEC.md:418-426 compute_losses; proj/src/codec.cpp:88-143 decoder).
//
//   l_rgb   = w_l1 L1(rgb, kf.rgb) + (1 - w_l1) (1 - SSIM) / 2     (11x11 Gaussian, sigma 1.5,
//             'valid' window positions, channel-averaged; oracle/loss.py documents the choice)
//   l_depth = mean over {measured depth valid, acc > 0.5} of |depth - kf.depth|
//   l_feat  = mean |decode(feat) - F_gt|,  decode(z) = W2 relu(W1 z + b1) + b2  (per pixel)
//   l_total = l_rgb + w_depth l_depth + w_feat l_feat
//
// Three kernels, all writing into the tape's cotangent buffer [H][W][4 + DP] that the backward
// blend reads (g_rgb 3 | g_depth | g_feat DP):
//   ssim_stats_kernel : 32x16 output tile + 5-pixel halo staged in shared memory; separable
//                       Gaussian blurs of x, y, x^2, y^2, xy; per valid window centre the SSIM and
//                       its partials A = dS/dmu_x, B = dS/dE[x^2], C = dS/dE[xy] (scaled by the
//                       loss weight) -> planar [9][H][W]; loss partial sums and the depth-mask count;
//   ssim_grad_kernel  : the adjoint blur of A, B, C (same halo tiling) ->
//                       g_x = blur(A) + 2 x blur(B) + y blur(C) + w_l1 sign(x - y) / (3HW);
//                       the masked depth cotangent (needs the count from the first kernel);
//   decoder_l1_kernel : one thread per pixel, decoder weights in shared memory (warp-uniform
//                       float4 broadcasts), hidden activations and their cotangents in registers,
//                       F_gt streamed once: y, sign(y - F_gt), W2^T g, ReLU mask, W1^T gh.
// Roofline: the stencils move ~130 B/pixel (HBM); the decoder does (d + D) * 2 * H FMAs per pixel
// (FP32 pipe; 6144 FMA/pixel at d = 16, H = 64, D = 32).
#include <algorithm>
#include <cmath>

#include "lgs_internal.cuh"
#include "lgs_kernels.h"
#include "dev_cache.h"

namespace lgs {

namespace {

constexpr int kR = 5;               // window radius (11 taps)
constexpr int kTW = 32, kTH = 16;   // output tile
constexpr int kRW = kTW + 2 * kR;   // staged region width (42)
constexpr int kRH = kTH + 2 * kR;   // staged region height (26)
constexpr float kC1 = 1e-4f, kC2 = 9e-4f;

__constant__ float c_win[2 * kR + 1];

// Shared-memory float4 load the compiler may not merge with an earlier load of the same address:
// the decoder reads each W2 row twice (y, then W2^T g) and must not keep 64 weights live across.
__device__ __forceinline__ float4 lds4_fresh(const float4* p) {
  float4 v;
  const unsigned a = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

__device__ __forceinline__ void block_sum_atomic(double v, double* dst, double* s_red) {
  // 256-thread block: warp shuffle then one atomic per block
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) s_red[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_red[w];
    if (t != 0.0) atomicAdd(dst, t);
  }
}

__global__ void __launch_bounds__(256) ssim_stats_kernel(const float* __restrict__ rgb, const float* __restrict__ gt,
                                                         const float* __restrict__ depth, const float* __restrict__ acc,
                                                         const float* __restrict__ kf_depth, int H, int W,
                                                         float kscale, float* __restrict__ abc,
                                                         double* __restrict__ sums) {
  __shared__ float sx[kRH][kRW], sy[kRH][kRW];
  __shared__ float hb[5][kRH][kTW];  // horizontal blurs of x, y, xx, yy, xy
  __shared__ double s_red[8];
  const int ox0 = blockIdx.x * kTW, oy0 = blockIdx.y * kTH;
  const int tid = threadIdx.x;
  const size_t plane = (size_t)H * W;
  double ssim_acc = 0.0, l1_acc = 0.0, dabs = 0.0, dcnt = 0.0;

  for (int ch = 0; ch < 3; ++ch) {
    __syncthreads();
    for (int i = tid; i < kRH * kRW; i += blockDim.x) {
      const int ry = i / kRW, rx = i % kRW;
      const int gy = oy0 - kR + ry, gx = ox0 - kR + rx;
      float xv = 0.f, yv = 0.f;
      if (gy >= 0 && gy < H && gx >= 0 && gx < W) {
        const size_t p = (size_t)gy * W + gx;
        xv = rgb[p * 3 + ch];
        yv = gt[p * 3 + ch];
      }
      sx[ry][rx] = xv;
      sy[ry][rx] = yv;
    }
    __syncthreads();
    for (int i = tid; i < kRH * kTW; i += blockDim.x) {
      const int ry = i / kTW, cx = i % kTW;
      float a = 0.f, b = 0.f, aa = 0.f, bb = 0.f, ab = 0.f;
#pragma unroll
      for (int k = 0; k < 2 * kR + 1; ++k) {
        const float w = c_win[k];
        const float xv = sx[ry][cx + k], yv = sy[ry][cx + k];
        a = fmaf(w, xv, a);
        b = fmaf(w, yv, b);
        aa = fmaf(w, xv * xv, aa);
        bb = fmaf(w, yv * yv, bb);
        ab = fmaf(w, xv * yv, ab);
      }
      hb[0][ry][cx] = a; hb[1][ry][cx] = b; hb[2][ry][cx] = aa; hb[3][ry][cx] = bb; hb[4][ry][cx] = ab;
    }
    __syncthreads();
    for (int i = tid; i < kTH * kTW; i += blockDim.x) {
      const int ty = i / kTW, tx = i % kTW;
      const int gy = oy0 + ty, gx = ox0 + tx;
      if (gy >= H || gx >= W) continue;
      const size_t p = (size_t)gy * W + gx;
      l1_acc += fabsf(sx[ty + kR][tx + kR] - sy[ty + kR][tx + kR]);
      float A = 0.f, B = 0.f, C = 0.f;
      if (gy >= kR && gy < H - kR && gx >= kR && gx < W - kR) {  // valid window centre
        float mx = 0.f, my = 0.f, exx = 0.f, eyy = 0.f, exy = 0.f;
#pragma unroll
        for (int k = 0; k < 2 * kR + 1; ++k) {
          const float w = c_win[k];
          mx = fmaf(w, hb[0][ty + k][tx], mx);
          my = fmaf(w, hb[1][ty + k][tx], my);
          exx = fmaf(w, hb[2][ty + k][tx], exx);
          eyy = fmaf(w, hb[3][ty + k][tx], eyy);
          exy = fmaf(w, hb[4][ty + k][tx], exy);
        }
        const float sxx = exx - mx * mx, syy = eyy - my * my, sxy = exy - mx * my;
        const float n1 = 2.f * mx * my + kC1, n2 = 2.f * sxy + kC2;
        const float d1 = mx * mx + my * my + kC1, d2 = sxx + syy + kC2;
        const float S = (n1 * n2) / (d1 * d2);
        ssim_acc += S;
        const float ks = kscale * S;  // kscale = d l_total / d S_p
        A = ks * (2.f * my / n1 - 2.f * my / n2 - 2.f * mx / d1 + 2.f * mx / d2);
        B = ks * (-1.f / d2);
        C = ks * (2.f / n2);
      }
      abc[(0 * 3 + ch) * plane + p] = A;
      abc[(1 * 3 + ch) * plane + p] = B;
      abc[(2 * 3 + ch) * plane + p] = C;
      if (ch == 0) {  // depth mask: valid measurement (finite, > 0) and acc > 0.5
        const float kd = kf_depth[p];
        if (isfinite(kd) && kd > 0.f && acc[p] > 0.5f) {
          dabs += fabsf(depth[p] - kd);
          dcnt += 1.0;
        }
      }
    }
  }
  block_sum_atomic(l1_acc, sums + LOSS_L1_RGB, s_red);
  block_sum_atomic(ssim_acc, sums + LOSS_SSIM, s_red);
  block_sum_atomic(dabs, sums + LOSS_DEPTH_ABS, s_red);
  block_sum_atomic(dcnt, sums + LOSS_DEPTH_CNT, s_red);
}

__global__ void __launch_bounds__(256) ssim_grad_kernel(const float* __restrict__ rgb, const float* __restrict__ gt,
                                                        const float* __restrict__ depth, const float* __restrict__ acc,
                                                        const float* __restrict__ kf_depth, int H, int W,
                                                        const float* __restrict__ abc, float l1_scale, float w_depth,
                                                        const double* __restrict__ sums, float* __restrict__ cot,
                                                        int cot_stride) {
  __shared__ float sm[3][kRH][kRW];
  __shared__ float hb[3][kRH][kTW];
  const int ox0 = blockIdx.x * kTW, oy0 = blockIdx.y * kTH;
  const int tid = threadIdx.x;
  const size_t plane = (size_t)H * W;
  const double cnt = sums[LOSS_DEPTH_CNT];
  const float gd = cnt > 0.0 ? (float)(w_depth / cnt) : 0.f;

  for (int ch = 0; ch < 3; ++ch) {
    __syncthreads();
    for (int i = tid; i < kRH * kRW; i += blockDim.x) {
      const int ry = i / kRW, rx = i % kRW;
      const int gy = oy0 - kR + ry, gx = ox0 - kR + rx;
      float a = 0.f, b = 0.f, c = 0.f;
      if (gy >= 0 && gy < H && gx >= 0 && gx < W) {
        const size_t p = (size_t)gy * W + gx;
        a = abc[(0 * 3 + ch) * plane + p];
        b = abc[(1 * 3 + ch) * plane + p];
        c = abc[(2 * 3 + ch) * plane + p];
      }
      sm[0][ry][rx] = a; sm[1][ry][rx] = b; sm[2][ry][rx] = c;
    }
    __syncthreads();
    for (int i = tid; i < kRH * kTW; i += blockDim.x) {
      const int ry = i / kTW, cx = i % kTW;
      float a = 0.f, b = 0.f, c = 0.f;
#pragma unroll
      for (int k = 0; k < 2 * kR + 1; ++k) {
        const float w = c_win[k];
        a = fmaf(w, sm[0][ry][cx + k], a);
        b = fmaf(w, sm[1][ry][cx + k], b);
        c = fmaf(w, sm[2][ry][cx + k], c);
      }
      hb[0][ry][cx] = a; hb[1][ry][cx] = b; hb[2][ry][cx] = c;
    }
    __syncthreads();
    for (int i = tid; i < kTH * kTW; i += blockDim.x) {
      const int ty = i / kTW, tx = i % kTW;
      const int gy = oy0 + ty, gx = ox0 + tx;
      if (gy >= H || gx >= W) continue;
      const size_t p = (size_t)gy * W + gx;
      float a = 0.f, b = 0.f, c = 0.f;
#pragma unroll
      for (int k = 0; k < 2 * kR + 1; ++k) {
        const float w = c_win[k];
        a = fmaf(w, hb[0][ty + k][tx], a);
        b = fmaf(w, hb[1][ty + k][tx], b);
        c = fmaf(w, hb[2][ty + k][tx], c);
      }
      const float x = rgb[p * 3 + ch], y = gt[p * 3 + ch];
      const float df = x - y;
      const float sg = df > 0.f ? l1_scale : (df < 0.f ? -l1_scale : 0.f);
      cot[p * cot_stride + ch] = sg + a + 2.f * x * b + y * c;
      if (ch == 0) {
        const float kd = kf_depth[p];
        float g = 0.f;
        if (isfinite(kd) && kd > 0.f && acc[p] > 0.5f) {
          const float dd = depth[p] - kd;
          g = dd > 0.f ? gd : (dd < 0.f ? -gd : 0.f);
        }
        cot[p * cot_stride + 3] = g;
      }
    }
  }
}

template <int DP, int HID>
__global__ void __launch_bounds__(128) decoder_l1_kernel(const float* __restrict__ feat, int d, int D,
                                                         const float* __restrict__ w1, const float* __restrict__ b1,
                                                         const float* __restrict__ w2, const float* __restrict__ b2,
                                                         const float* __restrict__ fgt, int64_t npix, float gscale,
                                                         float* __restrict__ cot, int cot_stride,
                                                         double* __restrict__ sums) {
  extern __shared__ float4 s_dyn4[];
  float* s = reinterpret_cast<float*>(s_dyn4);
  float* sw1 = s;                    // [HID][DP] (zero-padded columns)
  float* sb1 = sw1 + HID * DP;       // [HID]
  float* sb2 = sb1 + HID;            // [D] (padded to a multiple of 4)
  float* sw2 = sb2 + ((D + 3) & ~3); // [D][HID]
  __shared__ double s_red[4];
  for (int i = threadIdx.x; i < HID * DP; i += blockDim.x) {
    const int j = i / DP, k = i % DP;
    sw1[i] = k < d ? w1[j * d + k] : 0.f;
  }
  for (int i = threadIdx.x; i < HID; i += blockDim.x) sb1[i] = b1[i];
  for (int i = threadIdx.x; i < D; i += blockDim.x) sb2[i] = b2[i];
  for (int i = threadIdx.x; i < D * HID; i += blockDim.x) sw2[i] = w2[i];
  __syncthreads();

  double fsum = 0.0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npix; p += (int64_t)gridDim.x * blockDim.x) {
    float z[DP];
#pragma unroll
    for (int k = 0; k < DP; ++k) z[k] = k < d ? feat[p * d + k] : 0.f;
    float h[HID], gh[HID];
#pragma unroll
    for (int j = 0; j < HID; ++j) {
      float a = sb1[j];
      const float4* wr = reinterpret_cast<const float4*>(sw1 + j * DP);
#pragma unroll
      for (int q = 0; q < DP / 4; ++q) {
        const float4 wv = lds4_fresh(wr + q);
        a = fmaf(wv.x, z[4 * q + 0], a);
        a = fmaf(wv.y, z[4 * q + 1], a);
        a = fmaf(wv.z, z[4 * q + 2], a);
        a = fmaf(wv.w, z[4 * q + 3], a);
      }
      h[j] = fmaxf(a, 0.f);
      gh[j] = 0.f;
    }
    const float* fr = fgt + p * D;
    for (int c = 0; c < D; ++c) {
      const float4* wr = reinterpret_cast<const float4*>(sw2 + c * HID);
      float y = sb2[c];
#pragma unroll
      for (int q = 0; q < HID / 4; ++q) {
        const float4 wv = wr[q];
        y = fmaf(wv.x, h[4 * q + 0], y);
        y = fmaf(wv.y, h[4 * q + 1], y);
        y = fmaf(wv.z, h[4 * q + 2], y);
        y = fmaf(wv.w, h[4 * q + 3], y);
      }
      const float df = y - __ldg(fr + c);
      fsum += fabsf(df);
      const float g = df > 0.f ? gscale : (df < 0.f ? -gscale : 0.f);
#pragma unroll
      for (int q = 0; q < HID / 4; ++q) {
        const float4 wv = lds4_fresh(wr + q);
        gh[4 * q + 0] = fmaf(wv.x, g, gh[4 * q + 0]);
        gh[4 * q + 1] = fmaf(wv.y, g, gh[4 * q + 1]);
        gh[4 * q + 2] = fmaf(wv.z, g, gh[4 * q + 2]);
        gh[4 * q + 3] = fmaf(wv.w, g, gh[4 * q + 3]);
      }
    }
    float gz[DP];
#pragma unroll
    for (int k = 0; k < DP; ++k) gz[k] = 0.f;
#pragma unroll
    for (int j = 0; j < HID; ++j) {
      const float gm = h[j] > 0.f ? gh[j] : 0.f;  // ReLU mask: pre-activation > 0 (codec.cpp:136)
      const float4* wr = reinterpret_cast<const float4*>(sw1 + j * DP);
#pragma unroll
      for (int q = 0; q < DP / 4; ++q) {
        const float4 wv = lds4_fresh(wr + q);
        gz[4 * q + 0] = fmaf(wv.x, gm, gz[4 * q + 0]);
        gz[4 * q + 1] = fmaf(wv.y, gm, gz[4 * q + 1]);
        gz[4 * q + 2] = fmaf(wv.z, gm, gz[4 * q + 2]);
        gz[4 * q + 3] = fmaf(wv.w, gm, gz[4 * q + 3]);
      }
    }
    float4* co = reinterpret_cast<float4*>(cot + p * cot_stride + 4);
#pragma unroll
    for (int q = 0; q < DP / 4; ++q) co[q] = make_float4(gz[4 * q], gz[4 * q + 1], gz[4 * q + 2], gz[4 * q + 3]);
  }
  // block reduction of the feature L1 sum (128 threads)
  for (int off = 16; off > 0; off >>= 1) fsum += __shfl_xor_sync(0xffffffffu, fsum, off);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = fsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    const double t = s_red[0] + s_red[1] + s_red[2] + s_red[3];
    if (t != 0.0) atomicAdd(sums + LOSS_FEAT_ABS, t);
  }
}

template <int DP>
int launch_decoder_dp(const LossArgs& a, cudaStream_t s) {
  constexpr int HID = 64;
  const size_t smem = sizeof(float) * ((size_t)HID * DP + HID + ((a.D + 3) & ~3) + (size_t)a.D * HID);
  if (ensure_dyn_smem(reinterpret_cast<const void*>(decoder_l1_kernel<DP, HID>), (int)smem) != cudaSuccess) return 2;
  const int sms = device_sm_count();
  const int64_t npix = (int64_t)a.H * a.W;
  const int64_t blocks = std::min<int64_t>((npix + 127) / 128, (int64_t)sms * 8);
  const float gscale = (float)(a.w_feat / ((double)npix * a.D));
  decoder_l1_kernel<DP, HID><<<(unsigned)blocks, 128, smem, s>>>(a.feat, a.d, a.D, a.w1, a.b1, a.w2, a.b2, a.feat_gt,
                                                                 npix, gscale, a.cot, a.cot_stride, a.sums);
  return 0;
}

// Insertion coverage mask: pixel selected iff rendered acc < 0.5 OR the measured
// depth is valid (finite, > 0) and |rendered depth - measured| > max(0.05 m, 0.05 measured).
__global__ void __launch_bounds__(256) coverage_kernel(const float* __restrict__ acc, const float* __restrict__ depth,
                                                       const float* __restrict__ measured, int64_t npix,
                                                       uint8_t* __restrict__ mask, unsigned long long* __restrict__ count) {
  unsigned c = 0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npix; p += (int64_t)gridDim.x * blockDim.x) {
    const float m = measured[p];
    bool sel = acc[p] < 0.5f;
    if (!sel && isfinite(m) && m > 0.f) sel = fabsf(depth[p] - m) > fmaxf(0.05f, 0.05f * m);
    mask[p] = sel ? 1 : 0;
    c += sel ? 1u : 0u;
  }
  for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, (unsigned long long)c);
}

}  // namespace

void launch_coverage(const float* acc, const float* depth, const float* measured, int64_t npix, uint8_t* mask,
                     unsigned long long* count, cudaStream_t s) {
  cudaMemsetAsync(count, 0, sizeof(unsigned long long), s);
  if (npix == 0) return;
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t blocks = std::min<int64_t>((npix + 255) / 256, (int64_t)sms * 8);
  coverage_kernel<<<(unsigned)blocks, 256, 0, s>>>(acc, depth, measured, npix, mask, count);
}

bool decoder_supported(int hidden, int dp, int D) {
  return hidden == 64 && (dp == 4 || dp == 8 || dp == 16 || dp == 32) && D >= 1 &&
         (size_t)D * 64 * 4 + 64 * 33 * 4 <= 200 * 1024;
}

int launch_mapping_loss(const LossArgs& a, cudaStream_t s) {
  // Gaussian window, sigma 1.5, normalized (oracle/loss.py gauss_window); __constant__ is per device
  const bool win_ok = once_per_device(reinterpret_cast<const void*>(&c_win), [] {
    double w[2 * kR + 1], sum = 0.0;
    for (int k = 0; k <= 2 * kR; ++k) {
      const double x = k - kR;
      w[k] = std::exp(-(x * x) / (2.0 * 1.5 * 1.5));
      sum += w[k];
    }
    float wf[2 * kR + 1];
    for (int k = 0; k <= 2 * kR; ++k) wf[k] = (float)(w[k] / sum);
    return cudaMemcpyToSymbol(c_win, wf, sizeof wf) == cudaSuccess;
  });
  if (!win_ok) return 2;
  const dim3 grid((a.W + kTW - 1) / kTW, (a.H + kTH - 1) / kTH);
  const double npos = (double)(a.H - 2 * kR) * (double)(a.W - 2 * kR);
  // d l_total / d S_p = -(1 - w_l1) / 2 / (3 npos)
  const float kscale = (float)(-(1.0 - a.w_l1) / 2.0 / (3.0 * npos));
  const float l1_scale = (float)(a.w_l1 / (3.0 * (double)a.H * a.W));
  cudaMemsetAsync(a.sums, 0, sizeof(double) * LOSS_COUNT, s);
  ssim_stats_kernel<<<grid, 256, 0, s>>>(a.rgb, a.rgb_gt, a.depth, a.acc, a.depth_gt, a.H, a.W, kscale, a.abc, a.sums);
  ssim_grad_kernel<<<grid, 256, 0, s>>>(a.rgb, a.rgb_gt, a.depth, a.acc, a.depth_gt, a.H, a.W, a.abc, l1_scale,
                                        (float)a.w_depth, a.sums, a.cot, a.cot_stride);
  if (a.dp == 0) return 0;
  switch (a.dp) {
    case 4: return launch_decoder_dp<4>(a, s);
    case 8: return launch_decoder_dp<8>(a, s);
    case 16: return launch_decoder_dp<16>(a, s);
    default: return launch_decoder_dp<32>(a, s);
  }
}

}  // namespace lgs
