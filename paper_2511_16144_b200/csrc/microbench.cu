// microbench.cu -- measured FP32 (FFMA) peak of this device, the roofline denominator for the
// blend kernels (MEASURED_PEAKS.json only carries HBM and bf16 tensor figures).
#include <cuda_runtime.h>

#include "../../include/lgs.h"
#include "mma_tf32.cuh"

namespace {

// One warp: D = A (16x8) * B (8x8) through the fragment layouts documented in mma_tf32.cuh,
// with the 3xTF32 split (mode 1) or plain TF32 (mode 0).
__global__ void mma_selftest_kernel(const float* A, const float* B, float* D, int mode) {
  const int lane = threadIdx.x, gid = lane >> 2, tig = lane & 3;
  const float av[4] = {A[gid * 8 + tig], A[(gid + 8) * 8 + tig], A[gid * 8 + tig + 4], A[(gid + 8) * 8 + tig + 4]};
  const float bv[2] = {B[tig * 8 + gid], B[(tig + 4) * 8 + gid]};
  uint32_t ah[4], al[4], bh[2], bl[2];
  for (int i = 0; i < 4; ++i) lgs::split_tf32(av[i], ah[i], al[i]);
  for (int i = 0; i < 2; ++i) lgs::split_tf32(bv[i], bh[i], bl[i]);
  float d[4] = {0.f, 0.f, 0.f, 0.f};
  if (mode) lgs::mma_3xtf32(d, ah, al, bh, bl);
  else lgs::mma_tf32(d, ah, bh);
  D[gid * 8 + 2 * tig] = d[0];
  D[gid * 8 + 2 * tig + 1] = d[1];
  D[(gid + 8) * 8 + 2 * tig] = d[2];
  D[(gid + 8) * 8 + 2 * tig + 1] = d[3];
}

__global__ void ffma_peak_kernel(float* out, int iters, float a, float b) {
  float x0 = threadIdx.x * 1e-7f, x1 = x0 + 1e-7f, x2 = x0 + 2e-7f, x3 = x0 + 3e-7f;
  float x4 = x0 + 4e-7f, x5 = x0 + 5e-7f, x6 = x0 + 6e-7f, x7 = x0 + 7e-7f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  const float s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
  if (s == 12345.678f) out[0] = s;  // keep the chains alive
}

// legacy-path (mma.sync, SASS HMMA) TF32 throughput: 8 independent m16n8k8 chains per warp
__global__ void mma_peak_kernel(float* out, int iters) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = lgs::to_tf32(1e-3f * (threadIdx.x + i));
  for (int i = 0; i < 2; ++i) b[i] = lgs::to_tf32(1e-3f * (threadIdx.x - i));
  float d[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) lgs::mma_tf32(d[k], a, b);
  }
  float s = 0.f;
  for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1] + d[k][2] + d[k][3];
  if (s == 12345.678f) out[0] = s;
}

}  // namespace

// Legacy tensor-core (mma.sync m16n8k8 TF32) throughput of this device, TFLOP/s.
extern "C" LGS_API lgs_status lgs_measure_mma_tf32_peak(int32_t device, double* tflops) {
  if (!tflops) return LGS_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return LGS_ECUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* out = nullptr;
  if (cudaMalloc(&out, sizeof(float)) != cudaSuccess) return LGS_ENOMEM;
  const int threads = 256, blocks = sms * 4, iters = 2048;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mma_peak_kernel<<<blocks, threads>>>(out, 16);
  cudaEventRecord(e0);
  mma_peak_kernel<<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 16 * 8 * 8 * 8.0 * iters * (double)(threads / 32) * blocks;
  *tflops = flops / (ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? LGS_OK : LGS_ECUDA;
}

extern "C" LGS_API lgs_status lgs_debug_mma_selftest(int32_t device, const float* a16x8, const float* b8x8,
                                                     float* d16x8, int32_t split) {
  if (!a16x8 || !b8x8 || !d16x8) return LGS_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return LGS_ECUDA;
  float* buf = nullptr;
  if (cudaMalloc(&buf, sizeof(float) * (128 + 64 + 128)) != cudaSuccess) return LGS_ENOMEM;
  cudaMemcpy(buf, a16x8, sizeof(float) * 128, cudaMemcpyHostToDevice);
  cudaMemcpy(buf + 128, b8x8, sizeof(float) * 64, cudaMemcpyHostToDevice);
  mma_selftest_kernel<<<1, 32>>>(buf, buf + 128, buf + 192, split);
  const cudaError_t e = cudaMemcpy(d16x8, buf + 192, sizeof(float) * 128, cudaMemcpyDeviceToHost);
  cudaFree(buf);
  return e == cudaSuccess ? LGS_OK : LGS_ECUDA;
}

extern "C" LGS_API lgs_status lgs_measure_fp32_peak(int32_t device, double* tflops) {
  if (!tflops) return LGS_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return LGS_ECUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* out = nullptr;
  if (cudaMalloc(&out, sizeof(float)) != cudaSuccess) return LGS_ENOMEM;
  const int threads = 512, blocks = sms * 4, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  ffma_peak_kernel<<<blocks, threads>>>(out, 64, 1.0000001f, 1e-7f);  // warm-up
  cudaEventRecord(e0);
  ffma_peak_kernel<<<blocks, threads>>>(out, iters, 1.0000001f, 1e-7f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 8.0 * 16.0 * iters * (double)threads * blocks;
  *tflops = flops / (ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? LGS_OK : LGS_ECUDA;
}
