// dev_cache.h -- per-device launch facts cached for the host-side launchers, thread-safe.
//
// Each lgs_ctx binds its own device and several host threads may enqueue concurrently, so nothing
// device-specific may live in a plain function-local static: SM counts, kernel occupancies,
// dynamic-shared-memory opt-ins (cudaFuncSetAttribute) and __constant__ uploads are kept per
// (kernel or symbol, device) under one mutex.
#pragma once

#include <cuda_runtime.h>

#include <functional>

namespace lgs {

// SM count of the current device.
int device_sm_count();
// Max resident CTAs per SM of `kernel` at `threads` threads / `smem` dynamic bytes on the current
// device (at least 1).
int kernel_ctas_per_sm(const void* kernel, int threads, size_t smem);
// Raises `kernel`'s dynamic shared memory limit on the current device to at least `bytes`.
cudaError_t ensure_dyn_smem(const void* kernel, int bytes);
// Runs `init` once per (key, current device); later calls return the first call's result.
bool once_per_device(const void* key, const std::function<bool()>& init);

}  // namespace lgs
