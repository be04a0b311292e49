// dev_cache.cu -- see dev_cache.h.
#include <map>
#include <mutex>
#include <utility>

#include "dev_cache.h"

namespace lgs {

namespace {

std::mutex g_mu;
std::map<int, int> g_sms;                                  // device -> SM count
std::map<std::pair<const void*, int>, int> g_ctas;         // (kernel, device) -> CTAs per SM
std::map<std::pair<const void*, int>, int> g_smem;         // (kernel, device) -> dynamic smem limit set
std::map<std::pair<const void*, int>, bool> g_once;        // (key, device) -> init result

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

}  // namespace

int device_sm_count() {
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_sms.find(dev);
  if (it != g_sms.end()) return it->second;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms < 1) sms = 1;
  g_sms[dev] = sms;
  return sms;
}

int kernel_ctas_per_sm(const void* kernel, int threads, size_t smem) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(g_mu);
  const auto key = std::make_pair(kernel, dev * 4096 + threads);
  auto it = g_ctas.find(key);
  if (it != g_ctas.end()) return it->second;
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem);
  if (n < 1) n = 1;
  g_ctas[key] = n;
  return n;
}

cudaError_t ensure_dyn_smem(const void* kernel, int bytes) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(g_mu);
  int& have = g_smem[std::make_pair(kernel, dev)];
  if (have >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

bool once_per_device(const void* key, const std::function<bool()>& init) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lock(g_mu);
  const auto k = std::make_pair(key, dev);
  auto it = g_once.find(k);
  if (it != g_once.end()) return it->second;
  const bool ok = init();
  if (ok) g_once[k] = true;  // a failed init is retried on the next call
  return ok;
}

}  // namespace lgs
