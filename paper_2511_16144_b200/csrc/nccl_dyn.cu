// nccl_dyn.cu -- run-time binding of the NCCL entry points used by the multi-view gradient
// all-reduce (lgs_comm_* in lgs_capi.cu).  See nccl_dyn.h.
#include <dlfcn.h>

#include <mutex>

#include "nccl_dyn.h"

namespace lgs {

namespace {

NcclApi g_api;
bool g_ok = false;
std::string g_err;
std::once_flag g_once;

template <typename F>
bool resolve(void* h, const char* name, F& fn) {
  fn = reinterpret_cast<F>(dlsym(h, name));
  if (!fn) g_err = std::string("libnccl.so.2 lacks ") + name;
  return fn != nullptr;
}

void load() {
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's NCCL (torch), if any
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    const char* e = dlerror();
    g_err = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
    return;
  }
  g_ok = resolve(h, "ncclGetUniqueId", g_api.GetUniqueId) && resolve(h, "ncclCommInitRank", g_api.CommInitRank) &&
         resolve(h, "ncclCommDestroy", g_api.CommDestroy) && resolve(h, "ncclAllReduce", g_api.AllReduce) &&
         resolve(h, "ncclReduceScatter", g_api.ReduceScatter) && resolve(h, "ncclAllGather", g_api.AllGather) &&
         resolve(h, "ncclGroupStart", g_api.GroupStart) && resolve(h, "ncclGroupEnd", g_api.GroupEnd) &&
         resolve(h, "ncclGetErrorString", g_api.GetErrorString) && resolve(h, "ncclGetVersion", g_api.GetVersion) &&
         resolve(h, "ncclCommAbort", g_api.CommAbort) && resolve(h, "ncclCommGetAsyncError", g_api.CommGetAsyncError);
}

}  // namespace

const NcclApi* nccl_api(std::string* err) {
  std::call_once(g_once, load);
  if (!g_ok && err) *err = g_err;
  return g_ok ? &g_api : nullptr;
}

}  // namespace lgs
