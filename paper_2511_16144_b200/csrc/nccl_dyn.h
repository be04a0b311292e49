// nccl_dyn.h -- NCCL entry points resolved at run time (dlopen "libnccl.so.2").
//
// liblgs.so does not link NCCL: a process that already loaded NCCL (PyTorch's torch.distributed
// ships its own libnccl.so.2) must use that same copy, and a process that never touches the
// multi-GPU path should not need NCCL at all.  dlopen with RTLD_NOLOAD first picks up an already
// loaded libnccl.so.2; otherwise the system one is loaded.  Only the types come from <nccl.h>.
#pragma once

#include <nccl.h>

#include <string>

namespace lgs {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
  ncclResult_t (*GetVersion)(int*);
  ncclResult_t (*CommAbort)(ncclComm_t);
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*);
};

// nullptr (and *err set) when NCCL cannot be loaded.
const NcclApi* nccl_api(std::string* err);

}  // namespace lgs
