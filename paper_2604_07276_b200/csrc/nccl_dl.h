// Minimal runtime-loaded NCCL (dlopen "libnccl.so.2").  Loading lazily lets the library
// share the NCCL that torch has already mapped into the process (same soname) instead of
// linking a second copy; it is only needed when world_size > 1.
#pragma once
#include <cuda_runtime.h>

#include <string>

namespace nb {

struct NcclUid {
  char internal[128];
};
typedef void* NcclComm;

struct Nccl {
  bool ok = false;
  std::string err;
  int (*GetUniqueId)(NcclUid*) = nullptr;
  int (*CommInitRank)(NcclComm*, int, NcclUid, int) = nullptr;
  int (*CommDestroy)(NcclComm) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  int (*Broadcast)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  int (*Send)(const void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};

// ncclDataType_t / ncclRedOp_t values (nccl.h)
constexpr int kNcclInt32 = 2;
constexpr int kNcclInt64 = 4;
constexpr int kNcclFloat64 = 8;
constexpr int kNcclUint8 = 1;
constexpr int kNcclSum = 0;
constexpr int kNcclMax = 2;

const Nccl& nccl();

}  // namespace nb
