#include "nccl_dl.h"

#include <dlfcn.h>

#include <mutex>

namespace nb {

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    n.GetUniqueId = reinterpret_cast<int (*)(NcclUid*)>(sym("ncclGetUniqueId"));
    n.CommInitRank = reinterpret_cast<int (*)(NcclComm*, int, NcclUid, int)>(sym("ncclCommInitRank"));
    n.CommDestroy = reinterpret_cast<int (*)(NcclComm)>(sym("ncclCommDestroy"));
    n.AllReduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t)>(
        sym("ncclAllReduce"));
    n.Broadcast = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t)>(
        sym("ncclBroadcast"));
    n.Send = reinterpret_cast<int (*)(const void*, size_t, int, int, NcclComm, cudaStream_t)>(sym("ncclSend"));
    n.Recv = reinterpret_cast<int (*)(void*, size_t, int, int, NcclComm, cudaStream_t)>(sym("ncclRecv"));
    n.GroupStart = reinterpret_cast<int (*)()>(sym("ncclGroupStart"));
    n.GroupEnd = reinterpret_cast<int (*)()>(sym("ncclGroupEnd"));
    n.GetErrorString = reinterpret_cast<const char* (*)(int)>(sym("ncclGetErrorString"));
    n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.AllReduce && n.Broadcast && n.Send &&
           n.Recv && n.GroupStart && n.GroupEnd && n.GetErrorString;
    if (!n.ok) n.err = "libnccl.so.2 is missing required symbols";
  });
  return n;
}

}  // namespace nb
