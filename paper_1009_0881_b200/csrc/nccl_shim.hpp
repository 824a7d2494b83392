// nccl_shim.hpp -- NCCL loaded at run time (dlopen), so the single-GPU library
// has no hard NCCL dependency.  Resolves "libnccl.so.2" (the copy torch already
// loaded, if any) or the path baked in at build time (MLB_NCCL_PATH).
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <stdexcept>
#include <string>

namespace mlb {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;

  static NcclApi& get() {
    static NcclApi api;
    static bool loaded = false;
    if (!loaded) {
      // Single-node framework: bootstrap over loopback unless the user chose an
      // interface.  (On the GPU pool's boxes NCCL's default interface pick
      // fails its bootstrap -- "remote process exited or there was a network
      // error" -- while NVLink/P2P carries the data either way.)
      setenv("NCCL_SOCKET_IFNAME", "lo", 0);
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
#ifdef MLB_NCCL_PATH
      if (!h) h = dlopen(MLB_NCCL_PATH, RTLD_NOW | RTLD_GLOBAL);
#endif
      if (!h) throw std::runtime_error(std::string("NCCL not loadable: ") + dlerror());
      auto sym = [&](const char* n) {
        void* p = dlsym(h, n);
        if (!p) throw std::runtime_error(std::string("NCCL symbol missing: ") + n);
        return p;
      };
      api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
      api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
      api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
      api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
      api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
      api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
      api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
      loaded = true;
    }
    return api;
  }
};

inline void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw std::runtime_error(std::string("NCCL ") + what + ": " + NcclApi::get().GetErrorString(r));
}

}  // namespace mlb
