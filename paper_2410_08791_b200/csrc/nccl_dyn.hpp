// nccl_dyn.hpp — NCCL resolved at first use with dlopen instead of a link-time dependency.
//
// The executor shares its process with PyTorch, which ships its own libnccl.so.2 (2.28.x)
// while the system has 2.27.x; both have the same SONAME, so a link-time NEEDED entry would
// make whichever loads first win and break the other. Resolving lazily lets us bind to the
// NCCL already in the process (torch's) when there is one, else torch's bundled copy, else the
// system library. The C API used here is stable across these versions.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

namespace sp {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                  ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
    bool ok() const {
        return GetUniqueId && CommInitRank && CommDestroy && AllReduce && AllGather &&
               ReduceScatter && GetErrorString;
    }
};

inline const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        const char* candidates[] = {
            "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2",
            "libnccl.so.2", "libnccl.so"};
        for (const char* c : candidates) {
            if (h) break;
            h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
        }
        if (!h) {
            api.error = "libnccl.so.2 not found";
            return;
        }
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(h, "ncclAllGather"));
        api.ReduceScatter =
            reinterpret_cast<decltype(api.ReduceScatter)>(dlsym(h, "ncclReduceScatter"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
        if (!api.ok()) api.error = "libnccl.so.2 lacks required symbols";
    });
    return api;
}

}  // namespace sp
