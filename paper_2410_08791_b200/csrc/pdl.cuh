// pdl.cuh — programmatic dependent launch (PDL) for the compute stream's kernel chain.
//
// Each kernel is launched with cudaLaunchAttributeProgrammaticStreamSerialization, so the next
// kernel in the stream can be launched — and run its prologue (barrier init, TMEM allocation,
// tensor-map prefetch) on SMs the previous kernel's tail has already freed — before the
// previous kernel completes. Every kernel executes griddepcontrol.wait before its first global
// memory access that could depend on (or conflict with) the previous kernel, which blocks until
// that kernel has completed and its memory is visible; then griddepcontrol.launch_dependents
// lets the following kernel launch. In a kernel launched without the attribute both are no-ops.
// Off by default: measured on B200 it did not pay (C2 train step 19.1-19.2 ms without vs
// 19.6-20.1 ms with; C4 and small-layer inference unchanged within noise) — the early-launched
// dependents hold SM slots the GEMMs and the update stream need. SP_PDL=1 turns it on.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace sp {

__device__ __forceinline__ void pdl_wait_then_release() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SP_PDL");
        return e && e[0] == '1';
    }();
    return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace sp
