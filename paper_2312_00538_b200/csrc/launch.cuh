// Programmatic dependent launch (PDL) for the apply-path and saddle-solver
// kernels. Every kernel launched with launch_k lets its stream successor
// start at once (pdl_trigger), does its plan-only prologue (items, DWin, tile
// tables: immutable during an apply), and waits for its predecessor's
// results (pdl_wait) before touching any buffer an earlier kernel writes or
// reads. Every CTA waits before it exits, so grid completion stays
// transitive along the stream. KSVM_NFFT_PDL=0 launches without the
// attribute (the waits are then no-ops).
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>

namespace ksvm_nfft {

__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

inline bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("KSVM_NFFT_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <typename... KArgs, typename... Args>
void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    (void)cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);  // errors: cudaGetLastError
}

}  // namespace ksvm_nfft
