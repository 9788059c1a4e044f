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

// Data a predecessor kernel writes must be read after pdl_wait() with
// COHERENT loads (__ldcg / ld.global), never ld.global.nc (__ldg, or a plain
// load through a const __restrict__ pointer): ptxas treats .nc loads as
// reading memory that is invariant for the whole kernel and may schedule
// them above griddepcontrol.wait (observed: a v[perm] load issued before the
// wait; scripts/sass_pdl_check.py lists the .nc loads that precede the wait
// in every kernel, which must all be plan data). launder() additionally
// hides a pointer's value from the compiler, so address arithmetic on it
// cannot be hoisted either.
template <typename T>
__device__ __forceinline__ T* launder(T* p) {
    asm volatile("" : "+l"(p));
    return p;
}

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
