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

// L2 eviction-priority hints. Per apply the plan streams (window factors,
// cell codes: 40 B per point per window) are read once, while v (spread:
// gathered through each window's sort permutation) and the per-window
// outputs (gather: scattered through it) are touched in 8-byte pieces of
// 32-byte sectors by every window: streaming the plan data evict-first and
// keeping v / the outputs evict-last lets them stay in the 126 MB L2 instead
// of being re-fetched (or read-for-ownership) sector by sector.
__device__ __forceinline__ unsigned long long l2_evict_first() {
    unsigned long long p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long l2_evict_last() {
    unsigned long long p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// read-only plan data (may be issued before griddepcontrol.wait)
__device__ __forceinline__ double2 ld_plan(const double2* p, unsigned long long pol) {
    double2 r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
        : "=d"(r.x), "=d"(r.y) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ int2 ld_plan(const int2* p, unsigned long long pol) {
    int2 r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;"
        : "=r"(r.x), "=r"(r.y) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ float4 ld_plan(const float4* p, unsigned long long pol) {
    float4 r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
        : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p), "l"(pol));
    return r;
}
// coherent L2 load of data a predecessor kernel may have written (after pdl_wait)
__device__ __forceinline__ double ld_keep(const double* p, unsigned long long pol) {
    double r;
    asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol) : "memory");
    return r;
}
__device__ __forceinline__ void st_keep(double* p, double v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
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
