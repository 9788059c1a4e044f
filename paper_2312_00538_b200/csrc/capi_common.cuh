// Shared host-side plumbing of the C ABI (nfft_capi.cu, saddle.cu): error
// reporting (status codes of include/ksvm_nfft.h, thread-local message),
// device buffers, the current-device guard, the launch counter.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <cstdint>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ksvm_nfft.h"

namespace ksvm_nfft {

inline std::string& last_error_ref() {  // ksvm_nfft_last_error()
    thread_local std::string msg = "ok";
    return msg;
}

inline std::atomic<int64_t>& launch_counter() {  // ksvm_nfft_launch_count()
    static std::atomic<int64_t> count{0};
    return count;
}

struct DomainErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}
#define CK(x) ::ksvm_nfft::ck((x), #x)

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return KSVM_NFFT_OK;
    } catch (const DomainErr& e) {
        last_error_ref() = e.what();
        return KSVM_NFFT_ERR_DATA;
    } catch (const std::invalid_argument& e) {
        last_error_ref() = e.what();
        return KSVM_NFFT_ERR_CONFIG;
    } catch (const std::bad_alloc&) {
        last_error_ref() = "out of memory";
        return KSVM_NFFT_ERR_INTERNAL;
    } catch (const std::exception& e) {
        last_error_ref() = e.what();
        return KSVM_NFFT_ERR_INTERNAL;
    }
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
        o.p = nullptr;
        o.n = 0;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            reset();
            p = o.p;
            n = o.n;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    ~DevBuf() { reset(); }
    void reset() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void alloc(size_t count) {
        reset();
        if (count == 0) count = 1;
        CK(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    void upload(const T* h, size_t count, cudaStream_t st) {
        alloc(count);
        CK(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, st));
    }
};

// NVTX range (header-only NVTX3; a no-op unless a profiler such as Nsight
// Systems is attached). The apply path brackets each stage - spread_dK
// (spread, tile pre-reduction, node reduction), grid_dK (the convolution
// stages), gather_dK, combine - and the host-pointer copies (h2d / d2h), so a
// timeline shows the per-stage host enqueue and, under graph replay, the
// apply as one range. Stage GPU times: ksvm_nfft_op_set_stage_timing.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        CK(cudaGetDevice(&prev));
        if (prev != dev) CK(cudaSetDevice(dev));
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

// Exact kernel entries of an operator's window (or of the whole ANOVA
// kernel), for the preconditioner factorizations (lowrank.cu): the raw
// feature columns on the device plus the per-window weights (< 0: plain
// WindowOperator entry) and squared length scales. Filled by op_entry_view
// (nfft_capi.cu); `mu` / `stream` are the operator's.
struct EntryView {
    int device = 0;
    cudaStream_t stream = nullptr;
    std::mutex* mu = nullptr;
    int64_t n = 0;
    int nw = 0;
    const double* const* cols = nullptr;  // device: the windows' feature columns, in window order
    const int* wdim = nullptr;            // device: dimension of each of the nw windows
    std::vector<double> wgt, ell2;        // host, nw entries
};

}  // namespace ksvm_nfft
