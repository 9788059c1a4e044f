// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// Minimal FFTW3 API shim so the reference's own hot-path translation unit
// (/root/reference/proj/src/fastsum.cpp, compiled unmodified by path via
// oracle/Makefile) builds without libfftw3, which is absent from this image
// (SURVEY.md F5). Only the eight symbols fastsum.cpp uses are provided
// (P:src/fastsum.cpp:22-28, 161-172, 201-207, 273, 282); the arithmetic is
// oracle/offt.hpp's exact DFT.
#ifndef KSVM_ORACLE_FFTW3_SHIM_H
#define KSVM_ORACLE_FFTW3_SHIM_H

#include <cstdlib>
#include <vector>

#include "../offt.hpp"

typedef double fftw_complex[2];

struct fftw_plan_s {
    offt::PlanND plan;
    fftw_complex* in;
    fftw_complex* out;
};
typedef fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_ESTIMATE (1U << 6)
#define FFTW_PRESERVE_INPUT (1U << 4)

inline fftw_complex* fftw_alloc_complex(std::size_t n) {
    return static_cast<fftw_complex*>(std::malloc(sizeof(fftw_complex) * (n ? n : 1)));
}

inline void fftw_free(void* p) { std::free(p); }

inline fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex* in,
                               fftw_complex* out, int sign, unsigned /*flags*/) {
    std::vector<int> dims(n, n + rank);
    return new fftw_plan_s{offt::PlanND(dims, sign), in, out};
}

inline void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
    p->plan.execute(reinterpret_cast<const offt::cd*>(in), reinterpret_cast<offt::cd*>(out));
}

inline void fftw_execute(const fftw_plan p) { fftw_execute_dft(p, p->in, p->out); }

inline void fftw_destroy_plan(fftw_plan p) { delete p; }

#endif
