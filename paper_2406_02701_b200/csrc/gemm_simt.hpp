// Host interface of the SIMT GEMM (gemm_simt.cu).
#pragma once

#include "internal.hpp"

namespace mpcr {

struct SimtArgs {
    mp_precision pa, pb, pc;
    bool ta, tb;
    int64_t m, n, k;
    double alpha, beta;
    const void* A;
    int64_t lda;
    const void* B;
    int64_t ldb;
    void* C;
    int64_t ldc;
    bool lower_only;
    const TileProblem* problems;  // grouped launch when non-null
};

void launch_gemm_simt(Ctx* ctx, cudaStream_t s, const SimtArgs& g, int64_t count);

}  // namespace mpcr
