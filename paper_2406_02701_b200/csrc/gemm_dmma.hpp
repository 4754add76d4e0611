// Host interface of the FP64 DMMA GEMM (gemm_dmma.cu).
#pragma once

#include "internal.hpp"

namespace mpcr {

// C <- alpha op(A) op(B) + beta C in FP64, column-major (dense or grouped).
// A and B are FP64, or FP16 / FP32 storage widened exactly on load (each at
// its own precision); C is FP64, or FP32 rounded once from the FP64 result
// (FP16 / FP32 operands only, plus FP32 x FP64 for the panel TRSM).
struct DmmaArgs {
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
    mp_precision pin = MP_DOUBLE;  // operand storage precision (A, and B unless pin_b is set)
    bool exclusive = false;        // reserve the SM (latency-critical launches)
    int ksplit = 1;                // K split over a thread-block cluster (set by the launcher)
    int pin_b = -1;                // B storage precision when it differs from A's (-1: pin)
    mp_precision pout = MP_DOUBLE;  // C storage: FP64, or FP32 (rounded once from FP64, RNE)
    // op(B)[k][n] == 0 for k > n (B = L^T of a lower-triangular L, the TRSM
    // as X = A L^-T): each CTA stops its K loop at its last column
    bool k_tri = false;
    // lower-triangular operand (TRTRI levels): 1 = op(B)[k][n] == 0 for k < n
    // (each CTA starts its K loop at its first column), 2 = op(A)[m][k] == 0
    // for k > m (each CTA stops at its last row).  The skipped products are
    // exact zeros.
    int k_lower = 0;
    // The launcher may split K over a cluster when a launch leaves SMs idle;
    // that changes the summation order with the launch's problem COUNT, so
    // the scheduler's update and tail-TRSM lists (whose counts differ between
    // a single-GPU and a distributed run) turn it off: a tile's result then
    // depends only on its own operands.
    bool allow_ksplit = true;
};

void launch_dmma_gemm(Ctx* ctx, cudaStream_t s, const DmmaArgs& g, int64_t count);

}  // namespace mpcr
