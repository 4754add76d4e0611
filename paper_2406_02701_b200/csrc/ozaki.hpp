// Host interface of the FP64-from-INT8 (Ozaki) GEMM for FP16-valued operands
// (ozaki.cu).
#pragma once

#include <cstdint>

#include "internal.hpp"

namespace mpcr {

constexpr int OZ_SLICES = 6;  // 6 x 7-bit digits: exact for any FP16 row
// Longest contraction per launch: a digit group sums at most 6 pairs of
// products |d_p d_q| <= 64^2, so its int32 accumulator is exact for
// 6 * K * 2^12 < 2^31, i.e. K < 87381.
constexpr int64_t OZ_MAX_K = 65536;

// One problem of a grouped launch: digit tiles of A and B (indices into the
// slabs), the C tile, lower triangle only (SYRK).  A second pair of digit
// tiles (a_tile2 >= 0) is a second panel accumulated into the same output
// before C is read and written once: C += alpha (A B^T + A2 B2^T).
struct OzProblem {
    int32_t a_tile;
    int32_t b_tile;
    void* c;
    int32_t lower_only;
    int32_t a_tile2 = -1;
    int32_t b_tile2 = -1;
    int32_t pad = 0;
};

// Slice one FP16 matrix (rows x cols, element (r, c) at x[c * ld + r], or
// x[r * ld + c] when trans) into OZ_SLICES int8 digit planes [S][rows][kpad]
// (planes slice_stride bytes apart) and per-row exponents rexp[rows].  The
// number of planes each 128-row block needs (exactness needs only those; the
// others are not written) goes to ndig[block].
struct OzSliceItem {
    const void* x;
    void* out;
    int32_t* rexp;
    int32_t* ndig;  // optional: digits per 128-row block [ceil(rows / 128)] (without it every plane is written)
    int64_t ld, rows, cols, kpad, slice_stride;
    int32_t trans;
    int32_t pad;
};

// C = alpha * A B^T + beta * C with A (m x k), B (n x k) given as digit slabs
// [tiles][S][rows][kpad] and row exponents; C FP64 column-major (ldc).
struct OzGemm {
    const void* A = nullptr;
    const void* B = nullptr;
    int64_t a_tiles = 1, b_tiles = 1;
    int64_t a_slice_stride = 0, b_slice_stride = 0;  // bytes between digit planes
    int64_t kpad = 0;
    int64_t m = 0, n = 0, k = 0;
    void* C = nullptr;
    int64_t ldc = 0;
    double alpha = 1.0, beta = 0.0;
    bool lower_only = false;
    bool c_single = false;  // C is FP32 (else FP64)
    const OzProblem* problems = nullptr;  // device array (grouped) or nullptr
    int64_t count = 0;
    int64_t n_lower = 0;  // grouped: the first n_lower problems are lower_only (the rest are not)
    int64_t n_two = 0;    // grouped: problems with a second panel (profiling work count)
    const int32_t* rexp_a = nullptr;
    const int32_t* rexp_b = nullptr;
    const int32_t* ndig_a = nullptr;  // digits per 128-row block (<= OZ_SLICES), ndig_stride_* blocks per tile
    const int32_t* ndig_b = nullptr;
    int64_t ndig_stride_a = 0, ndig_stride_b = 0;
    int64_t rexp_stride_a = 0, rexp_stride_b = 0;  // between tiles

};

void launch_oz_slices(Ctx* ctx, cudaStream_t s, const OzSliceItem* items, int64_t count, int64_t max_rows,
                      int64_t max_cols);
// FP32 operands (column-major, no transpose, K <= 1024): the same digits,
// exact down to 2^(e_r - 41) of each row (OzSliceItem::x points to floats).
void launch_oz_slices_f32(Ctx* ctx, cudaStream_t s, const OzSliceItem* items, int64_t count, int64_t max_rows,
                          int64_t max_cols);
void launch_oz_gemm(Ctx* ctx, cudaStream_t s, const OzGemm& g);

}  // namespace mpcr
