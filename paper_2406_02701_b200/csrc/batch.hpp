// Host interface of the batched tile kernels (batch.cu).
#pragma once

#include "internal.hpp"

namespace mpcr {

struct CopyItem {
    const void* src;
    void* dst;
};

void launch_batched_convert(Ctx* ctx, cudaStream_t s, mp_precision pin, mp_precision pout,
                            const CopyItem* dev_items, int64_t count, int64_t elems);
void launch_batched_zero(Ctx* ctx, cudaStream_t s, mp_precision p, void* const* dev_ptrs,
                         int64_t count, int64_t elems, bool upper_only, int64_t nb);
struct SplitItem {
    const void* src;
    void* hi;
    void* lo;
};
// 3xTF32 operand split (hi = tf32(x), lo = tf32(x - hi)) of a column-major
// half/single rows x cols block into packed FP32 hi/lo buffers (ld = rows),
// or their transposes (ld = cols) when `trans`.
void launch_split_tf32(Ctx* ctx, cudaStream_t s, mp_precision pin, const void* src, int64_t lds,
                       int64_t rows, int64_t cols, float* hi, float* lo, bool trans);
// Same for a list of contiguous nb x nb FP32 tiles, always transposed.
void launch_batched_split_tf32_t(Ctx* ctx, cudaStream_t s, const SplitItem* dev_items, int64_t count,
                                 int64_t nb);
// hi/lo FP16 split of an FP64 array (hi + lo carries ~22 significant bits).
void launch_split_f16(Ctx* ctx, cudaStream_t s, const double* x, uint16_t* hi, uint16_t* lo,
                      int64_t n);
// Leaf (64x64 diagonal block) inverses of a lower-triangular FP64 matrix,
// written onto the diagonal blocks of Linv.
void launch_leaf_inverse(Ctx* ctx, cudaStream_t s, const double* L, int64_t ldl, int64_t n,
                         double* Linv, int64_t ldi);

// Row gather for mp_tile_get_rows: item q copies row `row` (0-based within
// the tile) of one nb x nb column-major tile of precision `prec`, widened to
// double, into dst[c * ldd] for c < nb.
struct RowItem {
    const void* tile;
    double* dst;
    int32_t row;
    int32_t prec;
};
void launch_gather_rows(Ctx* ctx, cudaStream_t s, const RowItem* dev_items, int64_t count, int64_t nb,
                        int64_t ldd);

}  // namespace mpcr
