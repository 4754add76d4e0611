// Host interface of the tcgen05 FP16 GEMM (gemm_tc.cu).
#pragma once

#include <cuda.h>

#include <cstdint>

#include "internal.hpp"

namespace mpcr {

// One problem of a grouped launch: tiles are indices into the third TMA
// dimension of the A, B and C slabs.
struct TcProblem {
    int32_t a_tile;
    int32_t b_tile;
    int32_t c_tile;
    int32_t lower_only;  // skip / keep C strictly above the diagonal
};

// C <- alpha op(A) op(B) + beta C with FP16 A, B and half/single C, or
// 3xTF32-split FP32 A, B and single C.
// Dense: *_tiles = 1, problems = nullptr.  Grouped: A, B and C are slabs of
// `*_tiles` column-major tiles `*_tile_stride` elements apart.
struct TcGemm {
    int kind = 0;  // 0: FP16 operands (kind::f16), 1: FP32 operands via TF32 (kind::tf32)
    mp_precision pc = MP_HALF;
    bool ta = false, tb = false;
    int64_t m = 0, n = 0, k = 0;
    double alpha = 1.0, beta = 0.0;
    const void* A = nullptr;
    int64_t lda = 0, a_tiles = 1, a_tile_stride = 0;
    const void* B = nullptr;
    int64_t ldb = 0, b_tiles = 1, b_tile_stride = 0;
    void* C = nullptr;
    int64_t ldc = 0, c_tiles = 1, c_tile_stride = 0;
    bool lower_only = false;
    const TcProblem* problems = nullptr;
    int64_t count = 0;
    // Optional lo parts, concatenated along K into one FP32 accumulator:
    //   kind 0, B2 only : C = alpha A (B + B2) + beta C   (split FP64 inverse)
    //   kind 1, A2 + B2 : 3xTF32, C = alpha (A B + A B2 + A2 B) + beta C
    // (A2/B2 share the layout, tiles and strides of A/B).
    const void* A2 = nullptr;
    const void* B2 = nullptr;
    // 0: fully persistent (one CTA per SM).  > 0: at most this many output
    // tiles per CTA, so SMs are handed back at that granularity and kernels
    // of a higher-priority stream (the Cholesky critical path) get in.
    int tiles_per_cta = 0;
    // op(B)[k][n] == 0 for k > n (B^T of a lower-triangular inverse: the
    // panel TRSM): a unit stops its K loop at its last column
    bool k_tri = false;
    // kind 0 with A2 and B2: C = alpha (A B + A2 B2) + beta C, the two K
    // segments in that order (two Cholesky steps' panels in one pass over C)
    bool two_panels = false;
};

bool tc_gemm_supported(const TcGemm& g);

// 3-D TMA map over [d2][d1][d0] elements (d0 contiguous, rows ld_elems
// apart, d2 slices tile_stride_elems apart), boxes of box0 x box1.
void tma_map_3d(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int esize, uint64_t d0,
                uint64_t d1, uint64_t d2, uint64_t ld_elems, uint64_t tile_stride_elems, uint32_t box0,
                uint32_t box1, CUtensorMapSwizzle swz);
void launch_tc_gemm(Ctx* ctx, cudaStream_t s, const TcGemm& g);

}  // namespace mpcr
