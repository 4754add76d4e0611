// GEMM dispatch: picks the kernel family from the precisions
// (linalg.cpp:340 branches on compute_precision(prec(C))).
//   A, B half and C half/single  -> tcgen05 FP16 tensor cores (gemm_tc.cu)
//   everything else              -> SIMT in C's compute type (gemm_simt.cu)
#include "batch.hpp"
#include "gemm_dmma.hpp"
#include "gemm_simt.hpp"
#include "gemm_tc.hpp"
#include "internal.hpp"

namespace mpcr {

void launch_gemm(Ctx* ctx, cudaStream_t s, const GemmDesc& g) {
    if (g.m == 0 || g.n == 0) return;
    if (g.pa == MP_HALF && g.pb == MP_HALF && (g.pc == MP_HALF || g.pc == MP_SINGLE) && g.k > 0) {
        TcGemm t;
        t.pc = g.pc;
        t.ta = g.ta;
        t.tb = g.tb;
        t.m = g.m;
        t.n = g.n;
        t.k = g.k;
        t.alpha = g.alpha;
        t.beta = g.beta;
        t.A = g.A;
        t.lda = g.lda;
        t.a_tile_stride = g.lda * (g.ta ? g.m : g.k);
        t.B = g.B;
        t.ldb = g.ldb;
        t.b_tile_stride = g.ldb * (g.tb ? g.k : g.n);
        t.C = g.C;
        t.ldc = g.ldc;
        t.c_tile_stride = g.ldc * g.n;
        t.lower_only = g.lower_only;
        if (tc_gemm_supported(t)) {
            launch_tc_gemm(ctx, s, t);
            return;
        }
    }
    // Single accumulator with half/single operands: 3xTF32 on tcgen05
    // (hi*hi + hi*lo + lo*hi of the TF32 splits), FP32 accumulate.
    if (g.pc == MP_SINGLE && g.pa != MP_DOUBLE && g.pb != MP_DOUBLE && g.k >= 32 &&
        g.m * g.n >= 128 * 256) {
        // kind::tf32 reads both operands K-major: hi/lo of A stored k x m and
        // of B stored k x n (transposing where the input is MN-major).
        const int64_t ar = g.ta ? g.k : g.m, ac = g.ta ? g.m : g.k;
        const int64_t br = g.tb ? g.n : g.k, bc = g.tb ? g.k : g.n;
        const size_t asz = static_cast<size_t>(g.m) * g.k, bsz = static_cast<size_t>(g.k) * g.n;
        float* w = static_cast<float*>(ctx->ensure_scratch((2 * asz + 2 * bsz) * 4 + 256, 2));
        float *ah = w, *al = w + asz, *bh = w + 2 * asz, *bl = w + 2 * asz + bsz;
        launch_split_tf32(ctx, s, g.pa, g.A, g.lda, ar, ac, ah, al, !g.ta);
        launch_split_tf32(ctx, s, g.pb, g.B, g.ldb, br, bc, bh, bl, g.tb);
        TcGemm t;
        t.kind = 1;
        t.pc = MP_SINGLE;
        t.ta = true;   // A^T stored k x m
        t.tb = false;  // B stored k x n
        t.m = g.m;
        t.n = g.n;
        t.k = g.k;
        t.alpha = g.alpha;
        t.beta = g.beta;
        t.A = ah;
        t.A2 = al;
        t.lda = g.k;
        t.a_tile_stride = asz;
        t.B = bh;
        t.B2 = bl;
        t.ldb = g.k;
        t.b_tile_stride = bsz;
        t.C = g.C;
        t.ldc = g.ldc;
        t.c_tile_stride = g.ldc * g.n;
        t.lower_only = g.lower_only;
        if (tc_gemm_supported(t)) {
            launch_tc_gemm(ctx, s, t);
            return;
        }
    }
    if (g.pa == MP_DOUBLE && g.pb == MP_DOUBLE && g.pc == MP_DOUBLE) {
        DmmaArgs d{g.ta, g.tb, g.m, g.n, g.k, g.alpha, g.beta, g.A, g.lda,
                   g.B, g.ldb, g.C, g.ldc, g.lower_only, nullptr};
        ProfScope ps(ctx, MP_PROF_GEMM_F64, s, 2.0 * g.m * g.n * g.k * (g.lower_only ? 0.5 : 1.0));
        launch_dmma_gemm(ctx, s, d, 1);
        return;
    }
    SimtArgs a{g.pa, g.pb, g.pc, g.ta, g.tb, g.m, g.n, g.k, g.alpha, g.beta, g.A, g.lda,
               g.B, g.ldb, g.C, g.ldc, g.lower_only, nullptr};
    const int cls = g.pc == MP_DOUBLE ? MP_PROF_GEMM_F64
                    : (g.pa == MP_HALF && g.pb == MP_HALF) ? MP_PROF_GEMM_F16
                                                            : MP_PROF_GEMM_F32;
    ProfScope ps(ctx, cls, s, 2.0 * g.m * g.n * g.k * (g.lower_only ? 0.5 : 1.0));
    launch_gemm_simt(ctx, s, a, 1);
}

void launch_grouped_gemm(Ctx* ctx, cudaStream_t s, const GroupedGemm& g) {
    if (g.count == 0) return;
    if (g.pc == MP_DOUBLE) {  // FP64 output: DMMA, narrow operands widened on load
        DmmaArgs d{false, g.tb, g.m, g.n, g.k, g.alpha, g.beta, nullptr, g.lda,
                   nullptr, g.ldb, nullptr, g.ldc, false, g.problems, g.pab};
        ProfScope ps(ctx, MP_PROF_GEMM_F64, s, 2.0 * g.m * g.n * g.k * g.count);
        launch_dmma_gemm(ctx, s, d, g.count);
        return;
    }
    SimtArgs a{g.pab, g.pab, g.pc, false, g.tb, g.m, g.n, g.k, g.alpha, g.beta, nullptr, g.lda,
               nullptr, g.ldb, nullptr, g.ldc, false, g.problems};
    const int cls = g.pc == MP_DOUBLE ? MP_PROF_GEMM_F64
                    : g.pab == MP_HALF ? MP_PROF_GEMM_F16 : MP_PROF_GEMM_F32;
    ProfScope ps(ctx, cls, s, 2.0 * g.m * g.n * g.k * g.count);
    launch_gemm_simt(ctx, s, a, g.count);
}

}  // namespace mpcr
