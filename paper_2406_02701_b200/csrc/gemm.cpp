// GEMM dispatch: picks the kernel family from the precisions
// (linalg.cpp:340 branches on compute_precision(prec(C))).
//   A, B half and C half/single  -> tcgen05 FP16 tensor cores (gemm_tc.cu)
//   C single, A/B not double     -> 3xTF32 on tcgen05
//   A, B half and C double       -> exact INT8 digit products (ozaki.cu)
//   all double                   -> DMMA (gemm_dmma.cu)
//   everything else              -> SIMT in C's compute type (gemm_simt.cu)
#include <algorithm>
#include <cstdlib>

#include "batch.hpp"
#include "gemm_dmma.hpp"
#include "gemm_simt.hpp"
#include "gemm_tc.hpp"
#include "internal.hpp"
#include "ozaki.hpp"

namespace mpcr {

bool ozaki_enabled() {
    static const bool on = [] {
        const char* e = getenv("MPCR_OZAKI");
        return !(e && e[0] == '0');
    }();
    return on;
}

// FP16 x FP16 -> FP64: exact 7-bit digit slicing + INT8 tensor cores (ozaki.cu).
static void launch_gemm_ozaki(Ctx* ctx, cudaStream_t s, const GemmDesc& g) {
    const int64_t kpad = (g.k + 15) / 16 * 16;
    const size_t sa = static_cast<size_t>(g.m) * kpad, sb = static_cast<size_t>(g.n) * kpad;
    const size_t dig = OZ_SLICES * (sa + sb);
    const size_t items_off = (dig + 255) / 256 * 256;
    const size_t rexp_off = items_off + 256;
    const int64_t mbk = (g.m + 127) / 128, nbk = (g.n + 127) / 128;  // digit counts per 128-row block
    char* w = static_cast<char*>(ctx->ensure_scratch(rexp_off + (g.m + g.n + mbk + nbk) * 4 + 256, 2));
    int8_t* da = reinterpret_cast<int8_t*>(w);
    int8_t* db = da + OZ_SLICES * sa;
    int32_t* ea = reinterpret_cast<int32_t*>(w + rexp_off);
    int32_t* eb = ea + g.m;
    int32_t* nd = eb + g.n;  // digits needed by the row blocks of A, then of B
    // op(A)(r = m, c = k); op(B)^T(r = n, c = k).  trans: element (r, c) at x[r * ld + c]
    OzSliceItem it[2] = {
        {g.A, da, ea, nd, g.lda, g.m, g.k, kpad, static_cast<int64_t>(sa), g.ta ? 1 : 0, 0},
        {g.B, db, eb, nd + mbk, g.ldb, g.n, g.k, kpad, static_cast<int64_t>(sb), g.tb ? 0 : 1, 0}};
    OzSliceItem* dit = reinterpret_cast<OzSliceItem*>(w + items_off);
    MP_CUDA(cudaMemcpyAsync(dit, it, sizeof(it), cudaMemcpyHostToDevice, s));
    launch_oz_slices(ctx, s, dit, 2, std::max(g.m, g.n), kpad);
    OzGemm o;
    o.A = da;
    o.B = db;
    o.a_slice_stride = static_cast<int64_t>(sa);
    o.b_slice_stride = static_cast<int64_t>(sb);
    o.kpad = kpad;
    o.m = g.m;
    o.n = g.n;
    o.k = g.k;
    o.C = g.C;
    o.ldc = g.ldc;
    o.alpha = g.alpha;
    o.beta = g.beta;
    o.lower_only = g.lower_only;
    o.rexp_a = ea;
    o.rexp_b = eb;
    o.ndig_a = nd;
    o.ndig_b = nd + mbk;
    launch_oz_gemm(ctx, s, o);
}

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
    if (g.pa == MP_HALF && g.pb == MP_HALF && g.pc == MP_DOUBLE && g.k > 0 && ozaki_enabled()) {
        // The int32 digit-group sums are exact while 6 pairs * K * 64^2 < 2^31
        // (K < 87381): longer contractions run in K chunks of OZ_MAX_K, each
        // chunk's FP64 result accumulated into C (beta applies once).
        for (int64_t k0 = 0; k0 < g.k; k0 += OZ_MAX_K) {
            GemmDesc c = g;
            c.k = std::min<int64_t>(OZ_MAX_K, g.k - k0);
            // op(A) columns / op(B) rows k0 .. k0 + c.k (elements of 2 bytes)
            c.A = static_cast<const uint16_t*>(g.A) + (g.ta ? k0 : k0 * g.lda);
            c.B = static_cast<const uint16_t*>(g.B) + (g.tb ? k0 * g.ldb : k0);
            if (k0 > 0) c.beta = 1.0;
            launch_gemm_ozaki(ctx, s, c);
        }
        return;
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
                   nullptr, g.ldb, nullptr, g.ldc, false, g.problems, g.pab, g.exclusive};
        d.k_lower = g.k_lower;
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
