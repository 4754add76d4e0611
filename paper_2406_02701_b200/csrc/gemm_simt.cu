// SIMT GEMM for every (A, B, C) precision combination and transpose flag —
// linalg::gemm semantics (linalg.cpp:316-357): operands widened exactly to the
// compute type of C (float for Half/Single, double for Double), alpha/beta
// cast to it, beta == 0 never reads C, result rounded to C's precision.
//
// 64x64 CTA tile, 16-deep K slab staged through shared memory in the compute
// type, 256 threads with a 4x4 register tile each.  blockIdx.z indexes the
// problem of a grouped launch (the MPCRTile scheduler's FP32/FP64 tiles).
#include <type_traits>

#include "device.cuh"
#include "gemm_simt.hpp"
#include "internal.hpp"

namespace mpcr {
namespace {

constexpr int TM = 64, TN = 64, TK = 16, NT = 256;

template <typename TA, typename TB, typename TC>
__global__ void __launch_bounds__(NT) gemm_simt_kernel(SimtArgs g) {
    using Acc = typename std::conditional<std::is_same<TC, double>::value, double, float>::type;
    const TileProblem pr = g.problems ? g.problems[blockIdx.z]
                                      : TileProblem{g.A, g.B, g.C, g.lower_only ? 1 : 0, 0};
    const int64_t m0 = static_cast<int64_t>(blockIdx.x) * TM;
    const int64_t n0 = static_cast<int64_t>(blockIdx.y) * TN;
    if (pr.lower_only && m0 + TM - 1 < n0) return;
    const TA* __restrict__ A = static_cast<const TA*>(pr.A);
    const TB* __restrict__ B = static_cast<const TB*>(pr.B);
    TC* __restrict__ C = static_cast<TC*>(pr.C);

    __shared__ Acc As[TK][TM + 4];
    __shared__ Acc Bs[TK][TN + 4];
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;
    Acc acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = Acc(0);

    for (int64_t k0 = 0; k0 < g.k; k0 += TK) {
#pragma unroll
        for (int r = 0; r < (TM * TK) / NT; ++r) {
            const int idx = tid + r * NT;
            int mm, kk;
            if (!g.ta) {
                mm = idx % TM;
                kk = idx / TM;
            } else {
                kk = idx % TK;
                mm = idx / TK;
            }
            const int64_t gm = m0 + mm, gk = k0 + kk;
            Acc v = Acc(0);
            if (gm < g.m && gk < g.k)
                v = load_as<Acc>(A, g.ta ? gm * g.lda + gk : gk * g.lda + gm);
            As[kk][mm] = v;
        }
#pragma unroll
        for (int r = 0; r < (TN * TK) / NT; ++r) {
            const int idx = tid + r * NT;
            int nn, kk;
            if (!g.tb) {
                kk = idx % TK;
                nn = idx / TK;
            } else {
                nn = idx % TN;
                kk = idx / TN;
            }
            const int64_t gn = n0 + nn, gk = k0 + kk;
            Acc v = Acc(0);
            if (gn < g.n && gk < g.k)
                v = load_as<Acc>(B, g.tb ? gk * g.ldb + gn : gn * g.ldb + gk);
            Bs[kk][nn] = v;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
            Acc a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][tx + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][ty + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
    const Acc alpha = static_cast<Acc>(g.alpha), beta = static_cast<Acc>(g.beta);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t gn = n0 + ty + 16 * j;
        if (gn >= g.n) continue;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t gm = m0 + tx + 16 * i;
            if (gm >= g.m || (pr.lower_only && gm < gn)) continue;
            const int64_t ci = gn * g.ldc + gm;
            Acc v = alpha * acc[i][j];
            if (beta != Acc(0)) v = v + beta * load_as<Acc>(C, ci);
            store_from(C, ci, v);
        }
    }
}

template <int P>
using ST = typename Storage<P>::T;

template <typename F>
void dispatch_p(mp_precision p, F&& f) {
    if (p == MP_HALF) f(std::integral_constant<int, 0>{});
    else if (p == MP_SINGLE) f(std::integral_constant<int, 1>{});
    else f(std::integral_constant<int, 2>{});
}

}  // namespace

void launch_gemm_simt(Ctx* ctx, cudaStream_t s, const SimtArgs& g, int64_t count) {
    if (g.m == 0 || g.n == 0) return;
    const dim3 grid(static_cast<unsigned>((g.m + TM - 1) / TM),
                    static_cast<unsigned>((g.n + TN - 1) / TN),
                    static_cast<unsigned>(g.problems ? count : 1));
    dispatch_p(g.pa, [&](auto pa) {
        dispatch_p(g.pb, [&](auto pb) {
            dispatch_p(g.pc, [&](auto pc) {
                constexpr int PA = decltype(pa)::value, PB = decltype(pb)::value,
                              PC = decltype(pc)::value;
                gemm_simt_kernel<ST<PA>, ST<PB>, ST<PC>><<<grid, NT, 0, s>>>(g);
            });
        });
    });
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

}  // namespace mpcr
