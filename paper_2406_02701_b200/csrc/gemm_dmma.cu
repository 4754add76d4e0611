// FP64 GEMM on the FP64 tensor path (DMMA, mma.sync m16n8k8 .f64).
//
// tcgen05 has no f64 kind, so FP64 tiles (the diagonal band of the
// mixed-precision Cholesky, its TRTRI, and linalg::gemm with a double C,
// linalg.cpp:349-356) run here.  Measured on B200: DMMA and DFMA both peak
// at 37.1 TFLOP/s (tools/micro/fp64_peak.cu); the SIMT kernel reached 15.5.
//
// CTA tile 128x128, K slab 16, 3-stage cp.async ring in shared memory;
// 16 warps as 4 (m) x 4 (n), warp tile 32x32 = 2 x 4 fragments of 16x8
// (32 FP64 accumulators per thread, 4 warps per scheduler).  Launches that
// would not fill the machine with 128x128 tiles (one SYRK tile on the
// Cholesky critical path, the TRTRI levels) use a 64x64 / 8-warp variant,
// several CTAs per SM.  Shared layouts follow global
// contiguity so every cp.async is 16 bytes; the padded strides make the
// fragment reads conflict-free (2 wavefronts per 256-byte warp load).
// blockIdx.z indexes the problem of a grouped launch; lower_only skips CTA
// tiles strictly above the diagonal and masks the rest (SYRK).
#include <algorithm>
#include <type_traits>

#include "gemm_dmma.hpp"
#include "device.cuh"
#include "internal.hpp"

namespace mpcr {
namespace {

template <int BT>
struct DCfg {
    // warp tile 32 x WTN: 32x32 for the 128 tile (16 warps); 32x16 for the 64
    // tile (8 warps).  The 64 tile serves latency-bound launches (one CTA per
    // SM): a 32-deep K slab keeps twice the bytes in flight per stage.
    static constexpr int WTN = BT == 64 ? 16 : 32;
    static constexpr int BM = BT, NTHR = BT * BT / WTN;
    static constexpr int BK = BT == 64 ? 32 : 16, NST = 3;
    static constexpr int SK_ = BK + 4;  // stride (doubles) of K-contiguous slabs [mn][k]
    static constexpr int SM_ = BT + 4;  // stride of MN-contiguous slabs [k][mn] (== 4 mod 16: conflict-free)
    static constexpr int SLAB = BT * SK_ > BK * SM_ ? BT * SK_ : BK * SM_;  // doubles per operand stage
    static constexpr int SMEM = NST * 2 * SLAB * 8;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int n = valid ? 16 : 0;  // src-size 0 zero-fills
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int n = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void dmma_k8(double (&d)[4], const double (&a)[4], const double (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

// Load one K slab [k0, k0+16) of op(X) rows [r0, r0+128) into smem.
//   mn_contig: X stored with the M/N index contiguous (ld between k) -> [k][mn]
//   else     : K contiguous (ld between m/n)                           -> [mn][k]
template <int BT>
__device__ __forceinline__ void load_slab(double* sm, const double* X, int64_t ldx, bool mn_contig,
                                          int64_t r0, int64_t rmax, int64_t k0, int64_t kmax,
                                          bool vec) {
    using CF = DCfg<BT>;
    constexpr int NTHR = CF::NTHR, SM_ = CF::SM_, SK_ = CF::SK_, BKd = CF::BK, CH = BT * BKd / 2;  // 16-byte chunks
    const int t = threadIdx.x;
    if (mn_contig) {
        // BK k-rows x BT mn
#pragma unroll
        for (int q = 0; q < CH / NTHR; ++q) {
            const int c = t + q * NTHR;
            const int kk = c / (BT / 2), mm = (c % (BT / 2)) * 2;
            const int64_t gk = k0 + kk, gm = r0 + mm;
            double* dst = sm + kk * SM_ + mm;
            if (vec) {
                const bool ok = gk < kmax && gm < rmax;  // rmax even when vec
                cp_async16(dst, ok ? X + gk * ldx + gm : X, ok);
            } else {
                for (int e = 0; e < 2; ++e) {
                    const bool ok = gk < kmax && gm + e < rmax;
                    cp_async8(dst + e, ok ? X + gk * ldx + gm + e : X, ok);
                }
            }
        }
    } else {
        // BT mn rows x BK k
#pragma unroll
        for (int q = 0; q < CH / NTHR; ++q) {
            const int c = t + q * NTHR;
            const int mm = c / (BKd / 2), kk = (c % (BKd / 2)) * 2;
            const int64_t gm = r0 + mm, gk = k0 + kk;
            double* dst = sm + mm * SK_ + kk;
            if (vec) {
                const bool ok = gm < rmax && gk < kmax;  // kmax even when vec
                cp_async16(dst, ok ? X + gm * ldx + gk : X, ok);
            } else {
                for (int e = 0; e < 2; ++e) {
                    const bool ok = gm < rmax && gk + e < kmax;
                    cp_async8(dst + e, ok ? X + gm * ldx + gk + e : X, ok);
                }
            }
        }
    }
}

// Narrow-storage operands (FP16 bits / FP32) are widened to FP64 on the way
// into shared memory (exact), so FP16/FP32 panel tiles feed the FP64 SYRK
// without a converted copy in HBM.  Register-staged: the next slab's global
// loads are in flight while the current slab is multiplied.
template <typename TI>
struct Stage4 {
    TI v[4];
};
__device__ __forceinline__ double widen(uint16_t h) { return h2d(h); }
__device__ __forceinline__ double widen(float f) { return static_cast<double>(f); }

template <int BT, typename TI>
struct NarrowSlab {
    static constexpr int NTHR = DCfg<BT>::NTHR, SM_ = DCfg<BT>::SM_, SK_ = DCfg<BT>::SK_, BKd = DCfg<BT>::BK;
    static constexpr int CH = BT * BKd / 4;  // 4-element chunks per slab
    static constexpr int PER = CH / NTHR;     // chunks per thread
    Stage4<TI> r[PER];

    __device__ __forceinline__ void load(const TI* X, int64_t ldx, bool mn_contig, int64_t r0,
                                         int64_t rmax, int64_t k0, int64_t kmax, bool vec) {
        const int t = threadIdx.x;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int c = t + q * NTHR;
            int mm, kk;
            if (mn_contig) {
                kk = c / (BT / 4);
                mm = (c % (BT / 4)) * 4;
            } else {
                mm = c / (BKd / 4);
                kk = (c % (BKd / 4)) * 4;
            }
            const int64_t gm = r0 + mm, gk = k0 + kk;
            const TI* src = mn_contig ? X + gk * ldx + gm : X + gm * ldx + gk;
            const bool full = mn_contig ? (gk < kmax && gm + 3 < rmax) : (gm < rmax && gk + 3 < kmax);
            if (vec && full) {
                r[q] = *reinterpret_cast<const Stage4<TI>*>(src);
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const bool ok = mn_contig ? (gk < kmax && gm + e < rmax) : (gm < rmax && gk + e < kmax);
                    r[q].v[e] = ok ? src[e] : TI(0);
                }
            }
        }
    }
    __device__ __forceinline__ void store(double* sm, bool mn_contig) const {
        const int t = threadIdx.x;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int c = t + q * NTHR;
            double d[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) d[e] = widen(r[q].v[e]);
            if (mn_contig) {
                const int kk = c / (BT / 4), mm = (c % (BT / 4)) * 4;
                double2* dst = reinterpret_cast<double2*>(sm + kk * SM_ + mm);
                dst[0] = make_double2(d[0], d[1]);
                dst[1] = make_double2(d[2], d[3]);
            } else {
                const int mm = c / (BKd / 4), kk = (c % (BKd / 4)) * 4;
                double2* dst = reinterpret_cast<double2*>(sm + mm * SK_ + kk);
                dst[0] = make_double2(d[0], d[1]);
                dst[1] = make_double2(d[2], d[3]);
            }
        }
    }
};

template <int BT>
__device__ __forceinline__ double sm_get(const double* sm, bool mn_contig, int mn, int k) {
    return mn_contig ? sm[k * DCfg<BT>::SM_ + mn] : sm[mn * DCfg<BT>::SK_ + k];
}

template <int BT, typename TA, typename TB, typename TC>
__global__ void __launch_bounds__(DCfg<BT>::NTHR, BT == 64 ? 2 : 1) dmma_gemm_kernel(DmmaArgs g) {
    using CF = DCfg<BT>;
    constexpr int BMd = BT, BNd = BT, SLAB = CF::SLAB, WTN = CF::WTN, WN = BT / WTN, NJ = WTN / 8;
    constexpr int BKd = CF::BK, NST = CF::NST;
    extern __shared__ __align__(16) double dsm[];
    const TileProblem pr = g.problems ? g.problems[blockIdx.z]
                                      : TileProblem{g.A, g.B, g.C, g.lower_only ? 1 : 0, 0};
    // split K: the S CTAs of a cluster (consecutive blockIdx.x) share one C
    // tile, each takes a K range, and the partial sums meet in the leader's
    // shared memory in rank order (deterministic)
    const int S = g.ksplit;
    const int rank = S > 1 ? static_cast<int>(blockIdx.x % S) : 0;
    const int64_t m0 = static_cast<int64_t>(S > 1 ? blockIdx.x / S : blockIdx.x) * BMd;
    const int64_t n0 = static_cast<int64_t>(blockIdx.y) * BNd;
    if (pr.lower_only && m0 + BMd - 1 < n0) return;  // the whole cluster leaves together
    int64_t kext = g.k_tri ? std::min<int64_t>(g.k, n0 + BNd) : g.k;
    if (g.k_lower == 2) kext = std::min<int64_t>(kext, m0 + BMd);
    const int64_t klo = g.k_lower == 1 ? std::min<int64_t>(kext, n0 / BKd * BKd) : 0;
    const int64_t kchunk = S > 1 ? ((kext - klo + S - 1) / S + BKd - 1) / BKd * BKd : kext - klo;
    const int64_t kbeg = klo + rank * kchunk, kend = std::min<int64_t>(kext, kbeg + kchunk);
    constexpr bool WA = std::is_same<TA, double>::value, WB = std::is_same<TB, double>::value;
    constexpr bool ANY_WIDE = WA || WB;
    const TA* __restrict__ A = static_cast<const TA*>(pr.A);
    const TB* __restrict__ B = static_cast<const TB*>(pr.B);
    TC* __restrict__ C = static_cast<TC*>(pr.C);
    const bool a_mn = !g.ta;  // op(A) = A: M contiguous
    const bool b_mn = g.tb;   // op(B) = B^T: N contiguous
    // vector copies (16 bytes of FP64, 4 narrow elements) need aligned
    // strides/offsets and extents along the contiguous index
    constexpr int VA = WA ? 2 : 4, VB = WB ? 2 : 4;
    const bool va = (g.lda % VA == 0) && ((reinterpret_cast<uintptr_t>(A) & (VA * sizeof(TA) - 1)) == 0) &&
                    (a_mn ? g.m % VA == 0 : g.k % VA == 0);
    const bool vb = (g.ldb % VB == 0) && ((reinterpret_cast<uintptr_t>(B) & (VB * sizeof(TB) - 1)) == 0) &&
                    (b_mn ? g.n % VB == 0 : g.k % VB == 0);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int wm = (warp / WN) * 32, wn = (warp % WN) * WTN;
    const int gq = lane / 4, tq = lane % 4;
    double acc[2][NJ][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;

    const int nk = kend > kbeg ? static_cast<int>((kend - kbeg + BKd - 1) / BKd) : 0;
    auto stage_a = [&](int s) { return dsm + s * 2 * SLAB; };
    auto stage_b = [&](int s) { return dsm + s * 2 * SLAB + SLAB; };
    [[maybe_unused]] NarrowSlab<BT, TA> ra;
    [[maybe_unused]] NarrowSlab<BT, TB> rb;
    auto issue = [&](int kb) {
        const int s = kb % NST;
        const int64_t k0 = kbeg + static_cast<int64_t>(kb) * BKd;
        if constexpr (WA)
            load_slab<BT>(stage_a(s), reinterpret_cast<const double*>(A), g.lda, a_mn, m0, g.m, k0, kend, va);
        else
            ra.load(A, g.lda, a_mn, m0, g.m, k0, kend, va);
        if constexpr (WB)
            load_slab<BT>(stage_b(s), reinterpret_cast<const double*>(B), g.ldb, b_mn, n0, g.n, k0, kend, vb);
        else
            rb.load(B, g.ldb, b_mn, n0, g.n, k0, kend, vb);
    };
    auto land = [&](int kb) {  // narrow operands: registers -> shared (FP64)
        if constexpr (!WA) ra.store(stage_a(kb % NST), a_mn);
        if constexpr (!WB) rb.store(stage_b(kb % NST), b_mn);
    };
#pragma unroll
    for (int s = 0; s < NST - 1; ++s) {
        if (s < nk) {
            issue(s);
            land(s);
        }
        if constexpr (ANY_WIDE) cp_commit();
    }
    for (int kb = 0; kb < nk; ++kb) {
        if constexpr (ANY_WIDE) cp_wait<NST - 2>();
        __syncthreads();
        const bool next = kb + NST - 1 < nk;
        if (next) issue(kb + NST - 1);
        if constexpr (ANY_WIDE) cp_commit();
        const double* sa = stage_a(kb % NST);
        const double* sb = stage_b(kb % NST);
#pragma unroll
        for (int ks = 0; ks < BKd; ks += 8) {
            double af[2][4], bf[NJ][2];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int mr = wm + i * 16 + gq;
#pragma unroll
                for (int v = 0; v < 4; ++v)  // a[v0 + 2 v1] = A[g + 8 v0][t + 4 v1]
                    af[i][v] = sm_get<BT>(sa, a_mn, mr + 8 * (v & 1), ks + tq + 4 * (v >> 1));
            }
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int nc = wn + j * 8 + gq;
#pragma unroll
                for (int v = 0; v < 2; ++v)  // b[v] = B[k = t + 4 v][n = g]
                    bf[j][v] = sm_get<BT>(sb, b_mn, nc, ks + tq + 4 * v);
            }
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < NJ; ++j) dmma_k8(acc[i][j], af[i], bf[j]);
        }
        if (next) land(kb + NST - 1);
    }
    if constexpr (ANY_WIDE) cp_wait<0>();
    if (S > 1) {
        // every CTA's stages are free once all have left the main loop
        asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
        constexpr int E = 2 * NJ * 4;  // accumulators per thread
        if (rank != 0) {
            const uint32_t local = static_cast<uint32_t>(
                __cvta_generic_to_shared(dsm + ((rank - 1) * CF::NTHR + threadIdx.x) * E));
            uint32_t remote;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(0));
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < NJ; ++j)
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(remote + 8 * ((i * NJ + j) * 4 + v)),
                                     "d"(acc[i][j][v])
                                     : "memory");
        }
        asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (rank != 0) return;
        for (int r = 1; r < S; ++r) {
            const double* part = dsm + ((r - 1) * CF::NTHR + threadIdx.x) * E;
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < NJ; ++j)
#pragma unroll
                    for (int v = 0; v < 4; ++v) acc[i][j][v] += part[(i * NJ + j) * 4 + v];
        }
    }
    // epilogue: c[v0 + 2 v1] at (g + 8 v1, 2 t + v0).  Per 16-row fragment
    // row i, the 16 C loads are issued before any store (a store may alias a
    // later load, so interleaving them would serialise the misses).
    const double alpha = g.alpha, beta = g.beta;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        double cold[NJ][4];
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int64_t gm = m0 + wm + i * 16 + gq + 8 * (v >> 1);
                const int64_t gn = n0 + wn + j * 8 + 2 * tq + (v & 1);
                const bool ok = gm < g.m && gn < g.n && !(pr.lower_only && gm < gn);
                cold[j][v] = (ok && beta != 0.0) ? static_cast<double>(C[gn * g.ldc + gm]) : 0.0;
            }
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int64_t gm = m0 + wm + i * 16 + gq + 8 * (v >> 1);
                const int64_t gn = n0 + wn + j * 8 + 2 * tq + (v & 1);
                if (gm < g.m && gn < g.n && !(pr.lower_only && gm < gn)) {
                    double r = alpha * acc[i][j][v];
                    if (beta != 0.0) r += beta * cold[j][v];
                    if constexpr (std::is_same<TC, double>::value)
                        C[gn * g.ldc + gm] = r;
                    else
                        C[gn * g.ldc + gm] = d2f(r);  // one rounding of the FP64 result
                }
            }
    }
}


template <int BT, typename TA, typename TB, typename TC>
void launch_bt(Ctx* ctx, cudaStream_t s, const DmmaArgs& g, int64_t count) {
    using CF = DCfg<BT>;
    static unsigned long long configured = 0;  // per-device bitmask
    if (first_on_device(configured)) {
        MP_CUDA(cudaFuncSetAttribute(dmma_gemm_kernel<BT, TA, TB, TC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     std::max(CF::SMEM, 160 * 1024)));
    }
    const int smem = g.exclusive ? std::max(CF::SMEM, 160 * 1024) : CF::SMEM;
    const unsigned S = static_cast<unsigned>(std::max(1, g.ksplit));
    const dim3 grid(static_cast<unsigned>((g.m + BT - 1) / BT) * S, static_cast<unsigned>((g.n + BT - 1) / BT),
                    static_cast<unsigned>(g.problems ? count : 1));
    if (S == 1) {
        dmma_gemm_kernel<BT, TA, TB, TC><<<grid, CF::NTHR, smem, s>>>(g);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(CF::NTHR);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = S;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    MP_CUDA(cudaLaunchKernelEx(&cfg, dmma_gemm_kernel<BT, TA, TB, TC>, g));
}

template <typename TA, typename TB, typename TC>
void launch_ti(Ctx* ctx, cudaStream_t s, const DmmaArgs& g, int64_t count, bool small) {
    if (small)
        launch_bt<64, TA, TB, TC>(ctx, s, g, count);
    else
        launch_bt<128, TA, TB, TC>(ctx, s, g, count);
}

}  // namespace

void launch_dmma_gemm(Ctx* ctx, cudaStream_t s, const DmmaArgs& g, int64_t count) {
    if (g.m == 0 || g.n == 0) return;
    // CTAs (at/below the diagonal for SYRK) a 128x128 launch would have
    const int64_t nprob = g.problems ? count : 1;
    const int64_t tm = (g.m + 127) / 128, tn = (g.n + 127) / 128;
    const int64_t ctas = nprob * (g.lower_only ? tm * (tn + 1) / 2 : tm * tn);  // lists live on the device
    // (k_tri: the K work per CTA shrinks, the CTA count does not)
    const bool small = ctas < ctx->sm_count;
    DmmaArgs h = g;
    h.ksplit = 1;
    if (small && g.allow_ksplit) {
        // latency-bound launches (TRTRI levels): split K over a cluster while
        // the 64x64 tiles leave most SMs idle, keeping >= 2 slabs per CTA
        const int64_t t64m = (g.m + 63) / 64, t64n = (g.n + 63) / 64;
        const int64_t c64 = nprob * (g.lower_only ? t64m * (t64n + 1) / 2 : t64m * t64n);
        for (int sp = 4; sp >= 2; sp /= 2)
            if (c64 * sp <= ctx->sm_count && g.k >= 64LL * sp) {
                h.ksplit = sp;
                break;
            }
    }
    const mp_precision pa = g.pin, pb = g.pin_b < 0 ? g.pin : static_cast<mp_precision>(g.pin_b);
    // storage type per precision: FP16 bits, float, double
    auto with_b = [&](auto ta, auto tc) {
        using TA = decltype(ta);
        using TC = decltype(tc);
        if (pb == MP_HALF)
            launch_ti<TA, uint16_t, TC>(ctx, s, h, count, small);
        else if (pb == MP_SINGLE)
            launch_ti<TA, float, TC>(ctx, s, h, count, small);
        else
            launch_ti<TA, double, TC>(ctx, s, h, count, small);
    };
    if (g.pout == MP_SINGLE) {
        if (pa == MP_SINGLE && pb == MP_DOUBLE)  // FP32 panel tile x FP64 inverse (TRSM)
            launch_ti<float, double, float>(ctx, s, h, count, small);
        else if (pa == MP_DOUBLE || pb == MP_DOUBLE)
            fail(MP_INTERNAL_ERROR, "dmma: FP32 output with an FP64 A operand is not built");
        else if (pa == MP_HALF)
            pb == MP_HALF ? launch_ti<uint16_t, uint16_t, float>(ctx, s, h, count, small)
                          : launch_ti<uint16_t, float, float>(ctx, s, h, count, small);
        else
            pb == MP_HALF ? launch_ti<float, uint16_t, float>(ctx, s, h, count, small)
                          : launch_ti<float, float, float>(ctx, s, h, count, small);
    } else if (g.pout == MP_DOUBLE) {
        if (pa == MP_HALF)
            with_b(uint16_t{}, double{});
        else if (pa == MP_SINGLE)
            with_b(float{}, double{});
        else
            with_b(double{}, double{});
    } else {
        fail(MP_INTERNAL_ERROR, "dmma: FP16 output is not built");
    }
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

}  // namespace mpcr
