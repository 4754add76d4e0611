// EXPERIMENT (not built into the library): the direct head-tile solve tried in
// round 2 to take TRTRI off the critical chain.  Wired
// into tile.cpp (head tile solved with L_kk and POTRF's leaf inverses, TRTRI
// moved to the lookahead stream) it made the chain slower, 1121 vs 1085 us per
// step at n = 131072, and the bench 1.5 % slower (tools/r02_gpu32.sh): each of
// the 64 CTAs streams all of L through one cp.async chunk in flight, so the
// solve is L2-latency bound (~190 us vs the inverse-based GEMM's ~100 us).
// Retried after the lookahead stream started updating the next head tile
// first (so the TRTRI path no longer waits for whole columns) and with three
// L chunks in flight: chain 1060 vs 1070 us per step, but the bench 1.8 %
// slower (TRTRI on the lookahead stream competes with the bulk; the solve
// itself ~300 us in situ; tools/r02_gpu37.sh).  A version worth wiring in
// needs the rows of a tile split over a cluster sharing L by multicast.
// Direct panel solve of the head tile: X = A L^-T with L the freshly factored
// diagonal tile (lower, FP64) and the 64 x 64 inverses of its diagonal blocks
// that POTRF leaves on the diagonal of the Linv workspace.
//
// Why: the head tile (k+1, k) feeds the SYRK that the next POTRF waits for.
// Solving it through the full inverse puts TRTRI (eight dependent GEMM
// launches) on the critical chain; solving it directly needs only the leaf
// inverses, so TRTRI moves to the lookahead stream, next to the tail TRSM
// that still uses it (tile.cpp).
//
// Blocked by 64 columns: X_j = (A_j - X_{<j} L_{j,<j}^T) Linv_jj^T.  Rows are
// independent: one CTA (4 warps, FP64 DMMA m16n8k8) owns 16 rows of the tile
// and walks the column blocks in order, keeping its X rows in shared memory.
// L chunks and the leaf inverse are staged by cp.async (double-buffered).
#include <cstdint>
#include <type_traits>

#include "device.cuh"
#include "internal.hpp"

namespace mpcr {
namespace {

constexpr int TH_ROWS = 16, TH_BLK = 64, TH_KC = 32, TH_P = 68;  // TH_P: staged pitch (doubles)

__device__ __forceinline__ void th_cp16(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void th_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void th_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void th_mma(double (&d)[4], const double (&a)[4], const double (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ double th_widen(uint16_t h) { return h2d(h); }
__device__ __forceinline__ double th_widen(float f) { return static_cast<double>(f); }
__device__ __forceinline__ double th_widen(double d) { return d; }
__device__ __forceinline__ void th_store(uint16_t* p, double v) { *p = d2h(v); }
__device__ __forceinline__ void th_store(float* p, double v) { *p = static_cast<float>(v); }
__device__ __forceinline__ void th_store(double* p, double v) { *p = v; }

// Stage rows [r0, r0 + 64) x columns [c0, c0 + kc) of column-major M (ld) as
// S[c][r] (pitch TH_P): column c's 64 rows are contiguous in both.
__device__ __forceinline__ void th_stage(double* S, const double* M, int64_t ld, int r0, int c0, int kc) {
    for (int e = threadIdx.x; e < kc * (TH_BLK / 2); e += blockDim.x) {
        const int c = e / (TH_BLK / 2), q = e % (TH_BLK / 2);
        th_cp16(S + c * TH_P + 2 * q, M + static_cast<int64_t>(c0 + c) * ld + r0 + 2 * q);
    }
}

template <typename TI>
__global__ void __launch_bounds__(128) trsm_head_kernel(const TI* __restrict__ A, TI* __restrict__ X,
                                                        const double* __restrict__ L,
                                                        const double* __restrict__ Linv, int nb) {
    extern __shared__ __align__(16) double th_sm[];
    const int XP = nb + 4;  // row pitch of the X rows (== 4 mod 16 doubles: conflict-light fragments)
    double* Xs = th_sm;                     // [16][XP]
    double* Ls = Xs + TH_ROWS * XP;         // [2][TH_KC][TH_P]
    double* Is = Ls + 2 * TH_KC * TH_P;     // [64][TH_P]: Linv_jj staged as [col][row]
    double* Ys = Is + TH_BLK * TH_P;        // [16][TH_P]
    const int r0 = blockIdx.x * TH_ROWS;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int g = lane / 4, t = lane % 4;
    const int nbw = 16 * warp;  // this warp's 16 columns of a 64-column block
    const int nblk = nb / TH_BLK;
    for (int j = 0; j < nblk; ++j) {
        const int j0 = j * TH_BLK;
        // the leaf inverse of block j (its own cp.async group, waited before the multiply)
        th_stage(Is, Linv + static_cast<int64_t>(j0) * nb + j0, nb, 0, 0, TH_BLK);
        th_commit();
        // acc = A[rows, j-block] (c fragment: row g + 8 v1, column 2 t + v0 of each n8 tile)
        double acc[2][4];
#pragma unroll
        for (int n8 = 0; n8 < 2; ++n8)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int rr = g + 8 * (v >> 1), cc = j0 + nbw + 8 * n8 + 2 * t + (v & 1);
                acc[n8][v] = th_widen(A[static_cast<int64_t>(cc) * nb + r0 + rr]);
            }
        // acc -= X[rows, 0:j0] L[j-block, 0:j0]^T, K in chunks of TH_KC
        const int nch = j0 / TH_KC;
        if (nch > 0) {
            th_stage(Ls, L + j0, nb, 0, 0, TH_KC);  // L[j0 + n][k] for k in [0, TH_KC)
            th_commit();
        }
        for (int ch = 0; ch < nch; ++ch) {
            if (ch + 1 < nch) {
                th_stage(Ls + ((ch + 1) & 1) * TH_KC * TH_P, L + j0, nb, 0, (ch + 1) * TH_KC, TH_KC);
                th_commit();
                th_wait<1>();
            } else {
                th_wait<0>();
            }
            __syncthreads();
            const double* lc = Ls + (ch & 1) * TH_KC * TH_P;
            const int kc0 = ch * TH_KC;
#pragma unroll
            for (int ks = 0; ks < TH_KC; ks += 8) {
                double a[4];
#pragma unroll
                for (int v = 0; v < 4; ++v)  // a[v] = X[g + 8 (v & 1)][k = t + 4 (v >> 1)]
                    a[v] = Xs[(g + 8 * (v & 1)) * XP + kc0 + ks + t + 4 * (v >> 1)];
#pragma unroll
                for (int n8 = 0; n8 < 2; ++n8) {
                    double b[2];
#pragma unroll
                    for (int v = 0; v < 2; ++v)  // b[v] = -L[j0 + n][k]: n = nbw + 8 n8 + g, k = t + 4 v
                        b[v] = -lc[(ks + t + 4 * v) * TH_P + nbw + 8 * n8 + g];
                    th_mma(acc[n8], a, b);
                }
            }
            __syncthreads();  // the buffer is restaged two chunks later
        }
        if (nch == 0) th_wait<0>();
        // Y = acc -> shared (row-major), then X_j = Y Linv_jj^T
#pragma unroll
        for (int n8 = 0; n8 < 2; ++n8)
#pragma unroll
            for (int v = 0; v < 4; ++v)
                Ys[(g + 8 * (v >> 1)) * TH_P + nbw + 8 * n8 + 2 * t + (v & 1)] = acc[n8][v];
        __syncthreads();
        double out[2][4] = {};
#pragma unroll
        for (int ks = 0; ks < TH_BLK; ks += 8) {
            double a[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) a[v] = Ys[(g + 8 * (v & 1)) * TH_P + ks + t + 4 * (v >> 1)];
#pragma unroll
            for (int n8 = 0; n8 < 2; ++n8) {
                double b[2];
#pragma unroll
                for (int v = 0; v < 2; ++v)  // b[v] = Linv_jj[n][k]: staged [col k][row n]
                    b[v] = Is[(ks + t + 4 * v) * TH_P + nbw + 8 * n8 + g];
                th_mma(out[n8], a, b);
            }
        }
        // X_j: shared (FP64, for the later blocks) and the output tile (rounded once)
#pragma unroll
        for (int n8 = 0; n8 < 2; ++n8)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int rr = g + 8 * (v >> 1), cc = j0 + nbw + 8 * n8 + 2 * t + (v & 1);
                Xs[rr * XP + cc] = out[n8][v];
                th_store(&X[static_cast<int64_t>(cc) * nb + r0 + rr], out[n8][v]);
            }
        __syncthreads();  // Xs, Ys and Is are read / rewritten by the next block
    }
}

}  // namespace

bool trsm_head_supported(int64_t nb) { return nb % TH_BLK == 0 && nb >= TH_BLK && nb <= 1024; }

void launch_trsm_head(Ctx* ctx, cudaStream_t s, mp_precision p, const void* A, void* X, const double* L,
                      const double* Linv, int64_t nb) {
    if (!trsm_head_supported(nb)) fail(MP_INVALID_PARAM, "trsm_head: nb must be a multiple of 64, <= 1024");
    const int smem = static_cast<int>((TH_ROWS * (nb + 4) + 2 * TH_KC * TH_P + TH_BLK * TH_P + TH_ROWS * TH_P) *
                                      sizeof(double));
    ProfScope ps(ctx, MP_PROF_TRSM, s, static_cast<double>(nb) * nb * nb);
    const dim3 grid(static_cast<unsigned>(nb / TH_ROWS));
    const int n = static_cast<int>(nb);
    static unsigned long long cfg[3] = {0, 0, 0};  // per-device bitmask per precision
    auto go = [&](auto* a, auto* x, const void* kfn) {
        if (first_on_device(cfg[p])) MP_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        using T = std::remove_const_t<std::remove_pointer_t<decltype(a)>>;
        trsm_head_kernel<T><<<grid, 128, smem, s>>>(a, x, L, Linv, n);
    };
    if (p == MP_HALF)
        go(static_cast<const uint16_t*>(A), static_cast<uint16_t*>(X), (const void*)trsm_head_kernel<uint16_t>);
    else if (p == MP_SINGLE)
        go(static_cast<const float*>(A), static_cast<float*>(X), (const void*)trsm_head_kernel<float>);
    else
        go(static_cast<const double*>(A), static_cast<double*>(X), (const void*)trsm_head_kernel<double>);
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

}  // namespace mpcr
