// Cholesky (POTRF), triangular inverse (TRTRI) and triangular solve kernels.
//
// POTRF: one cooperative launch per matrix/tile.  Right-looking, 64-wide
// blocks; per block step three phases separated by a grid barrier:
//   1. CTA 0 factors the 64x64 diagonal block in shared memory (checking the
//      pivots exactly like chol_kernel's `!(d > 0)`, linalg.cpp:121) and
//      inverts it (kept in `dinv` for the panel and for TRTRI);
//   2. panel rows below: X = A_panel * inv(L_kk)^T, one 64-row block per CTA;
//   3. trailing SYRK/GEMM update of the lower triangle, 64x64 blocks.
// The failing pivot is reported as the 0-based column (errors.hpp:25-31);
// every CTA stops at the next barrier.
//
// TRTRI: recursive 2x2 block inverse inv([[A,0],[B,C]]) = [[A^-1,0],
// [-C^-1 B A^-1, C^-1]] on top of POTRF's 64x64 leaf inverses, each level one
// grouped FP64 GEMM pair.  The MPCRTile scheduler turns the panel TRSM into a
// tensor-core GEMM with this inverse (see tile.cpp).
#include <cooperative_groups.h>

#include <algorithm>

#include <type_traits>
#include <cstdlib>
#include <vector>

#include "batch.hpp"
#include "device.cuh"
#include "internal.hpp"

namespace mpcr {
namespace {

constexpr int PB = 64;   // block size
constexpr int PT = 256;  // threads per CTA

struct GridBar {
    unsigned int count;
    unsigned int gen;
};

// Optional per-step clock trace of CTA 0 (MPCR_POTRF_TRACE=1, diagnostics).
__device__ int g_trace_on = 0;
__device__ long long g_trace[64 * 6];

#define PTRACE(kb, slot)                                                             \
    do {                                                                             \
        if (g_trace_on && blockIdx.x == 0 && threadIdx.x == 0 && (kb) < 64)          \
            g_trace[(kb) * 6 + (slot)] = clock64();                                  \
    } while (0)

__device__ __forceinline__ void grid_sync(GridBar* bar, unsigned int nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned int* vgen = &bar->gen;
        const unsigned int g = *vgen;
        __threadfence();
        if (atomicAdd(&bar->count, 1u) == nblocks - 1) {
            atomicExch(&bar->count, 0u);
            __threadfence();
            atomicAdd(&bar->gen, 1u);
        } else {
            while (*vgen == g) __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
}

// Arrive at a grid barrier without waiting for it (the CTA's prior global
// stores are published first).
__device__ __forceinline__ void grid_arrive(GridBar* bar, unsigned int nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&bar->count, 1u) == nblocks - 1) {
            atomicExch(&bar->count, 0u);
            __threadfence();
            atomicAdd(&bar->gen, 1u);
        }
    }
}

// acc(64x64 per CTA, 4x4 per thread) += P (64 x kk, ldp) * Q (64 x kk, ldq)^T
// with P/Q rows limited to pr/qr valid rows.  16-wide K slabs; the next
// slab's global loads are in flight (registers) while the current one is
// multiplied from shared memory.
template <typename T>
__device__ __forceinline__ void block_nt(T (&acc)[4][4], const T* P, int64_t ldp, int pr,
                                         const T* Q, int64_t ldq, int qr, int kk,
                                         T (*Ps)[PB + 1], T (*Qs)[PB + 1]) {
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    constexpr int PER = 16 * PB / PT;  // elements of each operand per thread and slab
    T pa[PER], qa[PER];
    auto gload = [&](int k0) {
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int idx = threadIdx.x + q * PT;
            const int r = idx % PB, k = k0 + idx / PB;
            pa[q] = (r < pr && k < kk) ? P[k * ldp + r] : T(0);
            qa[q] = (r < qr && k < kk) ? Q[k * ldq + r] : T(0);
        }
    };
    auto sstore = [&]() {
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int idx = threadIdx.x + q * PT;
            Ps[idx / PB][idx % PB] = pa[q];
            Qs[idx / PB][idx % PB] = qa[q];
        }
    };
    const int nk = (kk + 15) / 16;
    if (nk == 0) return;
    gload(0);
    sstore();
    __syncthreads();
    for (int sl = 0; sl < nk; ++sl) {
        const bool more = sl + 1 < nk;
        if (more) gload((sl + 1) * 16);
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            T a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = Ps[c][tx + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Qs[c][ty + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
        if (more) {
            sstore();
            __syncthreads();
        }
    }
}

#include "potrf_block.cuh"

// ---- FP64 trailing-update block on DMMA (mma.sync m16n8k8 .f64) ----
constexpr int US = 68;  // stride of the [k][row] operand slabs: conflict-free fragment loads

__device__ __forceinline__ void pcp_async16(void* smem, const void* gmem, bool valid) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void pcp_async8(void* smem, const void* gmem, bool valid) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(gmem), "r"(valid ? 8 : 0)
                 : "memory");
}

// Stage rows [r0, r0 + 64) x columns [k0, k0 + 64) of column-major A into
// U[k][row] (zero past `rows`), asynchronously.
__device__ __forceinline__ void stage_panel(double* U, const double* A, int64_t lda, int r0, int rows, int k0,
                                            bool vec) {
    for (int q = threadIdx.x; q < PB * (PB / 2); q += PT) {
        const int k = q / (PB / 2), rp = 2 * (q % (PB / 2));
        const double* src = A + (int64_t)(k0 + k) * lda + r0 + rp;
        double* dst = U + k * US + rp;
        if (vec && rp + 1 < rows) {
            pcp_async16(dst, src, true);
        } else {
            pcp_async8(dst, src, rp < rows);
            pcp_async8(dst + 1, src + 1, rp + 1 < rows);
        }
    }
}

// Stage the two panel blocks of trailing-update block (ib, jb) into U (two
// [k][row] slabs), asynchronously (one cp.async group).
__device__ __forceinline__ void stage_item(const double* A, int64_t lda, int n, int k0, int ib, int jb, double* U) {
    const bool vec = (lda % 2) == 0;
    stage_panel(U, A, lda, ib * PB, min(PB, n - ib * PB), k0, vec);
    stage_panel(U + PB * US, A, lda, jb * PB, min(PB, n - jb * PB), k0, vec);
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// C(r0.., c0..) -= P_i P_j^T for the 64 x 64 block (lower triangle only when
// ib == jb) from the slabs in U (staged by stage_item; `more`: one later
// group is still in flight).  8 warps, each a 32 x 16 tile of 2 x 2
// m16n8k8 fragments.
__device__ void update_block_dmma(double* A, int64_t lda, int n, int ib, int jb, const double* U, bool more) {
    const int r0 = ib * PB, c0 = jb * PB, rb = min(PB, n - r0), cb = min(PB, n - c0);
    const double* Pi = U;
    const double* Pj = U + PB * US;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, g = lane / 4, t = lane % 4;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
    // old values of this thread's fragment elements, loaded while the slabs land
    double old[2][2][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int r = wm + 16 * i + g + 8 * (v >> 1), c = wn + 8 * j + 2 * t + (v & 1);
                const bool ok = r < rb && c < cb && (ib != jb || r >= c);
                old[i][j][v] = ok ? A[(int64_t)(c0 + c) * lda + r0 + r] : 0.0;
            }
    double acc[2][2][4] = {};
    if (more)
        asm volatile("cp.async.wait_group 1;" ::: "memory");
    else
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < PB; ks += 8) {
        double af[2][4], bf[2][2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int v = 0; v < 4; ++v)  // a[v0 + 2 v1] = P_i[g + 8 v0][t + 4 v1]
                af[i][v] = Pi[(ks + t + 4 * (v >> 1)) * US + wm + 16 * i + g + 8 * (v & 1)];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int v = 0; v < 2; ++v)  // b[v] = P_j[n = g][k = t + 4 v]
                bf[j][v] = Pj[(ks + t + 4 * v) * US + wn + 8 * j + g];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j)
                asm volatile(
                    "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                    "{%0,%1,%2,%3};"
                    : "+d"(acc[i][j][0]), "+d"(acc[i][j][1]), "+d"(acc[i][j][2]), "+d"(acc[i][j][3])
                    : "d"(af[i][0]), "d"(af[i][1]), "d"(af[i][2]), "d"(af[i][3]), "d"(bf[j][0]), "d"(bf[j][1]));
    }
    // c[v0 + 2 v1] at (g + 8 v1, 2 t + v0)
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int r = wm + 16 * i + g + 8 * (v >> 1), c = wn + 8 * j + 2 * t + (v & 1);
                if (r < rb && c < cb && (ib != jb || r >= c))
                    A[(int64_t)(c0 + c) * lda + r0 + r] = old[i][j][v] - acc[i][j][v];
            }
    __syncthreads();  // this buffer is restaged two blocks later
}

// Factor the diagonal block kb held in D (lower, zeros above, identity
// padding; potrf_block.cuh): L_kk stays in D and goes to A, the inverses of
// its 16 x 16 diagonal pieces stay in Xs and go to xd (the other CTAs' panel
// solves read them).  Returns false (after flagging) on a failed pivot.
template <typename T>
__device__ bool diag_factor_store(T* A, int64_t lda, int n, int kb, T* xd, int64_t* info, int64_t info_off,
                                  int* abort_flag, T (*D)[PB + 1], T* Xs, int* s_fail) {
    const int k0 = kb * PB, bb = min(PB, n - k0);
    __shared__ T s_inv[PB];  // reciprocals of the pivots
    const int fail = factor_block_diag(D, Xs, s_fail, s_inv);
    if (fail >= 0 && fail < bb) {
        if (threadIdx.x == 0) {
            if (*info < 0) *info = info_off + k0 + fail;
            atomicExch(abort_flag, 1);
        }
        return false;
    }
    for (int idx = threadIdx.x; idx < bb * bb; idx += PT) {
        const int r = idx % bb, c = idx / bb;
        if (r >= c) A[(int64_t)(k0 + c) * lda + k0 + r] = D[r][c];
    }
    T* xk = xd + (int64_t)kb * 4 * 256;
    for (int idx = threadIdx.x; idx < 4 * 256; idx += PT) xk[idx] = Xs[idx];
    return true;
}

// Load L_kk (lower, zeros above) into Ls and its diagonal-piece inverses into Xs.
template <typename T>
__device__ void load_lkk(const T* A, int64_t lda, int n, int kb, const T* xd, T (*Ls)[PB + 1], T* Xs) {
    const int k0 = kb * PB, bb = min(PB, n - k0);
    for (int idx = threadIdx.x; idx < PB * PB; idx += PT) {
        const int r = idx % PB, c = idx / PB;
        Ls[r][c] = (r < bb && c < bb) ? (r >= c ? A[(int64_t)(k0 + c) * lda + k0 + r] : T(0)) : (r == c ? T(1) : T(0));
    }
    const T* xk = xd + (int64_t)kb * 4 * 256;
    for (int idx = threadIdx.x; idx < 4 * 256; idx += PT) Xs[idx] = xk[idx];
    __syncthreads();
}

// Panel block: As = A_{ib,kb} (rows r0.., zero padded), solved in place
// against L_kk (Ls, Xs) and written back.
template <typename T>
__device__ void panel_block(T* A, int64_t lda, int n, int kb, int ib, T (*As)[PB + 1], const T (*Ls)[PB + 1],
                            const T* Xs) {
    const int k0 = kb * PB, r0 = ib * PB, rb = min(PB, n - r0);
    for (int idx = threadIdx.x; idx < PB * PB; idx += PT) {
        const int r = idx % PB, c = idx / PB;
        As[r][c] = r < rb ? A[(int64_t)(k0 + c) * lda + r0 + r] : T(0);
    }
    __syncthreads();
    trsm_block(As, Ls, Xs);
    for (int idx = threadIdx.x; idx < PB * PB; idx += PT) {
        const int r = idx % PB, c = idx / PB;
        if (r < rb) A[(int64_t)(k0 + c) * lda + r0 + r] = As[r][c];
    }
}

// Full inverse of L_kk (for the TRTRI leaves) into linv_diag.
template <typename T>
__device__ void leaf_inverse(const T* A, int64_t lda, int n, int kb, const T* xd, T* linv_diag, int64_t ldi,
                             T (*Ls)[PB + 1], T* Xs, T (*Xf)[PB + 1], T* Tm) {
    load_lkk(A, lda, n, kb, xd, Ls, Xs);
    dinv_block(Ls, Xs, Xf, Tm);
    const int k0 = kb * PB, bb = min(PB, n - k0);
    for (int idx = threadIdx.x; idx < bb * bb; idx += PT) {
        const int r = idx % bb, c = idx / bb;
        linv_diag[(int64_t)(k0 + c) * ldi + k0 + r] = Xf[r][c];
    }
    __syncthreads();
}

// Shared memory of potrf_coop_kernel, in elements of T.
constexpr int POTRF_SMEM_ELEMS = 2 * PB * (PB + 1) + 4 * 256 + 3 * 256 + 2 * 16 * (PB + 1);
constexpr int POTRF_UPD_ELEMS = 4 * PB * US;  // double-buffered DMMA update slabs (double only)

// Cooperative blocked right-looking POTRF.  Per 64-block step kb:
//   CTA 0     panel block kb+1 = A_{kb+1,kb} L_kk^-T (L_kk and its diagonal
//             piece inverses still in shared memory), published with a
//             non-waiting arrive at barrier 1; then A_{kb+1,kb+1} -= P P^T
//             from shared memory and the factorization of that block: the
//             next step's diagonal work never waits for the other CTAs
//   others    panel blocks kb+2.. (same blocked solve), barrier 1, trailing
//             update of the lower triangle except block (kb+1, kb+1)
//   barrier 2 (all)
template <typename T>
__global__ void __launch_bounds__(PT, 1) potrf_coop_kernel(T* A, int64_t lda, int n, T* xd,
                                                        int64_t* info, int64_t info_off,
                                                        GridBar* bar, GridBar* bar1, int* abort_flag) {
    extern __shared__ __align__(16) unsigned char psm[];
    T* base = reinterpret_cast<T*>(psm);
    T (*D)[PB + 1] = reinterpret_cast<T (*)[PB + 1]>(base);
    T (*As)[PB + 1] = reinterpret_cast<T (*)[PB + 1]>(base + PB * (PB + 1));
    T* Xs = base + 2 * PB * (PB + 1);
    T* Tm = Xs + 4 * 256;
    T (*Ps)[PB + 1] = reinterpret_cast<T (*)[PB + 1]>(Tm + 3 * 256);
    T (*Qs)[PB + 1] = reinterpret_cast<T (*)[PB + 1]>(Tm + 3 * 256 + 16 * (PB + 1));
    // DMMA slabs of the trailing update (double only): two blocks' worth (2 x 2
    // x 64 x US elements) over the whole shared area, which the non-zero CTAs
    // only use for their panel solves before barrier 1
    double* Us = reinterpret_cast<double*>(base);

    __shared__ int s_fail;
    const int nblk = (n + PB - 1) / PB;
    const unsigned int G = gridDim.x;  // >= 2 whenever nblk >= 2
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;

    if (blockIdx.x == 0) {
        const int bb = min(PB, n);
        for (int idx = threadIdx.x; idx < PB * PB; idx += PT) {
            const int r = idx % PB, c = idx / PB;
            D[r][c] = (r < bb && c < bb) ? (r >= c ? A[(int64_t)c * lda + r] : T(0)) : (r == c ? T(1) : T(0));
        }
        __syncthreads();
        diag_factor_store(A, lda, n, 0, xd, info, info_off, abort_flag, D, Xs, &s_fail);
    }
    grid_sync(bar, G);
    if (*(volatile int*)abort_flag) return;
    for (int kb = 0; kb + 1 < nblk; ++kb) {
        const int k0 = kb * PB;  // a full block (not the last one)
        const int rest = nblk - kb - 1;
        PTRACE(kb, 0);
        if (blockIdx.x == 0) {
            const int r0 = k0 + PB, rb = min(PB, n - r0);
            T old[4][4];  // block (kb+1, kb+1), loaded early
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int r = tx + 16 * i, c = ty + 16 * j;
                    old[i][j] = (r < rb && c < rb && r >= c) ? A[(int64_t)(r0 + c) * lda + r0 + r] : T(0);
                }
            panel_block(A, lda, n, kb, kb + 1, As, D, Xs);
            grid_arrive(bar1, G);  // also orders the panel in As before the reads below
            PTRACE(kb, 1);
#pragma unroll 4
            for (int k = 0; k < PB; ++k) {
                T a[4], b[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) a[i] = As[tx + 16 * i][k];
#pragma unroll
                for (int j = 0; j < 4; ++j) b[j] = As[ty + 16 * j][k];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j <= i; ++j) old[i][j] = fma(-a[i], b[j], old[i][j]);  // lower only
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int r = tx + 16 * i, c = ty + 16 * j;
                    D[r][c] = (r < rb && c < rb) ? (r >= c ? old[i][j] : T(0)) : (r == c ? T(1) : T(0));
                }
            __syncthreads();
            PTRACE(kb, 2);
            diag_factor_store(A, lda, n, kb + 1, xd, info, info_off, abort_flag, D, Xs, &s_fail);
            PTRACE(kb, 3);
        } else {
            if (kb + 1 + (int)blockIdx.x < nblk) {
                load_lkk(A, lda, n, kb, xd, D, Xs);
                for (int ib = kb + 1 + blockIdx.x; ib < nblk; ib += G - 1) {
                    panel_block(A, lda, n, kb, ib, As, D, Xs);
                    __syncthreads();
                }
            }
            grid_sync(bar1, G);
            const int items = rest * (rest + 1) / 2;  // item 0 is (kb+1, kb+1): CTA 0's
            auto item_blocks = [&](int it, int& ib, int& jb) {
                int jj = 0, rem = it;
                while (rem >= rest - jj) {
                    rem -= rest - jj;
                    ++jj;
                }
                jb = kb + 1 + jj;
                ib = jb + rem;
            };
            if constexpr (std::is_same<T, double>::value) {
                // DMMA blocks, the next block's slabs staged while this one runs
                int q = 0;
                if (static_cast<int>(blockIdx.x) < items) {
                    int ib, jb;
                    item_blocks(blockIdx.x, ib, jb);
                    stage_item(A, lda, n, k0, ib, jb, Us);
                }
                for (int it = blockIdx.x; it < items; it += G - 1, ++q) {
                    const int nx = it + G - 1;
                    const bool more = nx < items;
                    if (more) {
                        int ib2, jb2;
                        item_blocks(nx, ib2, jb2);
                        stage_item(A, lda, n, k0, ib2, jb2, Us + ((q + 1) & 1) * 2 * PB * US);
                    }
                    int ib, jb;
                    item_blocks(it, ib, jb);
                    update_block_dmma(A, lda, n, ib, jb, Us + (q & 1) * 2 * PB * US, more);
                }
            }
            for (int it = blockIdx.x; !std::is_same<T, double>::value && it < items; it += G - 1) {
                int ib, jb;
                item_blocks(it, ib, jb);
                const int r0 = ib * PB, c0 = jb * PB;
                const int rb = min(PB, n - r0), cb = min(PB, n - c0);
                {
                    // the block's old values are loaded while block_nt runs (no aliasing
                    // with its reads: different columns), all before any store
                    T old[4][4];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int r = tx + 16 * i, c = ty + 16 * j;
                            old[i][j] = (r < rb && c < cb) ? A[(int64_t)(c0 + c) * lda + r0 + r] : T(0);
                        }
                    T acc[4][4] = {};
                    block_nt(acc, A + (int64_t)k0 * lda + r0, lda, rb, A + (int64_t)k0 * lda + c0, lda, cb, PB, Ps,
                             Qs);
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int r = tx + 16 * i, c = ty + 16 * j;
                            if (r < rb && c < cb && (ib != jb || r >= c))
                                A[(int64_t)(c0 + c) * lda + r0 + r] = old[i][j] - acc[i][j];
                        }
                    __syncthreads();
                }
            }
        }
        grid_sync(bar, G);
        PTRACE(kb, 4);
        if (*(volatile int*)abort_flag) return;
    }
}

// The full inverses of the diagonal blocks (TRTRI leaves), one CTA per block,
// from L and the diagonal-piece inverses the factorization left in xd.
__global__ void __launch_bounds__(PT, 1) leaf_inverse_kernel(const double* A, int64_t lda, int n, const double* xd,
                                                             double* linv_diag, int64_t ldi) {
    extern __shared__ __align__(16) unsigned char psm[];
    double* base = reinterpret_cast<double*>(psm);
    double (*Ls)[PB + 1] = reinterpret_cast<double (*)[PB + 1]>(base);
    double (*Xf)[PB + 1] = reinterpret_cast<double (*)[PB + 1]>(base + PB * (PB + 1));
    double* Xs = base + 2 * PB * (PB + 1);
    double* Tm = Xs + 4 * 256;
    leaf_inverse(A, lda, n, blockIdx.x, xd, linv_diag, ldi, Ls, Xs, Xf, Tm);
}

// ---- triangular solve (linalg.cpp:130-159), one thread per RHS vector ----
// Left:  op(T) x = alpha b for every column of B (rows n).
// Right: x op(T) = alpha b for every row of B, i.e. op(T)^T x^T = alpha b^T.
template <typename TT, typename TB, typename Acc>
__global__ void tri_solve_kernel(const TT* __restrict__ Tm, int64_t ldt, int64_t n, bool upper,
                                 bool trans, TB* __restrict__ B, int64_t ldb, int64_t nvec,
                                 Acc alpha, bool right) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= nvec) return;
    // element k of vector v
    auto bidx = [&](int64_t k) { return right ? k * ldb + v : v * ldb + k; };
    const bool tr = right ? !trans : trans;
    auto coef = [&](int64_t i, int64_t k) {
        return load_as<Acc>(Tm, tr ? i * ldt + k : k * ldt + i);
    };
    const bool eff_lower = (upper == tr);
    if (eff_lower) {
        for (int64_t i = 0; i < n; ++i) {
            Acc acc = load_as<Acc>(B, bidx(i)) * alpha;
            for (int64_t k = 0; k < i; ++k) acc -= coef(i, k) * load_as<Acc>(B, bidx(k));
            store_from(B, bidx(i), acc / coef(i, i));
        }
    } else {
        for (int64_t i = n; i-- > 0;) {
            Acc acc = load_as<Acc>(B, bidx(i)) * alpha;
            for (int64_t k = i + 1; k < n; ++k) acc -= coef(i, k) * load_as<Acc>(B, bidx(k));
            store_from(B, bidx(i), acc / coef(i, i));
        }
    }
}

template <typename TT, typename Acc>
__global__ void zero_diag_kernel(const TT* __restrict__ Tm, int64_t ldt, int64_t n,
                                 unsigned long long* first) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        if (load_as<Acc>(Tm, i * ldt + i) == Acc(0)) atomicMin(first, (unsigned long long)i);
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

void launch_potrf_lower(Ctx* ctx, cudaStream_t s, mp_precision p, void* A, int64_t lda,
                        int64_t n, int64_t* dev_info, int64_t info_offset, double* linv_diag,
                        int64_t ldi) {
    if (p == MP_HALF) fail(MP_INVALID_PARAM, "potrf: half storage must be widened first");
    if (n == 0) return;
    const int nblk = static_cast<int>((n + PB - 1) / PB);
    // scratch: barrier + abort flag + leaf inverses (kept for TRTRI)
    const size_t elem = p == MP_DOUBLE ? 8 : 4;
    const size_t dinv_bytes = static_cast<size_t>(nblk) * PB * PB * elem;
    char* scr = static_cast<char*>(ctx->ensure_scratch(256 + dinv_bytes, 1));
    MP_CUDA(cudaMemsetAsync(scr, 0, 256, s));
    GridBar* bar = reinterpret_cast<GridBar*>(scr);
    GridBar* bar1 = reinterpret_cast<GridBar*>(scr + 128);
    int* abort_flag = reinterpret_cast<int*>(scr + 64);
    void* dinv = scr + 256;
    // Few CTAs: the step is latency-bound (diagonal work on CTA 0 overlaps
    // the trailing update of the others); fewer CTAs make the grid barrier
    // cheaper.  MPCR_POTRF_CTAS overrides for tuning.
    static const int cap = [] {
        const char* e = getenv("MPCR_POTRF_CTAS");
        return e ? atoi(e) : 24;
    }();
    int grid = nblk * (nblk + 1) / 2;
    if (grid > cap) grid = cap;
    if (grid > ctx->sm_count) grid = ctx->sm_count;
    if (grid < 2) grid = nblk >= 2 ? 2 : 1;  // CTA 0's diagonal path needs a partner
    int ni = static_cast<int>(n);
    ProfScope ps(ctx, MP_PROF_POTRF, s, static_cast<double>(n) * n * n / 3.0);
    if (p == MP_DOUBLE) {
        static unsigned long long cfg = 0;  // per-device bitmask
        // The factorization is latency-bound: by default each CTA reserves
        // most of its SM's shared memory so no other kernel's CTAs share the
        // SM with it (MPCR_POTRF_EXCLUSIVE=0 turns this off).
        static const bool exclusive = [] {
            const char* e = getenv("MPCR_POTRF_EXCLUSIVE");
            return !(e && e[0] == '0');
        }();
        const size_t shm_need = std::max(POTRF_SMEM_ELEMS, POTRF_UPD_ELEMS) * sizeof(double);
        const size_t shm = exclusive ? std::max<size_t>(shm_need, 160 * 1024) : shm_need;
        if (first_on_device(cfg)) {
            MP_CUDA(cudaFuncSetAttribute((void*)potrf_coop_kernel<double>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
        }
        double* a = static_cast<double*>(A);
        double* d = static_cast<double*>(dinv);
        void* args[] = {&a, &lda, &ni, &d, &dev_info, &info_offset, &bar, &bar1, &abort_flag};
        static const bool trace = getenv("MPCR_POTRF_TRACE") != nullptr;
        if (trace) {
            const int on = 1;
            MP_CUDA(cudaMemcpyToSymbolAsync(g_trace_on, &on, sizeof(on), 0, cudaMemcpyHostToDevice, s));
        }
        MP_CUDA(cudaLaunchCooperativeKernel((void*)potrf_coop_kernel<double>, grid, PT, args, shm, s));
        if (linv_diag) {
            static unsigned long long cfg_l = 0;  // per-device bitmask
            const size_t shm_l = (2 * PB * (PB + 1) + 4 * 256 + 3 * 256) * sizeof(double);
            if (first_on_device(cfg_l)) {
                MP_CUDA(cudaFuncSetAttribute((void*)leaf_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)shm_l));
            }
            leaf_inverse_kernel<<<nblk, PT, shm_l, s>>>(a, lda, ni, d, linv_diag, ldi);
            count_launch(ctx);
        }
        if (trace) {
            long long tr[64 * 6];
            MP_CUDA(cudaMemcpyFromSymbolAsync(tr, g_trace, sizeof(tr), 0, cudaMemcpyDeviceToHost, s));
            MP_CUDA(cudaStreamSynchronize(s));
            double acc[4] = {};
            for (int kb = 0; kb + 1 < nblk && kb < 64; ++kb)
                for (int q = 0; q < 4; ++q) acc[q] += static_cast<double>(tr[kb * 6 + q + 1] - tr[kb * 6 + q]);
            fprintf(stderr, "potrf trace, CTA 0 (cycles, summed over %d steps): panel block %.0f syrk %.0f "
                    "factor+inverse %.0f barrier %.0f\n", nblk - 1, acc[0], acc[1], acc[2], acc[3]);
        }
    } else {
        const size_t shm = POTRF_SMEM_ELEMS * sizeof(float);
        static unsigned long long cfg_f = 0;  // per-device bitmask
        if (first_on_device(cfg_f)) {
            MP_CUDA(cudaFuncSetAttribute((void*)potrf_coop_kernel<float>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
        }
        float* a = static_cast<float*>(A);
        float* d = static_cast<float*>(dinv);
        void* args[] = {&a, &lda, &ni, &d, &dev_info, &info_offset, &bar, &bar1, &abort_flag};
        MP_CUDA(cudaLaunchCooperativeKernel((void*)potrf_coop_kernel<float>, grid, PT, args, shm, s));
    }
    count_launch(ctx);
}

// TRTRI plan: the recursive 2x2 block inverse inv([[A,0],[B,C]]) =
// [[A^-1,0],[-C^-1 B A^-1, C^-1]] level by level (grouped FP64 GEMMs), with
// every level's problem list uploaded once so a factorization issues its
// TRTRIs without host synchronisation.
struct TrtriPlan {
    const double* L;
    int64_t ldl;
    double* Linv;
    int64_t ldi, n;
    double* T = nullptr;           // workspace (n^2/2 doubles)
    TileProblem* dev = nullptr;    // device problem lists
    struct Rag {
        int64_t r, rows2;
    };
    struct Level {
        int64_t h, cnt;
        size_t off1, off2;
        std::vector<Rag> rag;
    };
    std::vector<Level> levels;
};

TrtriPlan* trtri_plan_create(Ctx* ctx, cudaStream_t s, const double* L, int64_t ldl, double* Linv,
                             int64_t ldi, int64_t n) {
    auto* P = new TrtriPlan{L, ldl, Linv, ldi, n};
    std::vector<TileProblem> all;
    MP_CUDA(cudaMalloc(&P->T, static_cast<size_t>(n) * n / 2 * sizeof(double) + 256));
    for (int64_t sz = 2 * PB; sz / 2 < n; sz *= 2) {
        TrtriPlan::Level lv;
        lv.h = sz / 2;
        const int64_t h = lv.h;
        std::vector<TileProblem> p1, p2;
        int64_t toff = 0;
        for (int64_t r = 0; r + h < n; r += sz) {
            const int64_t rows2 = (n - r - h) < h ? (n - r - h) : h;
            if (rows2 == h) {
                // T = B * Ainv (h x h), Linv21 = -Cinv * T
                p1.push_back(TileProblem{L + r * ldl + r + h, Linv + r * ldi + r, P->T + toff, 0, 0});
                p2.push_back(TileProblem{Linv + (r + h) * ldi + r + h, P->T + toff, Linv + r * ldi + r + h, 0, 0});
                toff += h * h;
            } else {
                lv.rag.push_back({r, rows2});
            }
        }
        lv.cnt = static_cast<int64_t>(p1.size());
        lv.off1 = all.size();
        all.insert(all.end(), p1.begin(), p1.end());
        lv.off2 = all.size();
        all.insert(all.end(), p2.begin(), p2.end());
        P->levels.push_back(lv);
    }
    if (!all.empty()) {
        MP_CUDA(cudaMalloc(&P->dev, all.size() * sizeof(TileProblem)));
        MP_CUDA(cudaMemcpyAsync(P->dev, all.data(), all.size() * sizeof(TileProblem),
                                cudaMemcpyHostToDevice, s));
        MP_CUDA(cudaStreamSynchronize(s));
    }
    return P;
}

void trtri_plan_destroy(TrtriPlan* P) {
    if (!P) return;
    if (P->T) cudaFree(P->T);
    if (P->dev) cudaFree(P->dev);
    delete P;
}

// Linv's strictly-upper part must already be zero; `leaves_done` means the
// 64x64 diagonal inverses were written by the POTRF that produced L.
void launch_trtri_plan(Ctx* ctx, cudaStream_t s, TrtriPlan* P, bool leaves_done) {
    const double* L = P->L;
    double* Linv = P->Linv;
    const int64_t ldl = P->ldl, ldi = P->ldi, n = P->n;
    if (!leaves_done) launch_leaf_inverse(ctx, s, L, ldl, n, Linv, ldi);
    for (const auto& lv : P->levels) {
        const int64_t h = lv.h;
        if (lv.cnt) {
            GroupedGemm g1{MP_DOUBLE, MP_DOUBLE, false, h, h, h, ldl, ldi, h, 1.0, 0.0,
                           P->dev + lv.off1, lv.cnt};
            g1.exclusive = true;  // TRTRI sits on the Cholesky critical path
            g1.k_lower = 1;       // Ainv lower: column block n0 needs K >= n0
            launch_grouped_gemm(ctx, s, g1);
            GroupedGemm g2{MP_DOUBLE, MP_DOUBLE, false, h, h, h, ldi, h, ldi, -1.0, 0.0,
                           P->dev + lv.off2, lv.cnt};
            g2.exclusive = true;
            g2.k_lower = 2;  // Cinv lower: row block m0 needs K < m0 + BM
            launch_grouped_gemm(ctx, s, g2);
        }
        for (const auto& rg : lv.rag) {
            const int64_t r = rg.r, rows2 = rg.rows2;
            GemmDesc g1{MP_DOUBLE, MP_DOUBLE, MP_DOUBLE, false, false, rows2, h, h, 1.0, 0.0,
                        L + r * ldl + r + h, ldl, Linv + r * ldi + r, ldi, P->T, rows2};
            launch_gemm(ctx, s, g1);
            GemmDesc g2{MP_DOUBLE, MP_DOUBLE, MP_DOUBLE, false, false, rows2, h, rows2, -1.0, 0.0,
                        Linv + (r + h) * ldi + r + h, ldi, P->T, rows2, Linv + r * ldi + r + h, ldi};
            launch_gemm(ctx, s, g2);
        }
    }
}

// One-shot inverse (zeroes Linv first).
void launch_trtri_lower(Ctx* ctx, cudaStream_t s, const double* L, int64_t ldl, double* Linv,
                        int64_t ldi, int64_t n) {
    launch_fill(ctx, s, MP_DOUBLE, Linv, ldi, n, n, 0.0);
    TrtriPlan* P = trtri_plan_create(ctx, s, L, ldl, Linv, ldi, n);
    launch_trtri_plan(ctx, s, P, false);
    MP_CUDA(cudaStreamSynchronize(s));
    trtri_plan_destroy(P);
}

void launch_tri_solve(Ctx* ctx, cudaStream_t s, mp_precision pt, const void* T, int64_t ldt,
                      int64_t n, bool upper, bool trans, mp_precision pb, void* B, int64_t ldb,
                      int64_t ncols, double alpha, bool right_side, int64_t brows) {
    const int64_t nvec = right_side ? brows : ncols;
    if (nvec == 0 || n == 0) return;
    const int threads = 128;
    const int grid = static_cast<int>((nvec + threads - 1) / threads);
    ProfScope ps(ctx, MP_PROF_TRSM, s, static_cast<double>(n) * n * nvec);
    dispatch_p(pt, [&](auto ptt) {
        dispatch_p(pb, [&](auto pbb) {
            constexpr int PT_ = decltype(ptt)::value, PB_ = decltype(pbb)::value;
            using Acc = typename std::conditional<PB_ == 2, double, float>::type;
            tri_solve_kernel<ST<PT_>, ST<PB_>, Acc><<<grid, threads, 0, s>>>(
                static_cast<const ST<PT_>*>(T), ldt, n, upper, trans, static_cast<ST<PB_>*>(B),
                ldb, nvec, static_cast<Acc>(alpha), right_side);
        });
    });
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

int64_t find_zero_diag(Ctx* ctx, cudaStream_t s, mp_precision p, const void* T, int64_t ldt,
                       int64_t n, mp_precision compute) {
    auto* first = static_cast<unsigned long long*>(ctx->ensure_scratch(64, 0));
    const unsigned long long init = ~0ull;
    MP_CUDA(cudaMemcpyAsync(first, &init, sizeof(init), cudaMemcpyHostToDevice, s));
    dispatch_p(p, [&](auto pp) {
        constexpr int P = decltype(pp)::value;
        if (compute == MP_DOUBLE)
            zero_diag_kernel<ST<P>, double><<<grid_for(n, 256, ctx->sm_count), 256, 0, s>>>(
                static_cast<const ST<P>*>(T), ldt, n, first);
        else
            zero_diag_kernel<ST<P>, float><<<grid_for(n, 256, ctx->sm_count), 256, 0, s>>>(
                static_cast<const ST<P>*>(T), ldt, n, first);
    });
    count_launch(ctx);
    unsigned long long r = 0;
    MP_CUDA(cudaMemcpyAsync(&r, first, sizeof(r), cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    return r == ~0ull ? -1 : static_cast<int64_t>(r);
}

}  // namespace mpcr
