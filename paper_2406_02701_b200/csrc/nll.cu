// Tiled forward solve w = L^{-1} z and the Gaussian negative log-likelihood
// (workloads.cpp:74-87) on a factored mixed-precision MPCRTile.
//
// The right-hand side lives in FP64 on the device; every tile is widened
// exactly to FP64 as it is read, so the solve is at least as accurate as the
// reference's forwardsolve at the factor's precision (workloads.cpp:83).
//   per tile row i:  w_i = L_ii^{-1} r_i      (one CTA, 32-column blocks:
//                                              warp-level substitution + update)
//                    r_j -= L_ji w_i, j > i   (one launch, HBM-bound GEMV)
#include "device.cuh"
#include "internal.hpp"

namespace mpcr {
namespace {

template <int P>
using ST = typename Storage<P>::T;

// In-place lower-triangular solve of one nb x nb tile against r (FP64),
// left-looking over 32-row blocks: the block's rows first take the dot
// products with all solved entries (8 threads per row, all loads of a thread
// independent), then warp 0 substitutes down the 32 x 32 diagonal block (one
// multiply, one shuffle and one FMA on the chain per column).
template <int P>
__global__ void __launch_bounds__(256) tile_trsv_kernel(const ST<P>* __restrict__ L, int64_t ld,
                                                        int nb, double* __restrict__ r) {
    extern __shared__ double wsol[];  // solved entries w[0 .. nb)
    __shared__ double rb[32];
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    for (int b0 = 0; b0 < nb; b0 += 32) {
        const int w = min(32, nb - b0);
        // (1) rb[row] = r[row] - sum_{c < b0} L[row][c] w[c]; thread = (row, part)
        {
            const int row = tid % 32, part = tid / 32;  // 8 parts over the columns
            double s0 = 0.0, s1 = 0.0;
            if (row < w) {
                const int64_t gr = b0 + row;
                int c = part;
                for (; c + 8 < b0; c += 16) {
                    s0 = fma(load_as<double>(L, (int64_t)c * ld + gr), wsol[c], s0);
                    s1 = fma(load_as<double>(L, (int64_t)(c + 8) * ld + gr), wsol[c + 8], s1);
                }
                for (; c < b0; c += 8) s0 = fma(load_as<double>(L, (int64_t)c * ld + gr), wsol[c], s0);
            }
            double sum = s0 + s1;
            // reduce the 8 parts (threads row, row+32, ..., row+224) through shared memory
            __shared__ double part_sum[8][33];
            part_sum[part][row] = sum;
            __syncthreads();
            if (tid < 32 && tid < w) {
                double t = 0.0;
#pragma unroll
                for (int q = 0; q < 8; ++q) t += part_sum[q][tid];
                rb[tid] = r[b0 + tid] - t;
            }
            __syncthreads();
        }
        // (2) warp 0: substitution down the diagonal block
        if (warp == 0) {
            double lrow[32];  // L[b0 + lane][b0 + j]
#pragma unroll
            for (int j = 0; j < 32; ++j)
                lrow[j] = (lane < w && j < w && j <= lane) ? load_as<double>(L, (int64_t)(b0 + j) * ld + b0 + lane)
                                                           : 0.0;
            double x = lane < w ? rb[lane] : 0.0;
            double dg = 1.0;
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (j == lane && lane < w) dg = lrow[j];
            const double inv = 1.0 / dg;  // one division per lane
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                if (j < w) {
                    if (lane == j) x *= inv;
                    const double xj = __shfl_sync(0xffffffffu, x, j);
                    if (lane > j) x = fma(-lrow[j], xj, x);
                }
            }
            if (lane < w) {
                r[b0 + lane] = x;
                wsol[b0 + lane] = x;
            }
        }
        __syncthreads();
    }
}

// r_j[rows] -= L_ji[rows, :] * w_i for a list of tiles (blockIdx.y = tile,
// blockIdx.x = 32-row chunk): lane = row (coalesced), the 8 warps split the
// columns, partial sums reduced in shared memory (deterministic order).
using GemvItem = TrsvItem;

template <int P>
__global__ void __launch_bounds__(256) tile_gemv_kernel(const GemvItem* __restrict__ items, int nb,
                                                        const double* __restrict__ w) {
    __shared__ double ws[1024];
    __shared__ double part_sum[8][33];
    const GemvItem it = items[blockIdx.y];
    const ST<P>* __restrict__ L = static_cast<const ST<P>*>(it.L);
    for (int c = threadIdx.x; c < nb && c < 1024; c += blockDim.x) ws[c] = w[c];
    __syncthreads();
    const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
    const int row = blockIdx.x * 32 + lane;
    const int chunk = (nb + 7) / 8, c0 = warp * chunk, c1 = min(nb, c0 + chunk);
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (row < nb) {
        int c = c0;
        for (; c + 8 <= c1; c += 8) {
#pragma unroll
            for (int u = 0; u < 8; ++u)
                acc[u] = fma(load_as<double>(L, (int64_t)(c + u) * nb + row), ws[c + u], acc[u]);
        }
        for (; c < c1; ++c) acc[0] = fma(load_as<double>(L, (int64_t)c * nb + row), ws[c], acc[0]);
    }
    part_sum[warp][lane] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    __syncthreads();
    if (warp == 0 && row < nb) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) t += part_sum[q][lane];
        it.r[row] -= t;
    }
}

__global__ void square_sum_kernel(const double* __restrict__ w, int64_t n, double* out) {
    __shared__ double s[256];
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += w[i] * w[i];
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int k = 128; k > 0; k >>= 1) {
        if (threadIdx.x < k) s[threadIdx.x] += s[threadIdx.x + k];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = s[0];
}

// A_ii <- round_p(A_ii + v) (chol_with_jitter's diagonal jitter,
// workloads.cpp:60-62: set(i, i, get(i, i) + jitter)).
template <int P>
__global__ void add_diag_kernel(ST<P>* __restrict__ A, int64_t ld, int n, double v) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        store_from(A, (int64_t)i * ld + i, load_as<double>(A, (int64_t)i * ld + i) + v);
}

template <typename F>
void dispatch_p(mp_precision p, F&& f) {
    if (p == MP_HALF) f(std::integral_constant<int, 0>{});
    else if (p == MP_SINGLE) f(std::integral_constant<int, 1>{});
    else f(std::integral_constant<int, 2>{});
}

}  // namespace

void launch_tile_trsv(Ctx* ctx, cudaStream_t s, mp_precision p, const void* L, int64_t ld, int nb,
                      double* r) {
    dispatch_p(p, [&](auto pp) {
        constexpr int P = decltype(pp)::value;
        tile_trsv_kernel<P><<<1, 256, nb * sizeof(double), s>>>(static_cast<const ST<P>*>(L), ld, nb, r);
    });
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

void launch_tile_gemv(Ctx* ctx, cudaStream_t s, mp_precision p, const void* dev_items,
                      int64_t count, int nb, const double* w) {
    if (count == 0) return;
    if (nb > 1024) fail(MP_INVALID_PARAM, "tile gemv: tile size above 1024");
    const dim3 grid(static_cast<unsigned>((nb + 31) / 32), static_cast<unsigned>(count));
    dispatch_p(p, [&](auto pp) {
        constexpr int P = decltype(pp)::value;
        tile_gemv_kernel<P><<<grid, 256, 0, s>>>(static_cast<const GemvItem*>(dev_items), nb, w);
    });
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

void launch_add_diag(Ctx* ctx, cudaStream_t s, mp_precision p, void* A, int64_t ld, int n,
                     double v) {
    dispatch_p(p, [&](auto pp) {
        constexpr int P = decltype(pp)::value;
        add_diag_kernel<P><<<(n + 255) / 256, 256, 0, s>>>(static_cast<ST<P>*>(A), ld, n, v);
    });
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

void launch_square_sum(Ctx* ctx, cudaStream_t s, const double* w, int64_t n, double* out) {
    square_sum_kernel<<<1, 256, 0, s>>>(w, n, out);
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

}  // namespace mpcr
