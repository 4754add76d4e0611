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

// In-place lower-triangular solve of one nb x nb tile against r (FP64).
template <int P>
__global__ void __launch_bounds__(256) tile_trsv_kernel(const ST<P>* __restrict__ L, int64_t ld,
                                                        int nb, double* __restrict__ r) {
    __shared__ double wb[32];
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    for (int b0 = 0; b0 < nb; b0 += 32) {
        const int w = min(32, nb - b0);
        if (warp == 0) {
            // lane i owns row b0 + i; substitution down the 32 x 32 block
            double x = lane < w ? r[b0 + lane] : 0.0;
            for (int j = 0; j < w; ++j) {
                const double lj = lane < w ? load_as<double>(L, (int64_t)(b0 + j) * ld + b0 + lane) : 0.0;
                const double xj = __shfl_sync(0xffffffffu, x, j) / __shfl_sync(0xffffffffu, lj, j);
                if (lane == j) x = xj;
                if (lane > j) x -= lj * xj;
            }
            if (lane < w) {
                r[b0 + lane] = x;
                wb[lane] = x;
            }
        }
        __syncthreads();
        for (int i = b0 + w + tid; i < nb; i += blockDim.x) {
            double s = 0.0;
            for (int c = 0; c < w; ++c) s += load_as<double>(L, (int64_t)(b0 + c) * ld + i) * wb[c];
            r[i] -= s;
        }
        __syncthreads();
    }
}

// r_j[rows] -= L_ji[rows, :] * w_i for a list of tiles (blockIdx.y = tile,
// blockIdx.x = 256-row chunk); thread = row, columns streamed coalesced.
using GemvItem = TrsvItem;

template <int P>
__global__ void __launch_bounds__(256) tile_gemv_kernel(const GemvItem* __restrict__ items, int nb,
                                                        const double* __restrict__ w) {
    __shared__ double ws[1024];
    const GemvItem it = items[blockIdx.y];
    const ST<P>* __restrict__ L = static_cast<const ST<P>*>(it.L);
    for (int c = threadIdx.x; c < nb && c < 1024; c += blockDim.x) ws[c] = w[c];
    __syncthreads();
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= nb) return;
    double s0 = 0.0, s1 = 0.0;
    int c = 0;
    for (; c + 1 < nb; c += 2) {
        s0 += load_as<double>(L, (int64_t)c * nb + row) * ws[c];
        s1 += load_as<double>(L, (int64_t)(c + 1) * nb + row) * ws[c + 1];
    }
    if (c < nb) s0 += load_as<double>(L, (int64_t)c * nb + row) * ws[c];
    it.r[row] -= s0 + s1;
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
        tile_trsv_kernel<P><<<1, 256, 0, s>>>(static_cast<const ST<P>*>(L), ld, nb, r);
    });
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

void launch_tile_gemv(Ctx* ctx, cudaStream_t s, mp_precision p, const void* dev_items,
                      int64_t count, int nb, const double* w) {
    if (count == 0) return;
    if (nb > 1024) fail(MP_INVALID_PARAM, "tile gemv: tile size above 1024");
    const dim3 grid(static_cast<unsigned>((nb + 255) / 256), static_cast<unsigned>(count));
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
