// linalg::solve (linalg.cpp:544-575) and chol2inv (linalg.cpp:383-408,
// 481-488) on the device.
//
// solve: exactly symmetric A (value comparison, linalg.cpp:443-448) takes the
// Cholesky path (chol, forwardsolve(U^T), backsolve(U)); otherwise, or when
// the factorization fails, LU with partial pivoting (lu_kernel,
// linalg.cpp:163-193) and two substitutions (lu_solve_impl, :451-476).
// The LU is one cooperative launch, right-looking one column at a time with
// the reference's operation order (pivot = first index of the largest
// magnitude, row swap, column scaled by an IEEE division, rank-1 update as a
// separate multiply and subtract), so the factors are bit-identical to the
// reference's in the same compute precision.
#include <cooperative_groups.h>

#include <cmath>
#include <vector>

#include "device.cuh"
#include "internal.hpp"

namespace mpcr {
namespace {

struct SolveBar {
    unsigned int count;
    unsigned int gen;
};

__device__ __forceinline__ void bar_sync(SolveBar* bar, unsigned int nblocks) {
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
            while (*vgen == g) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }

// Partial (value, index) of the pivot search; value -1 marks "none".
struct Piv {
    double v;
    long long i;
};

template <typename T>
__global__ void __launch_bounds__(256) lu_coop_kernel(T* __restrict__ a, int64_t n, int64_t* __restrict__ perm,
                                                      Piv* __restrict__ part, SolveBar* bar,
                                                      int64_t* __restrict__ fail_col) {
    const unsigned int G = gridDim.x;
    const int64_t gt = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nthreads = static_cast<int64_t>(G) * blockDim.x;
    __shared__ Piv sp[256];
    __shared__ long long s_piv;
    if (gt == 0)
        for (int64_t i = 0; i < n; ++i) perm[i] = i;
    for (int64_t j = 0; j < n; ++j) {
        T* colj = a + j * n;
        // (1) pivot: first index of the largest |a_ij|, i >= j (linalg.cpp:167-175);
        //     a NaN never wins a comparison, so it is skipped like the reference does
        Piv best{-1.0, -1};
        for (int64_t i = j + 1 + gt; i < n; i += nthreads) {
            const double v = fabs(static_cast<double>(colj[i]));
            if (v > best.v || (best.i >= 0 && v == best.v && i < best.i) || (best.i < 0 && v == v))
                best = Piv{v, i};
        }
        sp[threadIdx.x] = best;
        __syncthreads();
        for (int w = 128; w > 0; w >>= 1) {
            if (threadIdx.x < w) {
                const Piv o = sp[threadIdx.x + w];
                Piv& m = sp[threadIdx.x];
                if (o.i >= 0 && (m.i < 0 || o.v > m.v || (o.v == m.v && o.i < m.i))) m = o;
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) part[blockIdx.x] = sp[0];
        bar_sync(bar, G);
        if (threadIdx.x == 0) {
            // the reference starts from |a_jj| and takes a later row only if strictly larger
            const double d0 = fabs(static_cast<double>(colj[j]));
            double bv = d0;
            long long bi = j;
            Piv rest{-1.0, -1};
            for (unsigned int q = 0; q < G; ++q) {
                const Piv o = part[q];
                if (o.i >= 0 && (rest.i < 0 || o.v > rest.v || (o.v == rest.v && o.i < rest.i))) rest = o;
            }
            if (rest.i >= 0 && rest.v > bv) {  // d0 NaN: no row is ever larger
                bv = rest.v;
                bi = rest.i;
            }
            s_piv = (bv == 0.0) ? -1 : bi;
        }
        __syncthreads();
        const long long piv = s_piv;
        if (piv < 0) {
            if (gt == 0) *fail_col = j;
            return;  // every CTA sees the same value: uniform exit
        }
        // (2) swap rows j and piv over all columns
        if (piv != j) {
            for (int64_t c = gt; c < n; c += nthreads) {
                const T t = a[c * n + j];
                a[c * n + j] = a[c * n + piv];
                a[c * n + piv] = t;
            }
            if (gt == 0) {
                const int64_t t = perm[j];
                perm[j] = perm[piv];
                perm[piv] = t;
            }
        }
        bar_sync(bar, G);
        // (3) scale the column below the pivot
        const T d = colj[j];
        for (int64_t i = j + 1 + gt; i < n; i += nthreads) colj[i] = div_rn(colj[i], d);
        bar_sync(bar, G);
        // (4) rank-1 update, column by column (columns over CTAs, rows over threads)
        for (int64_t c = j + 1 + blockIdx.x; c < n; c += G) {
            T* colc = a + c * n;
            const T mult = colc[j];
            if (mult == T(0)) continue;
            for (int64_t i = j + 1 + threadIdx.x; i < n; i += blockDim.x)
                colc[i] = sub_rn(colc[i], mul_rn(colj[i], mult));
        }
        bar_sync(bar, G);
    }
}

// x = P b, then L y = x (unit diagonal), U x = y; one thread per right-hand
// side column, the reference's substitution order (tri_solve_kernel).
template <typename T>
__global__ void lu_substitute_kernel(const T* __restrict__ a, int64_t n, const int64_t* __restrict__ perm,
                                     const T* __restrict__ b, int64_t ldb, T* __restrict__ x, int64_t ldx,
                                     int64_t ncols) {
    const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= ncols) return;
    T* xc = x + c * ldx;
    for (int64_t i = 0; i < n; ++i) xc[i] = b[c * ldb + perm[i]];
    for (int64_t i = 0; i < n; ++i) {
        T acc = xc[i];
        for (int64_t k = 0; k < i; ++k) acc = sub_rn(acc, mul_rn(a[k * n + i], xc[k]));
        xc[i] = acc;  // unit diagonal
    }
    for (int64_t i = n; i-- > 0;) {
        T acc = xc[i];
        for (int64_t k = i + 1; k < n; ++k) acc = sub_rn(acc, mul_rn(a[k * n + i], xc[k]));
        xc[i] = div_rn(acc, a[i * n + i]);
    }
}

// a(i, j) == a(j, i) for all i < j (value comparison, linalg.cpp:443-448)
template <int P>
__global__ void symmetric_kernel(const typename Storage<P>::T* __restrict__ a, int64_t lda, int64_t n,
                                 int* __restrict__ asym) {
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n * n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = e / n, i = e - j * n;
        if (i < j && load_as<double>(a, j * lda + i) != load_as<double>(a, i * lda + j)) *asym = 1;
    }
}

}  // namespace

bool device_exactly_symmetric(Ctx* ctx, cudaStream_t s, mp_precision p, const void* a, int64_t lda, int64_t n) {
    int* flag = static_cast<int*>(ctx->ensure_scratch(64, 1));
    MP_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
    const int g = grid_for(n * n, 256, ctx->sm_count);
    if (p == MP_HALF)
        symmetric_kernel<0><<<g, 256, 0, s>>>(static_cast<const uint16_t*>(a), lda, n, flag);
    else if (p == MP_SINGLE)
        symmetric_kernel<1><<<g, 256, 0, s>>>(static_cast<const float*>(a), lda, n, flag);
    else
        symmetric_kernel<2><<<g, 256, 0, s>>>(static_cast<const double*>(a), lda, n, flag);
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
    int h = 0;
    MP_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    return h == 0;
}

// LU with partial pivoting of the n x n compute-precision matrix w (in place)
// and the substitutions for `ncols` right-hand sides (b -> x, compute
// precision, column-major).  Returns the zero-pivot column or -1.
int64_t lu_solve_device(Ctx* ctx, cudaStream_t s, mp_precision cp, void* w, int64_t n, const void* b,
                        int64_t ldb, void* x, int64_t ldx, int64_t ncols) {
    const int G = std::max(1, std::min(ctx->sm_count, static_cast<int>((n + 255) / 256) * 4));
    char* scr = static_cast<char*>(ctx->ensure_scratch(256 + G * sizeof(Piv) + n * sizeof(int64_t) + 256, 1));
    SolveBar* bar = reinterpret_cast<SolveBar*>(scr);
    int64_t* fail = reinterpret_cast<int64_t*>(scr + 64);
    Piv* part = reinterpret_cast<Piv*>(scr + 256);
    int64_t* perm = reinterpret_cast<int64_t*>(scr + 256 + G * sizeof(Piv));
    MP_CUDA(cudaMemsetAsync(scr, 0, 64, s));
    MP_CUDA(cudaMemsetAsync(fail, 0xFF, sizeof(int64_t), s));
    int64_t nn = n;
    void* args[] = {&w, &nn, &perm, &part, &bar, &fail};
    if (cp == MP_DOUBLE)
        MP_CUDA(cudaLaunchCooperativeKernel((void*)lu_coop_kernel<double>, G, 256, args, 0, s));
    else
        MP_CUDA(cudaLaunchCooperativeKernel((void*)lu_coop_kernel<float>, G, 256, args, 0, s));
    count_launch(ctx);
    int64_t hf = -1;
    MP_CUDA(cudaMemcpyAsync(&hf, fail, sizeof(hf), cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    if (hf >= 0) return hf;
    const int tb = 128, gb = static_cast<int>((ncols + tb - 1) / tb);
    if (cp == MP_DOUBLE)
        lu_substitute_kernel<double><<<gb, tb, 0, s>>>(static_cast<const double*>(w), n, perm,
                                                       static_cast<const double*>(b), ldb, static_cast<double*>(x),
                                                       ldx, ncols);
    else
        lu_substitute_kernel<float><<<gb, tb, 0, s>>>(static_cast<const float*>(w), n, perm,
                                                      static_cast<const float*>(b), ldb, static_cast<float*>(x), ldx,
                                                      ncols);
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
    return -1;
}

}  // namespace mpcr
