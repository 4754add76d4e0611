// Batched tile kernels for the MPCRTile scheduler: precision conversion of a
// list of equally sized contiguous tiles (the "cast panel tiles to their
// consumer precisions once" step, array.cpp:187-191 semantics), zero fill,
// triangle zeroing and the leaf inverses of TRTRI.  blockIdx.y = item.
#include "batch.hpp"
#include "device.cuh"
#include "internal.hpp"

namespace mpcr {
namespace {

template <typename TI, typename TO> __device__ __forceinline__ TO cv(TI x);
template <> __device__ __forceinline__ uint16_t cv<uint16_t, uint16_t>(uint16_t x) {
    return ((x & 0x7C00u) == 0x7C00u && (x & 0x3FFu)) ? uint16_t(0x7E00u) : x;
}
template <> __device__ __forceinline__ float cv<uint16_t, float>(uint16_t x) { return h2f(x); }
template <> __device__ __forceinline__ double cv<uint16_t, double>(uint16_t x) { return h2d(x); }
template <> __device__ __forceinline__ uint16_t cv<float, uint16_t>(float x) { return f2h(x); }
template <> __device__ __forceinline__ float cv<float, float>(float x) {
    return x != x ? __int_as_float(__float_as_int(x) | 0x00400000) : x;
}
template <> __device__ __forceinline__ double cv<float, double>(float x) { return f2d(x); }
template <> __device__ __forceinline__ uint16_t cv<double, uint16_t>(double x) { return d2h(x); }
template <> __device__ __forceinline__ float cv<double, float>(double x) { return d2f(x); }
template <> __device__ __forceinline__ double cv<double, double>(double x) { return x; }

// Eight elements per thread and step through 16-byte vector loads and
// stores when both tiles are 16-byte aligned (the scheduler's panel and
// matrix tiles always are); scalar tail / fallback otherwise.
template <typename T>
struct alignas(16) Vec8 {
    T v[8];
};

template <typename TI, typename TO>
__global__ void __launch_bounds__(256) batched_convert_kernel(const CopyItem* __restrict__ items,
                                                              int64_t n) {
    const CopyItem it = items[blockIdx.y];
    const TI* __restrict__ src = static_cast<const TI*>(it.src);
    TO* __restrict__ dst = static_cast<TO*>(it.dst);
    const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
    const int64_t n8 = vec ? n / 8 : 0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n8;
         t += (int64_t)gridDim.x * blockDim.x) {
        const Vec8<TI> a = reinterpret_cast<const Vec8<TI>*>(src)[t];
        Vec8<TO> b;
#pragma unroll
        for (int k = 0; k < 8; ++k) b.v[k] = cv<TI, TO>(a.v[k]);
        reinterpret_cast<Vec8<TO>*>(dst)[t] = b;
    }
    for (int64_t t = n8 * 8 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x)
        dst[t] = cv<TI, TO>(src[t]);
}

template <typename T>
__global__ void batched_zero_kernel(void* const* __restrict__ ptrs, int64_t n) {
    T* p = static_cast<T*>(ptrs[blockIdx.y]);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x)
        p[t] = T(0);
}

template <typename T>
__global__ void batched_zero_upper_kernel(void* const* __restrict__ ptrs, int64_t nb) {
    T* p = static_cast<T*>(ptrs[blockIdx.y]);
    const int64_t total = nb * nb;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / nb, i = t - j * nb;
        if (i < j) p[t] = T(0);
    }
}

// Inverse of each 64x64 diagonal block of a lower-triangular FP64 matrix:
// column c by forward substitution, all in shared memory.
__global__ void __launch_bounds__(64) leaf_inverse_kernel(const double* __restrict__ L,
                                                          int64_t ldl, int64_t n,
                                                          double* __restrict__ Linv,
                                                          int64_t ldi) {
    __shared__ double D[64][65];
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 64;
    const int bb = static_cast<int>(n - r0 < 64 ? n - r0 : 64);
    for (int c = 0; c < 64; ++c) {
        const int r = threadIdx.x;
        D[r][c] = (r < bb && c < bb) ? L[(r0 + c) * ldl + r0 + r] : 0.0;
    }
    __syncthreads();
    // column c of the inverse is private to thread c: written straight to
    // Linv and re-read from there (L1-resident).
    const int c = threadIdx.x;
    if (c < bb) {
        double* X = Linv + (r0 + c) * ldi + r0;
        for (int i = 0; i < bb; ++i) {
            double x = 0.0;
            if (i >= c) {
                double s = (i == c) ? 1.0 : 0.0;
                for (int k = c; k < i; ++k) s -= D[i][k] * X[k];
                x = s / D[i][i];
            }
            X[i] = x;
        }
    }
}

// hi = fp16(x), lo = fp16(x - hi): x ~= hi + lo to ~2^-22 relative.
__global__ void split_f16_kernel(const double* __restrict__ x, uint16_t* __restrict__ hi,
                                 uint16_t* __restrict__ lo, int64_t n) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const double v = x[t];
        const uint16_t h = d2h(v);
        hi[t] = h;
        lo[t] = d2h(v - h2d(h));
    }
}

__device__ __forceinline__ float to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// 3xTF32 operand split: hi = tf32(x), lo = tf32(x - hi) (x - hi is exact).
// One 32x32 block per CTA (blockDim 32x8); with `trans` the packed outputs
// hold the transpose (cols x rows, ld = cols) so the operand is K-major for
// kind::tf32 (which reads 128B-swizzled 32-bit data K-major only).
template <typename TI>
__device__ __forceinline__ void split_block(const TI* __restrict__ src, int64_t lds, int64_t rows,
                                            int64_t cols, float* __restrict__ hi,
                                            float* __restrict__ lo, bool trans,
                                            float (*th)[33], float (*tl)[33]) {
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * 32, j0 = static_cast<int64_t>(blockIdx.y) * 32;
    for (int r = threadIdx.y; r < 32; r += 8) {
        const int64_t i = i0 + threadIdx.x, j = j0 + r;
        if (i < rows && j < cols) {
            const float x = load_as<float>(src, j * lds + i);
            const float h = to_tf32(x);
            const float l = to_tf32(x - h);
            if (!trans) {
                hi[j * rows + i] = h;
                lo[j * rows + i] = l;
            } else {
                th[r][threadIdx.x] = h;
                tl[r][threadIdx.x] = l;
            }
        }
    }
    if (!trans) return;
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += 8) {
        const int64_t oj = i0 + r, oi = j0 + threadIdx.x;  // output (oi, oj) = input (oj, oi)
        if (oj < rows && oi < cols) {
            hi[oj * cols + oi] = th[threadIdx.x][r];
            lo[oj * cols + oi] = tl[threadIdx.x][r];
        }
    }
}

template <typename TI>
__global__ void split_tf32_2d_kernel(const TI* __restrict__ src, int64_t lds, int64_t rows,
                                     int64_t cols, float* __restrict__ hi, float* __restrict__ lo,
                                     bool trans) {
    __shared__ float th[32][33], tl[32][33];
    split_block(src, lds, rows, cols, hi, lo, trans, th, tl);
}

__global__ void batched_split_tf32_kernel(const SplitItem* __restrict__ items, int64_t nb) {
    __shared__ float th[32][33], tl[32][33];
    const SplitItem it = items[blockIdx.z];
    split_block(static_cast<const float*>(it.src), nb, nb, nb, static_cast<float*>(it.hi),
                static_cast<float*>(it.lo), true, th, tl);
}

template <int P>
using ST = typename Storage<P>::T;

}  // namespace

void launch_split_tf32(Ctx* ctx, cudaStream_t s, mp_precision pin, const void* src, int64_t lds,
                       int64_t rows, int64_t cols, float* hi, float* lo, bool trans) {
    if (rows == 0 || cols == 0) return;
    const dim3 grid(static_cast<unsigned>((rows + 31) / 32), static_cast<unsigned>((cols + 31) / 32));
    const dim3 block(32, 8);
    if (pin == MP_HALF)
        split_tf32_2d_kernel<<<grid, block, 0, s>>>(static_cast<const uint16_t*>(src), lds, rows, cols, hi, lo, trans);
    else if (pin == MP_SINGLE)
        split_tf32_2d_kernel<<<grid, block, 0, s>>>(static_cast<const float*>(src), lds, rows, cols, hi, lo, trans);
    else
        fail(MP_INVALID_PARAM, "split_tf32: double input");
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

void launch_batched_split_tf32_t(Ctx* ctx, cudaStream_t s, const SplitItem* dev_items, int64_t count,
                                 int64_t nb) {
    if (count == 0) return;
    const dim3 grid(static_cast<unsigned>((nb + 31) / 32), static_cast<unsigned>((nb + 31) / 32),
                    static_cast<unsigned>(count));
    batched_split_tf32_kernel<<<grid, dim3(32, 8), 0, s>>>(dev_items, nb);
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

void launch_split_f16(Ctx* ctx, cudaStream_t s, const double* x, uint16_t* hi, uint16_t* lo,
                      int64_t n) {
    split_f16_kernel<<<grid_for(n, 256, ctx->sm_count), 256, 0, s>>>(x, hi, lo, n);
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

void launch_batched_convert(Ctx* ctx, cudaStream_t s, mp_precision pin, mp_precision pout,
                            const CopyItem* dev_items, int64_t count, int64_t elems) {
    if (count == 0 || elems == 0) return;
    int gx = static_cast<int>((elems / 8 + 255) / 256);
    const int cap = static_cast<int>(8 * ctx->sm_count / (count < 1 ? 1 : count)) + 1;
    if (gx > cap) gx = cap;
    if (gx < 1) gx = 1;
    const dim3 grid(gx, static_cast<unsigned>(count));
    ProfScope ps(ctx, MP_PROF_CAST, s,
                 static_cast<double>(count) * elems * (elem_bytes(pin) + elem_bytes(pout)));
#define MP_BC(PI, PO)                                                                      \
    if (pin == PI && pout == PO) {                                                         \
        batched_convert_kernel<ST<PI>, ST<PO>><<<grid, 256, 0, s>>>(dev_items, elems);     \
    } else
    MP_BC(0, 0) MP_BC(0, 1) MP_BC(0, 2) MP_BC(1, 0) MP_BC(1, 1) MP_BC(1, 2) MP_BC(2, 0)
        MP_BC(2, 1) MP_BC(2, 2) fail(MP_INVALID_PARAM, "batched convert: precision");
#undef MP_BC
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

void launch_batched_zero(Ctx* ctx, cudaStream_t s, mp_precision p, void* const* dev_ptrs,
                         int64_t count, int64_t elems, bool upper_only, int64_t nb) {
    if (count == 0) return;
    int gx = static_cast<int>((elems + 255) / 256);
    if (gx > 64) gx = 64;
    const dim3 grid(gx, static_cast<unsigned>(count));
    if (upper_only) {
        if (p == MP_HALF) batched_zero_upper_kernel<uint16_t><<<grid, 256, 0, s>>>(dev_ptrs, nb);
        else if (p == MP_SINGLE) batched_zero_upper_kernel<float><<<grid, 256, 0, s>>>(dev_ptrs, nb);
        else batched_zero_upper_kernel<double><<<grid, 256, 0, s>>>(dev_ptrs, nb);
    } else {
        if (p == MP_HALF) batched_zero_kernel<uint16_t><<<grid, 256, 0, s>>>(dev_ptrs, elems);
        else if (p == MP_SINGLE) batched_zero_kernel<float><<<grid, 256, 0, s>>>(dev_ptrs, elems);
        else batched_zero_kernel<double><<<grid, 256, 0, s>>>(dev_ptrs, elems);
    }
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

void launch_leaf_inverse(Ctx* ctx, cudaStream_t s, const double* L, int64_t ldl, int64_t n,
                         double* Linv, int64_t ldi) {
    const int nblk = static_cast<int>((n + 63) / 64);
    leaf_inverse_kernel<<<nblk, 64, 0, s>>>(L, ldl, n, Linv, ldi);
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

namespace {
__global__ void __launch_bounds__(256) gather_rows_kernel(const RowItem* __restrict__ items, int64_t nb,
                                                          int64_t ldd) {
    const RowItem it = items[blockIdx.y];
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nb; c += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = c * nb + it.row;
        double v;
        if (it.prec == MP_HALF) v = h2d(static_cast<const uint16_t*>(it.tile)[e]);
        else if (it.prec == MP_SINGLE) v = f2d(static_cast<const float*>(it.tile)[e]);
        else v = static_cast<const double*>(it.tile)[e];
        it.dst[c * ldd] = v;
    }
}
}  // namespace

void launch_gather_rows(Ctx* ctx, cudaStream_t s, const RowItem* dev_items, int64_t count, int64_t nb,
                        int64_t ldd) {
    for (int64_t b = 0; b < count; b += 65535) {
        const int64_t cnt = count - b < 65535 ? count - b : 65535;
        const dim3 grid(static_cast<unsigned>((nb + 255) / 256), static_cast<unsigned>(cnt));
        gather_rows_kernel<<<grid, 256, 0, s>>>(dev_items + b, nb, ldd);
        count_launch(ctx);
    }
    MP_CUDA(cudaGetLastError());
}

}  // namespace mpcr
