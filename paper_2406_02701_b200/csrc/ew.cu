// Elementwise, reduction and layout kernels (array.cpp:228-429) plus the
// small helpers the factorizations need.  All HBM-streaming, grid-stride,
// grid sized to a multiple of the SM count.
#include <algorithm>
#include <cfloat>

#include "device.cuh"
#include "internal.hpp"

namespace mpcr {
namespace {

template <int P>
using ST = typename Storage<P>::T;

// ---- ew_binary (array.cpp:252-272) ----------------------------------------
template <int PA, int PB, int PO>
__global__ void ew_binary_kernel(int op, const ST<PA>* __restrict__ a, int64_t lda,
                                 const ST<PB>* __restrict__ b, int64_t ldb,
                                 ST<PO>* __restrict__ o, int64_t ldo, int64_t rows,
                                 int64_t cols) {
    using C = typename std::conditional<PO == 2, double, float>::type;
    const int64_t n = rows * cols;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / rows, i = t - j * rows;
        const C x = load_as<C>(a, j * lda + i);
        const C y = load_as<C>(b, j * ldb + i);
        store_from(o, j * ldo + i, op_rn(op, x, y));
    }
}

// ---- ew_scalar (array.cpp:274-291); y pre-rounded by the host ------------
template <int P>
__global__ void ew_scalar_kernel(int op, const ST<P>* __restrict__ a, int64_t lda,
                                 ST<P>* __restrict__ o, int64_t ldo, int64_t rows,
                                 int64_t cols, double yd) {
    using C = typename std::conditional<P == 2, double, float>::type;
    const C y = static_cast<C>(yd);
    const int64_t n = rows * cols;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / rows, i = t - j * rows;
        store_from(o, j * ldo + i, op_rn(op, load_as<C>(a, j * lda + i), y));
    }
}

// ---- ew_unary (array.cpp:293-322) -----------------------------------------
template <int P>
__global__ void ew_unary_kernel(int op, const ST<P>* __restrict__ a, int64_t lda,
                                ST<P>* __restrict__ o, int64_t ldo, int64_t rows,
                                int64_t cols) {
    const int64_t n = rows * cols;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / rows, i = t - j * rows;
        if (P == 2) {
            const double x = load_as<double>(a, j * lda + i);
            double v;
            switch (op) {
                case 0: v = log(x); break;
                case 1: v = exp(x); break;
                case 2: v = __dsqrt_rn(x); break;
                default: v = fabs(x); break;
            }
            store_from(o, j * ldo + i, v);
        } else {
            const double xd = load_as<double>(a, j * lda + i);
            const float x = d2f(xd);
            double v;
            switch (op) {
                case 0: v = f2d(logf(x)); break;
                case 1: v = f2d(expf(x)); break;
                case 2: v = f2d(__fsqrt_rn(x)); break;
                default: v = fabs(xd); break;
            }
            store_from(o, j * ldo + i, v);
        }
    }
}

// ---- reduce (array.cpp:336-369): deterministic two-pass -------------------
constexpr int kRedBlocks = 296;  // 2 x 148 SMs
constexpr int kRedThreads = 256;

struct MinMax {
    double v;
    int64_t i;
};

__device__ __forceinline__ MinMax better(MinMax a, MinMax b, bool is_min) {
    // Sequential std::min/std::max keeps the earliest element among equals
    // and never adopts a NaN after the first element.
    if (b.i < 0) return a;
    if (a.i < 0) return b;
    const bool b_wins = is_min ? (b.v < a.v) : (a.v < b.v);
    if (b_wins) return b;
    if (!(a.v < b.v) && !(b.v < a.v) && b.i < a.i && b.v == b.v && a.v == a.v) return b;
    return a;
}

template <int P>
__global__ void __launch_bounds__(kRedThreads) reduce_pass1(int op, const ST<P>* __restrict__ a,
                                                            int64_t lda, int64_t rows,
                                                            int64_t cols, double* part,
                                                            int64_t* part_i) {
    const int64_t n = rows * cols;
    const bool is_mm = (op == 2 || op == 3);
    double acc = 0.0;
    MinMax mm{0.0, -1};
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / rows, i = t - j * rows;
        const double x = load_as<double>(a, j * lda + i);
        if (is_mm) {
            if (x == x) mm = better(mm, MinMax{x, t}, op == 2);
        } else {
            acc += (op == 1) ? x * x : x;
        }
    }
    __shared__ double sacc[kRedThreads];
    __shared__ double sv[kRedThreads];
    __shared__ int64_t si[kRedThreads];
    sacc[threadIdx.x] = acc;
    sv[threadIdx.x] = mm.v;
    si[threadIdx.x] = mm.i;
    __syncthreads();
    for (int w = kRedThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            sacc[threadIdx.x] += sacc[threadIdx.x + w];
            MinMax r = better(MinMax{sv[threadIdx.x], si[threadIdx.x]},
                              MinMax{sv[threadIdx.x + w], si[threadIdx.x + w]}, op == 2);
            sv[threadIdx.x] = r.v;
            si[threadIdx.x] = r.i;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[blockIdx.x] = is_mm ? sv[0] : sacc[0];
        part_i[blockIdx.x] = si[0];
    }
}

__global__ void reduce_pass2(int op, const double* part, const int64_t* part_i, int nparts,
                             double first, double* out) {
    if (threadIdx.x != 0) return;
    if (op == 2 || op == 3) {
        MinMax mm{0.0, -1};
        for (int b = 0; b < nparts; ++b) mm = better(mm, MinMax{part[b], part_i[b]}, op == 2);
        // A leading NaN sticks (std::min/max never replace it); all-NaN -> NaN.
        *out = (first != first || mm.i < 0) ? first : mm.v;
    } else {
        double acc = 0.0;
        for (int b = 0; b < nparts; ++b) acc += part[b];
        *out = acc;
    }
}

// ---- transpose (array.cpp:422-429) via 32x33 smem tiles -------------------
template <typename T>
__global__ void transpose_kernel(const T* __restrict__ in, int64_t ldi, int64_t rows,
                                 int64_t cols, T* __restrict__ out, int64_t ldo) {
    __shared__ T tile[32][33];
    const int64_t i0 = blockIdx.x * 32, j0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t i = i0 + threadIdx.x, j = j0 + r;
        if (i < rows && j < cols) tile[r][threadIdx.x] = in[j * ldi + i];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t oi = j0 + threadIdx.x, oj = i0 + r;  // out is cols x rows
        if (oi < cols && oj < rows) out[oj * ldo + oi] = tile[threadIdx.x][r];
    }
}

template <typename T>
__global__ void diag_kernel(const T* __restrict__ a, int64_t lda, int64_t n, T* __restrict__ o) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x)
        o[t] = a[t * lda + t];
}

template <typename T>
__global__ void fill_kernel(T* __restrict__ a, int64_t lda, int64_t rows, int64_t cols, T v) {
    const int64_t n = rows * cols;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / rows, i = t - j * rows;
        a[j * lda + i] = v;
    }
}

template <typename T>
__global__ void zero_triangle_kernel(T* __restrict__ a, int64_t lda, int64_t n, bool upper) {
    const int64_t total = n * n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / n, i = t - j * n;
        if (upper ? (i < j) : (i > j)) a[j * lda + i] = T(0);
    }
}

template <typename T>
__global__ void mirror_lower_kernel(T* __restrict__ a, int64_t lda, int64_t n) {
    const int64_t total = n * n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / n, i = t - j * n;
        if (i < j) a[j * lda + i] = a[i * lda + j];
    }
}

template <int P>
__global__ void logdiag_kernel(const ST<P>* __restrict__ a, int64_t lda, int64_t n,
                               double* out) {
    __shared__ double s[256];
    double acc = 0.0;
    for (int64_t t = threadIdx.x; t < n; t += blockDim.x) acc += log(load_as<double>(a, t * lda + t));
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out += s[0];
}

// Matern closed forms (covariance.cpp:44-72).
__device__ __forceinline__ double matern_value(double d, double nu, double range, double var) {
    if (nu == 0.5) return var * exp(-d / range);
    if (nu == 1.5) {
        const double r = sqrt(3.0) * d / range;
        return var * (1.0 + r) * exp(-r);
    }
    const double r = sqrt(5.0) * d / range;
    return var * (1.0 + r + r * r / 3.0) * exp(-r);
}

// Unit grid with x fastest (covariance.cpp:15-21): point p has coordinates
// (p % side, p / side) / (side - 1), divided exactly as the reference does.
template <int P>
__global__ void matern_grid_kernel(ST<P>* __restrict__ dst, int64_t ld, int64_t row0,
                                   int64_t col0, int64_t rows, int64_t cols, int64_t side,
                                   double nu, double range, double var) {
    const int64_t n = rows * cols;
    const double den = static_cast<double>(side - 1);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / rows, i = t - j * rows;
        const int64_t pi = row0 + i, pj = col0 + j;
        const double dx = static_cast<double>(pi % side) / den - static_cast<double>(pj % side) / den;
        const double dy = static_cast<double>(pi / side) / den - static_cast<double>(pj / side) / den;
        store_from(dst, j * ld + i, matern_value(hypot(dx, dy), nu, range, var));
    }
}

// Arbitrary locations (x[p], y[p]); `nugget` added on the global diagonal.
template <int P>
__global__ void matern_points_kernel(ST<P>* __restrict__ dst, int64_t ld, int64_t row0,
                                     int64_t col0, int64_t rows, int64_t cols,
                                     const double* __restrict__ x, const double* __restrict__ y,
                                     double nu, double range, double var, double nugget) {
    const int64_t n = rows * cols;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / rows, i = t - j * rows;
        const int64_t pi = row0 + i, pj = col0 + j;
        double v = matern_value(hypot(x[pi] - x[pj], y[pi] - y[pj]), nu, range, var);
        if (pi == pj) v += nugget;
        store_from(dst, j * ld + i, v);
    }
}

// Batched symmetric generation for MPCRTile: one launch over the lower tiles
// (i >= j); a CTA computes a 32 x 32 block of tile (i, j) once and stores it
// to (i, j) and, transposed through shared memory, to (j, i) (each in its own
// precision, rounded from the double value as set_linear does).
struct MaternItem {
    void* lo;        // tile (i, j), column-major, ld = rows
    void* up;        // tile (j, i) or nullptr (diagonal / not stored here)
    int32_t p_lo, p_up;
    int64_t row0, col0;  // global row of tile row 0 / column of tile column 0
};

__device__ __forceinline__ void store_any(void* base, int p, int64_t i, double v) {
    if (p == MP_HALF) store_from(static_cast<uint16_t*>(base), i, v);
    else if (p == MP_SINGLE) store_from(static_cast<float*>(base), i, v);
    else static_cast<double*>(base)[i] = v;
}

// FP16 value of var * exp(-d / range) for an FP16 tile (nu = 1/2), equal to
// the reference's double value rounded by encode_f16: d from a branch-free
// FP64 reciprocal square root (relative error ~2^-46), an exact double range
// reduction t = fl + f, 2^-f on the SFU in FP32 (relative error < 2^-21
// overall), and the result accepted only when both v (1 +- 2^-19) round to
// the same half -- no rounding midpoint within reach of the error.  The rare
// rest falls back to the FP64 expression.  Returns false for a fallback.
__device__ __forceinline__ bool matern_half_fast(double dx, double dy, double c_log2, float var32,
                                                 uint16_t* h) {
    const double s2 = fma(dx, dx, dy * dy);
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(s2));
    r = r * fma(-0.5 * s2 * r, r, 1.5);  // one Newton step
    const double t = s2 * r * c_log2;      // d / range * log2(e)
    const double fl = floor(t);
    // NaN or coincident points: FP64 path.  Up to 2^-120 the FP32 scaling
    // below stays normal (tiny values round to +0 in half, exactly as the
    // reference's: no FP64 fallback for far-apart points)
    if (!(fl <= 120.0)) return false;
    float e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-static_cast<float>(t - fl)));
    const float v = e * __int_as_float((127 - static_cast<int>(fl)) << 23) * var32;  // exact 2^-fl
    if (!(fabsf(v) <= 6.0e4f)) return false;
    const uint16_t h1 = __half_as_ushort(__float2half_rn(v * (1.0f + 0x1p-19f)));
    const uint16_t h2 = __half_as_ushort(__float2half_rn(v * (1.0f - 0x1p-19f)));
    *h = h1;
    return h1 == h2;
}

// All-FP16 items (nu = 1/2): 32-bit indexing, the row point's coordinates
// loaded once per block, two tiles (i, j) and (j, i) written through a shared
// transpose of the half values.
template <bool GRID>
__device__ __forceinline__ void matern_half_tiles(const MaternItem& it, int nb, const double* __restrict__ x,
                                                  const double* __restrict__ y, int64_t side, double range,
                                                  double var, double nugget) {
    const int bpr = nb / 32;
    __shared__ uint16_t sh[32][34];
    const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
    const double den = static_cast<double>(side - 1);
    const double c_log2 = 1.4426950408889634 / range;
    const float var32 = static_cast<float>(var);
    const bool var_exact = static_cast<double>(var32) == var;
    uint16_t* lo = static_cast<uint16_t*>(it.lo);
    uint16_t* up = static_cast<uint16_t*>(it.up);
    auto coords = [&](int64_t p, double& cx, double& cy) {
        if (GRID) {
            cx = static_cast<double>(p % side) / den;
            cy = static_cast<double>(p / side) / den;
        } else {
            cx = x[p];
            cy = y[p];
        }
    };
    __shared__ int nfail;
    __shared__ uint16_t flist[32 * 32];  // elements left to the FP64 path (rare)
    __shared__ double cxs[32], cys[32];  // the block's column points
    const bool bpr_p2 = (bpr & (bpr - 1)) == 0;  // tile sizes of 32 x 2^k: shifts, not divisions
    const int bpr_lg = __ffs(bpr) - 1;
    for (int blk = blockIdx.x; blk < bpr * bpr; blk += gridDim.x) {
        const int bi = bpr_p2 ? (blk & (bpr - 1)) : blk % bpr;
        const int bj = bpr_p2 ? (blk >> bpr_lg) : blk / bpr;
        const int i = bi * 32 + tx;
        const int64_t pi = it.row0 + i, pc0 = it.col0 + bj * 32;
        double xi, yi;
        coords(pi, xi, yi);
        if (threadIdx.x < 32) coords(pc0 + threadIdx.x, cxs[threadIdx.x], cys[threadIdx.x]);
        if (threadIdx.x == 0) nfail = 0;
        __syncthreads();  // also: the previous block's transpose reads are done
        uint16_t* lob = lo + static_cast<int64_t>(bj * 32 + ty) * nb + bi * 32 + tx;  // column ty, row tx
        const int64_t step = 8 * static_cast<int64_t>(nb);
        // local column of this row's diagonal element in the block, or -1
        const int dcol = (pi >= pc0 && pi < pc0 + 32) ? static_cast<int>(pi - pc0) : -1;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int lj = ty + 8 * q;
            uint16_t h;
            if (var_exact && lj != dcol && matern_half_fast(xi - cxs[lj], yi - cys[lj], c_log2, var32, &h)) {
                lob[q * step] = h;
                sh[lj][tx] = h;
            } else {
                flist[atomicAdd(&nfail, 1)] = static_cast<uint16_t>(lj * 32 + tx);
            }
        }
        __syncthreads();
        // the failures, compacted: one element per thread on the FP64 path
        for (int f = threadIdx.x; f < nfail; f += blockDim.x) {
            const int e = flist[f], lj = e >> 5, li = e & 31;
            const int ii = bi * 32 + li, j = bj * 32 + lj;
            const int64_t pii = it.row0 + ii, pj = it.col0 + j;
            double xa, ya;
            coords(pii, xa, ya);
            double v = matern_value(hypot(xa - cxs[lj], ya - cys[lj]), 0.5, range, var);
            if (!GRID && pii == pj) v += nugget;
            const uint16_t h = d2h(v);
            lo[static_cast<int64_t>(j) * nb + ii] = h;
            sh[lj][li] = h;
        }
        if (!up) continue;
        __syncthreads();
        uint16_t* upb = up + static_cast<int64_t>(bi * 32 + ty) * nb + bj * 32 + tx;  // column bi*32+ty
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            *upb = sh[tx][ty + 8 * q];
            upb += 8 * static_cast<int64_t>(nb);
        }
    }
}

template <bool GRID>
__global__ void __launch_bounds__(256) matern_tiles_kernel(const MaternItem* __restrict__ items, int64_t nb,
                                                           const double* __restrict__ x,
                                                           const double* __restrict__ y, int64_t side,
                                                           double nu, double range, double var,
                                                           double nugget) {
    const MaternItem it = items[blockIdx.y];
    if (nu == 0.5 && it.p_lo == MP_HALF && (!it.up || it.p_up == MP_HALF)) {  // uniform per CTA
        matern_half_tiles<GRID>(it, static_cast<int>(nb), x, y, side, range, var, nugget);
        return;
    }
    const int64_t bpr = nb / 32;  // 32 x 32 blocks per tile row
    __shared__ double sv[32][33];
    const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // 8 row-groups of 32 lanes
    const double den = static_cast<double>(side - 1);
    // a CTA walks several blocks of its tile (few, long-lived CTAs: the block
    // scheduler, not the math, bounded the one-block-per-CTA version)
    for (int64_t blk = blockIdx.x; blk < bpr * bpr; blk += gridDim.x) {
    const int64_t bi = blk % bpr, bj = blk / bpr;
    if (blk != blockIdx.x) __syncthreads();  // the transpose buffers are reused
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int lj = ty + 8 * q;                    // column within the block
        const int64_t i = bi * 32 + tx, j = bj * 32 + lj;  // within the tile
        const int64_t pi = it.row0 + i, pj = it.col0 + j;
        double dx, dy;
        if (GRID) {
            dx = static_cast<double>(pi % side) / den - static_cast<double>(pj % side) / den;
            dy = static_cast<double>(pi / side) / den - static_cast<double>(pj / side) / den;
        } else {
            dx = x[pi] - x[pj];
            dy = y[pi] - y[pj];
        }
        double v = matern_value(hypot(dx, dy), nu, range, var);
        if (!GRID && pi == pj) v += nugget;
        store_any(it.lo, it.p_lo, j * nb + i, v);
        sv[lj][tx] = v;
    }
    if (!it.up) continue;
    __syncthreads();
    // (j, i) tile: element (row = global col pj, col = global row pi) = same value
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int li = ty + 8 * q;  // becomes the column of the transposed block
        const int64_t r = bj * 32 + tx, c = bi * 32 + li;
        store_any(it.up, it.p_up, c * nb + r, sv[tx][li]);
    }
    }
}

template <typename F>
void dispatch_p(mp_precision p, F&& f) {
    if (p == MP_HALF) f(std::integral_constant<int, 0>{});
    else if (p == MP_SINGLE) f(std::integral_constant<int, 1>{});
    else f(std::integral_constant<int, 2>{});
}

}  // namespace

void launch_ew_binary(Ctx* ctx, cudaStream_t s, int op, const Array& a, const Array& b,
                      Array& out) {
    const int g = grid_for(a.size(), 256, ctx->sm_count);
    dispatch_p(a.prec, [&](auto pa) {
        dispatch_p(b.prec, [&](auto pb) {
            constexpr int PA = decltype(pa)::value, PB = decltype(pb)::value;
            constexpr int PO = PA > PB ? PA : PB;
            ew_binary_kernel<PA, PB, PO><<<g, 256, 0, s>>>(
                op, static_cast<const ST<PA>*>(a.data), a.ld, static_cast<const ST<PB>*>(b.data),
                b.ld, static_cast<ST<PO>*>(out.data), out.ld, a.rows, a.cols);
        });
    });
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

void launch_ew_scalar(Ctx* ctx, cudaStream_t s, int op, const Array& a, double v, Array& out) {
    const int g = grid_for(a.size(), 256, ctx->sm_count);
    dispatch_p(a.prec, [&](auto pa) {
        constexpr int P = decltype(pa)::value;
        ew_scalar_kernel<P><<<g, 256, 0, s>>>(op, static_cast<const ST<P>*>(a.data), a.ld,
                                             static_cast<ST<P>*>(out.data), out.ld, a.rows,
                                             a.cols, v);
    });
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

void launch_ew_unary(Ctx* ctx, cudaStream_t s, int op, const Array& a, Array& out) {
    const int g = grid_for(a.size(), 256, ctx->sm_count);
    dispatch_p(a.prec, [&](auto pa) {
        constexpr int P = decltype(pa)::value;
        ew_unary_kernel<P><<<g, 256, 0, s>>>(op, static_cast<const ST<P>*>(a.data), a.ld,
                                            static_cast<ST<P>*>(out.data), out.ld, a.rows,
                                            a.cols);
    });
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

double run_reduce(Ctx* ctx, cudaStream_t s, int op, const Array& a) {
    auto* part = static_cast<double*>(ctx->ensure_scratch(
        kRedBlocks * (sizeof(double) + sizeof(int64_t)) + 64, 0));
    auto* part_i = reinterpret_cast<int64_t*>(part + kRedBlocks);
    double* out = reinterpret_cast<double*>(part_i + kRedBlocks);
    double first = 0.0;
    dispatch_p(a.prec, [&](auto pa) {
        constexpr int P = decltype(pa)::value;
        reduce_pass1<P><<<kRedBlocks, kRedThreads, 0, s>>>(op, static_cast<const ST<P>*>(a.data),
                                                          a.ld, a.rows, a.cols, part, part_i);
    });
    // first element (for the NaN-stickiness rule of min/max), as a double
    double* firstd = out + 1;
    launch_convert(ctx, s, a.prec, a.data, 1, MP_DOUBLE, firstd, 1, 1, 1);
    MP_CUDA(cudaMemcpyAsync(&first, firstd, sizeof(double), cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    reduce_pass2<<<1, 32, 0, s>>>(op, part, part_i, kRedBlocks, first, out);
    count_launch(ctx, 2);
    double r = 0.0;
    MP_CUDA(cudaMemcpyAsync(&r, out, sizeof(double), cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    if (op == 4) r /= static_cast<double>(a.size());
    return r;
}

void launch_transpose_raw(Ctx* ctx, cudaStream_t s, mp_precision p, const void* in,
                          int64_t ldi, int64_t rows, int64_t cols, void* out, int64_t ldo) {
    if (rows == 0 || cols == 0) return;
    dim3 grid(static_cast<unsigned>((rows + 31) / 32), static_cast<unsigned>((cols + 31) / 32));
    dim3 block(32, 8);
    dispatch_p(p, [&](auto pp) {
        constexpr int P = decltype(pp)::value;
        transpose_kernel<ST<P>><<<grid, block, 0, s>>>(static_cast<const ST<P>*>(in), ldi, rows,
                                                      cols, static_cast<ST<P>*>(out), ldo);
    });
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

void launch_transpose(Ctx* ctx, cudaStream_t s, const Array& a, Array& out) {
    launch_transpose_raw(ctx, s, a.prec, a.data, a.ld, a.rows, a.cols, out.data, out.ld);
}

void launch_diag(Ctx* ctx, cudaStream_t s, const Array& a, Array& out) {
    const int64_t n = a.rows < a.cols ? a.rows : a.cols;
    if (n == 0) return;
    dispatch_p(a.prec, [&](auto pp) {
        constexpr int P = decltype(pp)::value;
        diag_kernel<ST<P>><<<grid_for(n, 256, ctx->sm_count), 256, 0, s>>>(
            static_cast<const ST<P>*>(a.data), a.ld, n, static_cast<ST<P>*>(out.data));
    });
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

void launch_fill(Ctx* ctx, cudaStream_t s, mp_precision p, void* dst, int64_t ld, int64_t rows,
                 int64_t cols, double value) {
    if (rows * cols == 0) return;
    const int g = grid_for(rows * cols, 256, ctx->sm_count);
    if (p == MP_HALF) {
        // host-side encode of the constant (value is a plain literal here)
        const __half h = __double2half(value);
        fill_kernel<<<g, 256, 0, s>>>(static_cast<uint16_t*>(dst), ld, rows, cols,
                                      *reinterpret_cast<const uint16_t*>(&h));
    } else if (p == MP_SINGLE) {
        fill_kernel<<<g, 256, 0, s>>>(static_cast<float*>(dst), ld, rows, cols,
                                      static_cast<float>(value));
    } else {
        fill_kernel<<<g, 256, 0, s>>>(static_cast<double*>(dst), ld, rows, cols, value);
    }
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

void launch_zero_triangle(Ctx* ctx, cudaStream_t s, mp_precision p, void* A, int64_t lda,
                          int64_t n, bool upper) {
    if (n <= 1) return;
    const int g = grid_for(n * n, 256, ctx->sm_count);
    dispatch_p(p, [&](auto pp) {
        constexpr int P = decltype(pp)::value;
        zero_triangle_kernel<ST<P>><<<g, 256, 0, s>>>(static_cast<ST<P>*>(A), lda, n, upper);
    });
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

void launch_mirror_lower(Ctx* ctx, cudaStream_t s, mp_precision p, void* A, int64_t lda,
                         int64_t n) {
    if (n <= 1) return;
    const int g = grid_for(n * n, 256, ctx->sm_count);
    dispatch_p(p, [&](auto pp) {
        constexpr int P = decltype(pp)::value;
        mirror_lower_kernel<ST<P>><<<g, 256, 0, s>>>(static_cast<ST<P>*>(A), lda, n);
    });
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

void launch_logdiag_sum(Ctx* ctx, cudaStream_t s, mp_precision p, const void* A, int64_t lda,
                        int64_t n, double* dev_out) {
    dispatch_p(p, [&](auto pp) {
        constexpr int P = decltype(pp)::value;
        logdiag_kernel<P><<<1, 256, 0, s>>>(static_cast<const ST<P>*>(A), lda, n, dev_out);
    });
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

void launch_matern_tile(Ctx* ctx, cudaStream_t s, mp_precision p, void* dst, int64_t ld,
                        int64_t row0, int64_t col0, int64_t rows, int64_t cols, int64_t side,
                        double nu, double range, double variance) {
    const int g = grid_for(rows * cols, 256, ctx->sm_count);
    dispatch_p(p, [&](auto pp) {
        constexpr int P = decltype(pp)::value;
        matern_grid_kernel<P><<<g, 256, 0, s>>>(static_cast<ST<P>*>(dst), ld, row0, col0, rows,
                                                cols, side, nu, range, variance);
    });
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

}  // namespace mpcr

namespace mpcr {
void launch_matern_tiles(Ctx* ctx, cudaStream_t s, const void* items, int64_t count, int64_t nb,
                         const double* x, const double* y, int64_t side, double nu, double range,
                         double variance, double nugget) {
    if (count == 0) return;
    if (nb % 32) fail(MP_INVALID_PARAM, "matern: batched generation needs tiles of a multiple of 32");
    // ~64 CTAs per SM over the launch (balanced tail), each walking several blocks
    const int64_t blocks = (nb / 32) * (nb / 32);
    const int64_t per_item = std::max<int64_t>(1, std::min<int64_t>(blocks, (64LL * ctx->sm_count + count - 1) / count));
    const dim3 g(static_cast<unsigned>(per_item), static_cast<unsigned>(count));
    const auto* it = static_cast<const MaternItem*>(items);
    if (x)
        matern_tiles_kernel<false><<<g, 256, 0, s>>>(it, nb, x, y, side, nu, range, variance, nugget);
    else
        matern_tiles_kernel<true><<<g, 256, 0, s>>>(it, nb, x, y, side, nu, range, variance, nugget);
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

size_t matern_item_bytes() { return sizeof(MaternItem); }
void matern_item_fill(void* dst, void* lo, void* up, int p_lo, int p_up, int64_t row0, int64_t col0) {
    *static_cast<MaternItem*>(dst) = MaternItem{lo, up, p_lo, p_up, row0, col0};
}

void launch_matern_points(Ctx* ctx, cudaStream_t s, mp_precision p, void* dst, int64_t ld,
                          int64_t row0, int64_t col0, int64_t rows, int64_t cols, const double* x,
                          const double* y, double nu, double range, double variance,
                          double nugget) {
    const int g = grid_for(rows * cols, 256, ctx->sm_count);
    dispatch_p(p, [&](auto pp) {
        constexpr int P = decltype(pp)::value;
        matern_points_kernel<P><<<g, 256, 0, s>>>(static_cast<ST<P>*>(dst), ld, row0, col0, rows,
                                                  cols, x, y, nu, range, variance, nugget);
    });
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}
}  // namespace mpcr
