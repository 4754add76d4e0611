// Diagonal-block device routine of the cooperative POTRF (potrf.cu): factor
// a 64 x 64 block and invert the factor, one CTA of PT = 256 threads with the
// block in shared memory.  Included inside namespace mpcr::<anon> by potrf.cu
// (and by tools/micro/factor_bench.cu for timing); expects PB = 64, PT = 256.
#pragma once

#ifndef FB_MARK  // phase stamps for tools/micro/factor_bench.cu
#define FB_MARK(slot)
#endif

// 1 / sqrt(x) without a slow-path branch (the pivot chain stays one basic
// block): hardware approximation + two Newton steps.  Non-positive or NaN x
// gives NaN (the caller has already flagged the pivot).
__device__ __forceinline__ double rsqrt_nr(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x * y, y, 1.0);
    y = fma(0.5 * y, e, y);
    e = fma(-x * y, y, 1.0);
    return fma(0.5 * y, e, y);
}
__device__ __forceinline__ float rsqrt_nr(float x) { return rsqrtf(x); }

// Warp 0: factor the 64 x 16 panel at columns c0.. (rows >= c0 already
// updated by the columns left of it) right-looking in registers.  Lane l
// holds rows l and l + 32; the panel entries of each column are broadcast by
// shuffles.  The lane holding the next pivot's row updates that pivot from
// its own L entry first, so the pivot chain per column is one shuffle, the
// reciprocal square root and two FP64 operations.
// Pivot test as chol_kernel (`!(d > 0)`, linalg.cpp:121).
template <typename T>
__device__ __forceinline__ void panel_factor(T (*D)[PB + 1], int c0, int* s_fail, T* s_inv) {
    const int lane = threadIdx.x & 31;
    const bool hi = c0 >= 32;  // the panel's diagonal rows sit in the second slot
    const int r0 = lane, r1 = lane + 32;
    T v0[16], v1[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
        v0[c] = D[r0][c0 + c];  // entries above the diagonal are zero
        v1[c] = D[r1][c0 + c];
    }
    int fail = -1;
    T dnext = hi ? v1[0] : v0[0];  // this lane's candidate for the next pivot
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int gj = c0 + j;
        const T d = __shfl_sync(0xFFFFFFFFu, dnext, gj & 31);
        const T inv = rsqrt_nr(d);
        if (!(d > T(0)) && fail < 0) fail = gj;
        const T l0 = r0 > gj ? v0[j] * inv : (r0 == gj ? d * inv : T(0));
        const T l1 = r1 > gj ? v1[j] * inv : (r1 == gj ? d * inv : T(0));
        v0[j] = l0;
        v1[j] = l1;
        const T src = hi ? l1 : l0;
        if (j + 1 < 16) dnext = (hi ? v1[j + 1] : v0[j + 1]) - src * src;
#pragma unroll
        for (int c = j + 1; c < 16; ++c) {
            const T lc = __shfl_sync(0xFFFFFFFFu, src, (c0 + c) & 31);  // L(c0 + c, gj)
            v0[c] -= l0 * lc;
            v1[c] -= l1 * lc;
        }
        if (lane == 0) s_inv[gj] = inv;
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) {
        if (r0 >= c0 + c) D[r0][c0 + c] = v0[c];
        if (r1 >= c0 + c) D[r1][c0 + c] = v1[c];
    }
    if (lane == 0 && fail >= 0 && *s_fail < 0) *s_fail = fail;
}

// All threads: left-looking update of the panel at c0 by the columns left of it,
// D(r, c) -= sum_{t < c0} D(r, t) D(c, t) for r >= c, c in [c0, c0 + 16).
template <typename T>
__device__ __forceinline__ void panel_update(T (*D)[PB + 1], int c0) {
    for (int e = threadIdx.x; e < (PB - c0) * 16; e += PT) {
        const int r = c0 + e / 16, c = c0 + e % 16;
        if (r < c) continue;
        T s0 = D[r][c], s1 = T(0);
        for (int t = 0; t < c0; t += 2) {
            s0 -= D[r][t] * D[c][t];
            s1 -= D[r][t + 1] * D[c][t + 1];
        }
        D[r][c] = s0 + s1;
    }
}

// Warps 1..7: row block ib (rows 16 ib ..) of X = L^-1, once L's row block ib
// is final and X's row blocks above it are done:
//   X_ii = inv(L_ii)                           (warp 1, one column per lane)
//   T_j  = sum_{t = j}^{i-1} L_it X_tj, j < i  (warps 2..7, concurrently)
//   X_ij = -X_ii T_j
template <typename T>
__device__ __forceinline__ void xrow_block(const T (*D)[PB + 1], T (*X)[PB + 1], T* Tm, int ib, const T* s_inv) {
    const int tid = threadIdx.x - 32;  // 0..223
    const int r0 = 16 * ib;
    if (tid < 16) {
        // column cc of inv(L_ii), right-looking: one multiply-add per row on the chain
        const int cc = tid;
        T x[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = (i == cc) ? T(1) : T(0);
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            x[t] *= s_inv[r0 + t];
#pragma unroll
            for (int i = t + 1; i < 16; ++i) x[i] -= D[r0 + i][r0 + t] * x[t];
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) X[r0 + i][r0 + cc] = x[i];
    } else if (tid >= 32) {
        // 2 x 2 output patches of T_j (one patch per thread for ib <= 3)
        for (int e = tid - 32; e < ib * 64; e += PT - 64) {
            const int j = e / 64, pr = (e % 64) % 8, pc = (e % 64) / 8;
            const int cj = 16 * j, rr = r0 + 2 * pr, cc = cj + 2 * pc;
            T s00 = T(0), s01 = T(0), s10 = T(0), s11 = T(0);
            for (int t = cj; t < r0; ++t) {
                const T a0 = D[rr][t], a1 = D[rr + 1][t];
                const T b0 = X[t][cc], b1 = X[t][cc + 1];
                s00 += a0 * b0;
                s01 += a0 * b1;
                s10 += a1 * b0;
                s11 += a1 * b1;
            }
            T* tj = Tm + j * 256;  // T_j(r, c) at c * 16 + r
            tj[(2 * pc) * 16 + 2 * pr] = s00;
            tj[(2 * pc + 1) * 16 + 2 * pr] = s01;
            tj[(2 * pc) * 16 + 2 * pr + 1] = s10;
            tj[(2 * pc + 1) * 16 + 2 * pr + 1] = s11;
        }
    }
    asm volatile("bar.sync 1, 224;" ::: "memory");
    for (int e = tid; e < ib * 256; e += PT - 32) {
        const int j = e / 256, r = (e % 256) % 16, c = (e % 256) / 16;
        T s = T(0);
#pragma unroll
        for (int t = 0; t < 16; ++t) s += X[r0 + r][r0 + t] * Tm[j * 256 + c * 16 + t];
        X[r0 + r][16 * j + c] = -s;
    }
}

// Factor the SPD block in D (lower triangle valid, zeros above, padding rows
// and columns set to the identity) in place into L, and write X = L^-1 (lower,
// zeros above).  Left-looking over four 16-column panels: warp 0 factors
// panel i while warps 1..7 build row block i-1 of the inverse.  Returns the
// first failing column or -1; the pivot reciprocals go to s_inv.  Tm holds
// 3 x 256 elements.
template <typename T>
__device__ int factor_invert_block(T (*D)[PB + 1], T (*X)[PB + 1], T* Tm, int* s_fail, T* s_inv) {
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int idx = tid; idx < PB * (PB + 1); idx += PT) (&X[0][0])[idx] = T(0);
    if (tid == 0) *s_fail = -1;
    __syncthreads();
#pragma unroll 1
    for (int pi = 0; pi <= PB / 16; ++pi) {
        const int c0 = 16 * pi;
        FB_MARK(0);
        if (pi >= 1 && pi < PB / 16) {
            panel_update(D, c0);
            __syncthreads();
        }
        FB_MARK(1);
        if (warp == 0) {
            if (pi < PB / 16) panel_factor(D, c0, s_fail, s_inv);
        } else if (pi >= 1) {
            xrow_block<T>(D, X, Tm, pi - 1, s_inv);
        }
        FB_MARK(2);
        __syncthreads();
        FB_MARK(3);
    }
    return *s_fail;
}
