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
// holds rows l and l + 32.  Per pivot only the pivot itself is shuffled: the
// lane holding the next pivot's row updates that pivot from its own L entry
// first (so the chain per column is one shuffle, the reciprocal square root
// and two FP64 operations), and the column's 16 panel entries are broadcast
// through shared memory (cb, 2 x 16 elements) for the rank-1 update.
// Pivot test as chol_kernel (`!(d > 0)`, linalg.cpp:121).
template <typename T, bool HI>
__device__ __forceinline__ void panel_factor_t(T (*D)[PB + 1], int c0, int* s_fail, T* s_inv, T (*cb)[16]) {
    // HI: c0 >= 32, the panel's rows all sit in the second slot (rows 32..63)
    // and the first slot is zero -- it is skipped
    const int lane = threadIdx.x & 31;
    const int r0 = lane, r1 = lane + 32;
    const int pr = (HI ? r1 : r0) - c0;  // this lane's row within the panel's diagonal piece
    T v0[16], v1[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
        v0[c] = HI ? T(0) : D[r0][c0 + c];  // entries above the diagonal are zero
        v1[c] = D[r1][c0 + c];
    }
    int fail = -1;
    T dnext = HI ? v1[0] : v0[0];  // this lane's candidate for the next pivot
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int gj = c0 + j;
        const T d = __shfl_sync(0xFFFFFFFFu, dnext, gj & 31);
        const T inv = rsqrt_nr(d);
        if (!(d > T(0)) && fail < 0) fail = gj;
        T l0 = T(0);
        if (!HI) l0 = r0 > gj ? v0[j] * inv : (r0 == gj ? d * inv : T(0));
        const T l1 = r1 > gj ? v1[j] * inv : (r1 == gj ? d * inv : T(0));
        if (!HI) v0[j] = l0;
        v1[j] = l1;
        const T src = HI ? l1 : l0;
        if (j + 1 < 16) {
            dnext = (HI ? v1[j + 1] : v0[j + 1]) - src * src;
            if (pr > j && pr < 16) cb[j & 1][pr] = src;  // L(c0 + pr, gj)
            __syncwarp();
#pragma unroll
            for (int c = j + 1; c < 16; ++c) {
                const T lc = cb[j & 1][c];
                if (!HI) v0[c] -= l0 * lc;
                v1[c] -= l1 * lc;
            }
        }
        if (lane == 0) s_inv[gj] = inv;
    }
#pragma unroll
    for (int c = 0; c < 16; ++c) {
        if (!HI && r0 >= c0 + c) D[r0][c0 + c] = v0[c];
        if (r1 >= c0 + c) D[r1][c0 + c] = v1[c];
    }
    if (lane == 0 && fail >= 0 && *s_fail < 0) *s_fail = fail;
}

template <typename T>
__device__ __forceinline__ void panel_factor(T (*D)[PB + 1], int c0, int* s_fail, T* s_inv, T (*cb)[16]) {
    if (c0 >= 32) panel_factor_t<T, true>(D, c0, s_fail, s_inv, cb);
    else panel_factor_t<T, false>(D, c0, s_fail, s_inv, cb);
}

// All threads: left-looking update of the panel at C0 by the columns left of
// it, D(r, c) -= sum_{t < C0} D(r, t) D(c, t) for r >= c, c in [C0, C0 + 16).
// Compile-time trip counts: the loads of all of a thread's elements are in
// flight together.
template <typename T, int C0>
__device__ __forceinline__ void panel_update_t(T (*D)[PB + 1]) {
    constexpr int NE = (PB - C0) * 16 / PT;  // elements per thread
    int r[NE], c[NE];
    T s0[NE], s1[NE];
#pragma unroll
    for (int q = 0; q < NE; ++q) {
        const int e = threadIdx.x + q * PT;
        r[q] = C0 + e / 16;
        c[q] = C0 + e % 16;
        s0[q] = D[r[q]][c[q]];
        s1[q] = T(0);
    }
#pragma unroll
    for (int t = 0; t < C0; t += 2) {
#pragma unroll
        for (int q = 0; q < NE; ++q) {
            s0[q] -= D[r[q]][t] * D[c[q]][t];
            s1[q] -= D[r[q]][t + 1] * D[c[q]][t + 1];
        }
    }
#pragma unroll
    for (int q = 0; q < NE; ++q)
        if (r[q] >= c[q]) D[r[q]][c[q]] = s0[q] + s1[q];
}

template <typename T>
__device__ __forceinline__ void panel_update(T (*D)[PB + 1], int c0) {
    if (c0 == 16) panel_update_t<T, 16>(D);
    else if (c0 == 32) panel_update_t<T, 32>(D);
    else if (c0 == 48) panel_update_t<T, 48>(D);
}

// Warp 1, lanes 0..15: Xd_q = inv(L_qq) for the 16 x 16 diagonal piece q
// (one column per lane, right-looking: one multiply-add per row on the
// chain); Xd_q(r, c) at Xd[256 q + 16 r + c], zeros above the diagonal.
template <typename T>
__device__ __forceinline__ void diag_inverse16(const T (*D)[PB + 1], T* Xd, int q, const T* s_inv) {
    const int cc = threadIdx.x & 15, r0 = 16 * q;
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
    for (int i = 0; i < 16; ++i) Xd[256 * q + 16 * i + cc] = x[i];
}

// Factor the SPD block in D (lower triangle valid, zeros above, padding rows
// and columns set to the identity) in place into L, and write the inverses
// of its four 16 x 16 diagonal pieces to Xd.  Left-looking over 16-column
// panels: warp 0 factors panel i while warp 1 inverts the diagonal piece of
// panel i-1.  Returns the first failing column or -1; the pivot reciprocals
// go to s_inv.
template <typename T>
__device__ int factor_block_diag(T (*D)[PB + 1], T* Xd, int* s_fail, T* s_inv) {
    const int tid = threadIdx.x, warp = tid >> 5;
    __shared__ T cb[2][16];
    if (tid == 0) *s_fail = -1;
    __syncthreads();
#pragma unroll 1
    for (int pi = 0; pi <= PB / 16; ++pi) {
        const int c0 = 16 * pi;
        if (pi >= 1 && pi < PB / 16) {
            panel_update(D, c0);
            __syncthreads();
        }
        FB_MARK(0);
        if (warp == 0) {
            if (pi < PB / 16) panel_factor(D, c0, s_fail, s_inv, cb);
        } else if (warp == 1 && pi >= 1 && (tid & 31) < 16) {
            diag_inverse16<T>(D, Xd, pi - 1, s_inv);
        }
        FB_MARK(1);
        __syncthreads();
    }
    return *s_fail;
}

// In place X = A L^-T for the 64-row block in As, blocked by the 16-column
// pieces of L (lower, in Ls) with their inverses Xd:
//   Y_q = A_q - sum_{p < q} X_p L_qp^T,   X_q = Y_q Xd_q^T.
// Thread (r = tid % 64, g = tid / 64) owns columns g, g+4, g+8, g+12 of each piece.
template <typename T>
__device__ __forceinline__ void trsm_block(T (*As)[PB + 1], const T (*Ls)[PB + 1], const T* Xd) {
    const int r = threadIdx.x & 63, g = threadIdx.x >> 6;
#pragma unroll
    for (int q = 0; q < PB / 16; ++q) {
        const int q0 = 16 * q;
        T y[4], z[4] = {};
#pragma unroll
        for (int m = 0; m < 4; ++m) y[m] = As[r][q0 + g + 4 * m];
#pragma unroll
        for (int t = 0; t < q0; t += 2) {
            const T a0 = As[r][t], a1 = As[r][t + 1];
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                y[m] -= a0 * Ls[q0 + g + 4 * m][t];
                z[m] -= a1 * Ls[q0 + g + 4 * m][t + 1];
            }
        }
#pragma unroll
        for (int m = 0; m < 4; ++m) As[r][q0 + g + 4 * m] = y[m] + z[m];
        __syncthreads();
        T x[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const T* xr = Xd + 256 * q + 16 * (g + 4 * m);  // zeros above the diagonal
            T s0 = T(0), s1 = T(0);
#pragma unroll
            for (int u = 0; u < 16; u += 2) {
                s0 += As[r][q0 + u] * xr[u];
                s1 += As[r][q0 + u + 1] * xr[u + 1];
            }
            x[m] = s0 + s1;
        }
        __syncthreads();
#pragma unroll
        for (int m = 0; m < 4; ++m) As[r][q0 + g + 4 * m] = x[m];
        __syncthreads();
    }
}

// X = L^-1 (64 x 64, zeros above) from L (Ls) and the diagonal-piece
// inverses Xd, row block by row block: X_ij = -Xd_i sum_{t=j}^{i-1} L_it X_tj.
// Tm holds 3 x 256 elements.
template <typename T>
__device__ void dinv_block(const T (*Ls)[PB + 1], const T* Xd, T (*X)[PB + 1], T* Tm) {
    const int tid = threadIdx.x;
    for (int idx = tid; idx < PB * PB; idx += PT) {
        const int r = idx % PB, c = idx / PB;
        X[r][c] = (r / 16 == c / 16) ? Xd[256 * (r / 16) + 16 * (r % 16) + c % 16] : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int i = 1; i < PB / 16; ++i) {
        const int r0 = 16 * i;
        // T_j = sum_{t < r0} L(r0 + rr, t) X(t, 16 j + c): X is zero above the
        // diagonal, so the uniform range covers t in [16 j, r0)
#pragma unroll
        for (int q = 0; q < i; ++q) {
            const int e = tid + q * PT;  // 256 i elements
            const int j = e / 256, rr = e % 16, c = (e % 256) / 16;
            T s0 = T(0), s1 = T(0);
#pragma unroll
            for (int t = 0; t < r0; t += 2) {
                s0 += Ls[r0 + rr][t] * X[t][16 * j + c];
                s1 += Ls[r0 + rr][t + 1] * X[t + 1][16 * j + c];
            }
            Tm[e] = s0 + s1;  // T_j(rr, c) at 256 j + 16 c + rr
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < i; ++q) {
            const int e = tid + q * PT;
            const int j = e / 256, rr = e % 16, c = (e % 256) / 16;
            const T* xr = Xd + 256 * i + 16 * rr;  // zeros above the diagonal
            T s0 = T(0), s1 = T(0);
#pragma unroll
            for (int u = 0; u < 16; u += 2) {
                s0 += xr[u] * Tm[256 * j + 16 * c + u];
                s1 += xr[u + 1] * Tm[256 * j + 16 * c + u + 1];
            }
            X[r0 + rr][16 * j + c] = -(s0 + s1);
        }
        __syncthreads();
    }
}
