// Diagonal-block device routines of the cooperative POTRF (potrf.cu): the
// 64 x 64 block factorization and inverse, one CTA of PT threads with the
// block in shared memory.  Included inside namespace mpcr::<anon> by
// potrf.cu (and by tools/micro/factor_bench.cu for timing); expects PB, PT.
#pragma once

#ifndef FB_MARK  // phase markers for tools/micro/factor_bench.cu
#define FB_MARK(slot)
#endif

// ---- diagonal-block kernels (one CTA, 256 threads, D in shared memory) ----

// Factor the bb x bb lower block D in place, left-looking over 16-column
// panels, and leave the inverses of the 16 x 16 diagonal pieces in X:
//   (a) all threads: panel columns -= L(:, <c0) L(panel, <c0)^T
//   (b) warp 0: 16 x 16 diagonal piece in registers (one row per lane,
//       pivots by shuffles), then its inverse (one column per lane)
//   (c) all threads: rows below the piece times the piece's inverse^T
// Every step is parallel except (b).  Pivot test as chol_kernel
// (`!(d > 0)`, linalg.cpp:121).  Returns the failing local column or -1.
template <typename T>
__device__ int factor_block(T (*D)[PB + 1], T (*X)[PB + 1], int bb, int* s_fail, T* s_inv) {
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    if (tid == 0) *s_fail = -1;
    for (int c0 = 0; c0 < bb; c0 += 16) {
        const int w = min(16, bb - c0);
        // (a) left-looking update of the panel (rows c0..bb, columns c0..c0+w)
        if (c0 > 0) {
            const int rows = bb - c0;
            for (int e = tid; e < rows * w; e += PT) {
                const int r = c0 + e / w, c = c0 + e % w;
                if (r >= c) {
                    T s0 = D[r][c], s1 = T(0);
                    int t = 0;
                    for (; t + 1 < c0; t += 2) {
                        s0 -= D[r][t] * D[c][t];
                        s1 -= D[r][t + 1] * D[c][t + 1];
                    }
                    if (t < c0) s0 -= D[r][t] * D[c][t];
                    D[r][c] = s0 + s1;
                }
            }
        }
        __syncthreads();
        FB_MARK(0);
        // (b) diagonal piece: factor in registers, then invert
        if (warp == 0) {
            T r[16];
            const bool row_ok = lane < w;
#pragma unroll
            for (int j = 0; j < 16; ++j) r[j] = (row_ok && j <= lane) ? D[c0 + lane][c0 + j] : T(0);
            int fail = -1;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                if (j < w && fail < 0) {
                    const T djj = __shfl_sync(0xffffffffu, r[j], j);
                    if (!(djj > T(0))) {
                        fail = j;
                    } else {
                        const T inv = rsqrt(djj);  // one reciprocal per pivot
                        const T sd = djj * inv;
                        if (lane > j) r[j] = r[j] * inv;
                        if (lane == j) {
                            r[j] = sd;
                            s_inv[c0 + j] = inv;
                        }
#pragma unroll
                        for (int l = j + 1; l < 16; ++l) {
                            const T v = __shfl_sync(0xffffffffu, r[j], l);  // L[l][j]
                            if (lane >= l) r[l] -= r[j] * v;
                        }
                    }
                }
            }
            if (row_ok) {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (j <= lane) D[c0 + lane][c0 + j] = r[j];
            }
            if (lane == 0 && fail >= 0) *s_fail = c0 + fail;
            __syncwarp();
            FB_MARK(1);
            if (fail < 0 && lane < w) {
                // column `lane` of the piece's inverse: x_i = (e_ci - sum_{t<i} L_it x_t) / L_ii
                const int cc = lane;
                T x[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    T v = T(0);
                    if (i < w && i >= cc) {
                        T s = (i == cc) ? T(1) : T(0);
#pragma unroll
                        for (int t = 0; t < i; ++t)
                            if (t >= cc) s -= D[c0 + i][c0 + t] * x[t];
                        v = s * s_inv[c0 + i];
                    }
                    x[i] = v;
                }
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    if (i < w) X[c0 + i][c0 + cc] = x[i];
            }
        }
        __syncthreads();
        FB_MARK(2);
        if (*s_fail >= 0) return *s_fail;
        // (c) rows below the piece: L21 = A21 * inv(L11)^T, one row per thread
        for (int i = c0 + w + tid; i < bb; i += PT) {
            T a[16];
#pragma unroll
            for (int t = 0; t < 16; ++t) a[t] = t < w ? D[i][c0 + t] : T(0);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                if (j < w) {
                    T s = T(0);
#pragma unroll
                    for (int t = 0; t <= j; ++t) s += a[t] * X[c0 + j][c0 + t];
                    D[i][c0 + j] = s;
                }
            }
        }
        __syncthreads();
        FB_MARK(3);
    }
    return -1;
}

// X = D^-1 for the bb x bb lower block (zeros above the diagonal), from the
// 16 x 16 diagonal inverses factor_block left in X: off-diagonal 16-blocks by
// distance, X_ij = -X_ii * sum_{j<=t<i} D_it X_tj.  Uses Tm (16 x 16 x 3).
template <typename T>
__device__ void invert_block(const T (*D)[PB + 1], T (*X)[PB + 1], T* Tm, int bb, const T* /*s_inv*/) {
    const int tid = threadIdx.x;
    const int nsb = (bb + 15) / 16;
    // clear everything outside the diagonal 16-blocks
    for (int idx = tid; idx < PB * PB; idx += PT) {
        const int r = idx % PB, c = idx / PB;
        if (r / 16 != c / 16 || r >= bb || c >= bb || r < c) X[r][c] = T(0);
    }
    __syncthreads();
    for (int d = 1; d < nsb; ++d) {
        const int nblk = nsb - d;  // blocks (i, i - d)
        // T_b = sum_{t=j}^{i-1} D_it X_tj   (16 x 16 each)
        for (int e = tid; e < nblk * 256; e += PT) {
            const int b = e / 256, r = (e % 256) % 16, cc = (e % 256) / 16;
            const int bi = b + d, bj = b;
            const int row = bi * 16 + r, col = bj * 16 + cc;
            T s = T(0);
            if (row < bb && col < bb)
                for (int t = bj * 16; t < bi * 16; ++t) s += D[row][t] * X[t][col];
            Tm[e] = s;
        }
        __syncthreads();
        for (int e = tid; e < nblk * 256; e += PT) {
            const int b = e / 256, r = (e % 256) % 16, cc = (e % 256) / 16;
            const int bi = b + d, bj = b;
            const int row = bi * 16 + r, col = bj * 16 + cc;
            if (row < bb && col < bb) {
                T s = T(0);
                for (int t = 0; t < 16; ++t) s += X[row][bi * 16 + t] * Tm[b * 256 + cc * 16 + t];
                X[row][col] = -s;
            }
        }
        __syncthreads();
    }
}

