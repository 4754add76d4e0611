#include <cstdio>
#include <cuda_runtime.h>
constexpr int PB = 64, PT = 256;
template <typename T>
__device__ int factor_block(T (*D)[PB + 1], int bb, int* s_fail, T* s_inv, long long* tr) {
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    if (tid == 0) *s_fail = -1;
    __syncthreads();
    for (int c0 = 0; c0 < bb; c0 += 16) {
        const int w = min(16, bb - c0);
        if (tid == 0) tr[0] -= clock64();
        if (warp == 0) {
            T r[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) r[j] = (lane < w && j <= lane) ? D[c0 + lane][c0 + j] : T(0);
            int fail = -1;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                if (j < w && fail < 0) {
                    const T djj = __shfl_sync(0xffffffffu, r[j], j);
                    if (!(djj > T(0))) {
                        fail = j;
                    } else {
                        // one reciprocal per pivot instead of a divide per element
                        const T inv = rsqrt(djj);  // MUFU seed + Newton, ~1 ulp
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
            if (lane < w) {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (j <= lane) D[c0 + lane][c0 + j] = r[j];
            }
            if (lane == 0 && fail >= 0) *s_fail = c0 + fail;
        }
        __syncthreads();
        if (tid == 0) { long long c = clock64(); tr[0] += c; tr[1] -= c; }
        if (*s_fail >= 0) return *s_fail;
        // (ii) rows below: x * L_ss^T = D[i][c0..c0+w) by forward substitution
        // (4 threads per row, each an interleaved quarter of every dot product)
        {
            const int part = tid % 4;
            for (int i = c0 + w + tid / 4; i < bb; i += PT / 4) {
                T x[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    if (j < w) {
                        T s = T(0);
#pragma unroll
                        for (int t = 0; t < j; ++t)
                            if ((t & 3) == part) s += x[t] * D[c0 + j][c0 + t];
                        s += __shfl_xor_sync(0xffffffffu, s, 1);
                        s += __shfl_xor_sync(0xffffffffu, s, 2);
                        x[j] = (D[i][c0 + j] - s) * s_inv[c0 + j];
                    } else {
                        x[j] = T(0);
                    }
                }
                if (part == 0)
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (j < w) D[i][c0 + j] = x[j];
            }
        }
        __syncthreads();
        if (tid == 0) { long long c = clock64(); tr[1] += c; tr[2] -= c; }
        // (iii)
        // column oc and rows orow + 4q
        const int oc = tid % PB, orow = tid / PB;
        if (oc >= c0 + w && oc < bb) {
            T lc[16];
#pragma unroll
            for (int t = 0; t < 16; ++t) lc[t] = t < w ? D[oc][c0 + t] : T(0);
#pragma unroll 4
            for (int q = 0; q < PB / 4; ++q) {
                const int r = orow + 4 * q;
                if (r >= oc && r < bb) {
                    T s = D[r][oc];
#pragma unroll
                    for (int t = 0; t < 16; ++t) s -= D[r][c0 + t] * lc[t];
                    D[r][oc] = s;
                }
            }
        }
        __syncthreads();
        if (tid == 0) tr[2] += clock64();
    }
    return -1;
}


__global__ void kern(const double* A, double* out, long long* tr) {
    __shared__ double D[PB][PB + 1];
    __shared__ double s_inv[PB];
    __shared__ int s_fail;
    __shared__ long long t[3];
    if (threadIdx.x < 3) t[threadIdx.x] = 0;
    for (int rep = 0; rep < 10; ++rep) {
        for (int idx = threadIdx.x; idx < PB * PB; idx += PT) D[idx % PB][idx / PB] = A[idx];
        __syncthreads();
        factor_block<double>(D, PB, &s_fail, s_inv, t);
        __syncthreads();
    }
    for (int idx = threadIdx.x; idx < PB * PB; idx += PT) out[idx] = D[idx % PB][idx / PB];
    if (threadIdx.x < 3) tr[threadIdx.x] = t[threadIdx.x] / 10;
}
int main() {
    const int n = PB;
    double h[n * n];
    for (int j = 0; j < n; ++j) for (int i = 0; i < n; ++i) h[j * n + i] = (i == j ? n : 0.0) + 1.0 / (1 + i + j);
    double *A, *O; long long* tr;
    cudaMalloc(&A, sizeof(h)); cudaMalloc(&O, sizeof(h)); cudaMalloc(&tr, 64);
    cudaMemcpy(A, h, sizeof(h), cudaMemcpyHostToDevice);
    kern<<<1, PT>>>(A, O, tr);
    long long t[3]; cudaMemcpy(t, tr, 24, cudaMemcpyDeviceToHost);
    printf("factor_block 64x64 cycles: (i) warp piece %lld  (ii) panel solve %lld  (iii) update %lld  total %lld  err %s\n", t[0], t[1], t[2], t[0]+t[1]+t[2], cudaGetErrorString(cudaGetLastError()));
}
