// Times the POTRF diagonal-block routines (csrc/potrf_block.cuh) on one CTA:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2406_02701_b200/csrc \
//        tools/micro/factor_bench.cu -o tools/micro/factor_bench
#include <cstdio>
#include <cuda_runtime.h>

namespace bench {
__device__ long long g_fb[8];
__device__ long long g_last;
#ifdef FB_TRACE
#define FB_MARK(slot)                                   \
    do {                                                \
        if (threadIdx.x == 0) {                         \
            const long long now_ = clock64();           \
            g_fb[slot] += now_ - g_last;                \
            g_last = now_;                              \
        }                                               \
    } while (0)
#endif
constexpr int PB = 64, PT = 256;
#include "potrf_block.cuh"

__global__ void kern(const double* A, double* out, long long* tr) {
    extern __shared__ double dyn[];
    double (*D)[PB + 1] = reinterpret_cast<double (*)[PB + 1]>(dyn);
    double (*X)[PB + 1] = reinterpret_cast<double (*)[PB + 1]>(dyn + PB * (PB + 1));
    double* Tm = dyn + 2 * PB * (PB + 1);
    __shared__ double s_inv[PB];
    __shared__ int s_fail;
    long long tf = 0, ti = 0;
    for (int rep = 0; rep < 10; ++rep) {
        for (int idx = threadIdx.x; idx < PB * PB; idx += PT) D[idx % PB][idx / PB] = A[idx];
        __syncthreads();
        long long t0 = clock64();
        if (threadIdx.x == 0) g_last = t0;
        factor_block<double>(D, X, PB, &s_fail, s_inv);
        __syncthreads();
        long long t1 = clock64();
        invert_block<double>(D, X, Tm, PB, s_inv);
        __syncthreads();
        long long t2 = clock64();
        tf += t1 - t0;
        ti += t2 - t1;
    }
    for (int idx = threadIdx.x; idx < PB * PB; idx += PT) out[idx] = D[idx % PB][idx / PB];
    if (threadIdx.x == 0) {
        tr[0] = tf / 10;
        tr[1] = ti / 10;
        for (int q = 0; q < 4; ++q) tr[2 + q] = g_fb[q] / 10;
    }
}
}  // namespace bench

int main() {
    const int n = bench::PB;
    static double h[n * n], o[n * n];
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) h[j * n + i] = (i == j ? n : 0.0) + 1.0 / (1 + i + j);
    double *A, *O;
    long long* tr;
    cudaMalloc(&A, sizeof(h));
    cudaMalloc(&O, sizeof(h));
    cudaMalloc(&tr, 64);
    cudaMemcpy(A, h, sizeof(h), cudaMemcpyHostToDevice);
    const int shm = (2 * n * (n + 1) + 3 * 256) * 8;
    cudaFuncSetAttribute(bench::kern, cudaFuncAttributeMaxDynamicSharedMemorySize, shm);
    bench::kern<<<1, bench::PT, shm>>>(A, O, tr);
    long long t[6];
    cudaMemcpy(t, tr, 48, cudaMemcpyDeviceToHost);
    cudaMemcpy(o, O, sizeof(o), cudaMemcpyDeviceToHost);
    double err = 0;  // residual of L L^T vs A (lower)
    for (int i = 0; i < n; ++i)
        for (int j = 0; j <= i; ++j) {
            double s = 0;
            for (int k = 0; k <= j; ++k) s += o[k * n + i] * o[k * n + j];
            err = fmax(err, fabs(s - h[j * n + i]));
        }
    printf("64x64 factor %lld cycles (a %lld, b-factor %lld, b-inverse %lld, c %lld), invert %lld cycles, "
           "max|LL^T-A| %.2e  (%s)\n", t[0], t[2], t[3], t[4], t[5], t[1], err, cudaGetErrorString(cudaGetLastError()));
}
