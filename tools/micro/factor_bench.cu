// Times the POTRF diagonal-block routine (csrc/potrf_block.cuh) on one CTA:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2406_02701_b200/csrc \
//        tools/micro/factor_bench.cu -o tools/micro/factor_bench
// -DFB_STAMP=<tid> also prints per-phase clocks of that thread.
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>

namespace bench {
constexpr int PB = 64, PT = 256;
#ifdef FB_STAMP
__device__ long long g_st[8][4];
#define FB_MARK(slot)                                              \
    do {                                                           \
        if (threadIdx.x == FB_STAMP) g_st[pi][slot] = clock64();   \
    } while (0)
#endif
#include "potrf_block.cuh"

__global__ void __launch_bounds__(PT, 1) kern(const double* A, double* out, double* outx, long long* tr) {
    extern __shared__ double dyn[];
    double (*D)[PB + 1] = reinterpret_cast<double (*)[PB + 1]>(dyn);
    double (*X)[PB + 1] = reinterpret_cast<double (*)[PB + 1]>(dyn + PB * (PB + 1));
    double* Tm = dyn + 2 * PB * (PB + 1);
    __shared__ double s_inv[PB];
    __shared__ int s_fail;
    long long tf = 0;
    int fail = 0;
    for (int rep = 0; rep < 10; ++rep) {
        for (int idx = threadIdx.x; idx < PB * PB; idx += PT) {
            const int r = idx % PB, c = idx / PB;
            D[r][c] = r >= c ? A[idx] : 0.0;
        }
        __syncthreads();
        const long long t0 = clock64();
        fail = factor_invert_block<double>(D, X, Tm, &s_fail, s_inv);
        const long long t1 = clock64();
        tf += t1 - t0;
        __syncthreads();
    }
    for (int idx = threadIdx.x; idx < PB * PB; idx += PT) {
        const int r = idx % PB, c = idx / PB;
        out[idx] = r >= c ? D[r][c] : 0.0;
        outx[idx] = X[r][c];
    }
    if (threadIdx.x == 0) {
        tr[0] = tf / 10;
        tr[1] = fail;
    }
}
}  // namespace bench

int main() {
    const int n = bench::PB;
    static double h[n * n], o[n * n], ox[n * n];
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) h[j * n + i] = (i == j ? n : 0.0) + 1.0 / (1 + i + j);
    double *A, *O, *OX;
    long long* tr;
    cudaMalloc(&A, sizeof(h));
    cudaMalloc(&O, sizeof(h));
    cudaMalloc(&OX, sizeof(h));
    cudaMalloc(&tr, 64);
    cudaMemcpy(A, h, sizeof(h), cudaMemcpyHostToDevice);
    const int shm = (2 * n * (n + 1) + 3 * 256) * 8;
    cudaFuncSetAttribute(bench::kern, cudaFuncAttributeMaxDynamicSharedMemorySize, shm);
    bench::kern<<<1, bench::PT, shm>>>(A, O, OX, tr);
    long long t[2];
    cudaMemcpy(t, tr, 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(o, O, sizeof(o), cudaMemcpyDeviceToHost);
    cudaMemcpy(ox, OX, sizeof(ox), cudaMemcpyDeviceToHost);
    double err = 0, errx = 0;  // residuals of L L^T vs A (lower) and L X vs I
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            if (j <= i) {
                double s = 0;
                for (int k = 0; k <= j; ++k) s += o[k * n + i] * o[k * n + j];
                err = fmax(err, fabs(s - h[j * n + i]));
            }
            double s = 0;
            for (int k = 0; k < n; ++k) s += o[k * n + i] * ox[j * n + k];
            errx = fmax(errx, fabs(s - (i == j ? 1.0 : 0.0)));
        }
#ifdef FB_STAMP
    static long long st[8][4];
    cudaMemcpyFromSymbol(st, bench::g_st, sizeof(st));
    for (int p = 0; p <= 4; ++p)
        printf("thread %d phase %d: panel update %lld, own work %lld, wait %lld\n", FB_STAMP, p, st[p][1] - st[p][0],
               st[p][2] - st[p][1], st[p][3] - st[p][2]);
#endif
    printf("64x64 factor+inverse %lld cycles, fail %lld, max|LL^T-A| %.2e, max|LX-I| %.2e (%s)\n", t[0], t[1],
           err, errx, cudaGetErrorString(cudaGetLastError()));
}
