// Times the POTRF diagonal-block routines (csrc/potrf_block.cuh) on one CTA:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2406_02701_b200/csrc \
//        tools/micro/factor_bench.cu -o tools/micro/factor_bench
// Prints cycles of factor_block_diag and of its pieces (panel_update at each
// panel, panel_factor, diag_inverse16), trsm_block and dinv_block, and checks
// L L^T = A, L X = I and the panel solve.
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>

namespace bench {
constexpr int PB = 64, PT = 256;
#include "potrf_block.cuh"

__global__ void __launch_bounds__(PT, 1) kern(const double* A, const double* B, double* out, double* outx,
                                              double* outb, long long* tr) {
    extern __shared__ double dyn[];
    double (*D)[PB + 1] = reinterpret_cast<double (*)[PB + 1]>(dyn);
    double (*X)[PB + 1] = reinterpret_cast<double (*)[PB + 1]>(dyn + PB * (PB + 1));
    double (*As)[PB + 1] = reinterpret_cast<double (*)[PB + 1]>(dyn + 2 * PB * (PB + 1));
    double* Xd = dyn + 3 * PB * (PB + 1);
    double* Tm = Xd + 1024;
    __shared__ double s_inv[PB];
    __shared__ int s_fail;
    long long t[12] = {};
    int fail = 0;
    const int R = 10;
    for (int rep = 0; rep < R; ++rep) {
        for (int idx = threadIdx.x; idx < PB * PB; idx += PT) {
            const int r = idx % PB, c = idx / PB;
            D[r][c] = r >= c ? A[idx] : 0.0;
            As[r][c] = B[idx];
        }
        __syncthreads();
        long long t0 = clock64();
        fail = factor_block_diag<double>(D, Xd, &s_fail, s_inv);
        long long t1 = clock64();
        t[0] += t1 - t0;
        t0 = clock64();
        trsm_block<double>(As, D, Xd);
        __syncthreads();
        t1 = clock64();
        t[1] += t1 - t0;
        t0 = clock64();
        dinv_block<double>(D, Xd, X, Tm);
        __syncthreads();
        t1 = clock64();
        t[2] += t1 - t0;
        // pieces (timing only; X is scratch here and rebuilt below)
        for (int pi = 1; pi < 4; ++pi) {
            t0 = clock64();
            panel_update<double>(X, 16 * pi);
            __syncthreads();
            t1 = clock64();
            t[2 + pi] += t1 - t0;
        }
        __syncthreads();
        t0 = clock64();
        if (threadIdx.x < 32) panel_factor<double>(X, 0, &s_fail, s_inv, reinterpret_cast<double (*)[16]>(Tm));
        __syncthreads();
        t1 = clock64();
        t[6] += t1 - t0;
        t0 = clock64();
        if (threadIdx.x < 16) diag_inverse16<double>(D, Tm, 0, s_inv);
        __syncthreads();
        t1 = clock64();
        t[7] += t1 - t0;
        t0 = clock64();
        __syncthreads();
        t1 = clock64();
        t[8] += t1 - t0;
        dinv_block<double>(D, Xd, X, Tm);
        __syncthreads();
    }
    for (int idx = threadIdx.x; idx < PB * PB; idx += PT) {
        const int r = idx % PB, c = idx / PB;
        out[idx] = r >= c ? D[r][c] : 0.0;
        outx[idx] = X[r][c];
        outb[idx] = As[r][c];
    }
    if (threadIdx.x == 0) {
        for (int q = 0; q < 9; ++q) tr[q] = t[q] / R;
        tr[9] = fail;
    }
}
}  // namespace bench

int main() {
    const int n = bench::PB;
    static double h[n * n], hb[n * n], o[n * n], ox[n * n], ob[n * n];
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
            h[j * n + i] = (i == j ? n : 0.0) + 1.0 / (1 + i + j);
            hb[j * n + i] = std::sin(1.0 + i + 3.0 * j);
        }
    double *A, *B, *O, *OX, *OB;
    long long* tr;
    cudaMalloc(&A, sizeof(h));
    cudaMalloc(&B, sizeof(h));
    cudaMalloc(&O, sizeof(h));
    cudaMalloc(&OX, sizeof(h));
    cudaMalloc(&OB, sizeof(h));
    cudaMalloc(&tr, 128);
    cudaMemcpy(A, h, sizeof(h), cudaMemcpyHostToDevice);
    cudaMemcpy(B, hb, sizeof(h), cudaMemcpyHostToDevice);
    const int shm = (3 * n * (n + 1) + 1024 + 768) * 8;
    cudaFuncSetAttribute(bench::kern, cudaFuncAttributeMaxDynamicSharedMemorySize, shm);
    bench::kern<<<1, bench::PT, shm>>>(A, B, O, OX, OB, tr);
    long long t[10];
    cudaMemcpy(t, tr, sizeof(t), cudaMemcpyDeviceToHost);
    cudaMemcpy(o, O, sizeof(o), cudaMemcpyDeviceToHost);
    cudaMemcpy(ox, OX, sizeof(ox), cudaMemcpyDeviceToHost);
    cudaMemcpy(ob, OB, sizeof(ob), cudaMemcpyDeviceToHost);
    double err = 0, errx = 0, errb = 0;  // L L^T - A, L X - I, X_b L^T - B
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
            double sb = 0;  // (X_b L^T)(i, j) = sum_k X_b(i, k) L(j, k)
            for (int k = 0; k <= j; ++k) sb += ob[k * n + i] * o[k * n + j];
            errb = fmax(errb, fabs(sb - hb[j * n + i]));
        }
    printf("factor_block_diag %lld, trsm_block %lld, dinv_block %lld cycles; pieces: panel_update(16) %lld "
           "(32) %lld (48) %lld, panel_factor %lld, diag_inverse16 %lld, bare sync %lld\n",
           t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7], t[8]);
    printf("fail %lld, max|LL^T-A| %.2e, max|LX-I| %.2e, max|XL^T-B| %.2e (%s)\n", t[9], err, errx, errb,
           cudaGetErrorString(cudaGetLastError()));
}
