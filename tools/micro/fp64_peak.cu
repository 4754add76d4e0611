// Microbenchmark: FP64 throughput of DMMA (mma.sync f64 m16n8k4/k8/k16) vs DFMA on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void dmma_loop(double* out, int iters) {
    double a[K / 2], b[K / 4], c[4] = {0, 0, 0, 0};
    for (int i = 0; i < K / 2; ++i) a[i] = 1.0 + threadIdx.x * 1e-9 + i;
    for (int i = 0; i < K / 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            if (K == 4)
                asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                             : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
            else if (K == 8)
                asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                             : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
            else
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                             : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                             : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                               "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = c[0] + c[1] + c[2] + c[3];
}

__global__ void dfma_loop(double* out, int iters) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
    const double y = 1.0000001, z = 1e-7;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fma(x[i], y, z);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    double* out;
    cudaMalloc(&out, 148 * 8 * 1024 * sizeof(double));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int warps : {4, 8, 16}) {
        const int iters = 20000;
        auto run = [&](auto kern, double flop_per_iter_warp, const char* name) {
            kern<<<sms * 2, warps * 32>>>(out, 10);
            cudaEventRecord(a);
            kern<<<sms * 2, warps * 32>>>(out, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double fl = flop_per_iter_warp * iters * warps * sms * 2;
            printf("%-8s warps/CTA %2d: %.1f TFLOP/s (%.2f ms)\n", name, warps, fl / ms / 1e9, ms);
        };
        run(dmma_loop<4>, 8.0 * 2 * 16 * 8 * 4, "dmma k4");
        run(dmma_loop<8>, 8.0 * 2 * 16 * 8 * 8, "dmma k8");
        run(dmma_loop<16>, 8.0 * 2 * 16 * 8 * 16, "dmma k16");
        run(dfma_loop, 16.0 * 8 * 2 * 32, "dfma");
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
