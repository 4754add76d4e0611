// Latency probes on one CTA (cycles per dependent operation): DFMA, FFMA,
// double rsqrt, LDS.64, SHFL of a double, __syncthreads with 256 threads.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) probe(double* out, long long* t, int iters) {
    __shared__ double sm[512];
    const int tid = threadIdx.x;
    sm[tid] = tid;
    sm[tid + 256] = tid;
    __syncthreads();
    double x = 1.0 + tid * 1e-9, y = 0.999999;
    float xf = 1.0f + tid * 1e-6f, yf = 0.99999f;
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = fma(x, y, 1e-9);
    t1 = clock64();
    if (tid == 0) t[0] = (t1 - t0) / iters;
    // FFMA chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) xf = fmaf(xf, yf, 1e-6f);
    t1 = clock64();
    if (tid == 0) t[1] = (t1 - t0) / iters;
    // rsqrt chain
    double z = 2.0 + tid;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) z = rsqrt(z) + 1.5;
    t1 = clock64();
    if (tid == 0) t[2] = (t1 - t0) / iters;
    // LDS chain (pointer chasing through indices)
    int idx = tid;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) idx = ((int)sm[idx] + 1) & 255;
    t1 = clock64();
    if (tid == 0) t[3] = (t1 - t0) / iters;
    // SHFL chain (double)
    double s = tid;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) s = __shfl_sync(0xffffffffu, s, (tid + 1) & 31) + 1.0;
    t1 = clock64();
    if (tid == 0) t[4] = (t1 - t0) / iters;
    // syncthreads
    t0 = clock64();
    for (int i = 0; i < iters; ++i) __syncthreads();
    t1 = clock64();
    if (tid == 0) t[5] = (t1 - t0) / iters;
    // syncthreads with an STS -> LDS handoff (producer thread 0, all consume)
    double h = 0;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (tid == (i & 255)) sm[i & 1] = h + 1.0;
        __syncthreads();
        h = sm[i & 1];
    }
    t1 = clock64();
    if (tid == 0) t[6] = (t1 - t0) / iters;
    // DMUL chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = x * y;
    t1 = clock64();
    if (tid == 0) t[7] = (t1 - t0) / iters;
    out[tid] = x + xf + z + idx + s + h;
}

int main() {
    double* o;
    long long* t;
    cudaMalloc(&o, 256 * 8);
    cudaMalloc(&t, 8 * 8);
    probe<<<1, 256>>>(o, t, 1000);
    probe<<<1, 256>>>(o, t, 1000);
    long long h[8];
    cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
    printf("cycles: DFMA %lld  FFMA %lld  rsqrt(double)+add %lld  LDS %lld  SHFL.f64+add %lld  syncthreads %lld  "
           "sts-sync-lds %lld  DMUL %lld  (%s)\n",
           h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], cudaGetErrorString(cudaGetLastError()));
}
