// Half -> double widening variants at 32768^2 elements (write-heavy stream).
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ double h2d(uint16_t b) { return static_cast<double>(__half2float(__ushort_as_half(b))); }

// (a) output-centric: 16-byte store per group from a 4-byte load, U groups in flight
template <int U>
__global__ void __launch_bounds__(256) widen_out(const uint16_t* __restrict__ in, double* __restrict__ out, int64_t nq) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; t + (U - 1) * stride < nq; t += U * stride) {
        uint32_t v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcs(reinterpret_cast<const uint32_t*>(in) + t + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            double2 o = make_double2(h2d(v[u] & 0xffff), h2d(v[u] >> 16));
            __stcs(reinterpret_cast<double2*>(out) + t + u * stride, o);
        }
    }
}
// (b) input-centric: 16-byte load (8 halves) -> 4 contiguous 16-byte stores
__global__ void __launch_bounds__(256) widen_in(const uint16_t* __restrict__ in, double* __restrict__ out, int64_t n8) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n8; t += stride) {
        const uint4 v = __ldcs(reinterpret_cast<const uint4*>(in) + t);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
        double2* o = reinterpret_cast<double2*>(out) + 4 * t;
#pragma unroll
        for (int q = 0; q < 4; ++q) __stcs(o + q, make_double2(h2d(w[q] & 0xffff), h2d(w[q] >> 16)));
    }
}
// (c) 16-byte load per lane, staged through shared memory, lane-consecutive 16-byte stores
__global__ void __launch_bounds__(256) widen_smem(const uint16_t* __restrict__ in, double* __restrict__ out, int64_t n8) {
    __shared__ double2 buf[8][32 * 4 + 1];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t nwarps = (int64_t)gridDim.x * 8;
    for (int64_t wc = (int64_t)blockIdx.x * 8 + warp; wc * 32 < n8; wc += nwarps) {
        const int64_t t = wc * 32 + lane;
        if (t < n8) {
            const uint4 v = __ldcs(reinterpret_cast<const uint4*>(in) + t);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) buf[warp][lane * 4 + q] = make_double2(h2d(w[q] & 0xffff), h2d(w[q] >> 16));
        }
        __syncwarp();
        double2* o = reinterpret_cast<double2*>(out) + wc * 32 * 4;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t idx = (int64_t)q * 32 + lane;
            if (wc * 32 * 4 + idx < n8 * 4) __stcs(o + idx, buf[warp][q * 32 + lane]);
        }
        __syncwarp();
    }
}

int main() {
    const int64_t n = 32768LL * 32768LL;
    uint16_t* in; double* out;
    cudaMalloc(&in, n * 2); cudaMalloc(&out, n * 8);
    cudaMemset(in, 0x3c, n * 2);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](const char* name, auto launch) {
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(a);
        for (int i = 0; i < 10; ++i) launch();
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
        printf("%-28s %8.1f GB/s (%s)\n", name, n * 10.0 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    for (int blocks_per_sm : {4, 8, 16}) {
        const int g = sms * blocks_per_sm;
        char nm[64];
        snprintf(nm, 64, "out-centric U=4 g=%dx", blocks_per_sm); run(nm, [&] { widen_out<4><<<g, 256>>>(in, out, n / 2); });
        snprintf(nm, 64, "out-centric U=8 g=%dx", blocks_per_sm); run(nm, [&] { widen_out<8><<<g, 256>>>(in, out, n / 2); });
        snprintf(nm, 64, "in-centric g=%dx", blocks_per_sm); run(nm, [&] { widen_in<<<g, 256>>>(in, out, n / 8); });
        snprintf(nm, 64, "smem-staged g=%dx", blocks_per_sm); run(nm, [&] { widen_smem<<<g, 256>>>(in, out, n / 8); });
    }
}
