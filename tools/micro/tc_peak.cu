// Micro-benchmark: tcgen05 tensor-pipe throughput per kind on sm_100a (the
// roofline denominators the bench's blended roofline charges each kernel
// class at).  One CTA per SM; one elected thread issues back-to-back
// tcgen05.mma (M=128, N=256, cta_group::1) from shared-memory operands
// filled with random data (zeros would understate the power draw and
// overstate the clock) into two alternating TMEM accumulators; the pipe is
// never starved by loads, so this is the MMA issue-rate ceiling of a kind.
//   kind::f16  (FP16 in, FP32 acc):  K = 16 per instruction
//   kind::tf32 (TF32 in, FP32 acc):  K = 8
//   kind::i8   (INT8 in, INT32 acc): K = 32
// Usage: tc_peak [seconds_per_kind]  (prints TFLOP/s or TOPS per kind)
#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "../../paper_2406_02701_b200/csrc/tc_ptx.cuh"

using namespace mpcr;

enum Kind { F16 = 0, TF32 = 1, I8 = 2 };

__device__ __forceinline__ void mma_kind(int kind, uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if (kind == F16)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                     "l"(a), "l"(b), "r"(idesc), "r"(acc));
    else if (kind == TF32)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                     "l"(a), "l"(b), "r"(idesc), "r"(acc));
    else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                     "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <int KIND>
__global__ void __launch_bounds__(128, 1) tc_loop(int iters, unsigned seed, int* sink) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* A = sm;              // 128 rows x 128 B (SW128, K-major)
    unsigned char* B = sm + 128 * 128;  // 256 rows x 128 B
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_slot;
    // random operands: bounded finite values of the kind's input format
    for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) {
        unsigned x = (i + 1) * 2654435761u ^ seed ^ (blockIdx.x * 40503u);
        x ^= x >> 13;
        x *= 0x5bd1e995u;
        x ^= x >> 15;
        uint32_t v;
        if (KIND == F16)  // two halves in [-1, 1): sign, exponent 14/13, random mantissa
            v = ((x & 0x83FFu) | 0x3800u) | (((x >> 16) & 0x83FFu) | 0x3400u) << 16;
        else if (KIND == TF32)  // float in [-2, 2)
            v = (x & 0x807FFFFFu) | 0x3F800000u;
        else
            v = x;  // four random int8
        reinterpret_cast<uint32_t*>(sm)[i] = v;
    }
    ptx::fence_proxy_async_smem();
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_barrier_init();
    }
    if (threadIdx.x < 32) ptx::tmem_alloc<512>(&tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    if (threadIdx.x == 0) {
        uint32_t idesc;
        if (KIND == I8)
            idesc = (2u << 4) | (1u << 7) | (1u << 10) | (256u >> 3 << 17) | (128u >> 4 << 24);
        else
            idesc = ptx::umma_idesc(128, 256, false, false, KIND == F16 ? 0u : 2u);
        const uint32_t a0 = ptx::smem_u32(A), b0 = ptx::smem_u32(B);
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // 4 x 32 B K-slices of the 128 B rows
                const uint64_t ad = ptx::umma_desc_sw128(a0 + k * 32, 0, 1024);
                const uint64_t bd = ptx::umma_desc_sw128(b0 + k * 32, 0, 1024);
                mma_kind(KIND, tmem + (it & 1) * 256, ad, bd, idesc, (it > 1 || k > 0) ? 1u : 0u);
            }
        }
        ptx::mma_commit(&bar);
        ptx::mbar_wait(&bar, 0);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x == 0) sink[blockIdx.x] = iters;
    if (threadIdx.x < 32) ptx::tmem_dealloc<512>(tmem);
}

int main(int argc, char** argv) {
    const double secs = argc > 1 ? atof(argv[1]) : 2.0;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int* sink;
    cudaMalloc(&sink, sms * sizeof(int));
    const int smem = (128 + 256) * 128 + 1024;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[3] = {"f16 (FP16 in, FP32 acc)", "tf32 (TF32 in, FP32 acc)", "i8 (INT8 in, INT32 acc)"};
    const double kper[3] = {16, 8, 32};
    for (int kind = 0; kind < 3; ++kind) {
        void (*kern)(int, unsigned, int*) = kind == 0 ? tc_loop<F16> : kind == 1 ? tc_loop<TF32> : tc_loop<I8>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        // calibrate iterations to ~secs/10 per launch, then repeat for secs
        int iters = 20000;
        kern<<<sms, 128, smem>>>(100, 1u, sink);
        cudaEventRecord(e0);
        kern<<<sms, 128, smem>>>(iters, 2u, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        iters = static_cast<int>(iters * (secs * 100.0) / ms);
        if (iters < 1000) iters = 1000;
        double best = 0, sum = 0;
        int reps = 0;
        const auto t0 = std::chrono::steady_clock::now();
        while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < secs) {
            cudaEventRecord(e0);
            kern<<<sms, 128, smem>>>(iters, 3u + reps, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            const double ops = 2.0 * 128 * 256 * kper[kind] * 4.0 * iters * sms;
            const double r = ops / (ms * 1e-3) / 1e12;
            best = r > best ? r : best;
            sum += r;
            ++reps;
        }
        printf("tcgen05 kind::%-26s M=128 N=256: burst %.1f, mean over %.1f s %.1f T%s/s (%d launches)\n",
               names[kind], best, secs, sum / reps, kind == 2 ? "OP" : "FLOP", reps);
    }
    const cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
