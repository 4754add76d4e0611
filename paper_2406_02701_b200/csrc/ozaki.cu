// FP64 (or FP32-output) GEMM of FP16- or FP32-valued operands on the INT8
// tensor cores (Ozaki scheme, exact digit slicing).
//
// Where it serves: the FP64 tiles of the mixed-precision Cholesky are updated
// with panel tiles that are stored in FP16 (the reference converts them to
// double and calls an FP64 GEMM, linalg.cpp:349-356), FP32 tiles with FP32
// panel tiles, and linalg::gemm with FP16 operands and a double C.  B200 runs
// FP64 at 37 TFLOP/s but INT8 MMA at ~4.5 POPS, so the product is rebuilt
// from INT8 products:
//
//   every row r of an operand is scaled by 2^-e_r (e_r: exponent of its
//   largest magnitude) and split into up to S = 6 signed 7-bit digits
//     x = 2^e_r * sum_p d_p 2^(-6-7(p-1)),  d_p in [-64, 64]  (int8).
//   An FP16 row spans at most 40 significant bits below its maximum (2^5 ..
//   2^-24 plus 11 significand bits), and 6 digits hold 41, so the split is
//   EXACT (FP32 rows: exact down to 2^(e_r - 41)).  Only the digits a 128-row
//   block needs are produced and multiplied; int32 group sums are exact
//   (|sum| <= 6 * K * 64^2 < 2^31 for K < 87381; callers split longer K into
//   OZ_MAX_K chunks) and combined in FP64 with one rounding per group: the
//   result is as accurate as a correctly-ordered FP64 dot product.
//
// Kernel: persistent, warp-specialised, 128 x 128 output units drawn from a
// global counter (dynamic scheduling; a problem may carry two panels).
//   warp 0      TMA producer: 4-stage ring of {A 128x128, up to two B 128x128}
//               int8 digit tiles (128B swizzle); draws the units.
//   warp 1      TMEM allocator + MMA issuer (warp-uniform, elect.sync):
//               tcgen05.mma kind::i8 (M=128, N=128, K=32) into 4 rotating
//               int32 TMEM accumulators, one per digit group t = p + q (all
//               pairs of a group share the scale 2^(-12-7(t-2))), groups
//               issued in pairs (g, g-1) sharing the A digit plane.
//   warps 2-13  epilogue (three per TMEM lane quarter, 48/48/32 columns):
//               FP64 running sums in registers; per group sum += 2^(..) acc,
//               then C = alpha * 2^(e_r+e_c) * sum + beta * C rounded once
//               (lower triangle only for SYRK tiles).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "device.cuh"
#include "gemm_tc.hpp"
#include "internal.hpp"
#include "ozaki.hpp"
#include "tc_ptx.cuh"

namespace mpcr {
namespace oz {

constexpr int S = OZ_SLICES;  // digits per value
// A stage holds one A digit plane k-block and up to two B planes: the groups
// are issued in pairs (g, g-1), whose pairs (p, g-p) and (p, g-1-p) share A_p,
// so each A k-block feeds two MMAs (a quarter less operand ingress).
constexpr int BM = 128, BN = 128, BK = 128, STAGES = 4;
constexpr int A_STAGE = BM * BK, B_STAGE = BN * BK;  // 16 KB each
// + barriers, unit ring, the epilogue warps' column scales
// Epilogue: 12 warps, three per TMEM lane quarter, owning output columns
// [0, 48), [48, 96), [96, 128) of the unit (the sums of a thread's row live
// in registers: 48 doubles).
constexpr int EPI_WARPS = 12;
constexpr int CWMAX = 48;
__host__ __device__ constexpr int epi_col0(int g) { return g * 48; }
__host__ __device__ constexpr int epi_cols(int g) { return g < 2 ? 48 : 32; }
constexpr int SMEM_BYTES = STAGES * (A_STAGE + 2 * B_STAGE) + 1024 + 256 + EPI_WARPS * CWMAX * 8;
constexpr int NACC = 4;          // int32 accumulators in flight (MMA runs NACC groups ahead)
constexpr int TMEM_COLS = 512;  // NACC x 128 columns
constexpr int NTHREADS = 32 * (2 + EPI_WARPS);  // producer, MMA issuer, epilogue
constexpr int UR = 4;           // unit ring: the producer runs up to UR units ahead
constexpr int ROWEXP_NONFINITE = 0x7fffffff;

struct Params {
    CUtensorMap map_a, map_b;  // [tiles * S][rows][K] int8
    const OzProblem* problems;
    OzProblem single;
    int32_t nprob;
    int32_t nlower;  // the first nlower problems are lower_only: only their live units are enumerated
    int32_t M, N, K;
    int32_t mblocks, nblocks, kblocks;
    int64_t ldc;
    double alpha, beta;
    const int32_t* rexp_a;  // row exponents of A tile t at rexp_a + t * rexp_stride_a
    const int32_t* rexp_b;
    int64_t rexp_stride_a, rexp_stride_b;
    const int32_t* ndig_a;  // digits per 128-row block: tile t, block b at ndig_a[t * ndig_stride_a + b] (nullptr: all S)
    const int32_t* ndig_b;
    int32_t ndig_stride_a, ndig_stride_b;
    // dynamic unit scheduling: [0] next unit, [1] CTAs finished (the last
    // CTA resets both)
    unsigned int* sched;
    int32_t c_f32;  // C is FP32 (one rounding of the FP64 result), else FP64
    unsigned long long* stats;  // profiling: [0] += sa*sb per output tile, [1] += 1 (or nullptr)
};

// Digit counts of a problem: pairs (dp, dq) with dp <= sa, dq <= sb; groups
// g = sa + sb .. 2.
__device__ __forceinline__ void digits_of(const Params& p, int at, int bt, int m0, int n0, int& sa, int& sb) {
    sa = p.ndig_a ? max(1, min(S, p.ndig_a[at * p.ndig_stride_a + m0 / BM])) : S;
    sb = p.ndig_b ? max(1, min(S, p.ndig_b[bt * p.ndig_stride_b + n0 / BN])) : S;
}

__device__ __forceinline__ void mma_i8_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// kind::i8 instruction descriptor: S32 accumulator, signed 8-bit A and B,
// both K-major.
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
    return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}

// 2^e for |e| <= 1022 (built from the exponent bits; exact)
__device__ __forceinline__ double pow2(int e) {
    return __longlong_as_double(static_cast<long long>(1023 + e) << 52);
}

// One row's 64 (or ncol) outputs: C = sum * (2^e_r * alpha 2^e_c) + beta C,
// one rounding into TC.  All loads of a chunk of 8 precede its stores.
template <int CW, typename TC>
__device__ __forceinline__ void store_row(TC* Cr, int64_t ldc, const double (&sum)[CWMAX], const double* cs,
                                          double sr, double beta, int ncol) {
    if (ncol == CW) {
        // walking pointers keep one address live per chunk instead of eight
        TC* cp = Cr;
#pragma unroll
        for (int jb = 0; jb < CW; jb += 8) {
            double cv[8];
            if (beta != 0.0) {
                const TC* q = cp;
#pragma unroll
                for (int u = 0; u < 8; ++u, q += ldc) cv[u] = static_cast<double>(*q);
            }
            TC* q = cp;
#pragma unroll
            for (int u = 0; u < 8; ++u, q += ldc) {
                double out = sum[jb + u] * (sr * cs[jb + u]);
                if (beta != 0.0) out = fma(beta, cv[u], out);
                *q = static_cast<TC>(out);
            }
            cp = q;
        }
    } else {
#pragma unroll
        for (int j = 0; j < CW; ++j) {
            if (j >= ncol) break;
            double out = sum[j] * (sr * cs[j]);
            if (beta != 0.0) out = fma(beta, static_cast<double>(Cr[j * ldc]), out);
            Cr[j * ldc] = static_cast<TC>(out);
        }
    }
}

__device__ __forceinline__ bool skip_tile(const OzProblem& pr, int m0, int n0) {
    return pr.lower_only && (m0 + BM - 1 < n0);
}

__global__ void __launch_bounds__(NTHREADS, 1) oz_gemm_kernel(const __grid_constant__ Params p) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment (128B swizzle atoms) by an offset from the shared
    // array itself, so the compiler keeps shared-space addressing (LDS/STS)
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_STAGE;  // [STAGES][2][B_STAGE]
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * 2 * B_STAGE);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + NACC;
    uint64_t* ufull = tempty + NACC;
    uint64_t* uempty = ufull + UR;
    int32_t* uring = reinterpret_cast<int32_t*>(uempty + UR);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(uring + UR);
    double* colscale = reinterpret_cast<double*>(tmem_slot + 2);  // [EPI_WARPS][CWMAX]

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&p.map_a);
        ptx::tma_prefetch_desc(&p.map_b);
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < NACC; ++s) {
            ptx::mbar_init(&tfull[s], 1);
            ptx::mbar_init(&tempty[s], 32 * EPI_WARPS);
        }
        for (int s = 0; s < UR; ++s) {
            ptx::mbar_init(&ufull[s], 1);
            ptx::mbar_init(&uempty[s], 1 + EPI_WARPS);  // the MMA warp + the epilogue warps
        }
        ptx::fence_barrier_init();
    }
    if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    // Units: the live (lower-triangle) output blocks of the lower-only
    // problems, column by column, then every block of the others.  The
    // producer draws them from a global counter and passes them to the MMA
    // and epilogue warps through a shared ring: a CTA that starts late (its
    // SM held by another stream's kernel) simply takes fewer units.
    const int tiles_per_prob = p.mblocks * p.nblocks;
    const int jl = min(p.mblocks, p.nblocks);
    const int live_per_lower = jl * p.mblocks - jl * (jl - 1) / 2;
    const int64_t lower_units = static_cast<int64_t>(p.nlower) * live_per_lower;
    const int64_t total = lower_units + static_cast<int64_t>(p.nprob - p.nlower) * tiles_per_prob;
    // consumer side of the unit ring: the next unit (>= total: done)
    auto next_unit = [&](int it) -> int64_t {
        const int slot = it % UR;
        ptx::mbar_wait(&ufull[slot], static_cast<uint32_t>((it / UR) & 1));
        const int64_t t = *reinterpret_cast<volatile int32_t*>(&uring[slot]);
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&uempty[slot]);
        return t;
    };
    auto decode = [&](int64_t t, OzProblem& pr, int& m0, int& n0) {
        int64_t pi;
        if (t < lower_units) {
            pi = t / live_per_lower;
            const int u = static_cast<int>(t - pi * live_per_lower);
            // column j starts at j * mb - j (j - 1) / 2
            const double b = 2.0 * p.mblocks + 1.0;
            int j = static_cast<int>((b - sqrt(b * b - 8.0 * u)) * 0.5);
            j = max(0, min(j, jl - 1));
            auto start = [&](int c) { return c * p.mblocks - c * (c - 1) / 2; };
            while (j > 0 && start(j) > u) --j;
            while (j + 1 < jl && start(j + 1) <= u) ++j;
            m0 = (j + (u - start(j))) * BM;
            n0 = j * BN;
        } else {
            const int64_t t2 = t - lower_units;
            const int64_t q = t2 / tiles_per_prob;
            const int r = static_cast<int>(t2 - q * tiles_per_prob);
            pi = p.nlower + q;
            m0 = (r % p.mblocks) * BM;
            n0 = (r / p.mblocks) * BN;
        }
        pr = p.problems ? p.problems[pi] : p.single;
    };

    if (warp == 0) {
        // ===== TMA producer: groups t = 2S .. 2 (small magnitudes first) =====
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            // the next unit is drawn one unit ahead: the atomic's round trip
            // overlaps this unit's loads instead of stalling the MMA warp
            int64_t t_next = static_cast<int64_t>(atomicAdd(p.sched, 1u));
            for (int it = 0;; ++it) {
                const int slot = it % UR;
                const int64_t t = t_next;
                ptx::mbar_wait(&uempty[slot], static_cast<uint32_t>(((it / UR) & 1) ^ 1));
                uring[slot] = static_cast<int32_t>(t < total ? t : total);
                ptx::mbar_arrive(&ufull[slot]);
                if (t >= total) break;
                t_next = static_cast<int64_t>(atomicAdd(p.sched, 1u));
                OzProblem pr;
                int m0, n0;
                decode(t, pr, m0, n0);
                if (skip_tile(pr, m0, n0)) continue;
                const int np = pr.a_tile2 >= 0 ? 2 : 1;
                for (int ps = 0; ps < np; ++ps) {
                const int at = ps ? pr.a_tile2 : pr.a_tile, bt = ps ? pr.b_tile2 : pr.b_tile;
                int sa, sb;
                digits_of(p, at, bt, m0, n0, sa, sb);
                for (int g = sa + sb; g >= 2; g -= 2) {
                    const bool two = g - 1 >= 2;  // group g-1 rides along
                    const int lo = max(1, (two ? g - 1 : g) - sb), hi = min(sa, g - 1);
                    for (int dp = lo; dp <= hi; ++dp) {
                        const bool v1 = dp >= max(1, g - sb);                 // pair (dp, g - dp)
                        const bool v2 = two && dp <= min(sa, g - 2);          // pair (dp, g - 1 - dp)
                        const int za = at * S + dp - 1;
                        for (int kb = 0; kb < p.kblocks; ++kb) {
                            ptx::mbar_wait(&empty[stage], phase ^ 1);
                            ptx::mbar_arrive_expect_tx(&full[stage],
                                                       A_STAGE + (v1 ? B_STAGE : 0) + (v2 ? B_STAGE : 0));
                            ptx::tma_load_3d(sA + stage * A_STAGE, &p.map_a, &full[stage], kb * BK, m0, za);
                            if (v1)
                                ptx::tma_load_3d(sB + (stage * 2) * B_STAGE, &p.map_b, &full[stage], kb * BK, n0,
                                                 bt * S + (g - dp) - 1);
                            if (v2)
                                ptx::tma_load_3d(sB + (stage * 2 + 1) * B_STAGE, &p.map_b, &full[stage], kb * BK,
                                                 n0, bt * S + (g - 1 - dp) - 1);
                            if (++stage == STAGES) {
                                stage = 0;
                                phase ^= 1;
                            }
                        }
                    }
                }
                }  // panels
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer: one accumulator per digit group =====
        // The whole warp runs the (warp-uniform) loop so its state stays in
        // uniform registers; one elected lane issues the MMAs and commits.
        // (Issued from a lane-0 branch, every MMA paid ~20 instructions of
        // register-to-uniform moves and predicates: at 1 MOP per INT8 MMA the
        // issue loop, not the tensor pipe, set the pace -- 22 % tensor active
        // in situ.)
        constexpr uint32_t idesc = idesc_i8(BM, BN);
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int it = 0;; ++it) {
            const int64_t t = next_unit(it);
            if (t >= total) break;
            OzProblem pr;
            int m0, n0;
            decode(t, pr, m0, n0);
            if (skip_tile(pr, m0, n0)) continue;
            const int np = pr.a_tile2 >= 0 ? 2 : 1;
            for (int ps = 0; ps < np; ++ps) {
            int sa, sb;
            digits_of(p, ps ? pr.a_tile2 : pr.a_tile, ps ? pr.b_tile2 : pr.b_tile, m0, n0, sa, sb);
            if (p.stats && lane == 0) {
                atomicAdd(p.stats, static_cast<unsigned long long>(sa * sb));
                atomicAdd(p.stats + 1, 1ull);
            }
            for (int g = sa + sb; g >= 2; g -= 2) {
                const bool two = g - 1 >= 2;
                // accumulators of groups g and g-1 (the next one in the rotation)
                const int acc2 = acc + 1 == NACC ? 0 : acc + 1;
                const uint32_t ph2 = acc + 1 == NACC ? acc_phase ^ 1 : acc_phase;
                ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
                if (two) ptx::mbar_wait(&tempty[acc2], ph2 ^ 1);
                ptx::tc_fence_after();
                const uint32_t d1 = tmem_base + static_cast<uint32_t>(acc * BN);
                const uint32_t d2 = tmem_base + static_cast<uint32_t>(acc2 * BN);
                bool first1 = true, first2 = true;
                const int lo = max(1, (two ? g - 1 : g) - sb), hi = min(sa, g - 1);
                for (int dp = lo; dp <= hi; ++dp) {
                    const bool v1 = dp >= max(1, g - sb);
                    const bool v2 = two && dp <= min(sa, g - 2);
                    for (int kb = 0; kb < p.kblocks; ++kb) {
                        ptx::mbar_wait(&full[stage], phase);
                        ptx::tc_fence_after();
                        // K steps of 32 bytes advance the descriptors' start address field by 2
                        const uint64_t ad = ptx::umma_desc_sw128(ptx::smem_u32(sA + stage * A_STAGE), 0, 1024);
                        const uint64_t bd1 = ptx::umma_desc_sw128(ptx::smem_u32(sB + (stage * 2) * B_STAGE), 0, 1024);
                        const uint64_t bd2 =
                            ptx::umma_desc_sw128(ptx::smem_u32(sB + (stage * 2 + 1) * B_STAGE), 0, 1024);
                        const uint32_t acc1_0 = first1 ? 0u : 1u, acc2_0 = first2 ? 0u : 1u;
                        if (ptx::elect_one()) {
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                if (v1) mma_i8_ss(d1, ad + 2 * k, bd1 + 2 * k, idesc, k == 0 ? acc1_0 : 1u);
                                if (v2) mma_i8_ss(d2, ad + 2 * k, bd2 + 2 * k, idesc, k == 0 ? acc2_0 : 1u);
                            }
                            ptx::mma_commit(&empty[stage]);
                        }
                        __syncwarp();
                        if (v1) first1 = false;
                        if (v2) first2 = false;
                        if (++stage == STAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
                if (ptx::elect_one()) {
                    ptx::mma_commit(&tfull[acc]);
                    if (two) ptx::mma_commit(&tfull[acc2]);
                }
                __syncwarp();
                if (++acc == NACC) {
                    acc = 0;
                    acc_phase ^= 1;
                }
                if (two && ++acc == NACC) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
            }  // panels
        }
    } else {
        // ===== epilogue: warps 2 .. 2 + EPI_WARPS - 1 =====
        const int lg = warp & 3;            // TMEM lane group this warp may access
        const int cgi = (warp - 2) >> 2;    // column group
        const int cb = epi_col0(cgi), cw = epi_cols(cgi);
        const int r = lg * 32 + lane;       // tile row (TMEM lane)
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int it = 0;; ++it) {
            const int64_t t = next_unit(it);
            if (t >= total) break;
            OzProblem pr;
            int m0, n0;
            decode(t, pr, m0, n0);
            if (skip_tile(pr, m0, n0)) continue;
            const int np = pr.a_tile2 >= 0 ? 2 : 1;
            // C of this unit is read only after the last digit group: pull its
            // lines into L2 now, while the MMAs run (one lane per 16 rows, the
            // 64 columns of this warp's half), so the final pass does not wait
            // on DRAM latency per 8-column chunk
            if (p.beta != 0.0 && (lane & 15) == 0 && m0 + r < p.M) {
                const int64_t es = p.c_f32 ? 4 : 8;
                const char* Cp = static_cast<const char*>(pr.c) + (m0 + r) * es;
                for (int jb = 0; jb < cw; ++jb) {
                    const int col = n0 + cb + jb;
                    if (col < p.N)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(Cp + static_cast<int64_t>(col) * p.ldc * es));
                }
            }
            double* cs = colscale + (warp - 2) * CWMAX;
            const int c0 = n0 + cb;
            const int row = m0 + r;
            double sum[CWMAX];
#pragma unroll
            for (int j = 0; j < CWMAX; ++j) sum[j] = 0.0;
            for (int ps = 0; ps < np; ++ps) {
            int sa, sb;
            digits_of(p, ps ? pr.a_tile2 : pr.a_tile, ps ? pr.b_tile2 : pr.b_tile, m0, n0, sa, sb);
            for (int g = sa + sb; g >= 2; --g) {
                ptx::mbar_wait(&tfull[acc], acc_phase);
                ptx::tc_fence_after();
                const double w = __longlong_as_double(static_cast<long long>(1023 - 12 - 7 * (g - 2)) << 52);
                // 16-column TMEM loads, one wait each (the last group's third
                // load is skipped: 32 columns)
#pragma unroll
                for (int c = 0; c < CWMAX / 16; ++c) {
                    if (c * 16 >= cw) break;
                    uint32_t v[16];
                    ptx::tmem_ld_32x32b_x16(tmem_base + (static_cast<uint32_t>(lg * 32) << 16) +
                                                static_cast<uint32_t>(acc * BN + cb + c * 16),
                                            v);
                    ptx::tmem_ld_wait();
                    // int32 -> double exactly on the FP64 pipe: the bits (0x43300000,
                    // v ^ 2^31) are 2^52 + 2^31 + v (the conversion pipe's I2F.F64
                    // runs at a quarter of the DFMA rate)
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const double x = __hiloint2double(0x43300000, static_cast<int>(v[j] ^ 0x80000000u)) -
                                         4503601774854144.0;
                        sum[c * 16 + j] = fma(w, x, sum[c * 16 + j]);
                    }
                }
                ptx::tc_fence_before();
                ptx::mbar_arrive(&tempty[acc]);
                if (++acc == NACC) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
            if (ps + 1 < np) {
                // the first panel's sums to the second panel's scale: times
                // 2^(e_r - e_r2 + e_c - e_c2), exact (NaN if an exponent marks a
                // non-finite row or column of the first panel)
                const int32_t* ec1 = p.rexp_b + static_cast<int64_t>(pr.b_tile) * p.rexp_stride_b;
                const int32_t* ec2 = p.rexp_b + static_cast<int64_t>(pr.b_tile2) * p.rexp_stride_b;
#pragma unroll
                for (int q = lane; q < cw; q += 32) {
                    const int e1 = c0 + q < p.N ? __ldg(ec1 + c0 + q) : 0;
                    const int e2 = c0 + q < p.N ? __ldg(ec2 + c0 + q) : 0;
                    cs[q] = e1 == ROWEXP_NONFINITE ? __longlong_as_double(0x7ff8000000000000ll)
                            : e2 == ROWEXP_NONFINITE ? 0.0 : pow2(e1 - e2);
                }
                __syncwarp();
                if (row < p.M) {
                    const int er1 = p.rexp_a[static_cast<int64_t>(pr.a_tile) * p.rexp_stride_a + row];
                    const int er2 = p.rexp_a[static_cast<int64_t>(pr.a_tile2) * p.rexp_stride_a + row];
                    const double rf = er1 == ROWEXP_NONFINITE ? __longlong_as_double(0x7ff8000000000000ll)
                                      : er2 == ROWEXP_NONFINITE ? 0.0 : pow2(er1 - er2);
#pragma unroll
                    for (int j = 0; j < CWMAX; ++j)
                        if (j < cw) sum[j] *= rf * cs[j];
                }
                __syncwarp();
            }
            }  // panels
            // C = alpha * 2^(e_r + e_c) * sum + beta * C (the last panel's
            // exponents).  The warp's 64 column scales alpha 2^(e_c) (NaN for a
            // column holding Inf/NaN) go through shared memory once per unit;
            // 2^(e_r) 2^(e_c) is exact, so one product per element replaces
            // the two scalings.
            const int32_t* ecol =
                p.rexp_b + static_cast<int64_t>(np == 2 ? pr.b_tile2 : pr.b_tile) * p.rexp_stride_b;
#pragma unroll
            for (int q = lane; q < cw; q += 32) {
                const int e = c0 + q < p.N ? __ldg(ecol + c0 + q) : 0;
                cs[q] = e == ROWEXP_NONFINITE ? __longlong_as_double(0x7ff8000000000000ll) : p.alpha * pow2(e);
            }
            __syncwarp();
            if (row < p.M) {
                const int er = p.rexp_a[static_cast<int64_t>(np == 2 ? pr.a_tile2 : pr.a_tile) * p.rexp_stride_a + row];
                const double sr = er == ROWEXP_NONFINITE ? __longlong_as_double(0x7ff8000000000000ll) : pow2(er);
                // columns [c0, c0 + ncol) of this row (lower-only units: col <= row)
                int ncol = min(cw, p.N - c0);
                if (pr.lower_only) ncol = min(ncol, row - c0 + 1);
                float* Cf = static_cast<float*>(pr.c) + static_cast<int64_t>(c0) * p.ldc + row;
                double* Cd = static_cast<double*>(pr.c) + static_cast<int64_t>(c0) * p.ldc + row;
                if (cw == 48) {
                    if (p.c_f32) store_row<48>(Cf, p.ldc, sum, cs, sr, p.beta, ncol);
                    else store_row<48>(Cd, p.ldc, sum, cs, sr, p.beta, ncol);
                } else {
                    if (p.c_f32) store_row<32>(Cf, p.ldc, sum, cs, sr, p.beta, ncol);
                    else store_row<32>(Cd, p.ldc, sum, cs, sr, p.beta, ncol);
                }
            }
            __syncwarp();  // cs is rewritten for the next unit
        }
    }
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<TMEM_COLS>(tmem_base);
    }
    if (threadIdx.x == 0) {  // the last CTA out resets the counters for the next launch
        __threadfence();
        if (atomicAdd(p.sched + 1, 1u) == gridDim.x - 1) {
            p.sched[0] = 0;
            p.sched[1] = 0;
        }
    }
}

// ---- digit slicing -------------------------------------------------------------

// Digit counts are kept per 128-row block (the GEMM's BM = BN): the four
// 32-row stripes of a block run as one cluster, exchange their stripes' needs
// through distributed shared memory, and write only the digit planes their
// block needs (the GEMM reads no others).  Planes beyond a row's own need are
// zeros, so a block's planes are exact for each of its rows.
constexpr int OZ_BLOCK = 128, OZ_CLUSTER = OZ_BLOCK / 32;
static_assert(BM == OZ_BLOCK && BN == OZ_BLOCK, "digit counts are per GEMM block");

__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}

// max over the cluster of thread 0's `need`; the kernel started with
// cluster_arrive_relaxed() (peers must be running before their shared memory
// is written)
__device__ __forceinline__ int cluster_block_need(int need) {
    __shared__ int sneed[OZ_CLUSTER];
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    if (threadIdx.x == 0) {
        const uint32_t local = ptx::smem_u32(&sneed[ptx::cluster_ctarank()]);
#pragma unroll
        for (uint32_t r = 0; r < OZ_CLUSTER; ++r)
            asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(ptx::mapa_shared(local, r)), "r"(need) : "memory");
    }
    ptx::cluster_sync_all();
    int m = sneed[0];
#pragma unroll
    for (int r = 1; r < OZ_CLUSTER; ++r) m = max(m, sneed[r]);
    return max(1, min(m, S));
}

// Digits of one FP16 value: Y = x * 2^(41 - e_r) is an integer |Y| < 2^41
// with at most 11 significant bits, so it and every remainder Y - q 2^w (at
// most 13 significant bits) are exact FP32 values; balanced base-2^7 digits
// q = rint(Y 2^-w), most significant first (weights 2^35 .. 2^0), |q| <= 64.
// The rounding uses the 1.5 * 2^23 bias (FP32 adds, round-to-nearest-even),
// and q is read from the biased value's bits: no conversion-pipe ops.
// Digit planes 0 .. nd-1 of 16 consecutive FP16 values of one row, one
// 16-byte store per plane.  The low byte of the biased value's bits is q
// itself (two's complement), so packing is three byte permutes per four
// digits; planes past nd are neither computed nor stored.
// Y: the values already scaled by 2^(41 - e_r).
__device__ __forceinline__ void oz_digits16_y(float (&Y)[16], int nd, int8_t* out, int64_t stride) {
    constexpr float MAGIC = 12582912.0f;  // 1.5 * 2^23
#pragma unroll
    for (int d = 0; d < S; ++d) {
        if (d >= nd) break;
        uint32_t b[16];
        if (d < S - 1) {
            const float w = __int_as_float((127 + 35 - 7 * d) << 23), iw = __int_as_float((127 - 35 + 7 * d) << 23);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const float t = fmaf(Y[j], iw, MAGIC);  // rint(Y 2^-w) + 1.5 * 2^23, exact
                b[j] = __float_as_uint(t);
                Y[j] = fmaf(-(t - MAGIC), w, Y[j]);
            }
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) b[j] = __float_as_uint(Y[j] + MAGIC);  // |Y| <= 64, weight 2^0
        }
        uint4 v;
        v.x = __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
        v.y = __byte_perm(__byte_perm(b[4], b[5], 0x0040), __byte_perm(b[6], b[7], 0x0040), 0x5410);
        v.z = __byte_perm(__byte_perm(b[8], b[9], 0x0040), __byte_perm(b[10], b[11], 0x0040), 0x5410);
        v.w = __byte_perm(__byte_perm(b[12], b[13], 0x0040), __byte_perm(b[14], b[15], 0x0040), 0x5410);
        *reinterpret_cast<uint4*>(out + d * stride) = v;
    }
}

__device__ __forceinline__ void oz_digits16(const uint16_t (&h)[16], float scale, int nd, int8_t* out,
                                            int64_t stride) {
    float Y[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) Y[j] = __half2float(__ushort_as_half(h[j])) * scale;
    oz_digits16_y(Y, nd, out, stride);
}

// One CTA per 32-row stripe of one matrix: (1) row exponent e_r with
// |x| < 2^e_r for the whole row (frexp of the row max; rows holding Inf/NaN
// get ROWEXP_NONFINITE, their products become NaN), (2) the digits, one
// 32 x 128 block at a time, each thread writing 16 consecutive digits of one
// row per plane (16-byte stores).
__device__ __forceinline__ void oz_slice_generic(const OzSliceItem& it, int64_t r0) {
    const uint16_t* x = static_cast<const uint16_t*>(it.x);
    int need_stripe = 0;  // thread 0: digits this stripe's rows need
    __shared__ uint16_t sx[32][128 + 2];
    __shared__ uint32_t smax[8][33];
    __shared__ int sexp[32];
    auto at = [&](int64_t r, int64_t c) -> uint16_t {
        return it.trans ? x[r * it.ld + c] : x[c * it.ld + r];
    };
    // column-major stripes of 32 full rows, 16-byte aligned: 8 rows per load
    const bool vec = !it.trans && r0 + 32 <= it.rows && (it.ld % 8) == 0 &&
                     (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    if (vec) {
        if (threadIdx.x < 32) {
            smax[0][threadIdx.x] = 0;
            smax[1][threadIdx.x] = 31;
        }
        __syncthreads();
        const int rg = threadIdx.x % 4;  // rows rg*8 .. rg*8+7
        uint32_t mx[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        uint32_t mn[8] = {31, 31, 31, 31, 31, 31, 31, 31};  // min exponent field of nonzeros
#pragma unroll 4
        for (int64_t c = threadIdx.x / 4; c < it.cols; c += 64) {
            const uint4 v = *reinterpret_cast<const uint4*>(x + c * it.ld + r0 + rg * 8);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t lo = w[q] & 0x7fffu, hi = (w[q] >> 16) & 0x7fffu;
                mx[2 * q] = max(mx[2 * q], lo);
                mx[2 * q + 1] = max(mx[2 * q + 1], hi);
                if (lo) mn[2 * q] = min(mn[2 * q], max(lo >> 10, 1u));
                if (hi) mn[2 * q + 1] = min(mn[2 * q + 1], max(hi >> 10, 1u));
            }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            atomicMax(&smax[0][rg * 8 + j], mx[j]);
            atomicMin(&smax[1][rg * 8 + j], mn[j]);
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            const uint32_t m = smax[0][threadIdx.x];
            int e = 0, need = 0;
            if (m >= 0x7c00u) {
                e = ROWEXP_NONFINITE;
            } else if (m != 0) {
                frexp(h2d(static_cast<uint16_t>(m)), &e);
                // lowest set bit of the row is >= 2^(minexp - 25); digits reach
                // 2^(e - 6 - 7 (S - 1))
                const int lsb = static_cast<int>(smax[1][threadIdx.x]) - 25;
                need = 1 + (max(0, e - 6 - lsb) + 6) / 7;
            }
            sexp[threadIdx.x] = e;
            it.rexp[r0 + threadIdx.x] = e;
            for (int o = 16; o; o >>= 1) need = max(need, __shfl_xor_sync(0xffffffffu, need, o));
            need_stripe = need;
        }
        __syncthreads();
    } else {
        // (1) row max of |x| as FP16 magnitude bits (monotone in the value)
        int lr, cs;
        if (!it.trans) {  // warp = 32 consecutive rows of one column
            lr = threadIdx.x % 32;
            cs = threadIdx.x / 32;
        } else {  // warp = 32 consecutive columns of ... 8 threads per row chunk
            lr = threadIdx.x / 8;
            cs = threadIdx.x % 8;
        }
        const int64_t r = r0 + lr;
        uint32_t mx = 0;
        if (r < it.rows)
            for (int64_t c = cs; c < it.cols; c += 8) mx = max(mx, static_cast<uint32_t>(at(r, c) & 0x7fff));
        smax[cs][lr] = mx;
        __syncthreads();
        if (threadIdx.x < 32) {
            uint32_t m = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) m = max(m, smax[q][threadIdx.x]);
            int e = 0;
            if (m >= 0x7c00u)
                e = ROWEXP_NONFINITE;
            else if (m != 0)
                frexp(h2d(static_cast<uint16_t>(m)), &e);
            sexp[threadIdx.x] = e;
            if (r0 + threadIdx.x < it.rows) it.rexp[r0 + threadIdx.x] = e;
            need_stripe = S;  // no digit analysis here
        }
        __syncthreads();
    }
    // planes written: the block's need (all S when the caller keeps no counts)
    const int bn = cluster_block_need(need_stripe);  // every CTA of the cluster takes part
    const int bneed = it.ndig ? bn : S;
    if (it.ndig && threadIdx.x == 0 && ptx::cluster_ctarank() == 0) it.ndig[r0 / OZ_BLOCK] = bneed;
    // (2) digits
    const int lr = threadIdx.x / 8, cg = (threadIdx.x % 8) * 16;
    const int64_t gr = r0 + lr;
    const int er = sexp[lr];
    const bool zero = er == ROWEXP_NONFINITE;
    for (int64_t c0 = 0; c0 < it.kpad; c0 += 128) {
        if (vec) {
            for (int e = threadIdx.x; e < 128 * 4; e += 256) {  // 128 columns x 4 row groups
                const int b = e / 4, rg = e % 4;
                const int64_t cc = c0 + b;
                uint4 v = make_uint4(0, 0, 0, 0);
                if (cc < it.cols) v = *reinterpret_cast<const uint4*>(x + cc * it.ld + r0 + rg * 8);
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    sx[rg * 8 + 2 * q][b] = static_cast<uint16_t>(w[q] & 0xffffu);
                    sx[rg * 8 + 2 * q + 1][b] = static_cast<uint16_t>(w[q] >> 16);
                }
            }
        } else
        for (int e = threadIdx.x; e < 32 * 128; e += 256) {
            int a, b;
            if (!it.trans) {
                a = e % 32;
                b = e / 32;
            } else {
                b = e % 128;
                a = e / 128;
            }
            const int64_t rr = r0 + a, cc = c0 + b;
            sx[a][b] = (rr < it.rows && cc < it.cols) ? at(rr, cc) : static_cast<uint16_t>(0);
        }
        __syncthreads();
        if (gr < it.rows && c0 + cg < it.kpad) {
            const float scale = zero ? 0.0f : __int_as_float((127 + 41 - er) << 23);
            uint16_t hv[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) hv[j] = sx[lr][cg + j];
            oz_digits16(hv, scale, bneed, static_cast<int8_t*>(it.out) + gr * it.kpad + c0 + cg, it.slice_stride);
        }
        __syncthreads();
    }
}


__global__ void __cluster_dims__(OZ_CLUSTER, 1, 1) __launch_bounds__(256) oz_slice_kernel(const OzSliceItem* items) {
    cluster_arrive_relaxed();
    const OzSliceItem it = items[blockIdx.y];
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32;
    if (r0 >= it.rows) {  // past this matrix's rows: only the exchange
        cluster_block_need(0);
        return;
    }
    oz_slice_generic(it, r0);
}

// Tiles (K <= OZ_STRIPE_K): the whole 32-row stripe is staged in shared
// memory column by column by 16-byte cp.async copies (8 rows of one column
// each, every copy of the stripe in flight at once), then the row exponents
// and digit counts and the digits are cut from shared memory -- one HBM read
// of the operand, no register round trip.  Lane = row in both passes, so the
// column-major staging is read without bank conflicts.
constexpr int OZ_STRIPE_K = 1024;
constexpr int OZ_H_PITCH = 32;  // halves per staged column (64 bytes: 16-byte aligned, lane-per-row reads conflict-free)
__device__ __forceinline__ void cp_async16_zfill_h(void* smem, const void* gmem, bool valid) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(valid ? 16 : 0)
                 : "memory");
}
__global__ void __cluster_dims__(OZ_CLUSTER, 1, 1) __launch_bounds__(256)
    oz_slice_stripe_kernel(const OzSliceItem* items) {
    cluster_arrive_relaxed();
    const OzSliceItem it = items[blockIdx.y];
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32;
    if (r0 >= it.rows) {
        cluster_block_need(0);
        return;
    }
    const uint16_t* x = static_cast<const uint16_t*>(it.x);
    const bool vec = !it.trans && r0 + 32 <= it.rows && (it.ld % 8) == 0 &&
                     (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    extern __shared__ __align__(16) uint16_t sxh[];  // [kpad][OZ_H_PITCH]: column c's 32 rows at c * PITCH
    __shared__ uint32_t smax[8][33], smin[8][33];
    __shared__ int sexp[32];
    const int kp = static_cast<int>(it.kpad), cols = static_cast<int>(it.cols);
    const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
    if (vec) {
        for (int e = threadIdx.x; e < kp * 4; e += 256) {
            const int c = e / 4, q = e % 4;
            const bool ok = c < cols;
            cp_async16_zfill_h(sxh + c * OZ_H_PITCH + 8 * q,
                               ok ? x + static_cast<int64_t>(c) * it.ld + r0 + 8 * q : x, ok);
        }
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    } else {  // ragged last stripe, transposed or unaligned operand
        for (int e = threadIdx.x; e < kp * 32; e += 256) {
            const int c = e / 32, rr = e % 32;
            const int64_t gr = r0 + rr;
            sxh[c * OZ_H_PITCH + rr] =
                (c < cols && gr < it.rows) ? (it.trans ? x[gr * it.ld + c] : x[static_cast<int64_t>(c) * it.ld + gr])
                                           : static_cast<uint16_t>(0);
        }
    }
    __syncthreads();
    // (1) per row (lane): largest magnitude, smallest exponent field of a nonzero
    {
        uint32_t mx = 0, mn = 31;
#pragma unroll 8
        for (int c = w; c < kp; c += 8) {
            const uint32_t m = sxh[c * OZ_H_PITCH + lane] & 0x7fffu;
            mx = max(mx, m);
            if (m) mn = min(mn, max(m >> 10, 1u));
        }
        smax[w][lane] = mx;
        smin[w][lane] = mn;
    }
    __syncthreads();
    int need_stripe = 0;
    if (threadIdx.x < 32) {
        uint32_t m = 0, mn = 31;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            m = max(m, smax[q][threadIdx.x]);
            mn = min(mn, smin[q][threadIdx.x]);
        }
        int e = 0, need = 0;
        if (m >= 0x7c00u) {
            e = ROWEXP_NONFINITE;
        } else if (m != 0) {
            frexp(h2d(static_cast<uint16_t>(m)), &e);
            // lowest set bit of the row is >= 2^(minexp - 25); digits reach
            // 2^(e - 6 - 7 (S - 1))
            const int lsb = static_cast<int>(mn) - 25;
            need = 1 + (max(0, e - 6 - lsb) + 6) / 7;
        }
        sexp[threadIdx.x] = e;
        if (r0 + threadIdx.x < it.rows) it.rexp[r0 + threadIdx.x] = e;
        for (int o = 16; o; o >>= 1) need = max(need, __shfl_xor_sync(0xffffffffu, need, o));
        need_stripe = need;
    }
    __syncthreads();
    // planes written: the block's need (all S when the caller keeps no counts)
    const int bn = cluster_block_need(need_stripe);  // every CTA of the cluster takes part
    const int bneed = it.ndig ? bn : S;
    if (it.ndig && threadIdx.x == 0 && ptx::cluster_ctarank() == 0) it.ndig[r0 / OZ_BLOCK] = bneed;
    // (2) digits: lane = row, warp w takes 16-column groups w, w + 8, ...
    if (r0 + lane >= it.rows) return;
    const int er = sexp[lane];
    const float scale = er == ROWEXP_NONFINITE ? 0.0f : __int_as_float((127 + 41 - er) << 23);
    int8_t* outr = static_cast<int8_t*>(it.out) + (r0 + lane) * it.kpad;
    for (int c0 = 16 * w; c0 < kp; c0 += 128) {
        uint16_t hv[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) hv[j] = sxh[(c0 + j) * OZ_H_PITCH + lane];
        oz_digits16(hv, scale, bneed, outr + c0, it.slice_stride);
    }
}

// FP32 operands (FP32 destination tiles fed by FP32 panel tiles).  The same
// digits: Y = x 2^(41 - e_r) is exact (a power-of-two scaling, applied in two
// halves so the FP32 scale factors stay normal) and every remainder keeps
// Y's <= 24 significant bits, so the digits are exact down to 2^(e_r - 41).
// A row whose values reach below that (FP32 rows span up to 2^277) has its
// sixth digit rounded: the product error is then at most 2^-42 |row max| per
// term, far below the FP32 rounding of the result.  Column-major, no
// transpose (the tile scheduler's panel tiles), kpad <= OZ_STRIPE_K.
// The stripe (32 rows x kpad) is staged whole into shared memory by 16-byte
// cp.async copies (4 rows of one column each, all in flight at once): the
// FP32 head tile of every step is sliced on the critical path.
constexpr int OZ_F32_PITCH = 36;  // floats per staged column: 16-byte aligned, conflict-free row reads
__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, bool valid) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(valid ? 16 : 0)
                 : "memory");
}
__global__ void __cluster_dims__(OZ_CLUSTER, 1, 1) __launch_bounds__(256)
    oz_slice_f32_kernel(const OzSliceItem* items) {
    cluster_arrive_relaxed();
    const OzSliceItem it = items[blockIdx.y];
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32;
    if (r0 >= it.rows) {
        cluster_block_need(0);
        return;
    }
    const float* x = static_cast<const float*>(it.x);
    extern __shared__ __align__(16) float sxc[];  // [kpad][OZ_F32_PITCH], column c's rows at c * PITCH
    __shared__ uint32_t smax[8][33], smin[8][33];
    __shared__ int sexp[32];
    const int kp = static_cast<int>(it.kpad), cols = static_cast<int>(it.cols);
    const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
    const bool vec = r0 + 32 <= it.rows && (it.ld % 4) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    if (vec) {
        for (int e = threadIdx.x; e < kp * 8; e += 256) {
            const int c = e / 8, q = e % 8;
            const bool ok = c < cols;
            cp_async16_zfill(sxc + c * OZ_F32_PITCH + 4 * q, ok ? x + static_cast<int64_t>(c) * it.ld + r0 + 4 * q : x,
                             ok);
        }
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    } else {
        for (int e = threadIdx.x; e < kp * 32; e += 256) {
            const int c = e / 32, rr = e % 32;
            sxc[c * OZ_F32_PITCH + rr] =
                (c < cols && r0 + rr < it.rows) ? x[static_cast<int64_t>(c) * it.ld + r0 + rr] : 0.0f;
        }
    }
    __syncthreads();
    // (1) per row (lane): largest magnitude, smallest exponent field of a nonzero
    {
        uint32_t mx = 0, mn = 255;
        for (int c = w; c < kp; c += 8) {
            const uint32_t m = __float_as_uint(sxc[c * OZ_F32_PITCH + lane]) & 0x7fffffffu;
            mx = max(mx, m);
            if (m) mn = min(mn, max(m >> 23, 1u));
        }
        smax[w][lane] = mx;
        smin[w][lane] = mn;
    }
    __syncthreads();
    int need_stripe = 0;
    if (threadIdx.x < 32) {
        uint32_t m = 0, mn = 255;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            m = max(m, smax[q][threadIdx.x]);
            mn = min(mn, smin[q][threadIdx.x]);
        }
        int e = 0, need = 0;
        if (m >= 0x7f800000u) {
            e = ROWEXP_NONFINITE;
        } else if (m != 0) {
            frexpf(__uint_as_float(m), &e);
            const int lsb = static_cast<int>(mn) - 150;  // ulp of the smallest nonzero
            need = 1 + (max(0, e - 6 - lsb) + 6) / 7;
        }
        sexp[threadIdx.x] = e;
        if (r0 + threadIdx.x < it.rows) it.rexp[r0 + threadIdx.x] = e;
        for (int o = 16; o; o >>= 1) need = max(need, __shfl_xor_sync(0xffffffffu, need, o));
        need_stripe = need;
    }
    __syncthreads();
    const int bn = cluster_block_need(need_stripe);
    const int bneed = it.ndig ? bn : S;
    if (it.ndig && threadIdx.x == 0 && ptx::cluster_ctarank() == 0) it.ndig[r0 / OZ_BLOCK] = bneed;
    // (2) digits: lane = row, warp w takes 16-column groups w, w + 8, ...
    const int64_t gr = r0 + lane;
    if (gr >= it.rows) return;
    const int er = sexp[lane];
    const bool zero = er == ROWEXP_NONFINITE;
    const int sh = zero ? 0 : 41 - er, sh1 = sh / 2, sh2 = sh - sh / 2;
    const float s1 = zero ? 0.0f : __int_as_float((127 + sh1) << 23), s2 = __int_as_float((127 + sh2) << 23);
    int8_t* outr = static_cast<int8_t*>(it.out) + gr * it.kpad;
    for (int c0 = 16 * w; c0 < kp; c0 += 128) {
        float Y[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) Y[j] = (sxc[(c0 + j) * OZ_F32_PITCH + lane] * s1) * s2;
        oz_digits16_y(Y, bneed, outr + c0, it.slice_stride);
    }
}
}  // namespace oz

void launch_oz_slices(Ctx* ctx, cudaStream_t s, const OzSliceItem* items, int64_t count, int64_t max_rows,
                      int64_t max_cols) {
    if (count == 0) return;
    ProfScope ps(ctx, MP_PROF_CAST, s, 0.0);
    // 32-row stripes, whole 128-row blocks (clusters of four stripes)
    const dim3 grid(static_cast<unsigned>((max_rows + oz::OZ_BLOCK - 1) / oz::OZ_BLOCK * oz::OZ_CLUSTER),
                    static_cast<unsigned>(count));
    if (max_cols <= oz::OZ_STRIPE_K) {
        const int kpad = static_cast<int>((max_cols + 15) / 16 * 16);
        const int smem = kpad * oz::OZ_H_PITCH * 2;
        static unsigned long long cfg = 0;  // per-device bitmask
        if (first_on_device(cfg)) {
            MP_CUDA(cudaFuncSetAttribute(oz::oz_slice_stripe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         oz::OZ_STRIPE_K * oz::OZ_H_PITCH * 2));
        }
        oz::oz_slice_stripe_kernel<<<grid, 256, smem, s>>>(items);
    } else {
        oz::oz_slice_kernel<<<grid, 256, 0, s>>>(items);
    }
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

void launch_oz_slices_f32(Ctx* ctx, cudaStream_t s, const OzSliceItem* items, int64_t count, int64_t max_rows,
                          int64_t max_cols) {
    if (count == 0) return;
    if (max_cols > oz::OZ_STRIPE_K) fail(MP_INVALID_PARAM, "FP32 digit slicer: K > 1024");
    ProfScope ps(ctx, MP_PROF_CAST, s, 0.0);
    const dim3 grid(static_cast<unsigned>((max_rows + oz::OZ_BLOCK - 1) / oz::OZ_BLOCK * oz::OZ_CLUSTER),
                    static_cast<unsigned>(count));
    // the tile scheduler slices nb x nb panel tiles (kpad = nb <= OZ_STRIPE_K)
    const int smem = oz::OZ_STRIPE_K * oz::OZ_F32_PITCH * 4;
    static unsigned long long cfg = 0;  // per-device bitmask
    if (first_on_device(cfg))
        MP_CUDA(cudaFuncSetAttribute(oz::oz_slice_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    oz::oz_slice_f32_kernel<<<grid, 256, smem, s>>>(items);
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

void launch_oz_gemm(Ctx* ctx, cudaStream_t s, const OzGemm& g) {
    using namespace oz;
    Params p{};
    // [tiles * S][rows][K] int8 digits, rows kpad bytes apart
    tma_map_3d(&p.map_a, g.A, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, g.k, g.m, g.a_tiles * S, g.kpad,
               g.a_slice_stride, BK, BM, CU_TENSOR_MAP_SWIZZLE_128B);
    tma_map_3d(&p.map_b, g.B, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, g.k, g.n, g.b_tiles * S, g.kpad,
               g.b_slice_stride, BK, BN, CU_TENSOR_MAP_SWIZZLE_128B);
    p.problems = g.problems;
    p.single = OzProblem{0, 0, g.C, g.lower_only ? 1 : 0, -1, -1, 0};
    p.nprob = g.problems ? static_cast<int32_t>(g.count) : 1;
    p.nlower = g.problems ? static_cast<int32_t>(g.n_lower) : (g.lower_only ? 1 : 0);
    p.M = static_cast<int32_t>(g.m);
    p.N = static_cast<int32_t>(g.n);
    p.K = static_cast<int32_t>(g.k);
    p.mblocks = static_cast<int32_t>((g.m + BM - 1) / BM);
    p.nblocks = static_cast<int32_t>((g.n + BN - 1) / BN);
    p.kblocks = static_cast<int32_t>((g.k + BK - 1) / BK);
    p.ldc = g.ldc;
    p.alpha = g.alpha;
    p.beta = g.beta;
    p.rexp_a = g.rexp_a;
    p.rexp_b = g.rexp_b;
    p.rexp_stride_a = g.rexp_stride_a;
    p.rexp_stride_b = g.rexp_stride_b;
    p.ndig_a = g.ndig_a;
    p.ndig_b = g.ndig_b;
    p.ndig_stride_a = static_cast<int32_t>(g.ndig_stride_a);
    p.ndig_stride_b = static_cast<int32_t>(g.ndig_stride_b);
    p.c_f32 = g.c_single ? 1 : 0;
    p.stats = ctx->prof.enabled ? ctx->prof.dev_stats : nullptr;
    const int64_t jl = std::min(p.mblocks, p.nblocks);
    const int64_t total = static_cast<int64_t>(p.nlower) * (jl * p.mblocks - jl * (jl - 1) / 2) +
                          static_cast<int64_t>(p.nprob - p.nlower) * p.mblocks * p.nblocks;
    ProfScope ps(ctx, MP_PROF_GEMM_I8, s,
                 2.0 * static_cast<double>(g.m) * g.n * g.k * (p.nprob + g.n_two) * (g.lower_only ? 0.5 : 1.0));
    static unsigned long long configured = 0;  // per-device bitmask
    if (first_on_device(configured)) {
        MP_CUDA(cudaFuncSetAttribute(oz_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    }
    // one CTA per SM (or per unit), units drawn dynamically
    const int64_t grid = std::max<int64_t>(std::min<int64_t>(total, ctx->sm_count), 1);
    p.sched = ctx->sched_slot();
    oz_gemm_kernel<<<static_cast<unsigned>(grid), NTHREADS, SMEM_BYTES, s>>>(p);
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

}  // namespace mpcr
