// FP16 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// Serves linalg::gemm / matmul / crossprod (linalg.cpp:316-357, :284-314) when
// both operands are half and C is half or single (the reference computes
// these in float, linalg.cpp:340-348; FP16 x FP16 products are exact in FP32
// and the tensor core accumulates in FP32), and the FP16 trailing-update and
// panel-TRSM tiles of the MPCRTile Cholesky (grouped, one launch per step).
//
// Persistent, warp-specialised, one CTA per SM (grid <= 148):
//   warp 0      TMA producer: 4-stage ring of {A 128x64, B 256x64} FP16
//               tiles in 128B-swizzled shared memory (mbarrier full/empty).
//   warp 1      MMA issuer: one thread issues tcgen05.mma (M=128, N=256,
//               K=16) into a double-buffered TMEM accumulator (2 x 256 FP32
//               columns); tcgen05.commit frees smem stages / signals TMEM full.
//   warp 2      TMEM allocator (512 columns).
//   warp 3      C loader: TMA-loads the C tile chunk (128 x 256B) into a
//               shared buffer while the MMAs of that tile run (beta != 0 only).
//   warps 4-7   epilogue: tcgen05.ld 32 lanes x 32 columns, C = alpha*acc +
//               beta*C in FP32 (beta == 0 never reads C), rounded to C's
//               precision in the shared chunk, then one TMA store per chunk.
// Operand majorness follows the column-major storage: op(A) = A is MN-major,
// A^T K-major; op(B) = B is K-major, B^T MN-major.  All three matrices are
// addressed by 3-D TMA maps [tile][col][row], so a grouped launch can take any
// tiles of a slab by index.
#include <algorithm>
#include <cuda.h>
#include <cuda_fp16.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "device.cuh"
#include "gemm_tc.hpp"
#include "internal.hpp"
#include "tc_ptx.cuh"

namespace mpcr {
namespace tc {

// Every stage holds 128 bytes of K per row for either operand kind:
// 64 FP16 (kind::f16) or 32 FP32 (kind::tf32) elements.
constexpr int BM = 128, BN = 256, STAGES = 4;
constexpr int A_STAGE = BM * 128;  // 16 KB
constexpr int B_STAGE = BN * 128;  // 32 KB
constexpr int C_CHUNK = BM * 256;     // 32 KB: 128 rows x 256 bytes
constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) + C_CHUNK + 1024 /*align*/ + 256;
constexpr int TMEM_COLS = 512;

struct Params {
    CUtensorMap map_a[2];  // A, A_lo
    CUtensorMap map_b[2];  // B, B_lo
    CUtensorMap map_c;
    const TcProblem* problems;  // nullptr -> use `single`
    TcProblem single;
    int32_t nprob;
    int32_t M, N, K;
    float alpha, beta;
    int32_t mblocks, nblocks, kblocks;
    int32_t kblocks1;  // K blocks per segment; kblocks = nseg * kblocks1
    int32_t seg_a[3], seg_b[3];  // K segment s multiplies map_a[seg_a[s]] by map_b[seg_b[s]]
    int32_t c_evict_first;       // pair kernel: C loads/stores marked L2 evict_first
    // pair kernel unit assignment: cluster c takes units
    // (c / lanes) * lanes * per + c % lanes + r * lanes, r < per, so the
    // clusters resident together (one wave of `lanes`) work on neighbouring
    // units through one contiguous chunk of the list instead of striding it
    int32_t lanes, per;
    // B = L^-T of a lower-triangular L (the panel TRSM X = A L^-T): a unit
    // with output columns [n0, n0 + BN) needs only K < n0 + BN
    int32_t k_tri;
};

// K blocks per segment a unit with output columns from n0 runs, and the
// segment / K offset of its block kb.
__device__ __forceinline__ int unit_kb1(const Params& p, int n0, int bn, int bk) {
    return p.k_tri ? min(p.kblocks1, (n0 + bn + bk - 1) / bk) : p.kblocks1;
}

__device__ __forceinline__ bool skip_tile(const TcProblem& pr, int m0, int n0) {
    return pr.lower_only && (m0 + BM - 1 < n0);
}

// Epilogue conversions use the hardware cvt (round-to-nearest-even, IEEE
// subnormals and overflow to Inf — the reference's encode_f16 for every
// non-NaN value); the bit-exact software path (device.cuh) is kept for the
// cast kernels, where NaN payloads must match the reference too.
__device__ __forceinline__ float ld_c(const uint16_t* c, int i) { return __half2float(__ushort_as_half(c[i])); }
__device__ __forceinline__ float ld_c(const float* c, int i) { return c[i]; }
__device__ __forceinline__ void st_c(uint16_t* c, int i, float v) { c[i] = __half_as_ushort(__float2half_rn(v)); }
__device__ __forceinline__ void st_c(float* c, int i, float v) { c[i] = v; }

// KIND 0: kind::f16 (FP16 operands), KIND 1: kind::tf32 (FP32 storage).
constexpr int NTHREADS = 256;  // 4 role warps + 4 epilogue warps
constexpr int EPI_THREADS = 128;

template <int KIND, bool A_MN, bool B_MN, typename TC>
__global__ void __launch_bounds__(NTHREADS, 1) gemm_tc_kernel(const __grid_constant__ Params p) {
    constexpr int ES = KIND == 0 ? 2 : 4;      // operand element bytes
    constexpr int BK = 128 / ES;               // K elements per stage
    constexpr int BW = 128 / ES;               // MN elements per 128B swizzle row
    constexpr int BOX = BW * BK * ES;          // bytes of one MN-major TMA box
    constexpr int KSTEP_MN = (32 / ES) * 128;  // UMMA K (32 bytes of K) in MN-major rows
    constexpr uint32_t FMT = KIND == 0 ? 0u : 2u;
    constexpr int CW = 256 / sizeof(TC);  // chunk width in columns (128 half / 64 float)
    constexpr int NCHUNK = BN / CW;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment (128B swizzle atoms) by an offset from the shared
    // array itself, so the compiler keeps shared-space addressing (LDS/STS)
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_STAGE;
    TC* cbuf = reinterpret_cast<TC*>(sB + STAGES * B_STAGE);  // [CW cols][BM rows]
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(cbuf) + C_CHUNK);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* cfull = tempty + 2;
    uint64_t* cempty = cfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cempty + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&p.map_a[0]);
        ptx::tma_prefetch_desc(&p.map_a[1]);
        ptx::tma_prefetch_desc(&p.map_b[0]);
        ptx::tma_prefetch_desc(&p.map_b[1]);
        ptx::tma_prefetch_desc(&p.map_c);
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            ptx::mbar_init(&tfull[s], 1);
            ptx::mbar_init(&tempty[s], EPI_THREADS);
        }
        ptx::mbar_init(cfull, 1);
        ptx::mbar_init(cempty, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc<TMEM_COLS>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int tiles_per_prob = p.mblocks * p.nblocks;
    const int64_t total = static_cast<int64_t>(p.nprob) * tiles_per_prob;
    const bool read_c = p.beta != 0.0f;

    // grouped rasterization as in the pair kernel: 16 M-blocks per group
    constexpr int GROUP_M1 = 16;
    auto decode = [&](int64_t t, TcProblem& pr, int& m0, int& n0) {
        const int64_t pi = t / tiles_per_prob;
        const int r = static_cast<int>(t - pi * tiles_per_prob);
        pr = p.problems ? p.problems[pi] : p.single;
        const int per_group = GROUP_M1 * p.nblocks;
        const int g = r / per_group, rem = r - g * per_group;
        const int gm = min(GROUP_M1, p.mblocks - g * GROUP_M1);
        m0 = (g * GROUP_M1 + rem % gm) * BM;
        n0 = (rem / gm) * BN;
    };

    if (warp == 0) {
        // ===== TMA producer =====
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
                TcProblem pr;
                int m0, n0;
                decode(t, pr, m0, n0);
                if (skip_tile(pr, m0, n0)) continue;
                const int kb1 = unit_kb1(p, n0, BN, BK), nkb = (p.kblocks / p.kblocks1) * kb1;
                for (int kb = 0; kb < nkb; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    ptx::mbar_arrive_expect_tx(&full[stage], A_STAGE + B_STAGE);
                    uint8_t* a_dst = sA + stage * A_STAGE;
                    uint8_t* b_dst = sB + stage * B_STAGE;
                    // K segments: (A|A_lo) x (B|B_lo) products into one accumulator
                    const int sg = kb / kb1;
                    const int kk = (kb - sg * kb1) * BK;
                    const CUtensorMap* ma = &p.map_a[p.seg_a[sg]];
                    const CUtensorMap* mb = &p.map_b[p.seg_b[sg]];
                    if (A_MN) {
#pragma unroll
                        for (int j = 0; j < BM / BW; ++j)
                            ptx::tma_load_3d(a_dst + j * BOX, ma, &full[stage], m0 + j * BW, kk,
                                             pr.a_tile);
                    } else {
                        ptx::tma_load_3d(a_dst, ma, &full[stage], kk, m0, pr.a_tile);
                    }
                    if (B_MN) {
#pragma unroll
                        for (int j = 0; j < BN / BW; ++j)
                            ptx::tma_load_3d(b_dst + j * BOX, mb, &full[stage], n0 + j * BW, kk,
                                             pr.b_tile);
                    } else {
                        ptx::tma_load_3d(b_dst, mb, &full[stage], kk, n0, pr.b_tile);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer =====
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::umma_idesc(BM, BN, A_MN, B_MN, FMT);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
                TcProblem pr;
                int m0, n0;
                decode(t, pr, m0, n0);
                if (skip_tile(pr, m0, n0)) continue;
                ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
                const int nkb = (p.kblocks / p.kblocks1) * unit_kb1(p, n0, BN, BK);
                for (int kb = 0; kb < nkb; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t a_base = ptx::smem_u32(sA + stage * A_STAGE);
                    const uint32_t b_base = ptx::smem_u32(sB + stage * B_STAGE);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {  // 4 x 32 bytes of K per stage
                        const uint64_t ad = A_MN ? ptx::umma_desc_sw128(a_base + k * KSTEP_MN, BOX, 1024)
                                                 : ptx::umma_desc_sw128(a_base + k * 32, 0, 1024);
                        const uint64_t bd = B_MN ? ptx::umma_desc_sw128(b_base + k * KSTEP_MN, BOX, 1024)
                                                 : ptx::umma_desc_sw128(b_base + k * 32, 0, 1024);
                        if (KIND == 0)
                            ptx::mma_f16_ss(d_tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
                        else
                            ptx::mma_tf32_ss(d_tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
                    }
                    ptx::mma_commit(&empty[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                ptx::mma_commit(&tfull[acc]);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (warp == 3) {
        // ===== C loader: one chunk at a time into the shared C buffer =====
        if (lane == 0) {
            uint32_t cphase = 0;
            for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
                TcProblem pr;
                int m0, n0;
                decode(t, pr, m0, n0);
                if (skip_tile(pr, m0, n0)) continue;
                for (int h = 0; h < NCHUNK; ++h) {
                    ptx::mbar_wait(cempty, cphase ^ 1);
                    if (read_c) {
                        ptx::mbar_arrive_expect_tx(cfull, C_CHUNK);
                        ptx::tma_load_3d(cbuf, &p.map_c, cfull, m0, n0 + h * CW, pr.c_tile);
                    } else {
                        ptx::mbar_arrive(cfull);
                    }
                    cphase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        // ===== epilogue =====
        const int q = warp - 4;  // TMEM lane group this warp may access
        const int r = q * 32 + lane;  // tile row owned by this thread (TMEM lane)
        const bool is_leader = threadIdx.x == 128;
        int acc = 0;
        uint32_t acc_phase = 0, cphase = 0;
        for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
            TcProblem pr;
            int m0, n0;
            decode(t, pr, m0, n0);
            if (skip_tile(pr, m0, n0)) continue;
            ptx::mbar_wait(&tfull[acc], acc_phase);
            ptx::tc_fence_after();
            const int row = m0 + r;
#pragma unroll 1
            for (int h = 0; h < NCHUNK; ++h) {
                ptx::mbar_wait(cfull, cphase);
                cphase ^= 1;
#pragma unroll 1
                for (int c = 0; c < CW / 32; ++c) {
                    uint32_t v[32];
                    const int col0 = h * CW + c * 32;  // column within the tile
                    ptx::tmem_ld_32x32b_x32(
                        tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + col0, v);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int cc = c * 32 + j;  // column within the chunk
                        const float a = __fmul_rn(p.alpha, __uint_as_float(v[j]));
                        float out = a;
                        if (read_c) {
                            const float old = ld_c(cbuf, cc * BM + r);
                            out = (pr.lower_only && row < n0 + col0 + j)
                                      ? old
                                      : __fadd_rn(a, __fmul_rn(p.beta, old));
                        }
                        st_c(cbuf, cc * BM + r, out);
                    }
                }
                // chunk complete: hand it to the TMA unit, then release it
                ptx::fence_proxy_async_smem();
                ptx::named_bar_sync(1, EPI_THREADS);
                if (is_leader) {
                    ptx::tma_store_3d(&p.map_c, cbuf, m0, n0 + h * CW, pr.c_tile);
                    ptx::bulk_commit();
                    ptx::bulk_wait_read0();
                    ptx::mbar_arrive(cempty);
                }
            }
            ptx::tc_fence_before();
            ptx::mbar_arrive(&tempty[acc]);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
        if (is_leader) ptx::bulk_wait0();
    }
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<TMEM_COLS>(tmem_base);
    }
}


// ---- 2-CTA pair kernel (cta_group::2): 256 x 256 output tile per CTA pair ----
// Same warp roles; each CTA of the pair loads its 128 rows of A and its 128
// rows (half) of B per stage, so a CTA's shared-memory ingress per K step is
// 32 KB instead of 48 KB for the same FLOPs.  The even CTA issues the pair
// MMA (M=256, N=256); stage "full" barriers live in the even CTA, "empty"
// barriers in both (multicast commit); each CTA's epilogue reads its own 128
// TMEM lanes and signals the even CTA's tmem-empty barrier.
// 6 operand stages and two C chunk buffers: the C loader prefetches the next
// chunk (also the next unit's first one) while the epilogue works on the
// current, so the read-modify-write of C stays off the MMA's path.
// NST = 6 (default): six operand stages and two half-size C chunks (128 rows x
// 128 bytes) in the same shared memory; NST = 5 (MPCR_TC2_STAGES=5): five
// stages and two 128 x 256-byte chunks.  Six stages: +1.5 % on the n=65536
// Cholesky (770.5 -> 782 TF/s), dense GEMM unchanged.
constexpr int B2_STAGE = (BN / 2) * 128;  // 16 KB
template <int NST>
constexpr int c2_chunk() { return NST == 5 ? C_CHUNK : C_CHUNK / 2; }
template <int NST>
constexpr int smem2_bytes() { return NST * (A_STAGE + B2_STAGE) + 2 * c2_chunk<NST>() + 1024 + 256; }

// MC = 2: two pairs per cluster (4 CTAs) compute horizontally adjacent
// 256 x 256 tiles (same A rows, N-blocks 2q and 2q+1); each CTA loads half of
// its 128 A rows and multicasts them to the CTA of the other pair that needs
// the same rows, so the pair-of-pairs reads A from L2 once (48 KB of L2->SMEM
// traffic per pair and K step instead of 64 KB).  Requires MN-major A (64-row
// boxes) and an even number of N-blocks.  A stage is free again only once
// both pairs' MMAs have read it (empty barriers count MC commits).
template <bool A_MN, bool B_MN, typename TC, int STAGES2, int MC>
__global__ void __cluster_dims__(2 * MC, 1, 1) __launch_bounds__(NTHREADS, 1)
    gemm_tc2_kernel(const __grid_constant__ Params p) {
    static_assert(MC == 1 || (MC == 2 && A_MN), "multicast pairs need MN-major A");
    constexpr int ES = 2, BK = 64, BW = 64;
    constexpr int BOX = BW * BK * ES;          // 8 KB MN-major box
    constexpr int KSTEP_MN = (32 / ES) * 128;  // UMMA K (32 bytes) in MN-major rows
    constexpr int C2_CHUNK = c2_chunk<STAGES2>();
    constexpr int CW = C2_CHUNK / BM / sizeof(TC);
    constexpr int NCHUNK = BN / CW;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES2 * A_STAGE;
    TC* cbuf0 = reinterpret_cast<TC*>(sB + STAGES2 * B2_STAGE);  // two chunks of C2_CHUNK bytes
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(cbuf0) + 2 * C2_CHUNK);
    uint64_t* empty = full + STAGES2;
    uint64_t* tfull = empty + STAGES2;
    uint64_t* tempty = tfull + 2;
    uint64_t* cfull = tempty + 2;  // [2]
    uint64_t* cempty = cfull + 2;  // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cempty + 2);
    auto cbuf_of = [&](int b) { return reinterpret_cast<TC*>(reinterpret_cast<uint8_t*>(cbuf0) + b * C2_CHUNK); };

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t crank = ptx::cluster_ctarank();
    const uint32_t rank = crank & 1u;  // CTA within its pair
    const uint32_t pair = crank >> 1;  // pair within the cluster (MC == 2)
    const uint32_t lead = crank & ~1u;  // the pair's even CTA
    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&p.map_a[0]);
        ptx::tma_prefetch_desc(&p.map_a[1]);
        ptx::tma_prefetch_desc(&p.map_b[0]);
        ptx::tma_prefetch_desc(&p.map_b[1]);
        ptx::tma_prefetch_desc(&p.map_c);
        for (int s = 0; s < STAGES2; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], MC);  // one MMA commit per pair of the cluster
        }
        for (int s = 0; s < 2; ++s) {
            ptx::mbar_init(&tfull[s], 1);
            ptx::mbar_init(&tempty[s], 2);  // one arrival per CTA of the pair
            ptx::mbar_init(&cfull[s], 1);
            ptx::mbar_init(&cempty[s], 1);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc_2sm<TMEM_COLS>(tmem_slot);
    ptx::tc_fence_before();
    ptx::cluster_sync_all();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int mpairs = (p.mblocks + 1) / 2;  // an odd last block pairs with an out-of-range one
    const int nq = p.nblocks / MC;           // N-block groups (one block per pair)
    const int tiles_per_prob = mpairs * nq;
    const int64_t total = static_cast<int64_t>(p.nprob) * tiles_per_prob;
    const int64_t cid = blockIdx.x / (2 * MC);
    const int64_t wave0 = (cid / p.lanes) * static_cast<int64_t>(p.lanes) * p.per;
    const int64_t t_first = wave0 + cid % p.lanes;
    const int64_t t_end = min(total, wave0 + static_cast<int64_t>(p.lanes) * p.per);
    const int64_t ncl = p.lanes;
    const bool read_c = p.beta != 0.0f;
    // Units of a problem in groups of up to 8 M-pairs, N-blocks within a group:
    // the ~74 pairs in flight share 8 A and ~9 B slabs per K step, so large
    // GEMMs stream each operand from HBM a few times instead of once per
    // tile row (the Cholesky's 4 x 4-unit tiles keep the plain M-fastest order).
    constexpr int GROUP_M = 8;
    auto decode = [&](int64_t t, TcProblem& pr, int& m0, int& n0) {
        const int64_t pi = t / tiles_per_prob;
        const int r = static_cast<int>(t - pi * tiles_per_prob);
        pr = p.problems ? p.problems[pi] : p.single;
        const int per_group = GROUP_M * nq;
        const int g = r / per_group, rem = r - g * per_group;
        const int gm = min(GROUP_M, mpairs - g * GROUP_M);  // the last group may be narrower
        m0 = (g * GROUP_M + rem % gm) * (2 * BM) + static_cast<int>(rank) * BM;
        n0 = ((rem / gm) * MC + static_cast<int>(pair)) * BN;
    };

    if (warp == 0) {
        // ===== TMA producer (both CTAs): own A rows, own half of B =====
        if (lane == 0) {
            const uint32_t full0 = ptx::mapa_shared(ptx::smem_u32(full), lead);  // the pair's even CTA
            // multicast A: this CTA's A box `pair` also lands in the CTA of the
            // other pair holding the same rows (same `rank`)
            const uint16_t a_mask = static_cast<uint16_t>((1u << rank) | (1u << (rank + 2)));
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t t = t_first; t < t_end; t += ncl) {
                TcProblem pr;
                int m0, n0;
                decode(t, pr, m0, n0);
                const int nb0 = n0 + static_cast<int>(rank) * (BN / 2);
                // (multicast pairs run the whole K: the two pairs' units must stay in lockstep)
                const int kb1 = MC == 1 ? unit_kb1(p, n0, BN, BK) : p.kblocks1;
                const int nkb = (p.kblocks / p.kblocks1) * kb1;
                for (int kb = 0; kb < nkb; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], 2 * (A_STAGE + B2_STAGE));
                    const uint32_t fb = full0 + stage * 8;
                    uint8_t* a_dst = sA + stage * A_STAGE;
                    uint8_t* b_dst = sB + stage * B2_STAGE;
                    const int sg = kb / kb1;
                    const int kk = (kb - sg * kb1) * BK;
                    const CUtensorMap* ma = &p.map_a[p.seg_a[sg]];
                    const CUtensorMap* mb = &p.map_b[p.seg_b[sg]];
                    if (MC == 2) {
                        ptx::tma_load_3d_2sm_mc(a_dst + pair * BOX, ma, ptx::smem_u32(&full[stage]) & ptx::PEER_BIT_MASK,
                                                m0 + static_cast<int>(pair) * BW, kk, pr.a_tile, a_mask);
                    } else if (A_MN) {
#pragma unroll
                        for (int j = 0; j < BM / BW; ++j)
                            ptx::tma_load_3d_2sm(a_dst + j * BOX, ma, fb, m0 + j * BW, kk, pr.a_tile);
                    } else {
                        ptx::tma_load_3d_2sm(a_dst, ma, fb, kk, m0, pr.a_tile);
                    }
                    if (B_MN) {
#pragma unroll
                        for (int j = 0; j < (BN / 2) / BW; ++j)
                            ptx::tma_load_3d_2sm(b_dst + j * BOX, mb, fb, nb0 + j * BW, kk, pr.b_tile);
                    } else {
                        ptx::tma_load_3d_2sm(b_dst, mb, fb, kk, nb0, pr.b_tile);
                    }
                    if (++stage == STAGES2) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== pair MMA issuer (even CTA only) =====
        if (rank == 0 && lane == 0) {
            constexpr uint32_t idesc = ptx::umma_idesc(2 * BM, BN, A_MN, B_MN, 0u);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int64_t t = t_first; t < t_end; t += ncl) {
                ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
                TcProblem pr_;
                int m0_, n0_;
                decode(t, pr_, m0_, n0_);
                const int nkb = (p.kblocks / p.kblocks1) * (MC == 1 ? unit_kb1(p, n0_, BN, BK) : p.kblocks1);
                for (int kb = 0; kb < nkb; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t a_base = ptx::smem_u32(sA + stage * A_STAGE);
                    const uint32_t b_base = ptx::smem_u32(sB + stage * B2_STAGE);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint64_t ad = A_MN ? ptx::umma_desc_sw128(a_base + k * KSTEP_MN, BOX, 1024)
                                                 : ptx::umma_desc_sw128(a_base + k * 32, 0, 1024);
                        const uint64_t bd = B_MN ? ptx::umma_desc_sw128(b_base + k * KSTEP_MN, BOX, 1024)
                                                 : ptx::umma_desc_sw128(b_base + k * 32, 0, 1024);
                        ptx::mma_f16_ss_2sm(d_tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
                    }
                    // both pairs' producers write this stage (A multicast): free it in all CTAs
                    ptx::mma_commit_2sm_mc(&empty[stage], MC == 2 ? 0xF : 0x3);
                    if (++stage == STAGES2) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                ptx::mma_commit_2sm_mc(&tfull[acc], static_cast<uint16_t>(0x3u << lead));
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (warp == 3) {
        // ===== C loader (both CTAs, own rows) =====
        if (lane == 0) {
            uint32_t g = 0;  // running chunk count: buffer g & 1, phase (g >> 1) & 1
            for (int64_t t = t_first; t < t_end; t += ncl) {
                TcProblem pr;
                int m0, n0;
                decode(t, pr, m0, n0);
                for (int h = 0; h < NCHUNK; ++h, ++g) {
                    const int b = g & 1;
                    ptx::mbar_wait(&cempty[b], ((g >> 1) & 1) ^ 1);
                    if (read_c) {
                        ptx::mbar_arrive_expect_tx(&cfull[b], C2_CHUNK);
                        if (p.c_evict_first)
                            ptx::tma_load_3d_hint(cbuf_of(b), &p.map_c, &cfull[b], m0, n0 + h * CW, pr.c_tile,
                                                  ptx::l2_policy_evict_first());
                        else
                            ptx::tma_load_3d(cbuf_of(b), &p.map_c, &cfull[b], m0, n0 + h * CW, pr.c_tile);
                    } else {
                        ptx::mbar_arrive(&cfull[b]);
                    }
                }
            }
        }
    } else if (warp >= 4) {
        // ===== epilogue (both CTAs, own 128 TMEM lanes) =====
        const int q = warp - 4;
        const int r = q * 32 + lane;
        const bool is_leader = threadIdx.x == 128;
        const uint32_t tempty0 = ptx::mapa_shared(ptx::smem_u32(tempty), lead);
        int acc = 0;
        uint32_t acc_phase = 0, g = 0;
        for (int64_t t = t_first; t < t_end; t += ncl) {
            TcProblem pr;
            int m0, n0;
            decode(t, pr, m0, n0);
            ptx::mbar_wait(&tfull[acc], acc_phase);
            ptx::tc_fence_after();
            const int row = m0 + r;
#pragma unroll 1
            for (int h = 0; h < NCHUNK; ++h, ++g) {
                const int b = g & 1;
                TC* cbuf = cbuf_of(b);
                ptx::mbar_wait(&cfull[b], (g >> 1) & 1);
#pragma unroll 1
                for (int c = 0; c < CW / 32; ++c) {
                    uint32_t v[32];
                    const int col0 = h * CW + c * 32;
                    ptx::tmem_ld_32x32b_x32(
                        tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + col0, v);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int cc = c * 32 + j;
                        const float a = __fmul_rn(p.alpha, __uint_as_float(v[j]));
                        float out = a;
                        if (read_c) {
                            const float old = ld_c(cbuf, cc * BM + r);
                            out = (pr.lower_only && row < n0 + col0 + j)
                                      ? old
                                      : __fadd_rn(a, __fmul_rn(p.beta, old));
                        }
                        st_c(cbuf, cc * BM + r, out);
                    }
                }
                ptx::fence_proxy_async_smem();
                ptx::named_bar_sync(1, EPI_THREADS);
                if (is_leader) {
                    if (p.c_evict_first)
                        ptx::tma_store_3d_hint(&p.map_c, cbuf, m0, n0 + h * CW, pr.c_tile,
                                               ptx::l2_policy_evict_first());
                    else
                        ptx::tma_store_3d(&p.map_c, cbuf, m0, n0 + h * CW, pr.c_tile);
                    ptx::bulk_commit();
                    ptx::bulk_wait_read0();
                    ptx::mbar_arrive(&cempty[b]);
                }
            }
            // this CTA is done with accumulator `acc`: one arrival on the even CTA
            ptx::tc_fence_before();
            ptx::named_bar_sync(2, EPI_THREADS);
            if (is_leader) ptx::mbar_arrive_cluster(tempty0 + acc * 8);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
        if (is_leader) ptx::bulk_wait0();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync_all();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_2sm<TMEM_COLS>(tmem_base);
    }
}

// ---- host side ---------------------------------------------------------------
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    if (!fn) fail(MP_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

// 3-D map over [d2 tiles][d1][d0] elements; d0 contiguous.
void make_map(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int esize, uint64_t d0,
              uint64_t d1, uint64_t d2, uint64_t ld_elems, uint64_t tile_stride_elems,
              uint32_t box0, uint32_t box1, CUtensorMapSwizzle swz) {
    const cuuint64_t dims[3] = {d0, d1, d2 < 1 ? 1 : d2};
    const cuuint64_t strides[2] = {ld_elems * esize,
                                   (tile_stride_elems ? tile_stride_elems : ld_elems * d1) * esize};
    const cuuint32_t box[3] = {box0, box1, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = get_encode()(map, dt, 3, const_cast<void*>(base), dims, strides, box, estr,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(MP_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
}

}  // namespace tc

void tma_map_3d(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int esize, uint64_t d0,
                uint64_t d1, uint64_t d2, uint64_t ld_elems, uint64_t tile_stride_elems, uint32_t box0,
                uint32_t box1, CUtensorMapSwizzle swz) {
    tc::make_map(map, base, dt, esize, d0, d1, d2, ld_elems, tile_stride_elems, box0, box1, swz);
}

namespace tc {

// Operand map: 128-byte swizzled boxes of 128 bytes x box1 rows.
void make_op_map(CUtensorMap* map, int kind, const void* base, uint64_t d0, uint64_t d1,
                 uint64_t d2, uint64_t ld, uint64_t ts, uint32_t box1) {
    const int es = kind == 0 ? 2 : 4;
    make_map(map, base, kind == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
             es, d0, d1, d2, ld, ts, 128 / es, box1, CU_TENSOR_MAP_SWIZZLE_128B);
}

template <int KIND, bool A_MN, bool B_MN, typename TC>
void launch_kernel(Ctx* ctx, cudaStream_t s, const Params& p, int64_t total, int tiles_per_cta) {
    auto kern = gemm_tc_kernel<KIND, A_MN, B_MN, TC>;
    static unsigned long long configured = 0;  // per-device bitmask
    if (first_on_device(configured)) {
        MP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    }
    const int grid = static_cast<int>(std::min<int64_t>(persistent_grid(total, ctx->sm_count, tiles_per_cta), 1 << 30));
    kern<<<grid, NTHREADS, SMEM_BYTES, s>>>(p);
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}


template <bool A_MN, bool B_MN, typename TC, int NST, int MC>
void launch_kernel2(Ctx* ctx, cudaStream_t s, const Params& p, int64_t total_pairs, int tiles_per_cta) {
    auto kern = gemm_tc2_kernel<A_MN, B_MN, TC, NST, MC>;
    constexpr int SMEM2_BYTES = smem2_bytes<NST>();
    static unsigned long long configured = 0;  // per-device bitmask
    static int max_clusters[64] = {};
    int dev = 0;
    MP_CUDA(cudaGetDevice(&dev));
    if (first_on_device(configured)) {
        MP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2_BYTES));
        // clusters of 2 MC CTAs (one per SM) that fit at once: with MC = 2 a
        // GPC whose SM count is not a multiple of 4 leaves SMs unused
        cudaLaunchConfig_t oc = {};
        oc.gridDim = dim3(static_cast<unsigned>(2 * MC * (ctx->sm_count / (2 * MC))));
        oc.blockDim = dim3(NTHREADS);
        oc.dynamicSmemBytes = SMEM2_BYTES;
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, kern, &oc) != cudaSuccess || nc < 1) {
            (void)cudaGetLastError();
            nc = ctx->sm_count / (2 * MC);
        }
        max_clusters[dev & 63] = nc;
        static const bool dbg = getenv("MPCR_DEBUG_TC") != nullptr;
        if (dbg) std::fprintf(stderr, "[mpcr] pair kernel MC=%d: %d clusters resident\n", MC, nc);
    }
    const int resident = std::max(1, std::min(max_clusters[dev & 63], ctx->sm_count / (2 * MC)));
    const int64_t units = total_pairs / MC;  // a cluster takes MC horizontally adjacent pair tiles
    // bounded persistence counts pair tiles: a cluster unit holds MC of them
    const int tpc = tiles_per_cta > 0 ? std::max(1, tiles_per_cta / MC) : tiles_per_cta;
    const int64_t clusters = persistent_grid(units, resident, tpc);
    Params q = p;
    q.lanes = static_cast<int32_t>(std::min<int64_t>(resident, clusters));
    q.per = static_cast<int32_t>((units + clusters - 1) / clusters);
    static const bool strided = [] {  // MPCR_UNIT_STRIDED=1: classic grid-stride assignment
        const char* e = getenv("MPCR_UNIT_STRIDED");
        return e && e[0] == '1';
    }();
    if (strided) {
        q.lanes = static_cast<int32_t>(clusters);
        q.per = static_cast<int32_t>((units + clusters - 1) / clusters);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(2 * MC * clusters));
    cfg.blockDim = dim3(NTHREADS);
    cfg.dynamicSmemBytes = SMEM2_BYTES;
    cfg.stream = s;
    MP_CUDA(cudaLaunchKernelEx(&cfg, kern, q));
    count_launch(ctx);
    MP_CUDA(cudaGetLastError());
}

}  // namespace tc

bool tc_gemm_supported(const TcGemm& g) {
    // TMA: 16-byte aligned bases and leading strides for A, B and C.
    auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
    const int es = g.kind == 0 ? 2 : 4;
    if (!al(g.A) || !al(g.B) || !al(g.C) || (g.A2 && !al(g.A2)) || (g.B2 && !al(g.B2))) return false;
    if ((g.lda * es) % 16 || (g.ldb * es) % 16 || (g.ldc * elem_bytes(g.pc)) % 16) return false;
    if (g.m < 1 || g.n < 1 || g.k < 1) return false;
    if (g.m >= (1ll << 31) || g.n >= (1ll << 31) || g.k >= (1ll << 31)) return false;
    if (g.kind == 1 && g.pc != MP_SINGLE) return false;
    return g.pc == MP_HALF || g.pc == MP_SINGLE;
}

void launch_tc_gemm(Ctx* ctx, cudaStream_t s, const TcGemm& g) {
    using namespace tc;
    Params p;
    std::memset(&p, 0, sizeof(p));
    const bool a_mn = !g.ta, b_mn = g.tb;
    const int kind = g.kind;
    static const bool tc2_env = [] {
        const char* e = getenv("MPCR_TC2");
        return !(e && e[0] == '0');
    }();
    const bool pair = kind == 0 && tc2_env;  // FP16: 2-CTA pair kernel
    static const int tc2_stages = [] {
        const char* e = getenv("MPCR_TC2_STAGES");
        return (e && e[0] == '5') ? 5 : 6;
    }();
    const uint32_t rows_a = a_mn ? 0 : BM, rows_b = b_mn ? 0 : (pair ? BN / 2 : BN);
    const void* As[2] = {g.A, g.A2 ? g.A2 : g.A};
    const void* Bs[2] = {g.B, g.B2 ? g.B2 : g.B};
    for (int i = 0; i < 2; ++i) {
        // op(A): m x k.  MN-major: storage m x k (ld lda).  K-major: storage k x m.
        if (a_mn)
            make_op_map(&p.map_a[i], kind, As[i], g.m, g.k, g.a_tiles, g.lda, g.a_tile_stride, 128 / (kind ? 4 : 2));
        else
            make_op_map(&p.map_a[i], kind, As[i], g.k, g.m, g.a_tiles, g.lda, g.a_tile_stride, rows_a);
        if (b_mn)
            make_op_map(&p.map_b[i], kind, Bs[i], g.n, g.k, g.b_tiles, g.ldb, g.b_tile_stride, 128 / (kind ? 4 : 2));
        else
            make_op_map(&p.map_b[i], kind, Bs[i], g.k, g.n, g.b_tiles, g.ldb, g.b_tile_stride, rows_b);
    }
    // C: [c_tiles][n][m] with chunks of 128 rows x 256 bytes
    const bool half_c = g.pc == MP_HALF;
    make_map(&p.map_c, g.C, half_c ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
             half_c ? 2 : 4, g.m, g.n, g.c_tiles, g.ldc, g.c_tile_stride, BM,
             (half_c ? 128 : 64) / (pair && tc2_stages == 6 ? 2 : 1),
             CU_TENSOR_MAP_SWIZZLE_NONE);
    // K segments
    int nseg = 1;
    p.seg_a[0] = p.seg_b[0] = 0;
    // The tensor core's FP32 accumulator truncates on every MMA, so the error
    // grows with the accumulator's magnitude: the small lo segments go first
    // and hi*hi last.
    if (kind == 1 && g.A2 && g.B2) {  // 3xTF32: hi*lo + lo*hi + hi*hi
        nseg = 3;
        p.seg_a[0] = 0; p.seg_b[0] = 1;
        p.seg_a[1] = 1; p.seg_b[1] = 0;
        p.seg_a[2] = 0; p.seg_b[2] = 0;
    } else if (g.two_panels && g.A2 && g.B2) {  // A B (step k) then A2 B2 (step k+1)
        nseg = 2;
        p.seg_a[0] = 0; p.seg_b[0] = 0;
        p.seg_a[1] = 1; p.seg_b[1] = 1;
    } else if (g.B2) {  // A * B_lo + A * B
        nseg = 2;
        p.seg_a[0] = 0; p.seg_b[0] = 1;
        p.seg_a[1] = 0; p.seg_b[1] = 0;
    }
    static const int c_evict_first = [] {
        const char* e = getenv("MPCR_C_EVICT_FIRST");
        return (e && e[0] == '0') ? 0 : 1;
    }();
    p.c_evict_first = c_evict_first;
    p.problems = g.problems;
    p.single = TcProblem{0, 0, 0, g.lower_only ? 1 : 0};
    p.nprob = g.problems ? static_cast<int32_t>(g.count) : 1;
    p.M = static_cast<int32_t>(g.m);
    p.N = static_cast<int32_t>(g.n);
    p.K = static_cast<int32_t>(g.k);
    p.alpha = static_cast<float>(g.alpha);
    p.beta = static_cast<float>(g.beta);
    p.mblocks = static_cast<int32_t>((g.m + BM - 1) / BM);
    p.nblocks = static_cast<int32_t>((g.n + BN - 1) / BN);
    const int bk = kind == 0 ? 64 : 32;
    p.kblocks1 = static_cast<int32_t>((g.k + bk - 1) / bk);
    p.kblocks = nseg * p.kblocks1;
    p.k_tri = g.k_tri ? 1 : 0;
    const int64_t total = static_cast<int64_t>(p.nprob) * p.mblocks * p.nblocks;
    ProfScope ps(ctx, kind == 0 ? MP_PROF_GEMM_F16 : MP_PROF_GEMM_F32, s,
                 2.0 * static_cast<double>(g.m) * g.n * g.k * p.nprob * (g.two_panels ? 2 : 1) *
                     (g.lower_only ? 0.5 : 1.0));
    if (pair) {
        const int64_t pairs = static_cast<int64_t>(p.nprob) * ((p.mblocks + 1) / 2) * p.nblocks;
        // MPCR_DEBUG_TC: one line per pair-kernel launch in issue order (picks
        // the launch index of an ncu capture and its tile count)
        static const bool dbg_tc = getenv("MPCR_DEBUG_TC") != nullptr;
        static int64_t dbg_idx = 0;
        if (dbg_tc)
            std::fprintf(stderr, "[mpcr] tc2 launch %lld: C %s, %d problem(s) of %dx%dx%d, beta %g\n",
                         static_cast<long long>(dbg_idx++), half_c ? "half" : "single", p.nprob, p.M,
                         p.N, p.K, p.beta);
        // MPCR_TC4=1: clusters of two pairs with A multicast (even N-block
        // count, MN-major A, six stages)
        static const bool tc4_env = [] {
            const char* e = getenv("MPCR_TC4");
            return e && e[0] == '1';
        }();
        if (tc4_env && a_mn && p.nblocks % 2 == 0 && tc2_stages == 6) {
            if (b_mn)
                half_c ? launch_kernel2<true, true, uint16_t, 6, 2>(ctx, s, p, pairs, g.tiles_per_cta)
                       : launch_kernel2<true, true, float, 6, 2>(ctx, s, p, pairs, g.tiles_per_cta);
            else
                half_c ? launch_kernel2<true, false, uint16_t, 6, 2>(ctx, s, p, pairs, g.tiles_per_cta)
                       : launch_kernel2<true, false, float, 6, 2>(ctx, s, p, pairs, g.tiles_per_cta);
            return;
        }
#define MP_TC2(AM, BMJ)                                                                 \
        if (a_mn == AM && b_mn == BMJ) {                                                \
            if (tc2_stages == 6) {                                                      \
                if (half_c)                                                             \
                    launch_kernel2<AM, BMJ, uint16_t, 6, 1>(ctx, s, p, pairs, g.tiles_per_cta); \
                else                                                                    \
                    launch_kernel2<AM, BMJ, float, 6, 1>(ctx, s, p, pairs, g.tiles_per_cta); \
            } else if (half_c) {                                                        \
                launch_kernel2<AM, BMJ, uint16_t, 5, 1>(ctx, s, p, pairs, g.tiles_per_cta); \
            } else {                                                                    \
                launch_kernel2<AM, BMJ, float, 5, 1>(ctx, s, p, pairs, g.tiles_per_cta);   \
            }                                                                           \
            return;                                                                     \
        }
        MP_TC2(true, true)
        MP_TC2(true, false)
        MP_TC2(false, true)
        MP_TC2(false, false)
#undef MP_TC2
    }
#define MP_TC(AM, BMJ)                                                                  \
    if (a_mn == AM && b_mn == BMJ) {                                                    \
        if (kind == 1)                                                                  \
            launch_kernel<1, AM, BMJ, float>(ctx, s, p, total, g.tiles_per_cta);        \
        else if (half_c)                                                                \
            launch_kernel<0, AM, BMJ, uint16_t>(ctx, s, p, total, g.tiles_per_cta);     \
        else                                                                            \
            launch_kernel<0, AM, BMJ, float>(ctx, s, p, total, g.tiles_per_cta);        \
        return;                                                                         \
    }
    MP_TC(true, true)
    MP_TC(true, false)
    MP_TC(false, true)
    MP_TC(false, false)
#undef MP_TC
}

}  // namespace mpcr
