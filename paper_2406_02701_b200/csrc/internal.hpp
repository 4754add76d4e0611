// Internal types of the B200-native MPCR engine (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "mpcr_b200.h"

struct mp_tile_s;

namespace mpcr {

// Thrown inside the library, converted to mp_status at the C-ABI edge.
struct Error : std::runtime_error {
    mp_status status;
    int64_t info;
    Error(mp_status s, const std::string& msg, int64_t inf = -1)
        : std::runtime_error(msg), status(s), info(inf) {}
};

[[noreturn]] inline void fail(mp_status s, const std::string& msg) { throw Error(s, msg); }

#define MP_CUDA(expr)                                                                   \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess)                                                          \
            ::mpcr::fail(e_ == cudaErrorMemoryAllocation ? MP_OUT_OF_MEMORY : MP_CUDA_ERROR, \
                         std::string(#expr) + ": " + cudaGetErrorString(e_));           \
    } while (0)

inline int elem_bytes(mp_precision p) { return p == MP_HALF ? 2 : p == MP_SINGLE ? 4 : 8; }
inline mp_precision promote(mp_precision a, mp_precision b) { return a >= b ? a : b; }
// array.hpp:109-111 — Half kernels compute in Single.
inline mp_precision compute_precision(mp_precision p) { return p == MP_HALF ? MP_SINGLE : p; }
inline const char* prec_name(mp_precision p) {
    return p == MP_HALF ? "half" : p == MP_SINGLE ? "single" : "double";
}

struct Ctx;

// Event-pair profiler per kernel class (mp_prof_*).
struct Prof {
    bool enabled = false;
    struct Rec {
        cudaEvent_t a, b;
        int cls;
        double work;
        cudaStream_t s;
    };
    std::vector<Rec> pending;
    // optional timeline (mp_prof_trace): per-launch start/end relative to base
    bool trace = false;
    cudaEvent_t base = nullptr;
    struct Span {
        int cls, stream;
        float t0, t1;
    };
    std::vector<Span> spans;
    std::vector<cudaEvent_t> pool;
    double ms[MP_PROF_NUM_CLASSES] = {};
    int64_t launches[MP_PROF_NUM_CLASSES] = {};
    double work[MP_PROF_NUM_CLASSES] = {};
    // device counters while profiling: [0] INT8 digit-pair MMAs issued per
    // 128-row k-extent, summed over output tiles; [1] those output tiles
    unsigned long long* dev_stats = nullptr;
};

struct Ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;   // current (own or external)
    cudaStream_t aux[4] = {};        // scheduler side streams
    cudaStream_t hi = nullptr;       // high-priority critical-path stream
    cudaStream_t hi2 = nullptr;      // second high-priority stream (lookahead side work)
    int64_t launches = 0;            // kernels launched by this library
    Prof prof;
    // Scratch device memory (grown on demand, freed with the context).
    // slot 0: op-level work buffers, 1: staging / POTRF barriers, 2: GEMM
    // operand splits (3xTF32), 3: spare
    void* scr[4] = {nullptr, nullptr, nullptr, nullptr};
    size_t scr_bytes[4] = {0, 0, 0, 0};
    // bumped whenever a scratch slot is (re)allocated: CUDA graphs captured
    // over scratch pointers are stale once it changes
    uint64_t scr_gen = 0;
    void* ensure_scratch(size_t bytes, int which = 0);
    // Work counters of dynamically scheduled persistent kernels: one pair
    // [next unit, CTAs finished] per launch, handed out round robin; the last
    // CTA of a launch resets its pair, so captured graphs replay unchanged.
    static constexpr int SCHED_SLOTS = 8192;  // > the INT8-digit launches of any captured factorization
    unsigned int* sched_pool = nullptr;  // 2 * SCHED_SLOTS, zeroed at context creation
    int sched_next = 0;
    unsigned int* sched_slot() { return sched_pool + 2 * (sched_next++ % SCHED_SLOTS); }
};

// Make ctx's device current for this thread (every C-ABI entry point does
// this through its handle accessors before any allocation or launch).
inline void bind_device(const Ctx* c) {
    int d = -1;
    if (cudaGetDevice(&d) != cudaSuccess || d != c->device) {
        const cudaError_t e = cudaSetDevice(c->device);
        if (e != cudaSuccess) throw std::runtime_error(std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    }
}

struct Array {
    Ctx* ctx = nullptr;
    mp_precision prec = MP_DOUBLE;
    int64_t rows = 0, cols = 0, ld = 0;
    bool is_matrix = false;
    bool owner = true;
    void* data = nullptr;
    int64_t size() const { return rows * cols; }
    size_t bytes() const { return static_cast<size_t>(ld * cols) * elem_bytes(prec); }
};

// Begin/end an event-timed region for kernel class `cls` on `s`.
struct ProfScope {
    Ctx* ctx;
    int cls;
    cudaStream_t s;
    double work;
    cudaEvent_t a = nullptr;
    ProfScope(Ctx* c, int k, cudaStream_t st, double w);
    ~ProfScope();
};

// Fold finished event pairs into the totals (blocking: wait for all).
void prof_collect(Ctx* ctx, bool blocking = true);

// ---- kernels (each returns after enqueueing on stream s) -----------------
// casts: cast.cu
void launch_convert(Ctx* ctx, cudaStream_t s, mp_precision pin, const void* src, int64_t lds,
                    mp_precision pout, void* dst, int64_t ldd, int64_t rows, int64_t cols);
void launch_from_doubles(Ctx* ctx, cudaStream_t s, const double* src, mp_precision pout,
                         void* dst, int64_t n);
// ew.cu
void launch_ew_binary(Ctx* ctx, cudaStream_t s, int op, const Array& a, const Array& b,
                      Array& out);
void launch_ew_scalar(Ctx* ctx, cudaStream_t s, int op, const Array& a, double v, Array& out);
void launch_ew_unary(Ctx* ctx, cudaStream_t s, int op, const Array& a, Array& out);
double run_reduce(Ctx* ctx, cudaStream_t s, int op, const Array& a);
void launch_transpose(Ctx* ctx, cudaStream_t s, const Array& a, Array& out);
void launch_diag(Ctx* ctx, cudaStream_t s, const Array& a, Array& out);
void launch_fill(Ctx* ctx, cudaStream_t s, mp_precision p, void* dst, int64_t ld,
                 int64_t rows, int64_t cols, double value);

// GEMM: gemm.cu.  Dense column-major C <- alpha op(A) op(B) + beta C, computed
// in compute_precision(pc).  lower_only: skip C entries strictly above the
// diagonal (SYRK on the lower triangle).
struct GemmDesc {
    mp_precision pa, pb, pc;
    bool ta, tb;
    int64_t m, n, k;
    double alpha, beta;
    const void* A;
    int64_t lda;
    const void* B;
    int64_t ldb;
    void* C;
    int64_t ldc;
    bool lower_only = false;
};
void launch_gemm(Ctx* ctx, cudaStream_t s, const GemmDesc& g);
// solve.cu: exact symmetry test and LU (partial pivoting) solve
bool device_exactly_symmetric(Ctx* ctx, cudaStream_t s, mp_precision p, const void* a, int64_t lda, int64_t n);
int64_t lu_solve_device(Ctx* ctx, cudaStream_t s, mp_precision cp, void* w, int64_t n, const void* b,
                        int64_t ldb, void* x, int64_t ldx, int64_t ncols);
// Grid of a persistent tile kernel (one CTA per SM resident): fully
// persistent when tiles_per_cta <= 0, else whole waves of SMs with at most
// ~tiles_per_cta tiles per CTA (so SMs are handed back at that granularity
// without a ragged last wave).
inline int64_t persistent_grid(int64_t total, int sms, int tiles_per_cta) {
    if (total <= sms) return total < 1 ? 1 : total;
    if (tiles_per_cta <= 0) return sms;
    const int64_t waves = (total + static_cast<int64_t>(sms) * tiles_per_cta - 1) /
                          (static_cast<int64_t>(sms) * tiles_per_cta);
    const int64_t g = waves * sms;
    return g < total ? g : total;
}
bool ozaki_enabled();  // MPCR_OZAKI=0 turns the INT8 FP64 path off

// Grouped tile GEMM used by the MPCRTile scheduler: every problem is
// C_p <- alpha A_p op(B_p) + beta C_p with identical shapes.
struct TileProblem {
    const void* A;  // m x k, column-major, lda
    const void* B;  // (tb ? n x k : k x n), column-major, ldb
    void* C;        // m x n, column-major, ldc
    int32_t lower_only;
    int32_t pad;
};
struct GroupedGemm {
    mp_precision pab;   // operand precision (A and B)
    mp_precision pc;    // output precision
    bool tb;            // B transposed (the tiled-chol update is NT)
    int64_t m, n, k, lda, ldb, ldc;
    double alpha, beta;
    const TileProblem* problems;  // device array
    int64_t count;
    // Optional: all operand tiles are slices of one slab (enables TMA maps).
    const void* slab = nullptr;
    int64_t slab_tiles = 0;
    // Critical-path launch: each CTA reserves its SM (no co-resident CTAs).
    bool exclusive = false;
    int k_lower = 0;  // FP64: lower-triangular operand, see DmmaArgs::k_lower
};
void launch_grouped_gemm(Ctx* ctx, cudaStream_t s, const GroupedGemm& g);

// Cholesky / triangular kernels: potrf.cu, trsm.cu
// In-place lower Cholesky of a column-major n x n matrix (compute in the
// compute precision of p); writes the failing column (or -1) to dev_info.
// FP64 only: when linv_diag is given, the inverses of the 64x64 diagonal
// blocks of L are written onto the diagonal blocks of linv_diag (ld ldi).
void launch_potrf_lower(Ctx* ctx, cudaStream_t s, mp_precision p, void* A, int64_t lda,
                        int64_t n, int64_t* dev_info, int64_t info_offset,
                        double* linv_diag = nullptr, int64_t ldi = 0);
// Inverse of a lower triangular FP64 matrix, out of place.  The strictly
// upper part of Linv is written with zeros.
void launch_trtri_lower(Ctx* ctx, cudaStream_t s, const double* L, int64_t ldl, double* Linv,
                        int64_t ldi, int64_t n);
struct TrtriPlan;
TrtriPlan* trtri_plan_create(Ctx* ctx, cudaStream_t s, const double* L, int64_t ldl, double* Linv,
                             int64_t ldi, int64_t n);
void trtri_plan_destroy(TrtriPlan* P);
void launch_trtri_plan(Ctx* ctx, cudaStream_t s, TrtriPlan* P, bool leaves_done);
// General triangular solve (linalg.cpp:130-159 semantics): op(T) X = B for
// every column of B (in place), computing in compute type of pb.
void launch_tri_solve(Ctx* ctx, cudaStream_t s, mp_precision pt, const void* T, int64_t ldt,
                      int64_t n, bool upper, bool trans, mp_precision pb, void* B,
                      int64_t ldb, int64_t ncols, double alpha, bool right_side,
                      int64_t brows);
// Scan the diagonal of T for exact zeros; returns first index or -1 (syncs).
int64_t find_zero_diag(Ctx* ctx, cudaStream_t s, mp_precision p, const void* T, int64_t ldt,
                       int64_t n, mp_precision compute);
// Zero the strictly-upper (upper=true) or strictly-lower part.
void launch_zero_triangle(Ctx* ctx, cudaStream_t s, mp_precision p, void* A, int64_t lda,
                          int64_t n, bool upper);
// out = in^T for square or rectangular (generic, precision preserving).
void launch_transpose_raw(Ctx* ctx, cudaStream_t s, mp_precision p, const void* in,
                          int64_t ldi, int64_t rows, int64_t cols, void* out, int64_t ldo);
// Mirror the lower triangle into the upper (exact symmetry).
void launch_mirror_lower(Ctx* ctx, cudaStream_t s, mp_precision p, void* A, int64_t lda,
                         int64_t n);
// sum of log(diag) over n entries with stride (double accumulate) into dev_out.
void launch_logdiag_sum(Ctx* ctx, cudaStream_t s, mp_precision p, const void* A, int64_t lda,
                        int64_t n, double* dev_out);
// Matern fill of a column-major tile block.
void launch_matern_tile(Ctx* ctx, cudaStream_t s, mp_precision p, void* dst, int64_t ld,
                        int64_t row0, int64_t col0, int64_t rows, int64_t cols,
                        int64_t side, double nu, double range, double variance);

// Batched symmetric Matern fill of square nb-tiles (items built with
// matern_item_fill); x == nullptr selects the unit grid of `side` points.
void launch_matern_tiles(Ctx* ctx, cudaStream_t s, const void* items, int64_t count, int64_t nb,
                         const double* x, const double* y, int64_t side, double nu, double range,
                         double variance, double nugget);
size_t matern_item_bytes();
void matern_item_fill(void* dst, void* lo, void* up, int p_lo, int p_up, int64_t row0, int64_t col0);
void launch_matern_points(Ctx* ctx, cudaStream_t s, mp_precision p, void* dst, int64_t ld,
                          int64_t row0, int64_t col0, int64_t rows, int64_t cols, const double* x,
                          const double* y, double nu, double range, double variance,
                          double nugget);

// nll.cu: tiled forward solve pieces (FP64 right-hand side)
struct TrsvItem {
    const void* L;  // tile (j, i), nb x nb column-major
    double* r;      // r_j
};
void launch_tile_trsv(Ctx* ctx, cudaStream_t s, mp_precision p, const void* L, int64_t ld, int nb,
                      double* r);
void launch_tile_gemv(Ctx* ctx, cudaStream_t s, mp_precision p, const void* dev_items,
                      int64_t count, int nb, const double* w);
void launch_square_sum(Ctx* ctx, cudaStream_t s, const double* w, int64_t n, double* out);
void launch_add_diag(Ctx* ctx, cudaStream_t s, mp_precision p, void* A, int64_t ld, int n,
                     double v);

inline void count_launch(Ctx* ctx, int n = 1) { ctx->launches += n; }

// One-time per-device setup (kernel attribute opt-ins): true the first time
// it is called for the current device with this mask.
inline bool first_on_device(unsigned long long& mask) {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) d = 0;
    const unsigned long long bit = 1ull << (d & 63);
    if (mask & bit) return false;
    mask |= bit;
    return true;
}

extern thread_local std::string g_last_error;
double host_round(double x, mp_precision p);
int64_t tile_chol_inplace(Ctx* c, ::mp_tile_s& t);

}  // namespace mpcr

struct mp_ctx_s : mpcr::Ctx {};
struct mp_array_s : mpcr::Array {};
