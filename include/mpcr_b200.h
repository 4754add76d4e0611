/*
 * mpcr_b200.h — C ABI of the B200-native MPCR multi-precision engine.
 *
 * Drop-in boundary for the reference's C++ core (`mpnum`, /root/reference/proj)
 * and the paper's MPCRTile API.  Every entry point cites the
 * reference interface it replaces.  Plain pointers and sizes only; no C++ or
 * torch types.  All matrices are column-major (array.hpp:18).
 *
 * Error convention: every call returns mp_status, a 1:1 mirror of the
 * reference exception classes (errors.hpp:8-76).  Argument/shape/precision
 * checks run before any device work, as in the reference.  A human-readable
 * message for the last failure on the calling thread is in mp_last_error().
 * NotPositiveDefinite reports the 0-based global failing pivot column through
 * the `info` out-parameter (errors.hpp:25-31, LAPACK-style).
 *
 * Execution: every compute call is enqueued on the context's stream (settable
 * with mp_ctx_set_stream) and returns without a host sync, except calls that
 * return a host value (mp_reduce, mp_*_logdet, info-reporting factorizations)
 * which synchronise the stream.  Results are deterministic run to run.
 */
#ifndef MPCR_B200_H
#define MPCR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* precision.hpp:11 — same integer values. */
typedef enum { MP_HALF = 0, MP_SINGLE = 1, MP_DOUBLE = 2 } mp_precision;

/* errors.hpp:8-76, one code per exception class. */
typedef enum {
    MP_OK = 0,
    MP_SHAPE_MISMATCH = 1,        /* ShapeMismatch        errors.hpp:8   */
    MP_INDEX_OUT_OF_RANGE = 2,    /* IndexOutOfRange      errors.hpp:12  */
    MP_NOT_A_MATRIX = 3,          /* NotAMatrix           errors.hpp:16  */
    MP_EMPTY_ARRAY = 4,           /* EmptyArray           errors.hpp:20  */
    MP_NOT_POSITIVE_DEFINITE = 5, /* NotPositiveDefinite  errors.hpp:25  */
    MP_SINGULAR_MATRIX = 6,       /* SingularMatrix       errors.hpp:33  */
    MP_NO_CONVERGENCE = 7,        /* NoConvergence        errors.hpp:37  */
    MP_UNKNOWN_OPERATION = 8,     /* UnknownOperation     errors.hpp:41  */
    MP_BACKEND_UNAVAILABLE = 9,   /* BackendUnavailable   errors.hpp:46  */
    MP_PRECISION_MISMATCH = 10,   /* PrecisionMismatch    errors.hpp:50  */
    MP_INVALID_PARAM = 11,        /* InvalidParam         errors.hpp:54  */
    MP_IO_ERROR = 12,             /* IoError              errors.hpp:58  */
    MP_CUDA_ERROR = 100,
    MP_NCCL_ERROR = 101,
    MP_OUT_OF_MEMORY = 102,
    MP_INTERNAL_ERROR = 103
} mp_status;

/* array.hpp:94-97 */
typedef enum { MP_ADD = 0, MP_SUB = 1, MP_MUL = 2, MP_DIV = 3 } mp_binary_op;
typedef enum { MP_LOG = 0, MP_EXP = 1, MP_SQRT = 2, MP_ABS = 3 } mp_unary_op;
typedef enum { MP_SUM = 0, MP_SQUARE_SUM = 1, MP_MIN = 2, MP_MAX = 3, MP_MEAN = 4 } mp_reduce_op;
/* linalg.hpp:21 */
typedef enum { MP_LEFT = 0, MP_RIGHT = 1 } mp_side;

typedef struct mp_ctx_s* mp_ctx;     /* device, streams, workspace, comms        */
typedef struct mp_array_s* mp_array; /* device-resident MPArray (array.hpp:18)   */
typedef struct mp_tile_s* mp_tile;   /* device-resident MPCRTile  */

/* ------------------------------------------------------------------------- */
/* Library / context                                                          */
/* ------------------------------------------------------------------------- */
const char* mp_last_error(void);
const char* mp_version(void);
/* Device compute capability; fails with MP_BACKEND_UNAVAILABLE if not sm_100. */
mp_status mp_device_check(int device, int* major, int* minor, int* sm_count);

mp_status mp_ctx_create(int device, mp_ctx* out);
mp_status mp_ctx_destroy(mp_ctx ctx);
/* Use an external cudaStream_t (0 = the context's own stream). */
mp_status mp_ctx_set_stream(mp_ctx ctx, void* cuda_stream);
mp_status mp_ctx_get_stream(mp_ctx ctx, void** cuda_stream);
mp_status mp_ctx_synchronize(mp_ctx ctx);
/* Deterministic kernel-class profiling with CUDA events on the launching
 * streams.  Classes: see mp_prof_class.  Query returns summed device ms,
 * launch count and algorithmic flops (or bytes) of that class. */
typedef enum {
    MP_PROF_GEMM_F16 = 0,
    MP_PROF_GEMM_F32 = 1,
    MP_PROF_GEMM_F64 = 2,
    MP_PROF_POTRF = 3,
    MP_PROF_TRSM = 4,
    MP_PROF_CAST = 5,
    MP_PROF_OTHER = 6,
    MP_PROF_GEMM_I8 = 7, /* FP64 products of FP16 operands on INT8 digits */
    MP_PROF_NUM_CLASSES = 8
} mp_prof_class;
mp_status mp_prof_enable(mp_ctx ctx, int enable);
mp_status mp_prof_reset(mp_ctx ctx);
mp_status mp_prof_query(mp_ctx ctx, int cls, double* ms, int64_t* launches, double* work);
/* While profiling: INT8 digit-pair MMAs the FP64-from-FP16 (Ozaki) kernel
 * issued, summed over its 128 x 128 output tiles (pair_mmas / tiles = mean
 * digit products per FP64 tile product), since the last mp_prof_reset. */
mp_status mp_prof_digit_products(mp_ctx ctx, int64_t* pair_mmas, int64_t* tiles);
/* Timeline capture (profiling must be enabled): every timed launch's start
 * and end in ms relative to the moment tracing was enabled, with its stream
 * (0 = context stream, 1 = critical-path stream); dumped as CSV. */
mp_status mp_prof_trace(mp_ctx ctx, int enable);
mp_status mp_prof_trace_dump(mp_ctx ctx, const char* path);
/* Number of this library's kernels launched since context creation. */
mp_status mp_launch_count(mp_ctx ctx, int64_t* launches);

/* Pinned host memory (for end-to-end transfers). */
mp_status mp_host_alloc(size_t bytes, void** ptr);
mp_status mp_host_free(void* ptr);

/* ------------------------------------------------------------------------- */
/* MPArray (array.hpp:18-82)                                                  */
/* ------------------------------------------------------------------------- */
/* MPArray::zeros / zeros_matrix (array.hpp:23-29).  is_matrix = 0 makes a
 * vector of rows elements (cols must be 1). */
mp_status mp_array_create(mp_ctx ctx, mp_precision p, int64_t rows, int64_t cols,
                          int is_matrix, mp_array* out);
/* Non-owning view of caller device memory (ld >= rows). */
mp_status mp_array_wrap(mp_ctx ctx, mp_precision p, int64_t rows, int64_t cols, int64_t ld,
                        void* device_ptr, mp_array* out);
mp_status mp_array_destroy(mp_array a);
mp_status mp_array_info(mp_array a, mp_precision* p, int64_t* rows, int64_t* cols,
                        int64_t* ld, int* is_matrix, void** device_ptr);
/* to_matrix (array.hpp:48): reshape in place. */
mp_status mp_array_to_matrix(mp_array a, int64_t rows, int64_t cols);
/* Raw storage bytes (2/4/8 per element, column-major, ld == rows). */
mp_status mp_array_upload(mp_array a, const void* host, size_t bytes);
mp_status mp_array_download(mp_array a, void* host, size_t bytes);
/* from_doubles / to_doubles (array.cpp:66-76, :169-173): host doubles are
 * copied up and rounded on the device with set_linear semantics. */
mp_status mp_array_from_doubles(mp_array a, const double* host, int64_t count);
mp_status mp_array_to_doubles(mp_array a, double* host, int64_t count);
/* Element get/set (array.hpp:52-55), 0-based, bounds-checked. */
mp_status mp_array_get(mp_array a, int64_t i, int64_t j, double* value);
mp_status mp_array_set(mp_array a, int64_t i, int64_t j, double value);

/* MPArray::converted (array.cpp:187-191): bit-exact re-rounding into dst's
 * precision (encode_f16 semantics, NaN -> 0x7E00). dst must match shape. */
mp_status mp_convert(mp_ctx ctx, mp_array src, mp_array dst);
/* Raw-pointer cast of n contiguous elements (the kernel the MPArray form uses). */
mp_status mp_convert_raw(mp_ctx ctx, mp_precision pin, const void* src, mp_precision pout,
                         void* dst, int64_t n);

/* ew_binary (array.cpp:252-272): out precision must be promote(a, b). */
mp_status mp_ew_binary(mp_ctx ctx, mp_binary_op op, mp_array a, mp_array b, mp_array out);
/* ew_scalar (array.cpp:274-291). */
mp_status mp_ew_scalar(mp_ctx ctx, mp_binary_op op, mp_array a, double s, mp_array out);
/* ew_unary (array.cpp:293-322). */
mp_status mp_ew_unary(mp_ctx ctx, mp_unary_op op, mp_array a, mp_array out);
/* reduce (array.cpp:336-369): double accumulation; synchronises. */
mp_status mp_reduce(mp_ctx ctx, mp_reduce_op op, mp_array a, double* result);
/* transpose (array.cpp:422-429), diag (array.cpp:371-378). */
mp_status mp_transpose(mp_ctx ctx, mp_array a, mp_array out);
mp_status mp_diag(mp_ctx ctx, mp_array a, mp_array out);

/* ------------------------------------------------------------------------- */
/* Dense kernels (linalg.hpp:23-54)                                           */
/* ------------------------------------------------------------------------- */
/* linalg::gemm (linalg.cpp:316-357): C <- alpha op(A) op(B) + beta C in C's
 * precision; MP_PRECISION_MISMATCH if prec(C) < promote(A, B); beta == 0
 * never reads C. */
mp_status mp_gemm(mp_ctx ctx, mp_array a, mp_array b, mp_array c, int trans_a, int trans_b,
                  double alpha, double beta);
/* Raw-pointer GEMM (same semantics; lda/ldb/ldc column-major leading dims). */
mp_status mp_gemm_raw(mp_ctx ctx, mp_precision pa, mp_precision pb, mp_precision pc,
                      int trans_a, int trans_b, int64_t m, int64_t n, int64_t k, double alpha,
                      const void* A, int64_t lda, const void* B, int64_t ldb, double beta,
                      void* C, int64_t ldc);
/* linalg::matmul (linalg.cpp:284-297): out precision promote(a, b). */
mp_status mp_matmul(mp_ctx ctx, mp_array a, mp_array b, mp_array out);
/* linalg::crossprod (linalg.cpp:299-314); b == NULL gives A^T A (SYRK,
 * exactly symmetric: lower triangle computed, mirrored). */
mp_status mp_crossprod(mp_ctx ctx, mp_array a, mp_array b, mp_array out);
/* linalg::chol (linalg.cpp:359-378): upper U with A = U^T U, lower zeroed.
 * info = first failing pivot column (0-based) or -1; synchronises. */
mp_status mp_chol(mp_ctx ctx, mp_array a, mp_array out, int64_t* info);
/* linalg::trsm (linalg.cpp:498-542): computes in B's precision; B overwritten;
 * exact-zero diagonal -> MP_SINGULAR_MATRIX. */
mp_status mp_trsm(mp_ctx ctx, mp_array a, mp_array b, mp_side side, int upper, int trans,
                  double alpha);
/* forwardsolve / backsolve (linalg.cpp:490-496): out precision promote. */
mp_status mp_forwardsolve(mp_ctx ctx, mp_array l, mp_array b, mp_array out);
mp_status mp_backsolve(mp_ctx ctx, mp_array u, mp_array b, mp_array out);
/* solve(a, b) (linalg.cpp:551-575): exactly symmetric a -> Cholesky path,
 * otherwise / not positive definite -> LU with partial pivoting (lu_kernel,
 * linalg.cpp:163-193); out = a^-1 b in promote(a, b); zero pivot ->
 * MP_SINGULAR_MATRIX. */
mp_status mp_solve(mp_ctx ctx, mp_array a, mp_array b, mp_array out);
/* chol2inv(u) (linalg.cpp:383-408, 481-488): (U^T U)^-1 from the upper
 * factor, exactly symmetric, in u's precision. */
mp_status mp_chol2inv(mp_ctx ctx, mp_array u, mp_array out);

/* ------------------------------------------------------------------------- */
/* Rng (rng.cpp:9-53): the reference's seeded stream, host-side, bit for bit */
/* ------------------------------------------------------------------------- */
/* n uniforms on [0, 1) of Rng(seed) after discarding `skip` draws (B of the
 * acceptance inputs is the draws after A's n^2: skip = n^2).  No device work. */
mp_status mp_rng_uniform(uint64_t seed, int64_t skip, int64_t n, double* out);
/* n standard normals of Rng(seed) (Box-Muller, rng.cpp:38-50). */
mp_status mp_rng_normal(uint64_t seed, int64_t n, double* out);

/* ------------------------------------------------------------------------- */
/* Op-name dispatch (dispatch.hpp, dispatch.cpp:46-137)                       */
/* ------------------------------------------------------------------------- */
/* KernelKey: input precisions and the promoted output; in_b = -1 for the
 * unary form.  Registered ops, in the reference's order: add sub mul div
 * rbind cbind matmul crossprod (binary), log exp sqrt abs transpose chol
 * solve (unary). */
typedef struct {
    int in_a;
    int in_b;
    int out;
} mp_kernel_key;
/* KernelRegistry::is_unary; MP_UNKNOWN_OPERATION for an unregistered name. */
mp_status mp_op_is_unary(const char* op, int* unary);
/* dispatch::resolve (dispatch.cpp:102-114): prec_b < 0 for the unary form;
 * out = promote(a, b).  MP_UNKNOWN_OPERATION for an unregistered name. */
mp_status mp_resolve(const char* op, int prec_a, int prec_b, mp_kernel_key* key);
/* dispatch::execute (dispatch.cpp:116-137): MP_PRECISION_MISMATCH when the
 * inputs' precisions differ from the key; b = NULL for unary ops.  *out is a
 * new device array (mp_array_destroy it). */
mp_status mp_execute(mp_ctx ctx, const mp_kernel_key* key, const char* op, mp_array a, mp_array b,
                     mp_array* out);

/* ------------------------------------------------------------------------- */
/* MPCRTile                                                */
/* ------------------------------------------------------------------------- */
/* new(MPCRTile, rows, cols, rows_per_tile, cols_per_tile, values, precisions)
 * (PAPER.md:346-356).  precisions: tiles_r x tiles_c column-major grid.
 * Tiles are stored one contiguous column-major buffer per tile. */
mp_status mp_tile_create(mp_ctx ctx, int64_t rows, int64_t cols, int64_t rows_per_tile,
                         int64_t cols_per_tile, const int* precisions, mp_tile* out);
mp_status mp_tile_destroy(mp_tile t);
mp_status mp_tile_info(mp_tile t, int64_t* rows, int64_t* cols, int64_t* rows_per_tile,
                       int64_t* cols_per_tile, int64_t* tiles_r, int64_t* tiles_c);
/* Whole-matrix values (column-major doubles), rounded per tile precision. */
mp_status mp_tile_set_values(mp_tile t, const double* host);
mp_status mp_tile_get_values(mp_tile t, double* host);
/* Rows rows[0..count) of the whole matrix widened to double, row-major
 * (host[q * cols + c]).  No reference counterpart: checking a factor too
 * large to download (sampled residuals of L L^T - A at n = 131072). */
mp_status mp_tile_get_rows(mp_tile t, const int64_t* rows, int64_t count, double* host);
/* Same, device-resident double source (n x n column-major, ld). */
mp_status mp_tile_set_values_device(mp_tile t, const double* dev, int64_t ld);
/* MPCRTile.GetTile, 0-based; returns a non-owning view. */
mp_status mp_tile_get_tile(mp_tile t, int64_t i, int64_t j, mp_array* view);
mp_status mp_tile_precision(mp_tile t, int64_t i, int64_t j, mp_precision* p);
/* MPCRTile.gemm: C overwritten, per-tile precision of C. */
mp_status mp_tile_gemm(mp_ctx ctx, mp_tile a, mp_tile b, mp_tile c, int trans_a, int trans_b,
                       double alpha, double beta);
/* chol(MPCRTile, overwrite_input): lower L, upper tiles
 * zeroed.  overwrite_input != 0 factors in place (out may be NULL); else a new
 * MPCRTile is returned in *out.  info = global failing column or -1. */
mp_status mp_tile_chol(mp_ctx ctx, mp_tile a, int overwrite_input, mp_tile* out,
                       int64_t* info);
/* MPCRTile.trsm: B overwritten. */
mp_status mp_tile_trsm(mp_ctx ctx, mp_tile a, mp_tile b, mp_side side, int upper, int trans,
                       double alpha);
/* logdet = 2 sum log L_ii of a factored MPCRTile (workloads.cpp:76-80). */
mp_status mp_tile_logdet(mp_ctx ctx, mp_tile l, double* logdet);

/* Matern covariance generated on the device straight into tile storage
 * (covariance.cpp:9-31 grid + :44-72 closed forms; first n points of a
 * side x side unit grid, x fastest).  Each tile rounded to its precision. */
mp_status mp_tile_fill_matern(mp_ctx ctx, mp_tile t, int64_t grid_side, double nu,
                              double range, double variance);
/* Same closed forms for arbitrary 2-D locations given in HOST memory
 * (x[0..n), y[0..n); n = rows = cols), copied up on the context stream;
 * `nugget` is added to the diagonal before rounding (0 for none). */
mp_status mp_tile_fill_matern_points(mp_ctx ctx, mp_tile t, const double* host_x,
                                     const double* host_y, int64_t n, double nu, double range,
                                     double variance, double nugget);
/* Tile-wise converted(): each tile of src rounded/widened into the precision
 * dst holds for that tile (same grid; array.cpp:187-191 per tile). */
mp_status mp_tile_convert(mp_ctx ctx, mp_tile dst, mp_tile src);
/* Device copy of all tile values (identical grids and precisions). */
mp_status mp_tile_copy(mp_ctx ctx, mp_tile dst, mp_tile src);
/* gaussian_nll (workloads.cpp:74-87) of host vector z under the covariance
 * held in `cov`, which is factored in place (lower L):
 *   chol_with_jitter (workloads.cpp:54-70): when jitter > 0 it is added to
 *   the diagonal first and multiplied by 10 after every NotPositiveDefinite
 *   failure while <= max_jitter (the input is restored between attempts);
 *   logdet = 2 sum log L_ii; w = L^{-1} z (FP64 vector, tiles widened);
 *   nll = 0.5 w'w + 0.5 logdet + 0.5 n log(2 pi).
 * Any of the outputs may be NULL.  jitter_used receives the final jitter. */
mp_status mp_tile_gaussian_nll(mp_ctx ctx, mp_tile cov, const double* host_z, double jitter,
                               double max_jitter, double* nll, double* logdet, double* quad,
                               double* jitter_used);

/* matern_mle (workloads.cpp:89-110, optimize.cpp:9-95): Nelder-Mead over
 * (log range, log sigma2) of a Matern(nu) Gaussian process at the host
 * points (x, y) with observations z; every objective evaluation regenerates
 * the covariance into `cov` on the device and evaluates mp_tile_gaussian_nll
 * (jitter policy as given).  max_iter / tol as NelderMeadConfig (the
 * reference's matern_mle default: 200 / 1e-4). */
mp_status mp_tile_matern_mle(mp_ctx ctx, mp_tile cov, const double* host_x, const double* host_y,
                             const double* host_z, int64_t n, double nu, double init_log_range,
                             double init_log_sigma2, int max_iter, double tol, double jitter,
                             double max_jitter, double* range_hat, double* sigma2_hat, double* nll,
                             int* iterations, int* converged);

/* ------------------------------------------------------------------------- */
/* Multi-GPU: 2D block-cyclic MPCRTile over a P x Q process grid (one process */
/* per GPU).  Tile (i, j), i >= j, lives on rank (i mod P) * Q + (j mod Q);   */
/* panel tiles and the diagonal inverse are broadcast with NCCL over NVLink.  */
/* ------------------------------------------------------------------------- */
typedef struct mp_dist_s* mp_dist;
/* 128-byte ncclUniqueId, made on one rank and shared by the caller (e.g.
 * torch.distributed); NCCL is resolved with dlopen at first use. */
mp_status mp_nccl_unique_id(unsigned char* out128);
mp_status mp_dist_create(mp_ctx ctx, int rank, int world, int P, int Q,
                         const unsigned char* uid128, mp_dist* out);
mp_status mp_dist_destroy(mp_dist d);
/* Test harness: `world` ranks simulated on ONE GPU in one process (rank r on
 * ctxs[r], each context with its own streams), collectives as event-ordered
 * device copies; the ranks must run concurrently from `world` host threads.
 * Exercises the multi-rank executor bit for bit without a second GPU. */
mp_status mp_dist_create_sim(mp_ctx* ctxs, int world, int P, int Q, mp_dist* out);
/* Owner rank of tile (i, j). */
int mp_dist_owner(int64_t i, int64_t j, int P, int Q);
/* The per-rank action list the distributed chol executes, as int32 records
 * {op, k, i, j, root, prec, comm} (op: 1 POTRF, 2 BCAST_DIAG, 3 TRSM, 4
 * BCAST_PANEL, 5 UPDATE; root: global rank; comm: 0 world, 1 this rank's
 * process row, 2 its process column).  L_kk^-1 goes down process column
 * k mod Q; panel tile L_ik along process row i mod P, then down process
 * column i mod Q (P + Q - 2 copies).  actions may be NULL to query *count. */
mp_status mp_dist_schedule(int rank, int P, int Q, int64_t tiles, const int* precisions,
                           int32_t* actions, int64_t capacity, int64_t* count);
/* MPCRTile whose lower-triangle tiles are distributed; this rank stores only
 * the tiles it owns (rows must equal cols).  mp_tile_chol on it runs the
 * distributed factorization; mp_tile_logdet / mp_tile_gaussian_nll reduce
 * over the ranks; get/set/fill touch owned tiles only. */
mp_status mp_tile_create_dist(mp_ctx ctx, mp_dist dist, int64_t n, int64_t tile,
                              const int* precisions, mp_tile* out);
/* 1 if this rank stores tile (i, j). */
int mp_tile_owns(mp_tile t, int64_t i, int64_t j);

#ifdef __cplusplus
}
#endif
#endif /* MPCR_B200_H */
