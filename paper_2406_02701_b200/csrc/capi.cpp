// C-ABI implementation: context, MPArray, elementwise and dense linalg entry
// points (include/mpcr_b200.h).  Argument checks mirror the reference's
// exception behaviour (array.cpp, linalg.cpp) and run before any device work.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "internal.hpp"

using namespace mpcr;

namespace mpcr {

thread_local std::string g_last_error;

void* Ctx::ensure_scratch(size_t bytes, int which) {
    void*& p = scr[which];
    size_t& cap = scr_bytes[which];
    if (bytes <= cap) return p;
    if (p) {
        MP_CUDA(cudaStreamSynchronize(stream));
        MP_CUDA(cudaFree(p));
        p = nullptr;
        cap = 0;
    }
    MP_CUDA(cudaMalloc(&p, bytes));
    cap = bytes;
    ++scr_gen;
    return p;
}

ProfScope::ProfScope(Ctx* c, int k, cudaStream_t st, double w) : ctx(c), cls(k), s(st), work(w) {
    if (!ctx->prof.enabled) return;
    if (ctx->prof.pool.empty()) {
        cudaEvent_t e;
        MP_CUDA(cudaEventCreate(&e));
        a = e;
    } else {
        a = ctx->prof.pool.back();
        ctx->prof.pool.pop_back();
    }
    MP_CUDA(cudaEventRecord(a, s));
}

ProfScope::~ProfScope() {
    if (!a) return;
    cudaEvent_t b;
    if (ctx->prof.pool.empty()) {
        if (cudaEventCreate(&b) != cudaSuccess) return;
    } else {
        b = ctx->prof.pool.back();
        ctx->prof.pool.pop_back();
    }
    if (cudaEventRecord(b, s) != cudaSuccess) return;
    ctx->prof.pending.push_back({a, b, cls, work, s});
    if (ctx->prof.pending.size() > 8192) prof_collect(ctx, false);
}

// Fold finished event pairs into the totals.  Non-blocking mode only takes
// pairs that already completed (in order) so profiling never stalls the host.
void prof_collect(Ctx* ctx, bool blocking) {
    size_t done = 0;
    for (auto& r : ctx->prof.pending) {
        if (!blocking && cudaEventQuery(r.b) != cudaSuccess) break;
        MP_CUDA(cudaEventSynchronize(r.b));
        ++done;
        float ms = 0.f;
        MP_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
        ctx->prof.ms[r.cls] += ms;
        ctx->prof.launches[r.cls] += 1;
        ctx->prof.work[r.cls] += r.work;
        if (ctx->prof.trace && ctx->prof.base) {
            float t0 = 0.f, t1 = 0.f;
            MP_CUDA(cudaEventElapsedTime(&t0, ctx->prof.base, r.a));
            MP_CUDA(cudaEventElapsedTime(&t1, ctx->prof.base, r.b));
            ctx->prof.spans.push_back({r.cls, r.s == ctx->hi ? 1 : r.s == ctx->hi2 ? 2 : 0, t0, t1});
        }
        ctx->prof.pool.push_back(r.a);
        ctx->prof.pool.push_back(r.b);
    }
    ctx->prof.pending.erase(ctx->prof.pending.begin(), ctx->prof.pending.begin() + done);
}

// Host restatement of encode_f16 rounding for scalars (precision.cpp:49-93),
// used to pre-round ew_scalar's operand (array.cpp:280).
double host_round_half(double x) {
    if (std::isnan(x)) return x;
    uint64_t d;
    std::memcpy(&d, &x, 8);
    const uint64_t sign = d >> 63;
    const int dexp = static_cast<int>((d >> 52) & 0x7FF);
    const uint64_t frac = d & ((uint64_t{1} << 52) - 1);
    if (dexp == 0x7FF) return x;
    if (dexp == 0) return sign ? -0.0 : 0.0;
    const int e = dexp - 1023;
    const uint64_t m = (uint64_t{1} << 52) | frac;
    int shift = 42;
    if (e < -14) {
        shift = 42 + (-14 - e);
        if (shift >= 64) return sign ? -0.0 : 0.0;
    }
    uint64_t keep = m >> shift;
    const uint64_t rem = m & ((uint64_t{1} << shift) - 1);
    const uint64_t half = uint64_t{1} << (shift - 1);
    if (rem > half || (rem == half && (keep & 1))) ++keep;
    double mag;
    if (e >= -14) {
        int he = e + 15;
        if (keep == 0x800) {
            keep = 0x400;
            ++he;
        }
        if (he >= 31) return sign ? -INFINITY : INFINITY;
        mag = std::ldexp(static_cast<double>(keep), he - 25);
    } else {
        mag = std::ldexp(static_cast<double>(keep), -24);
    }
    return sign ? -mag : mag;
}

double host_round(double x, mp_precision p) {
    if (p == MP_HALF) return host_round_half(x);
    if (p == MP_SINGLE) return static_cast<double>(static_cast<float>(x));
    return x;
}

}  // namespace mpcr

#define MP_API_BEGIN try {
#define MP_API_END                                        \
    return MP_OK;                                         \
    }                                                     \
    catch (const mpcr::Error& e) {                        \
        mpcr::g_last_error = e.what();                    \
        return e.status;                                  \
    }                                                     \
    catch (const std::bad_alloc&) {                       \
        mpcr::g_last_error = "host allocation failed";    \
        return MP_OUT_OF_MEMORY;                          \
    }                                                     \
    catch (const std::exception& e) {                     \
        mpcr::g_last_error = e.what();                    \
        return MP_INTERNAL_ERROR;                         \
    }

namespace {

Ctx* C_(mp_ctx c) {
    if (!c) fail(MP_INVALID_PARAM, "null context");
    bind_device(c);
    return c;
}
Array& A_(mp_array a, const char* what) {
    if (!a) fail(MP_INVALID_PARAM, std::string(what) + ": null array");
    if (a->ctx) bind_device(a->ctx);
    return *a;
}
void require_matrix(const Array& a, const char* what) {
    if (!a.is_matrix) fail(MP_NOT_A_MATRIX, std::string(what) + ": input is not a matrix");
}
void require_prec(const Array& out, mp_precision want, const char* what) {
    if (out.prec != want)
        fail(MP_PRECISION_MISMATCH, std::string(what) + ": output precision must be " +
                                        prec_name(want));
}
void require_shape(const Array& a, int64_t r, int64_t c, const char* what) {
    if (a.rows != r || a.cols != c)
        fail(MP_SHAPE_MISMATCH, std::string(what) + ": expected " + std::to_string(r) + "x" +
                                    std::to_string(c) + ", got " + std::to_string(a.rows) + "x" +
                                    std::to_string(a.cols));
}
void require_contiguous(const Array& a, const char* what) {
    if (a.ld != a.rows && a.cols > 1)
        fail(MP_INVALID_PARAM, std::string(what) + ": strided array not supported here");
}

}  // namespace

extern "C" {

const char* mp_last_error(void) { return mpcr::g_last_error.c_str(); }
const char* mp_version(void) { return "mpcr_b200 0.1 (sm_100a)"; }

mp_status mp_device_check(int device, int* major, int* minor, int* sm_count) {
    MP_API_BEGIN
    cudaDeviceProp prop;
    const cudaError_t e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess)
        fail(MP_BACKEND_UNAVAILABLE, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (major) *major = prop.major;
    if (minor) *minor = prop.minor;
    if (sm_count) *sm_count = prop.multiProcessorCount;
    if (prop.major != 10 || prop.minor != 0)
        fail(MP_BACKEND_UNAVAILABLE, "device is not sm_100 (B200); this build targets sm_100a");
    MP_API_END
}

mp_status mp_ctx_create(int device, mp_ctx* out) {
    MP_API_BEGIN
    if (!out) fail(MP_INVALID_PARAM, "null out");
    int maj = 0, mn = 0, sms = 0;
    const mp_status st = mp_device_check(device, &maj, &mn, &sms);
    if (st != MP_OK) return st;
    MP_CUDA(cudaSetDevice(device));
    auto* c = new mp_ctx_s();
    c->device = device;
    c->sm_count = sms;
    MP_CUDA(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    c->stream = c->own_stream;
    int lo = 0, hi = 0;
    MP_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    MP_CUDA(cudaStreamCreateWithPriority(&c->hi, cudaStreamNonBlocking, hi));
    MP_CUDA(cudaStreamCreateWithPriority(&c->hi2, cudaStreamNonBlocking, hi));
    for (auto& s : c->aux) MP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    MP_CUDA(cudaMalloc(&c->sched_pool, 2 * Ctx::SCHED_SLOTS * sizeof(unsigned int)));
    MP_CUDA(cudaMemset(c->sched_pool, 0, 2 * Ctx::SCHED_SLOTS * sizeof(unsigned int)));
    // the context's streams are non-blocking: the zeroing must be complete
    // before any of them can launch a kernel that draws from the pool
    MP_CUDA(cudaDeviceSynchronize());
    *out = c;
    MP_API_END
}

mp_status mp_ctx_destroy(mp_ctx ctx) {
    MP_API_BEGIN
    if (!ctx) return MP_OK;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    for (auto& r : ctx->prof.pending) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : ctx->prof.pool) cudaEventDestroy(e);
    for (void* p : ctx->scr)
        if (p) cudaFree(p);
    if (ctx->prof.dev_stats) cudaFree(ctx->prof.dev_stats);
    if (ctx->sched_pool) cudaFree(ctx->sched_pool);
    for (auto& s : ctx->aux) cudaStreamDestroy(s);
    cudaStreamDestroy(ctx->hi);
    cudaStreamDestroy(ctx->hi2);
    cudaStreamDestroy(ctx->own_stream);
    delete ctx;
    MP_API_END
}

mp_status mp_ctx_set_stream(mp_ctx ctx, void* s) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    c->stream = s ? static_cast<cudaStream_t>(s) : c->own_stream;
    MP_API_END
}

mp_status mp_ctx_get_stream(mp_ctx ctx, void** s) {
    MP_API_BEGIN
    *s = C_(ctx)->stream;
    MP_API_END
}

mp_status mp_ctx_synchronize(mp_ctx ctx) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    MP_CUDA(cudaSetDevice(c->device));
    MP_CUDA(cudaStreamSynchronize(c->stream));
    MP_CUDA(cudaDeviceSynchronize());
    MP_API_END
}

mp_status mp_prof_enable(mp_ctx ctx, int enable) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    if (enable && !c->prof.dev_stats) {
        MP_CUDA(cudaMalloc(&c->prof.dev_stats, 64));
        MP_CUDA(cudaMemsetAsync(c->prof.dev_stats, 0, 64, c->stream));
    }
    c->prof.enabled = enable != 0;
    MP_API_END
}

mp_status mp_prof_digit_products(mp_ctx ctx, int64_t* pair_mmas, int64_t* tiles) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    unsigned long long h[2] = {0, 0};
    if (c->prof.dev_stats) {
        MP_CUDA(cudaStreamSynchronize(c->stream));
        MP_CUDA(cudaDeviceSynchronize());
        MP_CUDA(cudaMemcpy(h, c->prof.dev_stats, sizeof(h), cudaMemcpyDeviceToHost));
    }
    if (pair_mmas) *pair_mmas = static_cast<int64_t>(h[0]);
    if (tiles) *tiles = static_cast<int64_t>(h[1]);
    MP_API_END
}

mp_status mp_prof_reset(mp_ctx ctx) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    prof_collect(c);
    for (int i = 0; i < MP_PROF_NUM_CLASSES; ++i) {
        c->prof.ms[i] = 0;
        c->prof.launches[i] = 0;
        c->prof.work[i] = 0;
    }
    if (c->prof.dev_stats) {
        MP_CUDA(cudaDeviceSynchronize());
        MP_CUDA(cudaMemset(c->prof.dev_stats, 0, 64));
    }
    MP_API_END
}

mp_status mp_prof_query(mp_ctx ctx, int cls, double* ms, int64_t* launches, double* work) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    if (cls < 0 || cls >= MP_PROF_NUM_CLASSES) fail(MP_INVALID_PARAM, "bad profile class");
    prof_collect(c);
    if (ms) *ms = c->prof.ms[cls];
    if (launches) *launches = c->prof.launches[cls];
    if (work) *work = c->prof.work[cls];
    MP_API_END
}

mp_status mp_prof_trace(mp_ctx ctx, int enable) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    prof_collect(c);
    c->prof.spans.clear();
    c->prof.trace = enable != 0;
    if (enable) {
        if (!c->prof.base) MP_CUDA(cudaEventCreate(&c->prof.base));
        MP_CUDA(cudaEventRecord(c->prof.base, c->stream));
    }
    MP_API_END
}

mp_status mp_prof_trace_dump(mp_ctx ctx, const char* path) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    prof_collect(c);
    FILE* f = std::fopen(path, "w");
    if (!f) fail(MP_IO_ERROR, std::string("cannot open ") + path);
    std::fprintf(f, "cls,stream,start_ms,end_ms\n");
    for (const auto& sp : c->prof.spans) std::fprintf(f, "%d,%d,%.4f,%.4f\n", sp.cls, sp.stream, sp.t0, sp.t1);
    std::fclose(f);
    MP_API_END
}

mp_status mp_launch_count(mp_ctx ctx, int64_t* launches) {
    MP_API_BEGIN
    *launches = C_(ctx)->launches;
    MP_API_END
}

mp_status mp_host_alloc(size_t bytes, void** ptr) {
    MP_API_BEGIN
    MP_CUDA(cudaHostAlloc(ptr, bytes, cudaHostAllocDefault));
    MP_API_END
}

mp_status mp_host_free(void* ptr) {
    MP_API_BEGIN
    if (ptr) MP_CUDA(cudaFreeHost(ptr));
    MP_API_END
}

// ---- MPArray -----------------------------------------------------------------
mp_status mp_array_create(mp_ctx ctx, mp_precision p, int64_t rows, int64_t cols, int is_matrix,
                          mp_array* out) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    if (p < MP_HALF || p > MP_DOUBLE) fail(MP_INVALID_PARAM, "bad precision");
    if (rows < 0 || cols < 0) fail(MP_INVALID_PARAM, "negative dimension");
    if (!is_matrix) {
        if (rows < 1) fail(MP_INVALID_PARAM, "zeros: size must be >= 1");  // array.cpp:57
        if (cols != 1) fail(MP_INVALID_PARAM, "vector must have cols == 1");
    }
    auto* a = new mp_array_s();
    a->ctx = c;
    a->prec = p;
    a->rows = rows;
    a->cols = cols;
    a->ld = rows > 0 ? rows : 1;
    a->is_matrix = is_matrix != 0;
    const size_t bytes = static_cast<size_t>(rows * cols) * elem_bytes(p);
    if (bytes) {
        try {
            MP_CUDA(cudaMalloc(&a->data, bytes));
            MP_CUDA(cudaMemsetAsync(a->data, 0, bytes, c->stream));
        } catch (...) {
            delete a;
            throw;
        }
    }
    *out = a;
    MP_API_END
}

mp_status mp_array_wrap(mp_ctx ctx, mp_precision p, int64_t rows, int64_t cols, int64_t ld,
                        void* ptr, mp_array* out) {
    MP_API_BEGIN
    auto* a = new mp_array_s();
    a->ctx = C_(ctx);
    a->prec = p;
    a->rows = rows;
    a->cols = cols;
    a->ld = ld;
    a->is_matrix = true;
    a->owner = false;
    a->data = ptr;
    if (ld < rows) {
        delete a;
        fail(MP_INVALID_PARAM, "ld < rows");
    }
    *out = a;
    MP_API_END
}

mp_status mp_array_destroy(mp_array a) {
    MP_API_BEGIN
    if (!a) return MP_OK;
    // cudaFree synchronises the device; the owning context may already be gone.
    if (a->owner && a->data) cudaFree(a->data);
    delete a;
    MP_API_END
}

mp_status mp_array_info(mp_array a, mp_precision* p, int64_t* rows, int64_t* cols, int64_t* ld,
                        int* is_matrix, void** ptr) {
    MP_API_BEGIN
    Array& x = A_(a, "info");
    if (p) *p = x.prec;
    if (rows) *rows = x.rows;
    if (cols) *cols = x.cols;
    if (ld) *ld = x.ld;
    if (is_matrix) *is_matrix = x.is_matrix;
    if (ptr) *ptr = x.data;
    MP_API_END
}

mp_status mp_array_to_matrix(mp_array a, int64_t rows, int64_t cols) {
    MP_API_BEGIN
    Array& x = A_(a, "to_matrix");
    if (rows * cols != x.size())
        fail(MP_SHAPE_MISMATCH, "to_matrix: " + std::to_string(rows) + "x" + std::to_string(cols) +
                                    " does not hold " + std::to_string(x.size()) + " elements");
    require_contiguous(x, "to_matrix");
    x.rows = rows;
    x.cols = cols;
    x.ld = rows > 0 ? rows : 1;
    x.is_matrix = true;
    MP_API_END
}

mp_status mp_array_upload(mp_array a, const void* host, size_t bytes) {
    MP_API_BEGIN
    Array& x = A_(a, "upload");
    const size_t need = static_cast<size_t>(x.size()) * elem_bytes(x.prec);
    if (bytes != need) fail(MP_SHAPE_MISMATCH, "upload: byte count mismatch");
    if (x.ld == x.rows || x.cols <= 1)
        MP_CUDA(cudaMemcpyAsync(x.data, host, bytes, cudaMemcpyHostToDevice, x.ctx->stream));
    else
        MP_CUDA(cudaMemcpy2DAsync(x.data, x.ld * elem_bytes(x.prec), host,
                                  x.rows * elem_bytes(x.prec), x.rows * elem_bytes(x.prec), x.cols,
                                  cudaMemcpyHostToDevice, x.ctx->stream));
    MP_CUDA(cudaStreamSynchronize(x.ctx->stream));
    MP_API_END
}

mp_status mp_array_download(mp_array a, void* host, size_t bytes) {
    MP_API_BEGIN
    Array& x = A_(a, "download");
    const size_t need = static_cast<size_t>(x.size()) * elem_bytes(x.prec);
    if (bytes != need) fail(MP_SHAPE_MISMATCH, "download: byte count mismatch");
    if (x.ld == x.rows || x.cols <= 1)
        MP_CUDA(cudaMemcpyAsync(host, x.data, bytes, cudaMemcpyDeviceToHost, x.ctx->stream));
    else
        MP_CUDA(cudaMemcpy2DAsync(host, x.rows * elem_bytes(x.prec), x.data,
                                  x.ld * elem_bytes(x.prec), x.rows * elem_bytes(x.prec), x.cols,
                                  cudaMemcpyDeviceToHost, x.ctx->stream));
    MP_CUDA(cudaStreamSynchronize(x.ctx->stream));
    MP_API_END
}

mp_status mp_array_from_doubles(mp_array a, const double* host, int64_t count) {
    MP_API_BEGIN
    Array& x = A_(a, "from_doubles");
    if (count != x.size())
        fail(MP_SHAPE_MISMATCH, "from_doubles: " + std::to_string(count) + " values cannot fill " +
                                    std::to_string(x.rows) + "x" + std::to_string(x.cols));
    if (count == 0) return MP_OK;
    Ctx* c = x.ctx;
    double* tmp = static_cast<double*>(c->ensure_scratch(count * sizeof(double), 1));
    MP_CUDA(cudaMemcpyAsync(tmp, host, count * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    launch_convert(c, c->stream, MP_DOUBLE, tmp, x.rows, x.prec, x.data, x.ld, x.rows, x.cols);
    MP_CUDA(cudaStreamSynchronize(c->stream));
    MP_API_END
}

mp_status mp_array_to_doubles(mp_array a, double* host, int64_t count) {
    MP_API_BEGIN
    Array& x = A_(a, "to_doubles");
    if (count != x.size()) fail(MP_SHAPE_MISMATCH, "to_doubles: count mismatch");
    if (count == 0) return MP_OK;
    Ctx* c = x.ctx;
    double* tmp = static_cast<double*>(c->ensure_scratch(count * sizeof(double), 1));
    launch_convert(c, c->stream, x.prec, x.data, x.ld, MP_DOUBLE, tmp, x.rows, x.rows, x.cols);
    MP_CUDA(cudaMemcpyAsync(host, tmp, count * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    MP_CUDA(cudaStreamSynchronize(c->stream));
    MP_API_END
}

mp_status mp_array_get(mp_array a, int64_t i, int64_t j, double* value) {
    MP_API_BEGIN
    Array& x = A_(a, "get");
    if (i < 0 || j < 0 || i >= x.rows || j >= x.cols)
        fail(MP_INDEX_OUT_OF_RANGE, "index (" + std::to_string(i) + ", " + std::to_string(j) +
                                        ") out of range for " + std::to_string(x.rows) + "x" +
                                        std::to_string(x.cols));
    Ctx* c = x.ctx;
    double* tmp = static_cast<double*>(c->ensure_scratch(64, 1));
    const char* src = static_cast<const char*>(x.data) + (j * x.ld + i) * elem_bytes(x.prec);
    launch_convert(c, c->stream, x.prec, src, 1, MP_DOUBLE, tmp, 1, 1, 1);
    MP_CUDA(cudaMemcpyAsync(value, tmp, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    MP_CUDA(cudaStreamSynchronize(c->stream));
    MP_API_END
}

mp_status mp_array_set(mp_array a, int64_t i, int64_t j, double value) {
    MP_API_BEGIN
    Array& x = A_(a, "set");
    if (i < 0 || j < 0 || i >= x.rows || j >= x.cols)
        fail(MP_INDEX_OUT_OF_RANGE, "index (" + std::to_string(i) + ", " + std::to_string(j) +
                                        ") out of range");
    Ctx* c = x.ctx;
    double* tmp = static_cast<double*>(c->ensure_scratch(64, 1));
    MP_CUDA(cudaMemcpyAsync(tmp, &value, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    char* dst = static_cast<char*>(x.data) + (j * x.ld + i) * elem_bytes(x.prec);
    launch_convert(c, c->stream, MP_DOUBLE, tmp, 1, x.prec, dst, 1, 1, 1);
    MP_CUDA(cudaStreamSynchronize(c->stream));
    MP_API_END
}

mp_status mp_convert(mp_ctx ctx, mp_array src, mp_array dst) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    Array& s = A_(src, "convert");
    Array& d = A_(dst, "convert");
    if (s.rows != d.rows || s.cols != d.cols) fail(MP_SHAPE_MISMATCH, "convert: shape mismatch");
    launch_convert(c, c->stream, s.prec, s.data, s.ld, d.prec, d.data, d.ld, s.rows, s.cols);
    MP_API_END
}

mp_status mp_convert_raw(mp_ctx ctx, mp_precision pin, const void* src, mp_precision pout,
                         void* dst, int64_t n) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    if (n < 0) fail(MP_INVALID_PARAM, "negative count");
    launch_convert(c, c->stream, pin, src, n, pout, dst, n, n, 1);
    MP_API_END
}

// ---- elementwise (array.cpp:228-429) -------------------------------------------
static void check_same_shape(const Array& a, const Array& b, const char* what) {
    if (a.rows != b.rows || a.cols != b.cols || a.is_matrix != b.is_matrix)
        fail(MP_SHAPE_MISMATCH, std::string(what) + ": shapes " + std::to_string(a.rows) + "x" +
                                    std::to_string(a.cols) + " and " + std::to_string(b.rows) +
                                    "x" + std::to_string(b.cols) + " do not match");
}

mp_status mp_ew_binary(mp_ctx ctx, mp_binary_op op, mp_array a, mp_array b, mp_array out) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    Array &x = A_(a, "ew_binary"), &y = A_(b, "ew_binary"), &o = A_(out, "ew_binary");
    if (op < MP_ADD || op > MP_DIV) fail(MP_UNKNOWN_OPERATION, "ew_binary: unknown op");
    check_same_shape(x, y, "ew_binary");
    require_shape(o, x.rows, x.cols, "ew_binary");
    require_prec(o, promote(x.prec, y.prec), "ew_binary");
    launch_ew_binary(c, c->stream, op, x, y, o);
    MP_API_END
}

mp_status mp_ew_scalar(mp_ctx ctx, mp_binary_op op, mp_array a, double s, mp_array out) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    Array &x = A_(a, "ew_scalar"), &o = A_(out, "ew_scalar");
    if (op < MP_ADD || op > MP_DIV) fail(MP_UNKNOWN_OPERATION, "ew_scalar: unknown op");
    require_shape(o, x.rows, x.cols, "ew_scalar");
    require_prec(o, x.prec, "ew_scalar");
    // array.cpp:280: the scalar is rounded to the array precision on the float path
    const double v = x.prec == MP_DOUBLE ? s : static_cast<double>(static_cast<float>(host_round(s, x.prec)));
    launch_ew_scalar(c, c->stream, op, x, v, o);
    MP_API_END
}

mp_status mp_ew_unary(mp_ctx ctx, mp_unary_op op, mp_array a, mp_array out) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    Array &x = A_(a, "ew_unary"), &o = A_(out, "ew_unary");
    if (op < MP_LOG || op > MP_ABS) fail(MP_UNKNOWN_OPERATION, "ew_unary: unknown op");
    require_shape(o, x.rows, x.cols, "ew_unary");
    require_prec(o, x.prec, "ew_unary");
    launch_ew_unary(c, c->stream, op, x, o);
    MP_API_END
}

mp_status mp_reduce(mp_ctx ctx, mp_reduce_op op, mp_array a, double* result) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    Array& x = A_(a, "reduce");
    if (op < MP_SUM || op > MP_MEAN) fail(MP_UNKNOWN_OPERATION, "reduce: unknown op");
    if (x.size() == 0) fail(MP_EMPTY_ARRAY, "reduce: empty array");
    *result = run_reduce(c, c->stream, op, x);
    MP_API_END
}

mp_status mp_transpose(mp_ctx ctx, mp_array a, mp_array out) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    Array &x = A_(a, "transpose"), &o = A_(out, "transpose");
    require_matrix(x, "transpose");
    require_shape(o, x.cols, x.rows, "transpose");
    require_prec(o, x.prec, "transpose");
    launch_transpose(c, c->stream, x, o);
    MP_API_END
}

mp_status mp_diag(mp_ctx ctx, mp_array a, mp_array out) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    Array &x = A_(a, "diag"), &o = A_(out, "diag");
    require_matrix(x, "diag");
    const int64_t n = x.rows < x.cols ? x.rows : x.cols;
    if (o.size() != n) fail(MP_SHAPE_MISMATCH, "diag: output length");
    require_prec(o, x.prec, "diag");
    launch_diag(c, c->stream, x, o);
    MP_API_END
}

// ---- dense linalg (linalg.cpp) -------------------------------------------------
mp_status mp_gemm_raw(mp_ctx ctx, mp_precision pa, mp_precision pb, mp_precision pc, int ta,
                      int tb, int64_t m, int64_t n, int64_t k, double alpha, const void* A,
                      int64_t lda, const void* B, int64_t ldb, double beta, void* Cp,
                      int64_t ldc) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    if (pc < promote(pa, pb))
        fail(MP_PRECISION_MISMATCH, std::string("gemm: accumulator precision ") + prec_name(pc) +
                                        " is below the promoted input precision " +
                                        prec_name(promote(pa, pb)));
    if (m < 0 || n < 0 || k < 0) fail(MP_INVALID_PARAM, "gemm: negative size");
    GemmDesc g{pa, pb, pc, ta != 0, tb != 0, m, n, k, alpha, beta, A, lda, B, ldb, Cp, ldc};
    launch_gemm(c, c->stream, g);
    MP_API_END
}

mp_status mp_gemm(mp_ctx ctx, mp_array a, mp_array b, mp_array cc, int ta, int tb, double alpha,
                  double beta) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    Array &x = A_(a, "gemm"), &y = A_(b, "gemm"), &z = A_(cc, "gemm");
    require_matrix(x, "gemm");
    require_matrix(y, "gemm");
    require_matrix(z, "gemm");
    const int64_t m = ta ? x.cols : x.rows, k = ta ? x.rows : x.cols;
    const int64_t kb = tb ? y.cols : y.rows, n = tb ? y.rows : y.cols;
    if (k != kb || z.rows != m || z.cols != n)
        fail(MP_SHAPE_MISMATCH, "gemm: op(a) is " + std::to_string(m) + "x" + std::to_string(k) +
                                    ", op(b) is " + std::to_string(kb) + "x" + std::to_string(n) +
                                    ", c is " + std::to_string(z.rows) + "x" +
                                    std::to_string(z.cols));
    if (z.prec < promote(x.prec, y.prec))
        fail(MP_PRECISION_MISMATCH, std::string("gemm: accumulator precision ") +
                                        prec_name(z.prec) +
                                        " is below the promoted input precision " +
                                        prec_name(promote(x.prec, y.prec)));
    GemmDesc g{x.prec, y.prec, z.prec, ta != 0, tb != 0, m, n, k, alpha, beta,
               x.data, x.ld, y.data, y.ld, z.data, z.ld};
    launch_gemm(c, c->stream, g);
    MP_API_END
}

mp_status mp_matmul(mp_ctx ctx, mp_array a, mp_array b, mp_array out) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    Array &x = A_(a, "matmul"), &y = A_(b, "matmul"), &o = A_(out, "matmul");
    require_matrix(x, "matmul");
    require_matrix(y, "matmul");
    if (x.cols != y.rows)
        fail(MP_SHAPE_MISMATCH, "matmul: inner dimensions " + std::to_string(x.cols) + " and " +
                                    std::to_string(y.rows) + " differ");
    require_shape(o, x.rows, y.cols, "matmul");
    require_prec(o, promote(x.prec, y.prec), "matmul");
    GemmDesc g{x.prec, y.prec, o.prec, false, false, x.rows, y.cols, x.cols, 1.0, 0.0,
               x.data, x.ld, y.data, y.ld, o.data, o.ld};
    launch_gemm(c, c->stream, g);
    MP_API_END
}

mp_status mp_crossprod(mp_ctx ctx, mp_array a, mp_array b, mp_array out) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    Array& x = A_(a, "crossprod");
    Array& y = b ? A_(b, "crossprod") : x;
    Array& o = A_(out, "crossprod");
    require_matrix(x, "crossprod");
    require_matrix(y, "crossprod");
    if (x.rows != y.rows)
        fail(MP_SHAPE_MISMATCH, "crossprod: row counts " + std::to_string(x.rows) + " and " +
                                    std::to_string(y.rows) + " differ");
    require_shape(o, x.cols, y.cols, "crossprod");
    require_prec(o, promote(x.prec, y.prec), "crossprod");
    const bool syrk = (b == nullptr) || (b == a);
    GemmDesc g{x.prec, y.prec, o.prec, true, false, x.cols, y.cols, x.rows, 1.0, 0.0,
               x.data, x.ld, y.data, y.ld, o.data, o.ld, syrk};
    launch_gemm(c, c->stream, g);
    // crossprod_kernel is exactly symmetric for b == a (linalg.cpp:94-95):
    // compute the lower triangle once and mirror it.
    if (syrk) launch_mirror_lower(c, c->stream, o.prec, o.data, o.ld, o.rows);
    MP_API_END
}

mp_status mp_chol(mp_ctx ctx, mp_array a, mp_array out, int64_t* info) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    Array &x = A_(a, "chol"), &o = A_(out, "chol");
    if (info) *info = -1;
    require_matrix(x, "chol");
    if (x.rows != x.cols)
        fail(MP_SHAPE_MISMATCH, "chol: matrix is " + std::to_string(x.rows) + "x" +
                                    std::to_string(x.cols) + ", not square");
    require_shape(o, x.rows, x.cols, "chol");
    require_prec(o, x.prec, "chol");
    const int64_t n = x.rows;
    if (n == 0) return MP_OK;
    const mp_precision cp = compute_precision(x.prec);
    const size_t nn = static_cast<size_t>(n) * n;
    char* scr = static_cast<char*>(c->ensure_scratch(2 * nn * elem_bytes(cp) + 64, 0));
    int64_t* dinfo = reinterpret_cast<int64_t*>(scr);
    void* w1 = scr + 64;
    void* w2 = scr + 64 + nn * elem_bytes(cp);
    const int64_t neg = -1;
    MP_CUDA(cudaMemcpyAsync(dinfo, &neg, sizeof(neg), cudaMemcpyHostToDevice, c->stream));
    // widen, then transpose so the factor reads the reference's upper
    // triangle (chol_kernel reads u_ij, i <= j; linalg.cpp:110-127)
    launch_convert(c, c->stream, x.prec, x.data, x.ld, cp, w2, n, n, n);
    launch_transpose_raw(c, c->stream, cp, w2, n, n, n, w1, n);
    launch_potrf_lower(c, c->stream, cp, w1, n, n, dinfo, 0);
    int64_t hinfo = -1;
    MP_CUDA(cudaMemcpyAsync(&hinfo, dinfo, sizeof(hinfo), cudaMemcpyDeviceToHost, c->stream));
    MP_CUDA(cudaStreamSynchronize(c->stream));
    if (hinfo >= 0) {
        if (info) *info = hinfo;
        throw Error(MP_NOT_POSITIVE_DEFINITE,
                    "matrix is not positive definite at pivot column " + std::to_string(hinfo),
                    hinfo);
    }
    launch_zero_triangle(c, c->stream, cp, w1, n, n, /*upper=*/true);
    launch_transpose_raw(c, c->stream, cp, w1, n, n, n, w2, n);  // U = L^T
    launch_convert(c, c->stream, cp, w2, n, o.prec, o.data, o.ld, n, n);
    MP_API_END
}

mp_status mp_trsm(mp_ctx ctx, mp_array a, mp_array b, mp_side side, int upper, int trans,
                  double alpha) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    Array &x = A_(a, "trsm"), &y = A_(b, "trsm");
    require_matrix(x, "trsm");
    require_matrix(y, "trsm");
    if (x.rows != x.cols) fail(MP_SHAPE_MISMATCH, "trsm: a is not square");
    const int64_t n = x.rows;
    if (side == MP_LEFT ? y.rows != n : y.cols != n)
        fail(MP_SHAPE_MISMATCH, "trsm: b is " + std::to_string(y.rows) + "x" +
                                    std::to_string(y.cols) + ", incompatible with " +
                                    std::to_string(n) + "x" + std::to_string(n) +
                                    (side == MP_LEFT ? " on the left" : " on the right"));
    const mp_precision cp = compute_precision(y.prec);
    const int64_t z = find_zero_diag(c, c->stream, x.prec, x.data, x.ld, n, cp);
    if (z >= 0)
        fail(MP_SINGULAR_MATRIX, "triangular solve: zero diagonal at index " + std::to_string(z));
    launch_tri_solve(c, c->stream, x.prec, x.data, x.ld, n, upper != 0, trans != 0, y.prec,
                     y.data, y.ld, y.cols, alpha, side == MP_RIGHT, y.rows);
    MP_API_END
}

static mp_status tri_solve_api(mp_ctx ctx, mp_array t, mp_array b, mp_array out, bool upper,
                               const char* what) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    Array &x = A_(t, what), &y = A_(b, what), &o = A_(out, what);
    require_matrix(x, what);
    if (x.rows != x.cols) fail(MP_SHAPE_MISMATCH, std::string(what) + ": triangular matrix is not square");
    if (y.rows != x.rows)
        fail(MP_SHAPE_MISMATCH, std::string(what) + ": rhs has " + std::to_string(y.rows) +
                                    " rows, expected " + std::to_string(x.rows));
    require_shape(o, y.rows, y.cols, what);
    const mp_precision po = promote(x.prec, y.prec);
    require_prec(o, po, what);
    const mp_precision cp = compute_precision(po);
    const int64_t z = find_zero_diag(c, c->stream, x.prec, x.data, x.ld, x.rows, cp);
    if (z >= 0)
        fail(MP_SINGULAR_MATRIX, "triangular solve: zero diagonal at index " + std::to_string(z));
    launch_convert(c, c->stream, y.prec, y.data, y.ld, o.prec, o.data, o.ld, y.rows, y.cols);
    launch_tri_solve(c, c->stream, x.prec, x.data, x.ld, x.rows, upper, false, o.prec, o.data,
                     o.ld, o.cols, 1.0, false, o.rows);
    MP_API_END
}

mp_status mp_forwardsolve(mp_ctx ctx, mp_array l, mp_array b, mp_array out) {
    return tri_solve_api(ctx, l, b, out, false, "forwardsolve");
}

mp_status mp_backsolve(mp_ctx ctx, mp_array u, mp_array b, mp_array out) {
    return tri_solve_api(ctx, u, b, out, true, "backsolve");
}


// chol2inv (linalg.cpp:383-408): (U^T U)^-1 for the upper factor U, exactly
// symmetric.  X = U^-1 = (L^-1)^T with L = U^T inverted by the FP64 TRTRI,
// then X X^T = Linv^T Linv (lower half computed once, mirrored), rounded to
// U's precision.  Exact zero diagonal -> SingularMatrix.
mp_status mp_chol2inv(mp_ctx ctx, mp_array u, mp_array out) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    Array &x = A_(u, "chol2inv"), &o = A_(out, "chol2inv");
    require_matrix(x, "chol2inv");
    if (x.rows != x.cols) fail(MP_SHAPE_MISMATCH, "chol2inv: matrix is not square");
    require_shape(o, x.rows, x.cols, "chol2inv");
    require_prec(o, x.prec, "chol2inv");
    const int64_t n = x.rows;
    if (n == 0) return MP_OK;
    const int64_t z = find_zero_diag(c, c->stream, x.prec, x.data, x.ld, n, compute_precision(x.prec));
    if (z >= 0) fail(MP_SINGULAR_MATRIX, "chol2inv: zero diagonal at index " + std::to_string(z));
    const size_t nn = static_cast<size_t>(n) * n;
    double* w = static_cast<double*>(c->ensure_scratch(3 * nn * sizeof(double), 0));
    double *wu = w, *wl = w + nn, *wi = w + 2 * nn;
    launch_convert(c, c->stream, x.prec, x.data, x.ld, MP_DOUBLE, wu, n, n, n);
    launch_zero_triangle(c, c->stream, MP_DOUBLE, wu, n, n, /*upper=*/false);  // U's lower part is unused
    launch_transpose_raw(c, c->stream, MP_DOUBLE, wu, n, n, n, wl, n);          // L = U^T
    launch_trtri_lower(c, c->stream, wl, n, wi, n, n);                          // Linv
    GemmDesc g{MP_DOUBLE, MP_DOUBLE, MP_DOUBLE, true, false, n, n, n, 1.0, 0.0, wi, n, wi, n, wu, n, true};
    launch_gemm(c, c->stream, g);  // lower of Linv^T Linv
    launch_mirror_lower(c, c->stream, MP_DOUBLE, wu, n, n);
    launch_convert(c, c->stream, MP_DOUBLE, wu, n, o.prec, o.data, o.ld, n, n);
    MP_API_END
}

// solve(a, b) (linalg.cpp:551-575): out = a^-1 b in promote(a, b).  Exactly
// symmetric a: chol(a.converted(out_prec)), forwardsolve(U^T), backsolve(U);
// otherwise (or not positive definite) LU with partial pivoting in the
// compute precision (lu_solve_impl, :451-476).  Zero pivot -> SingularMatrix.
mp_status mp_solve(mp_ctx ctx, mp_array a, mp_array b, mp_array out) {
    MP_API_BEGIN
    Ctx* c = C_(ctx);
    Array &x = A_(a, "solve"), &y = A_(b, "solve"), &o = A_(out, "solve");
    require_matrix(x, "solve");
    if (x.rows != x.cols) fail(MP_SHAPE_MISMATCH, "solve: matrix is not square");
    if (y.rows != x.rows)
        fail(MP_SHAPE_MISMATCH, "solve: rhs has " + std::to_string(y.rows) + " rows, expected " +
                                    std::to_string(x.rows));
    require_shape(o, y.rows, y.cols, "solve");
    const mp_precision po = promote(x.prec, y.prec);
    require_prec(o, po, "solve");
    const int64_t n = x.rows;
    if (n == 0 || y.cols == 0) return MP_OK;
    if (device_exactly_symmetric(c, c->stream, x.prec, x.data, x.ld, n)) {
        // SPD fast path through the public entry points (same semantics as the reference)
        mp_array ac = nullptr, uu = nullptr, lt = nullptr, yy = nullptr;
        auto cleanup = [&] {
            for (mp_array h : {ac, uu, lt, yy})
                if (h) mp_array_destroy(h);
        };
        bool ok = mp_array_create(ctx, po, n, n, 1, &ac) == MP_OK && mp_array_create(ctx, po, n, n, 1, &uu) == MP_OK &&
                  mp_array_create(ctx, po, n, n, 1, &lt) == MP_OK &&
                  mp_array_create(ctx, po, y.rows, y.cols, 1, &yy) == MP_OK;
        if (!ok) {
            cleanup();
            fail(MP_OUT_OF_MEMORY, "solve: workspace");
        }
        mp_status st = mp_convert(ctx, a, ac);
        int64_t info = -1;
        if (st == MP_OK) st = mp_chol(ctx, ac, uu, &info);
        if (st == MP_OK) {
            st = mp_transpose(ctx, uu, lt);
            if (st == MP_OK) st = mp_forwardsolve(ctx, lt, b, yy);
            if (st == MP_OK) st = mp_backsolve(ctx, uu, yy, out);
            cleanup();
            if (st != MP_OK) throw Error(st, g_last_error);
            return MP_OK;
        }
        cleanup();
        if (st != MP_NOT_POSITIVE_DEFINITE) throw Error(st, g_last_error);
        // not positive definite: fall through to LU
    }
    const mp_precision cp = compute_precision(po);
    const size_t es = elem_bytes(cp);
    const size_t nn = static_cast<size_t>(n) * n, nb = static_cast<size_t>(y.rows) * y.cols;
    char* w = static_cast<char*>(c->ensure_scratch((nn + 2 * nb) * es + 512, 0));
    void* wa = w;
    void* wb = w + ((nn * es + 255) / 256) * 256;
    void* wx = static_cast<char*>(wb) + ((nb * es + 255) / 256) * 256;
    launch_convert(c, c->stream, x.prec, x.data, x.ld, cp, wa, n, n, n);
    launch_convert(c, c->stream, y.prec, y.data, y.ld, cp, wb, y.rows, y.rows, y.cols);
    const int64_t zp = lu_solve_device(c, c->stream, cp, wa, n, wb, y.rows, wx, y.rows, y.cols);
    if (zp >= 0) fail(MP_SINGULAR_MATRIX, "solve: zero pivot at column " + std::to_string(zp));
    launch_convert(c, c->stream, cp, wx, y.rows, o.prec, o.data, o.ld, y.rows, y.cols);
    MP_API_END
}

}  // extern "C"
