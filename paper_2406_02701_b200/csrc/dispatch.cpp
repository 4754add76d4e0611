// Op-name dispatch on device arrays: the reference's KernelRegistry /
// resolve / execute (proj/core/src/dispatch.cpp:46-137, dispatch.hpp) over
// the C ABI.  The table holds the same names with the same arity; resolve
// promotes the two input precisions (dispatch.cpp:102-107); execute checks
// the key against the inputs (PrecisionMismatch, :116-137) and returns a new
// device array from the op's kernel.
#include <cstring>
#include <string>

#include "internal.hpp"

using namespace mpcr;

namespace {

enum OpKind { EW, CONCAT_ROWS, CONCAT_COLS, MATMUL, CROSSPROD, UNARY_EW, TRANSPOSE, CHOL, SOLVE };

struct OpEntry {
    const char* name;
    OpKind kind;
    int arg;  // mp_binary_op / mp_unary_op for the elementwise kinds
    bool unary;
};

// registration order of KernelRegistry::KernelRegistry (dispatch.cpp:48-77)
constexpr OpEntry kOps[] = {
    {"add", EW, MP_ADD, false},          {"sub", EW, MP_SUB, false},
    {"mul", EW, MP_MUL, false},          {"div", EW, MP_DIV, false},
    {"rbind", CONCAT_ROWS, 0, false},    {"cbind", CONCAT_COLS, 0, false},
    {"matmul", MATMUL, 0, false},        {"crossprod", CROSSPROD, 0, false},
    {"log", UNARY_EW, MP_LOG, true},     {"exp", UNARY_EW, MP_EXP, true},
    {"sqrt", UNARY_EW, MP_SQRT, true},   {"abs", UNARY_EW, MP_ABS, true},
    {"transpose", TRANSPOSE, 0, true},   {"chol", CHOL, 0, true},
    {"solve", SOLVE, 0, true},
};

const OpEntry* lookup(const char* op) {
    if (!op) fail(MP_INVALID_PARAM, "null operation name");
    for (const auto& e : kOps)
        if (std::strcmp(e.name, op) == 0) return &e;
    throw Error(MP_UNKNOWN_OPERATION, std::string("unknown operation: ") + op);
}

void check_status(mp_status st) {
    if (st != MP_OK) throw Error(st, mp_last_error());
}

}  // namespace

#define MP_API_BEGIN try {
#define MP_API_END                                        \
    return MP_OK;                                         \
    }                                                     \
    catch (const mpcr::Error& e) {                        \
        mpcr::g_last_error = e.what();                    \
        return e.status;                                  \
    }                                                     \
    catch (const std::exception& e) {                     \
        mpcr::g_last_error = e.what();                    \
        return MP_INTERNAL_ERROR;                         \
    }

extern "C" {

mp_status mp_op_is_unary(const char* op, int* unary) {
    MP_API_BEGIN
    const OpEntry* e = lookup(op);
    if (unary) *unary = e->unary ? 1 : 0;
    MP_API_END
}

mp_status mp_resolve(const char* op, int prec_a, int prec_b, mp_kernel_key* key) {
    MP_API_BEGIN
    lookup(op);
    if (!key) fail(MP_INVALID_PARAM, "null key");
    if (prec_a < MP_HALF || prec_a > MP_DOUBLE || prec_b > MP_DOUBLE)
        fail(MP_INVALID_PARAM, "resolve: bad precision");
    key->in_a = prec_a;
    key->in_b = prec_b < 0 ? -1 : prec_b;
    key->out = prec_b < 0 ? prec_a : (prec_a >= prec_b ? prec_a : prec_b);
    MP_API_END
}

mp_status mp_execute(mp_ctx ctx, const mp_kernel_key* key, const char* op, mp_array a, mp_array b,
                     mp_array* out) {
    MP_API_BEGIN
    const OpEntry* e = lookup(op);
    if (!ctx || !key || !a || !out) fail(MP_INVALID_PARAM, "execute: null argument");
    bind_device(ctx);
    *out = nullptr;
    const Array& x = *a;
    const bool binary_call = b != nullptr;
    if (binary_call != (key->in_b >= 0) || x.prec != key->in_a || (binary_call && b->prec != key->in_b))
        fail(MP_PRECISION_MISMATCH, std::string("execute(") + op + "): input precision" +
                                        (binary_call ? "s do" : " does") + " not match the kernel key");
    if (binary_call == e->unary)
        fail(MP_INVALID_PARAM, std::string("execute(") + op + "): wrong number of operands");
    const mp_precision po = static_cast<mp_precision>(key->out);
    mp_array o = nullptr;
    auto make = [&](int64_t r, int64_t c, int is_matrix) {
        check_status(mp_array_create(ctx, po, r, c, is_matrix, &o));
    };
    try {
        switch (e->kind) {
            case EW:
                make(x.rows, x.cols, x.is_matrix);
                check_status(mp_ew_binary(ctx, static_cast<mp_binary_op>(e->arg), a, b, o));
                break;
            case UNARY_EW:
                make(x.rows, x.cols, x.is_matrix);
                check_status(mp_ew_unary(ctx, static_cast<mp_unary_op>(e->arg), a, o));
                break;
            case MATMUL:
                if (!x.is_matrix || !b->is_matrix) fail(MP_NOT_A_MATRIX, "matmul: input is not a matrix");
                make(x.rows, b->cols, 1);
                check_status(mp_matmul(ctx, a, b, o));
                break;
            case CROSSPROD:
                if (!x.is_matrix || !b->is_matrix) fail(MP_NOT_A_MATRIX, "crossprod: input is not a matrix");
                make(x.cols, b->cols, 1);
                check_status(mp_crossprod(ctx, a, b, o));
                break;
            case TRANSPOSE:
                if (!x.is_matrix) fail(MP_NOT_A_MATRIX, "transpose: input is not a matrix");
                make(x.cols, x.rows, 1);
                check_status(mp_transpose(ctx, a, o));
                break;
            case CHOL: {
                if (!x.is_matrix) fail(MP_NOT_A_MATRIX, "chol: input is not a matrix");
                make(x.rows, x.cols, 1);
                int64_t info = -1;
                const mp_status st = mp_chol(ctx, a, o, &info);
                if (st == MP_NOT_POSITIVE_DEFINITE) throw Error(st, mp_last_error(), info);
                check_status(st);
                break;
            }
            case SOLVE: {  // solve(a) = a^-1 (linalg.cpp:544-549)
                if (!x.is_matrix) fail(MP_NOT_A_MATRIX, "solve: input is not a matrix");
                if (x.rows != x.cols) fail(MP_SHAPE_MISMATCH, "solve: matrix is not square");
                mp_array eye = nullptr;
                check_status(mp_array_create(ctx, po, x.rows, x.rows, 1, &eye));
                launch_fill(ctx, ctx->stream, po, eye->data, eye->ld, x.rows, x.rows, 0.0);
                launch_add_diag(ctx, ctx->stream, po, eye->data, eye->ld, static_cast<int>(x.rows), 1.0);
                make(x.rows, x.rows, 1);
                const mp_status st = mp_solve(ctx, a, eye, o);
                mp_array_destroy(eye);
                check_status(st);
                break;
            }
            case CONCAT_ROWS:
            case CONCAT_COLS: {  // concat (array.cpp:391-420): exact widening into promote(a, b)
                const Array& y = *b;
                const bool rows = e->kind == CONCAT_ROWS;
                if (rows && x.cols != y.cols)
                    fail(MP_SHAPE_MISMATCH, "rbind: column counts " + std::to_string(x.cols) + " and " +
                                                std::to_string(y.cols) + " differ");
                if (!rows && x.rows != y.rows)
                    fail(MP_SHAPE_MISMATCH, "cbind: row counts " + std::to_string(x.rows) + " and " +
                                                std::to_string(y.rows) + " differ");
                make(rows ? x.rows + y.rows : x.rows, rows ? x.cols : x.cols + y.cols, 1);
                char* base = static_cast<char*>(o->data);
                launch_convert(ctx, ctx->stream, x.prec, x.data, x.ld, po, base, o->ld, x.rows, x.cols);
                const int64_t off = rows ? x.rows : x.cols * o->ld;
                launch_convert(ctx, ctx->stream, y.prec, y.data, y.ld, po, base + off * elem_bytes(po), o->ld,
                               y.rows, y.cols);
                break;
            }
        }
    } catch (...) {
        if (o) mp_array_destroy(o);
        throw;
    }
    *out = o;
    MP_API_END
}

}  // extern "C"
