// C++ façade: the reference core's call signatures (proj/core/include/mpnum/
// linalg.hpp, array.hpp, workloads.hpp, dispatch.hpp) running on the B200
// engine through the C ABI (mpcr_b200.h).  Header-only; a maintainer of the
// reference includes it next to the mpnum headers and swaps
//     mpnum::linalg::gemm(a, b, c, p)   ->  mpcr_b200::linalg::gemm(eng, a, b, c, p)
// (same arguments plus an Engine), keeping the reference's MPArray on the
// host side.  mp_status codes are rethrown as the reference's exception types
// (errors.hpp:8-76), so existing handlers such as the
//     catch (const NotPositiveDefinite&)
// of chol_with_jitter (workloads.cpp:54-70) work unchanged.
//
// Needs the reference headers on the include path (-I proj/core/include) and
// links -lmpcr_b200.  tests/cpp/facade_test.cpp compiles and runs it against
// the reference library (test infrastructure) under `pytest -m gpu`.
#pragma once

#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "mpcr_b200.h"
#include "mpnum/array.hpp"
#include "mpnum/errors.hpp"
#include "mpnum/linalg.hpp"
#include "mpnum/workloads.hpp"

namespace mpcr_b200 {

// mp_status -> the reference exception (errors.hpp:8-76).
[[noreturn]] inline void rethrow(mp_status s, int64_t info = -1) {
    const std::string msg = mp_last_error();
    switch (s) {
        case MP_SHAPE_MISMATCH: throw mpnum::ShapeMismatch(msg);
        case MP_INDEX_OUT_OF_RANGE: throw mpnum::IndexOutOfRange(msg);
        case MP_NOT_A_MATRIX: throw mpnum::NotAMatrix(msg);
        case MP_EMPTY_ARRAY: throw mpnum::EmptyArray(msg);
        case MP_NOT_POSITIVE_DEFINITE: throw mpnum::NotPositiveDefinite(static_cast<int>(info));
        case MP_SINGULAR_MATRIX: throw mpnum::SingularMatrix(msg);
        case MP_NO_CONVERGENCE: throw mpnum::NoConvergence(msg);
        case MP_UNKNOWN_OPERATION: throw mpnum::UnknownOperation(msg);
        case MP_BACKEND_UNAVAILABLE: throw mpnum::BackendUnavailable(msg);
        case MP_PRECISION_MISMATCH: throw mpnum::PrecisionMismatch(msg);
        case MP_IO_ERROR: throw mpnum::IoError(msg);
        default: throw mpnum::InvalidParam(msg);
    }
}
inline void check(mp_status s, int64_t info = -1) {
    if (s != MP_OK) rethrow(s, info);
}

// One device context (streams, scratch) per GPU; owns the mp_ctx.
class Engine {
public:
    explicit Engine(int device = 0) { check(mp_ctx_create(device, &ctx_)); }
    ~Engine() { mp_ctx_destroy(ctx_); }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;
    mp_ctx get() const { return ctx_; }

private:
    mp_ctx ctx_ = nullptr;
};

// A device copy of a reference MPArray (set_linear rounding on upload).
class DeviceArray {
public:
    DeviceArray(Engine& e, const mpnum::MPArray& x) : DeviceArray(e, x.precision(), x.rows(), x.cols(), x.is_matrix()) {
        const std::vector<double> v = x.to_doubles();
        check(mp_array_from_doubles(h_, v.data(), static_cast<int64_t>(v.size())));
    }
    DeviceArray(Engine& e, mpnum::Precision p, std::size_t rows, std::size_t cols, bool is_matrix = true) {
        check(mp_array_create(e.get(), static_cast<mp_precision>(p), static_cast<int64_t>(rows),
                              static_cast<int64_t>(cols), is_matrix ? 1 : 0, &h_));
    }
    explicit DeviceArray(mp_array h) : h_(h) {}
    ~DeviceArray() {
        if (h_) mp_array_destroy(h_);
    }
    DeviceArray(const DeviceArray&) = delete;
    DeviceArray& operator=(const DeviceArray&) = delete;
    mp_array get() const { return h_; }

    // Back to a host MPArray of the same precision and shape (exact).
    mpnum::MPArray to_host() const {
        mp_precision p;
        int64_t r = 0, c = 0, ld = 0;
        int m = 0;
        void* dptr = nullptr;
        check(mp_array_info(h_, &p, &r, &c, &ld, &m, &dptr));
        std::vector<double> v(static_cast<std::size_t>(r * c));
        check(mp_array_to_doubles(h_, v.data(), static_cast<int64_t>(v.size())));
        const auto prec = static_cast<mpnum::Precision>(p);
        return m ? mpnum::MPArray::from_doubles(v, r, c, prec) : mpnum::MPArray::vector_from_doubles(v, prec);
    }
    // Copy into an existing host array of the same shape (c of gemm / trsm).
    void to_host(mpnum::MPArray& out) const {
        std::vector<double> v(out.size());
        check(mp_array_to_doubles(h_, v.data(), static_cast<int64_t>(v.size())));
        for (std::size_t i = 0; i < v.size(); ++i) out.set_linear(i, v[i]);
    }

private:
    mp_array h_ = nullptr;
};

// MPArray::converted (array.cpp:187-191).
inline mpnum::MPArray converted(Engine& e, const mpnum::MPArray& a, mpnum::Precision p) {
    DeviceArray da(e, a), out(e, p, a.rows(), a.cols(), a.is_matrix());
    check(mp_convert(e.get(), da.get(), out.get()));
    return out.to_host();
}

namespace linalg {

using mpnum::linalg::GemmParams;
using mpnum::linalg::Side;

// linalg::gemm (linalg.cpp:316-357): c <- alpha op(a) op(b) + beta c in c's precision.
inline void gemm(Engine& e, const mpnum::MPArray& a, const mpnum::MPArray& b, mpnum::MPArray& c,
                 const GemmParams& p) {
    DeviceArray da(e, a), db(e, b), dc(e, c);
    check(mp_gemm(e.get(), da.get(), db.get(), dc.get(), p.trans_a, p.trans_b, p.alpha, p.beta));
    dc.to_host(c);
}

// linalg::matmul (linalg.cpp:284-296): output in promote(a, b).
inline mpnum::MPArray matmul(Engine& e, const mpnum::MPArray& a, const mpnum::MPArray& b) {
    DeviceArray da(e, a), db(e, b), out(e, mpnum::promote(a.precision(), b.precision()), a.rows(), b.cols());
    check(mp_matmul(e.get(), da.get(), db.get(), out.get()));
    return out.to_host();
}

// linalg::crossprod (linalg.cpp:298-314): a^T a (exactly symmetric) or a^T b.
inline mpnum::MPArray crossprod(Engine& e, const mpnum::MPArray& a) {
    DeviceArray da(e, a), out(e, a.precision(), a.cols(), a.cols());
    check(mp_crossprod(e.get(), da.get(), nullptr, out.get()));
    return out.to_host();
}
inline mpnum::MPArray crossprod(Engine& e, const mpnum::MPArray& a, const mpnum::MPArray& b) {
    DeviceArray da(e, a), db(e, b), out(e, mpnum::promote(a.precision(), b.precision()), a.cols(), b.cols());
    check(mp_crossprod(e.get(), da.get(), db.get(), out.get()));
    return out.to_host();
}

// linalg::chol (linalg.cpp:359-378): upper u with a = u^T u; throws
// mpnum::NotPositiveDefinite(first failing column).
inline mpnum::MPArray chol(Engine& e, const mpnum::MPArray& a) {
    DeviceArray da(e, a), out(e, a.precision(), a.rows(), a.cols());
    int64_t info = -1;
    const mp_status st = mp_chol(e.get(), da.get(), out.get(), &info);  // info is set by the call
    check(st, info);
    return out.to_host();
}

// linalg::trsm (linalg.cpp:498-542): b overwritten with x.
inline void trsm(Engine& e, const mpnum::MPArray& a, mpnum::MPArray& b, Side side, bool upper, bool trans,
                 double alpha) {
    DeviceArray da(e, a), db(e, b);
    check(mp_trsm(e.get(), da.get(), db.get(), side == Side::Left ? MP_LEFT : MP_RIGHT, upper, trans, alpha));
    db.to_host(b);
}

// linalg::forwardsolve / backsolve (linalg.cpp:490-496).
inline mpnum::MPArray forwardsolve(Engine& e, const mpnum::MPArray& l, const mpnum::MPArray& b) {
    DeviceArray dl(e, l), db(e, b), out(e, mpnum::promote(l.precision(), b.precision()), b.rows(), b.cols());
    check(mp_forwardsolve(e.get(), dl.get(), db.get(), out.get()));
    return out.to_host();
}
inline mpnum::MPArray backsolve(Engine& e, const mpnum::MPArray& u, const mpnum::MPArray& b) {
    DeviceArray du(e, u), db(e, b), out(e, mpnum::promote(u.precision(), b.precision()), b.rows(), b.cols());
    check(mp_backsolve(e.get(), du.get(), db.get(), out.get()));
    return out.to_host();
}

}  // namespace linalg

// dispatch::resolve / execute (dispatch.cpp:102-137) by op name.
namespace dispatch {

inline mp_kernel_key resolve(const std::string& op, mpnum::Precision a, mpnum::Precision b) {
    mp_kernel_key k;
    check(mp_resolve(op.c_str(), static_cast<int>(a), static_cast<int>(b), &k));
    return k;
}
inline mp_kernel_key resolve(const std::string& op, mpnum::Precision a) {
    mp_kernel_key k;
    check(mp_resolve(op.c_str(), static_cast<int>(a), -1, &k));
    return k;
}
inline mpnum::MPArray execute(Engine& e, const mp_kernel_key& key, const std::string& op,
                              const mpnum::MPArray& a, const mpnum::MPArray* b = nullptr) {
    DeviceArray da(e, a);
    mp_array out = nullptr;
    if (b) {
        DeviceArray db(e, *b);
        check(mp_execute(e.get(), &key, op.c_str(), da.get(), db.get(), &out));
    } else {
        check(mp_execute(e.get(), &key, op.c_str(), da.get(), nullptr, &out));
    }
    return DeviceArray(out).to_host();
}

}  // namespace dispatch

// MPCRTile resident on the device.
class Tile {
public:
    // new(MPCRTile, rows, cols, rows_per_tile, cols_per_tile, values, precisions):
    // precisions is the tiles_r x tiles_c grid, column-major.
    Tile(Engine& e, std::size_t rows, std::size_t cols, std::size_t rpt, std::size_t cpt,
         const std::vector<int>& precisions, const std::vector<double>& values)
        : e_(e) {
        check(mp_tile_create(e.get(), rows, cols, rpt, cpt, precisions.data(), &t_));
        if (!values.empty()) check(mp_tile_set_values(t_, values.data()));
    }
    ~Tile() {
        if (t_) mp_tile_destroy(t_);
    }
    Tile(const Tile&) = delete;
    Tile& operator=(const Tile&) = delete;
    // chol(MPCRTile) in place; NotPositiveDefinite carries
    // the global failing column.
    void chol() {
        int64_t info = -1;
        const mp_status st = mp_tile_chol(e_.get(), t_, 1, nullptr, &info);
        check(st, info);
    }
    double logdet() const {
        double v = 0;
        check(mp_tile_logdet(e_.get(), t_, &v));
        return v;
    }
    std::vector<double> values() const {
        int64_t r = 0, c = 0;
        check(mp_tile_info(t_, &r, &c, nullptr, nullptr, nullptr, nullptr));
        std::vector<double> v(static_cast<std::size_t>(r * c));
        check(mp_tile_get_values(t_, v.data()));
        return v;
    }
    mp_tile get() const { return t_; }

private:
    Engine& e_;
    mp_tile t_ = nullptr;
};

namespace stats {

// stats::gaussian_nll (workloads.cpp:74-87) with chol_with_jitter
// (workloads.cpp:54-70) written exactly as the reference writes it, its
// Cholesky on the GPU: the NotPositiveDefinite rethrown by linalg::chol
// drives the x10 jitter escalation.
inline double gaussian_nll(Engine& e, const mpnum::MPArray& z, const mpnum::MPArray& cov, mpnum::Precision prec,
                           const mpnum::stats::JitterPolicy& policy = {}) {
    using mpnum::MPArray;
    const std::size_t n = cov.rows();
    const MPArray v = cov.precision() == prec ? cov : converted(e, cov, prec);
    MPArray u;
    if (prec == mpnum::Precision::Double) {
        u = linalg::chol(e, v);
    } else {
        double jitter = policy.initial;
        for (;;) {
            MPArray jittered = v;
            for (std::size_t i = 0; i < v.rows(); ++i) jittered.set(i, i, v.get(i, i) + jitter);
            try {
                u = linalg::chol(e, jittered);
                break;
            } catch (const mpnum::NotPositiveDefinite&) {
                jitter *= 10.0;
                if (jitter > policy.max_jitter) throw;
            }
        }
    }
    double log_det = 0.0;
    for (std::size_t i = 0; i < n; ++i) log_det += std::log(u.get(i, i));
    log_det *= 2.0;
    const MPArray zc = z.precision() == prec ? z : converted(e, z, prec);
    const MPArray rhs = MPArray::from_doubles(zc.to_doubles(), n, 1, prec);
    // forwardsolve(t(u), rhs): t(u) on the device
    DeviceArray du(e, u), ut(e, prec, n, n);
    check(mp_transpose(e.get(), du.get(), ut.get()));
    DeviceArray drhs(e, rhs), w(e, prec, n, 1);
    check(mp_forwardsolve(e.get(), ut.get(), drhs.get(), w.get()));
    double quad = 0.0;
    check(mp_reduce(e.get(), MP_SQUARE_SUM, w.get(), &quad));
    return 0.5 * quad + 0.5 * log_det + 0.5 * static_cast<double>(n) * std::log(2.0 * M_PI);
}

}  // namespace stats

}  // namespace mpcr_b200
