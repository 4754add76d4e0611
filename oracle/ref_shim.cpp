// TEST INFRASTRUCTURE ONLY — the CPU oracle. Nothing in the product path
// (paper_2406_02701_b200/) links, loads or calls this file. Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// use it, as the checker or as the timed CPU reference arm.
//
// extern "C" shim over the UNMODIFIED reference library `mpnum`
// (/root/reference/proj/core/src/*.cpp compiled by oracle/Makefile into
// oracle/_ref/libmpnum_ref.so).  Values cross the boundary as column-major
// doubles that are exactly representable in the stated precision, plus raw
// storage bytes for the cast path.  Every entry point returns the status code
// of include/mpcr_b200.h (mp_status) so the parity tests compare error
// behaviour 1:1 with the CUDA library.
//
// The only non-trivial code here is the MPCRTile composition
// (ref_tile_chol / ref_tile_trsm / ref_tile_gemm): the reference ships no
// MPCRTile implementation (SPEC.md:13, PAPER.md:344-717 is commented out), so
// the tiled oracle composes reference primitives exactly as SURVEY.md §8c
// prescribes: linalg::chol (linalg.cpp:359), linalg::trsm (linalg.cpp:498),
// linalg::gemm (linalg.cpp:316) and MPArray::converted (array.cpp:187).

#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <vector>

#include "mpnum/array.hpp"
#include "mpnum/covariance.hpp"
#include "mpnum/errors.hpp"
#include "mpnum/linalg.hpp"
#include "mpnum/precision.hpp"
#include "mpnum/rng.hpp"
#include "mpnum/workloads.hpp"

using namespace mpnum;

namespace {

// Mirrors mp_status in include/mpcr_b200.h.
enum {
    S_OK = 0,
    S_SHAPE = 1,
    S_INDEX = 2,
    S_NOT_MATRIX = 3,
    S_EMPTY = 4,
    S_NOT_PD = 5,
    S_SINGULAR = 6,
    S_NO_CONV = 7,
    S_UNKNOWN_OP = 8,
    S_BACKEND = 9,
    S_PREC = 10,
    S_INVALID = 11,
    S_IO = 12,
    S_INTERNAL = 99,
};

thread_local int g_info = -1;

int guard(const std::function<void()>& fn) {
    g_info = -1;
    try {
        fn();
        return S_OK;
    } catch (const NotPositiveDefinite& e) {
        g_info = e.column;
        return S_NOT_PD;
    } catch (const ShapeMismatch&) {
        return S_SHAPE;
    } catch (const IndexOutOfRange&) {
        return S_INDEX;
    } catch (const NotAMatrix&) {
        return S_NOT_MATRIX;
    } catch (const EmptyArray&) {
        return S_EMPTY;
    } catch (const SingularMatrix&) {
        return S_SINGULAR;
    } catch (const NoConvergence&) {
        return S_NO_CONV;
    } catch (const UnknownOperation&) {
        return S_UNKNOWN_OP;
    } catch (const BackendUnavailable&) {
        return S_BACKEND;
    } catch (const PrecisionMismatch&) {
        return S_PREC;
    } catch (const InvalidParam&) {
        return S_INVALID;
    } catch (...) {
        return S_INTERNAL;
    }
}

Precision P(int p) { return static_cast<Precision>(p); }

MPArray mat(const double* v, std::size_t r, std::size_t c, int p) {
    return MPArray::from_doubles(std::vector<double>(v, v + r * c), r, c, P(p));
}

void out_doubles(const MPArray& a, double* out) {
    const auto v = a.to_doubles();
    std::memcpy(out, v.data(), v.size() * sizeof(double));
}

// Raw storage element i of `a` into `dst` (storage format of a's precision).
void store_raw(const MPArray& a, std::size_t i, unsigned char* dst) {
    switch (a.precision()) {
        case Precision::Half: {
            const Half16Bits b = a.half_bits(i);
            std::memcpy(dst + 2 * i, &b, 2);
            break;
        }
        case Precision::Single: {
            const float f = static_cast<float>(a.at_linear(i));
            std::memcpy(dst + 4 * i, &f, 4);
            break;
        }
        default: {
            const double d = a.at_linear(i);
            std::memcpy(dst + 8 * i, &d, 8);
            break;
        }
    }
}

double load_raw(const unsigned char* src, std::size_t i, int p) {
    switch (p) {
        case 0: {
            Half16Bits b;
            std::memcpy(&b, src + 2 * i, 2);
            return decode_f16(b);
        }
        case 1: {
            float f;
            std::memcpy(&f, src + 4 * i, 4);
            return static_cast<double>(f);
        }
        default: {
            double d;
            std::memcpy(&d, src + 8 * i, 8);
            return d;
        }
    }
}

}  // namespace

extern "C" {

int ref_last_info() { return g_info; }

void ref_set_num_threads(int t) { linalg::set_num_threads(t); }

// precision.cpp:49-93 / :95-109
void ref_encode_f16(const double* x, std::uint16_t* out, std::int64_t n) {
    for (std::int64_t i = 0; i < n; ++i) out[i] = encode_f16(x[i]);
}
void ref_decode_f16(const std::uint16_t* b, double* out, std::int64_t n) {
    for (std::int64_t i = 0; i < n; ++i) out[i] = decode_f16(b[i]);
}

// MPArray::converted (array.cpp:187-191) on raw storage bytes.  The input is
// loaded through set_linear of its decoded value, exactly the state an
// MPArray of precision `pin` holding those bytes would be in.
int ref_convert(int pin, int pout, const void* in, void* out, std::int64_t n) {
    return guard([&] {
        MPArray a = MPArray::zeros(static_cast<std::size_t>(n), P(pin));
        const auto* src = static_cast<const unsigned char*>(in);
        for (std::int64_t i = 0; i < n; ++i) a.set_linear(i, load_raw(src, i, pin));
        const MPArray b = a.converted(P(pout));
        auto* dst = static_cast<unsigned char*>(out);
        for (std::int64_t i = 0; i < n; ++i) store_raw(b, i, dst);
    });
}

// linalg::gemm (linalg.cpp:316-357): C <- alpha op(A) op(B) + beta C in C's
// precision.  A is ar x ac, B is br x bc, C is cr x cc (column-major doubles).
int ref_gemm(int pa, int pb, int pc, std::int64_t ar, std::int64_t ac, std::int64_t br,
             std::int64_t bc, std::int64_t cr, std::int64_t cc, int ta, int tb,
             double alpha, double beta, const double* A, const double* B, double* C) {
    return guard([&] {
        const MPArray a = mat(A, ar, ac, pa);
        const MPArray b = mat(B, br, bc, pb);
        MPArray c = mat(C, cr, cc, pc);
        linalg::gemm(a, b, c, {ta != 0, tb != 0, alpha, beta});
        out_doubles(c, C);
    });
}

// linalg::matmul (linalg.cpp:284-297); output precision promote(pa, pb).
int ref_matmul(int pa, int pb, std::int64_t m, std::int64_t k, std::int64_t k2,
               std::int64_t n, const double* A, const double* B, double* out) {
    return guard([&] {
        out_doubles(linalg::matmul(mat(A, m, k, pa), mat(B, k2, n, pb)), out);
    });
}

// linalg::crossprod (linalg.cpp:299-314); B == nullptr means crossprod(A).
int ref_crossprod(int pa, int pb, std::int64_t m, std::int64_t na, std::int64_t mb,
                  std::int64_t nb, const double* A, const double* B, double* out) {
    return guard([&] {
        const MPArray a = mat(A, m, na, pa);
        if (B == nullptr) {
            out_doubles(linalg::crossprod(a), out);
        } else {
            out_doubles(linalg::crossprod(a, mat(B, mb, nb, pb)), out);
        }
    });
}

// linalg::chol (linalg.cpp:359-378): upper U, lower zeroed; NotPositiveDefinite
// column available through ref_last_info().
int ref_chol(int p, std::int64_t r, std::int64_t c, const double* A, double* out) {
    return guard([&] { out_doubles(linalg::chol(mat(A, r, c, p)), out); });
}

// linalg::trsm (linalg.cpp:498-542); B overwritten.
int ref_trsm(int pa, int pb, std::int64_t ar, std::int64_t ac, std::int64_t br,
             std::int64_t bc, int side_right, int upper, int trans, double alpha,
             const double* A, double* B) {
    return guard([&] {
        const MPArray a = mat(A, ar, ac, pa);
        MPArray b = mat(B, br, bc, pb);
        linalg::trsm(a, b, side_right ? linalg::Side::Right : linalg::Side::Left,
                     upper != 0, trans != 0, alpha);
        out_doubles(b, B);
    });
}

// forwardsolve / backsolve (linalg.cpp:490-496, :424-441).
int ref_trisolve(int upper, int pt, int pb, std::int64_t n, std::int64_t tn,
                 std::int64_t br, std::int64_t bc, const double* T, const double* B,
                 double* out) {
    return guard([&] {
        const MPArray t = mat(T, n, tn, pt);
        const MPArray b = mat(B, br, bc, pb);
        out_doubles(upper ? linalg::backsolve(t, b) : linalg::forwardsolve(t, b), out);
    });
}

// linalg::solve (linalg.cpp:551-575) and chol2inv (linalg.cpp:481-488).
int ref_solve(int pa, int pb, std::int64_t n, std::int64_t bc, const double* A, const double* B,
              double* out) {
    return guard([&] { out_doubles(linalg::solve(mat(A, n, n, pa), mat(B, n, bc, pb)), out); });
}

int ref_chol2inv(int p, std::int64_t n, const double* U, double* out) {
    return guard([&] { out_doubles(linalg::chol2inv(mat(U, n, n, p)), out); });
}

// ew_binary / ew_scalar / ew_unary (array.cpp:252-322).
int ref_ew_binary(int op, int pa, int pb, std::int64_t r, std::int64_t c, std::int64_t r2,
                  std::int64_t c2, const double* A, const double* B, double* out) {
    return guard([&] {
        out_doubles(ew_binary(static_cast<BinaryOp>(op), mat(A, r, c, pa), mat(B, r2, c2, pb)),
                    out);
    });
}
int ref_ew_scalar(int op, int p, std::int64_t r, std::int64_t c, const double* A, double s,
                  double* out) {
    return guard([&] {
        out_doubles(ew_scalar(static_cast<BinaryOp>(op), mat(A, r, c, p), s), out);
    });
}
int ref_ew_unary(int op, int p, std::int64_t r, std::int64_t c, const double* A,
                 double* out) {
    return guard([&] {
        out_doubles(ew_unary(static_cast<UnaryOp>(op), mat(A, r, c, p)), out);
    });
}

// reduce (array.cpp:336-369).
int ref_reduce(int op, int p, std::int64_t r, std::int64_t c, const double* A,
               double* result) {
    return guard([&] { *result = reduce(static_cast<ReduceOp>(op), mat(A, r, c, p)); });
}

// transpose (array.cpp:422-429), diag (array.cpp:371-378).
int ref_transpose(int p, std::int64_t r, std::int64_t c, const double* A, double* out) {
    return guard([&] { out_doubles(transpose(mat(A, r, c, p)), out); });
}
int ref_diag(int p, std::int64_t r, std::int64_t c, const double* A, double* out) {
    return guard([&] { out_doubles(diag(mat(A, r, c, p)), out); });
}

// Rng (rng.cpp:9-53): the synthetic-input stream shared by GPU and oracle.
void ref_rng_uniform(std::uint64_t seed, std::int64_t n, double* out) {
    Rng rng(seed);
    for (std::int64_t i = 0; i < n; ++i) out[i] = rng.uniform();
}
void ref_rng_normal(std::uint64_t seed, std::int64_t n, double* out) {
    Rng rng(seed);
    for (std::int64_t i = 0; i < n; ++i) out[i] = rng.normal();
}

// Matern covariance over the first n points of a side x side unit grid
// (covariance.cpp:9-31 grid, :44-72 closed forms; mpnum_cli.cpp:73-82 for the
// "first n points of the smallest square grid" convention), rounded to prec.
int ref_grid_matern(std::int64_t side, std::int64_t n, double nu, double range,
                    double sigma2, int prec, double* out) {
    return guard([&] {
        const auto g = stats::grid_locations(static_cast<std::size_t>(side));
        MPArray d = MPArray::zeros_matrix(n, n, Precision::Double);
        for (std::int64_t j = 0; j < n; ++j)
            for (std::int64_t i = 0; i < n; ++i) d.set(i, j, g.distances.get(i, j));
        out_doubles(stats::matern_cov(d, {nu, range, sigma2}, P(prec)), out);
    });
}

// gaussian_nll (workloads.cpp:74-87) with the default JitterPolicy.
int ref_gaussian_nll(int prec, std::int64_t n, const double* z, const double* cov,
                     double* result) {
    return guard([&] {
        const MPArray zz = MPArray::vector_from_doubles(std::vector<double>(z, z + n),
                                                        Precision::Double);
        *result = stats::gaussian_nll(zz, mat(cov, n, n, 2), P(prec));
    });
}

// matern_mle (workloads.cpp:89-110): Nelder-Mead over (log range, log sigma2)
// on the unit-grid distances of `side`, first n points.
int ref_matern_mle(int prec, std::int64_t side, std::int64_t n, const double* z, double init_log_range,
                   double init_log_sigma2, int max_iter, double tol, double* range_hat, double* sigma2_hat,
                   double* nll, int* iterations) {
    return guard([&] {
        const auto g = stats::grid_locations(static_cast<std::size_t>(side));
        MPArray d = MPArray::zeros_matrix(n, n, Precision::Double);
        for (std::int64_t j = 0; j < n; ++j)
            for (std::int64_t i = 0; i < n; ++i) d.set(i, j, g.distances.get(i, j));
        const MPArray zz = MPArray::vector_from_doubles(std::vector<double>(z, z + n), Precision::Double);
        stats::NelderMeadConfig cfg;
        cfg.max_iter = max_iter;
        cfg.tol = tol;
        const auto r = stats::matern_mle(zz, d, P(prec), init_log_range, init_log_sigma2, cfg);
        *range_hat = r.range_hat;
        *sigma2_hat = r.sigma2_hat;
        *nll = r.nll;
        *iterations = r.iterations;
    });
}

// sample_gp (workloads.cpp:41-49).
int ref_sample_gp(std::int64_t n, const double* cov, std::uint64_t seed, double* out) {
    return guard([&] {
        Rng rng(seed);
        out_doubles(stats::sample_gp(mat(cov, n, n, 2), rng), out);
    });
}

// ---------------------------------------------------------------------------
// MPCRTile oracle (paper-only API), composed from reference
// primitives.  Tiles are nb x nb (nt = n / nb per side), prec[j * nt + i] is
// the precision of tile (i, j) (column-major tile grid, like R's matrix()).
// ---------------------------------------------------------------------------

namespace {

struct TileGrid {
    std::int64_t nt_r, nt_c, br, bc;
    std::vector<MPArray> t;  // column-major tile grid
    MPArray& at(std::int64_t i, std::int64_t j) { return t[j * nt_r + i]; }
};

TileGrid make_grid(std::int64_t rows, std::int64_t cols, std::int64_t br, std::int64_t bc,
                   const int* prec, const double* values) {
    TileGrid g{rows / br, cols / bc, br, bc, {}};
    g.t.reserve(g.nt_r * g.nt_c);
    for (std::int64_t tj = 0; tj < g.nt_c; ++tj) {
        for (std::int64_t ti = 0; ti < g.nt_r; ++ti) {
            std::vector<double> v(br * bc);
            for (std::int64_t j = 0; j < bc; ++j)
                for (std::int64_t i = 0; i < br; ++i)
                    v[j * br + i] = values[(tj * bc + j) * rows + ti * br + i];
            g.t.push_back(MPArray::from_doubles(v, br, bc, P(prec[tj * g.nt_r + ti])));
        }
    }
    return g;
}

void grid_out(TileGrid& g, std::int64_t rows, double* out) {
    for (std::int64_t tj = 0; tj < g.nt_c; ++tj)
        for (std::int64_t ti = 0; ti < g.nt_r; ++ti) {
            const MPArray& a = g.at(ti, tj);
            for (std::int64_t j = 0; j < g.bc; ++j)
                for (std::int64_t i = 0; i < g.br; ++i)
                    out[(tj * g.bc + j) * rows + ti * g.br + i] = a.get(i, j);
        }
}

MPArray as_prec(const MPArray& a, Precision p) {
    return a.precision() == p ? a : a.converted(p);
}

}  // namespace

// Right-looking tiled Cholesky, lower L: for each k
//   U_kk = chol(A_kk)                          (linalg.cpp:359, FP of tile kk)
//   A_ik = trsm(U_kk -> p_ik, A_ik, Right, upper, notrans)   i > k
//   A_ij = gemm(A_ik -> p_ij, A_jk -> p_ij, A_ij, {F, T, -1, 1})  i >= j > k
// Upper tiles are zeroed, as the paper's printout shows.  On failure the
// global failing column is in ref_last_info().
int ref_tile_chol(std::int64_t n, std::int64_t nb, const int* prec, const double* A,
                  double* L) {
    int local_info = -1;
    const int st = guard([&] {
        if (n % nb != 0) throw ShapeMismatch("tile size must divide n");
        TileGrid g = make_grid(n, n, nb, nb, prec, A);
        const std::int64_t nt = g.nt_r;
        for (std::int64_t k = 0; k < nt; ++k) {
            MPArray u;
            try {
                u = linalg::chol(g.at(k, k));
            } catch (const NotPositiveDefinite& e) {
                local_info = static_cast<int>(k * nb + e.column);
                throw NotPositiveDefinite(local_info);
            }
            g.at(k, k) = transpose(u);
            for (std::int64_t i = k + 1; i < nt; ++i) {
                MPArray& b = g.at(i, k);
                linalg::trsm(as_prec(u, b.precision()), b, linalg::Side::Right, true, false,
                             1.0);
            }
            for (std::int64_t j = k + 1; j < nt; ++j) {
                for (std::int64_t i = j; i < nt; ++i) {
                    MPArray& c = g.at(i, j);
                    linalg::gemm(as_prec(g.at(i, k), c.precision()),
                                 as_prec(g.at(j, k), c.precision()), c,
                                 {false, true, -1.0, 1.0});
                }
            }
        }
        for (std::int64_t j = 1; j < nt; ++j)
            for (std::int64_t i = 0; i < j; ++i)
                g.at(i, j) = MPArray::zeros_matrix(nb, nb, g.at(i, j).precision());
        grid_out(g, n, L);
    });
    return st;
}

// MPCRTile.gemm: C_ij = alpha * sum_l op(A)_il op(B)_lj +
// beta * C_ij, every tile product in C_ij's precision; the first product of a
// tile carries beta, later ones accumulate with beta = 1.
int ref_tile_gemm(std::int64_t ar, std::int64_t ac, std::int64_t abr, std::int64_t abc,
                  const int* pa, const double* A, std::int64_t brr, std::int64_t bcc,
                  std::int64_t bbr, std::int64_t bbc, const int* pb, const double* B,
                  std::int64_t cr, std::int64_t cc, std::int64_t cbr, std::int64_t cbc,
                  const int* pc, double* C, int ta, int tb, double alpha, double beta) {
    return guard([&] {
        TileGrid a = make_grid(ar, ac, abr, abc, pa, A);
        TileGrid b = make_grid(brr, bcc, bbr, bbc, pb, B);
        TileGrid c = make_grid(cr, cc, cbr, cbc, pc, C);
        const std::int64_t kt = ta ? a.nt_r : a.nt_c;
        const std::int64_t kb = tb ? b.nt_c : b.nt_r;
        if (kt != kb || (ta ? a.nt_c : a.nt_r) != c.nt_r || (tb ? b.nt_r : b.nt_c) != c.nt_c)
            throw ShapeMismatch("tile gemm: incompatible tile grids");
        for (std::int64_t j = 0; j < c.nt_c; ++j)
            for (std::int64_t i = 0; i < c.nt_r; ++i) {
                MPArray& t = c.at(i, j);
                for (std::int64_t l = 0; l < kt; ++l) {
                    const MPArray& x = ta ? a.at(l, i) : a.at(i, l);
                    const MPArray& y = tb ? b.at(j, l) : b.at(l, j);
                    linalg::gemm(as_prec(x, t.precision()), as_prec(y, t.precision()), t,
                                 {ta != 0, tb != 0, alpha, l == 0 ? beta : 1.0});
                }
            }
        grid_out(c, cr, C);
    });
}

// MPCRTile.trsm: op(A) X = alpha B (Left) or
// X op(A) = alpha B (Right), tile substitution in B-tile precision.  The first
// update of each B tile carries beta = alpha; a tile with no update gets alpha
// through the diagonal trsm.
int ref_tile_trsm(std::int64_t n, std::int64_t nb, const int* pa, const double* A,
                  std::int64_t br, std::int64_t bc, std::int64_t bbr, std::int64_t bbc,
                  const int* pb, double* B, int side_right, int upper, int trans,
                  double alpha) {
    return guard([&] {
        TileGrid a = make_grid(n, n, nb, nb, pa, A);
        TileGrid b = make_grid(br, bc, bbr, bbc, pb, B);
        const std::int64_t nt = a.nt_r;
        const bool eff_lower = (upper != 0) == (trans != 0);
        // opA(r, k) as a stored tile plus a transpose flag.
        auto op_tile = [&](std::int64_t r, std::int64_t k) -> const MPArray& {
            return trans ? a.at(k, r) : a.at(r, k);
        };
        if (!side_right) {
            if (b.nt_r != nt || bbr != nb) throw ShapeMismatch("tile trsm: B row tiling");
            for (std::int64_t s = 0; s < nt; ++s) {
                const std::int64_t r = eff_lower ? s : nt - 1 - s;
                for (std::int64_t c = 0; c < b.nt_c; ++c) {
                    MPArray& t = b.at(r, c);
                    bool first = true;
                    for (std::int64_t q = 0; q < s; ++q) {
                        const std::int64_t k = eff_lower ? q : nt - 1 - q;
                        linalg::gemm(as_prec(op_tile(r, k), t.precision()),
                                     as_prec(b.at(k, c), t.precision()), t,
                                     {trans != 0, false, -1.0, first ? alpha : 1.0});
                        first = false;
                    }
                    linalg::trsm(as_prec(a.at(r, r), t.precision()), t, linalg::Side::Left,
                                 upper != 0, trans != 0, first ? alpha : 1.0);
                }
            }
        } else {
            if (b.nt_c != nt || bbc != nb) throw ShapeMismatch("tile trsm: B col tiling");
            // X op(A) = B: column c of X depends on columns already solved;
            // op(A) lower => solve the last column first.
            for (std::int64_t s = 0; s < nt; ++s) {
                const std::int64_t c = eff_lower ? nt - 1 - s : s;
                for (std::int64_t r = 0; r < b.nt_r; ++r) {
                    MPArray& t = b.at(r, c);
                    bool first = true;
                    for (std::int64_t q = 0; q < s; ++q) {
                        const std::int64_t k = eff_lower ? nt - 1 - q : q;
                        // X_rk * opA(k, c)
                        linalg::gemm(as_prec(b.at(r, k), t.precision()),
                                     as_prec(op_tile(k, c), t.precision()), t,
                                     {false, trans != 0, -1.0, first ? alpha : 1.0});
                        first = false;
                    }
                    linalg::trsm(as_prec(a.at(c, c), t.precision()), t, linalg::Side::Right,
                                 upper != 0, trans != 0, first ? alpha : 1.0);
                }
            }
        }
        grid_out(b, br, B);
    });
}

}  // extern "C"
