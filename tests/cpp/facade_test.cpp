// TEST INFRASTRUCTURE: the drop-in boundary compiled from C++.
//
// The reference's own host types (mpnum::MPArray, GemmParams, JitterPolicy,
// the exception hierarchy; linked from oracle/_ref/libmpnum_ref.so, the
// unmodified reference sources) drive the B200 engine through the façade
// include/mpcr_b200_mpnum.hpp, and every result is compared with the
// reference's CPU call on the same inputs.  Built by tests/cpp/Makefile
// (__graft_entry__.build() when /root/reference is present); run by
// tests/test_cpp_boundary.py under `pytest -m gpu`.  Prints one line per
// check and "facade ok" when all pass; exits non-zero otherwise.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "mpcr_b200_mpnum.hpp"
#include "mpnum/dispatch.hpp"
#include "mpnum/rng.hpp"

using mpnum::MPArray;
using mpnum::Precision;

static int failures = 0;

static void expect(bool ok, const std::string& what) {
    std::printf("%s %s\n", ok ? "ok  " : "FAIL", what.c_str());
    if (!ok) ++failures;
}

static double rel_frob(const MPArray& a, const MPArray& b) {
    double num = 0, den = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        const double d = a.at_linear(i) - b.at_linear(i);
        num += d * d;
        den += b.at_linear(i) * b.at_linear(i);
    }
    return std::sqrt(num / den);
}

// acceptance criterion 4 inputs: Rng(1000 + n), column-major uniform draws
static MPArray random_uniform(std::size_t r, std::size_t c, Precision p, mpnum::Rng& rng) {
    std::vector<double> v(r * c);
    for (auto& x : v) x = rng.uniform();
    return MPArray::from_doubles(v, r, c, p);
}

static MPArray spd(std::size_t n, Precision p, mpnum::Rng& rng) {
    const MPArray b = random_uniform(n, n, Precision::Double, rng);
    MPArray a = mpnum::linalg::crossprod(b);
    std::vector<double> v = a.to_doubles();
    for (std::size_t i = 0; i < n; ++i) v[i * n + i] += static_cast<double>(n);
    return MPArray::from_doubles(v, n, n, p);
}

int main() {
    mpcr_b200::Engine eng(0);
    const std::size_t n = 512;
    mpnum::Rng rng(1000 + n);

    // 1. linalg::gemm, FP32 (config 1's call shape) and FP16 inputs into FP32 / FP64
    for (Precision pa : {Precision::Single, Precision::Half}) {
        for (Precision pc : {Precision::Single, Precision::Double}) {
            const MPArray a = random_uniform(n, n, pa, rng), b = random_uniform(n, n, pa, rng);
            MPArray c_ref = MPArray::zeros_matrix(n, n, pc), c_gpu = MPArray::zeros_matrix(n, n, pc);
            mpnum::linalg::GemmParams p;
            p.trans_b = true;
            mpnum::linalg::gemm(a, b, c_ref, p);
            mpcr_b200::linalg::gemm(eng, a, b, c_gpu, p);
            const double err = rel_frob(c_gpu, c_ref);
            const double tol = pc == Precision::Single ? 4.0 * n * 5.96e-8 : 1e-13;
            expect(err <= tol, "gemm " + mpnum::precision_name(pa) + "->" + mpnum::precision_name(pc) +
                                   " rel err " + std::to_string(err));
        }
    }
    // 2. crossprod, exactly symmetric
    {
        const MPArray a = random_uniform(n, 256, Precision::Single, rng);
        const MPArray g = mpcr_b200::linalg::crossprod(eng, a), r = mpnum::linalg::crossprod(a);
        bool sym = true;
        for (std::size_t j = 0; j < g.cols(); ++j)
            for (std::size_t i = 0; i < j; ++i) sym = sym && g.get(i, j) == g.get(j, i);
        expect(sym && rel_frob(g, r) < 1e-5, "crossprod symmetric, rel err " + std::to_string(rel_frob(g, r)));
    }
    // 3. linalg::chol (upper) vs the reference, double and single
    for (Precision p : {Precision::Double, Precision::Single}) {
        const MPArray a = spd(n, p, rng);
        const MPArray u = mpcr_b200::linalg::chol(eng, a), ur = mpnum::linalg::chol(a);
        const double u_p = p == Precision::Double ? 1.11e-16 : 5.96e-8;
        expect(rel_frob(u, ur) <= 100.0 * n * u_p,
               "chol " + mpnum::precision_name(p) + " rel err " + std::to_string(rel_frob(u, ur)));
    }
    // 4. NotPositiveDefinite is rethrown with the reference's failing column
    {
        std::vector<double> v(n * n, 0.0);
        for (std::size_t i = 0; i < n; ++i) v[i * n + i] = 1.0;
        v[300 * n + 300] = -1.0;
        const MPArray a = MPArray::from_doubles(v, n, n, Precision::Double);
        int gpu_col = -2, ref_col = -3;
        try {
            mpcr_b200::linalg::chol(eng, a);
        } catch (const mpnum::NotPositiveDefinite& e) {
            gpu_col = e.column;
        }
        try {
            mpnum::linalg::chol(a);
        } catch (const mpnum::NotPositiveDefinite& e) {
            ref_col = e.column;
        }
        expect(gpu_col == 300 && gpu_col == ref_col,
               "NotPositiveDefinite column gpu " + std::to_string(gpu_col) + " ref " + std::to_string(ref_col));
    }
    // 5. gaussian_nll with chol_with_jitter: pivot 5 is -5e-6 (uncoupled, so
    // its Schur complement is exactly that), the first jitter 1e-6 leaves it
    // negative and the NotPositiveDefinite rethrown by the GPU chol must be
    // caught by the façade's copy of workloads.cpp:54-70 and escalate to 1e-5,
    // as the reference does; compared with stats::gaussian_nll
    {
        const std::size_t m = 256;
        std::vector<double> x(m * m, 0.0);
        for (std::size_t j = 10; j < m; ++j)  // an SPD exponential block on rows/cols 10..m-1
            for (std::size_t i = 10; i < m; ++i)
                x[j * m + i] = 0.5 * std::exp(-std::fabs(static_cast<double>(i) - static_cast<double>(j)) / 8.0);
        for (std::size_t i = 0; i < m; ++i) x[i * m + i] += 1.0;
        x[5 * m + 5] = -5e-6;
        const MPArray cov = MPArray::from_doubles(x, m, m, Precision::Double);
        std::vector<double> zv(m);
        for (auto& z : zv) z = rng.normal();
        const MPArray z = MPArray::vector_from_doubles(zv, Precision::Double);
        int first_fail = -1;
        try {
            MPArray j1 = cov.converted(Precision::Single);
            for (std::size_t i = 0; i < m; ++i) j1.set(i, i, j1.get(i, i) + 1e-6);
            mpcr_b200::linalg::chol(eng, j1);
        } catch (const mpnum::NotPositiveDefinite& e) {
            first_fail = e.column;
        }
        const double g = mpcr_b200::stats::gaussian_nll(eng, z, cov, Precision::Single);
        const double r = mpnum::stats::gaussian_nll(z, cov, Precision::Single);
        expect(first_fail == 5 && std::fabs(g - r) <= 1e-5 * std::fabs(r),
               "gaussian_nll single with jitter escalation (first try fails at column " +
                   std::to_string(first_fail) + "): " + std::to_string(g) + " ref " + std::to_string(r));
        bool threw = false;  // prec Double: no jitter, the exception reaches the caller
        try {
            mpcr_b200::stats::gaussian_nll(eng, z, cov, Precision::Double);
        } catch (const mpnum::NotPositiveDefinite& e) {
            threw = e.column == 5;
        }
        expect(threw, "gaussian_nll double (no jitter) throws NotPositiveDefinite(5)");
    }
    // 6. dispatch by op name: same key and result as the reference registry
    {
        const MPArray a = random_uniform(64, 48, Precision::Half, rng), b = random_uniform(48, 32, Precision::Single, rng);
        const mp_kernel_key k = mpcr_b200::dispatch::resolve("matmul", a.precision(), b.precision());
        const mpnum::dispatch::KernelKey kr = mpnum::dispatch::resolve("matmul", a.precision(), b.precision());
        const MPArray g = mpcr_b200::dispatch::execute(eng, k, "matmul", a, &b);
        const MPArray r = mpnum::dispatch::execute(kr, "matmul", a, b);
        expect(k.out == static_cast<int>(kr.out) && g.precision() == r.precision() && rel_frob(g, r) < 1e-6,
               "dispatch matmul key/out precision/values");
        bool unknown = false;
        try {
            mpcr_b200::dispatch::resolve("qr", Precision::Double);
        } catch (const mpnum::UnknownOperation&) {
            unknown = true;
        }
        expect(unknown, "dispatch unknown op -> UnknownOperation");
    }
    // 7. MPCRTile chol + logdet (PAPER.md:585-646 example)
    {
        const std::vector<double> m4 = {1.0, 0.36787944117144233, 0.36787944117144233, 0.24311673443421421,
                                        0.36787944117144233, 1.0, 0.24311673443421421, 0.36787944117144233,
                                        0.36787944117144233, 0.24311673443421421, 1.0, 0.36787944117144233,
                                        0.24311673443421421, 0.36787944117144233, 0.36787944117144233, 1.0};
        mpcr_b200::Tile t(eng, 4, 4, 2, 2, {2, 1, 1, 2}, m4);
        t.chol();
        const std::vector<double> l = t.values();
        expect(std::fabs(l[1 * 4 + 1] - 0.9298735) < 1e-6 && std::fabs(l[0 * 4 + 2] - 0.3678795) < 5e-8,
               "MPCRTile chol reproduces the paper printout (PAPER.md:643-646)");
    }
    std::printf("%s\n", failures ? "facade FAILED" : "facade ok");
    return failures ? 1 : 0;
}
