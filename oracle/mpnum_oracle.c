/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement ("port") of the reference
 * algorithms on the MPCR hot path.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it, as the checker.  The product
 * library never links it.
 *
 * Parity is PINNED: tests/test_oracle.py checks every function below
 * bit-for-bit against the unmodified reference compiled into
 * oracle/_ref/libmpnum_ref.so (oracle/Makefile) and against the committed
 * golden vectors in tests/golden/ (made by tests/golden/make_golden.py).
 *
 * Arithmetic follows the reference loop order exactly; build with
 * -ffp-contract=off (no FMA contraction) like the reference's x86-64 build.
 * Matrices are column-major; values are passed as doubles that are exactly
 * representable in the stated precision (0 half, 1 single, 2 double).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { ST_OK = 0, ST_SHAPE = 1, ST_NOT_PD = 5, ST_SINGULAR = 6, ST_PREC = 10, ST_NOMEM = 102 };

static int g_info = -1;
int mpo_last_info(void) { return g_info; }

/* ---- precision.cpp:49-93 encode_f16 (RNE straight from double) ---------- */
uint16_t mpo_encode_f16(double x) {
    uint64_t d;
    memcpy(&d, &x, 8);
    const uint16_t sign = (uint16_t)((d >> 63) << 15);
    const int dexp = (int)((d >> 52) & 0x7FF);
    const uint64_t dfrac = d & ((UINT64_C(1) << 52) - 1);
    if (dexp == 0x7FF) return dfrac ? (uint16_t)0x7E00 : (uint16_t)(sign | 0x7C00);
    if (dexp == 0) return sign; /* zero or double subnormal -> signed zero */
    const int e = dexp - 1023;
    const uint64_t m = (UINT64_C(1) << 52) | dfrac;
    int shift = 42;
    if (e < -14) {
        shift = 42 + (-14 - e);
        if (shift >= 64) return sign;
    }
    uint64_t keep = m >> shift;
    const uint64_t rem = m & ((UINT64_C(1) << shift) - 1);
    const uint64_t half = UINT64_C(1) << (shift - 1);
    if (rem > half || (rem == half && (keep & 1))) ++keep;
    if (e >= -14) {
        int he = e + 15;
        if (keep == 0x800) {
            keep = 0x400;
            ++he;
        }
        if (he >= 31) return (uint16_t)(sign | 0x7C00);
        return (uint16_t)(sign | (he << 10) | (keep & 0x3FF));
    }
    return (uint16_t)(sign | keep);
}

/* ---- precision.cpp:95-109 decode_f16 ------------------------------------- */
double mpo_decode_f16(uint16_t bits) {
    const int sign = (bits >> 15) & 1;
    const int ex = (bits >> 10) & 0x1F;
    const int frac = bits & 0x3FF;
    double mag;
    if (ex == 0x1F) {
        if (frac) return NAN;
        mag = INFINITY;
    } else if (ex == 0) {
        mag = ldexp((double)frac, -24);
    } else {
        mag = ldexp((double)(0x400 | frac), ex - 25);
    }
    return sign ? -mag : mag;
}

/* set_linear / at_linear (array.cpp:97-133): round a double to storage p. */
static double round_p(double v, int p) {
    if (p == 0) return mpo_decode_f16(mpo_encode_f16(v));
    if (p == 1) return (double)(float)v;
    return v;
}

/* ---- MPArray::converted (array.cpp:187-191) on raw storage bytes -------- */
static double load_raw(const unsigned char* s, int64_t i, int p) {
    if (p == 0) {
        uint16_t b;
        memcpy(&b, s + 2 * i, 2);
        return mpo_decode_f16(b);
    }
    if (p == 1) {
        float f;
        memcpy(&f, s + 4 * i, 4);
        return (double)f;
    }
    double d;
    memcpy(&d, s + 8 * i, 8);
    return d;
}
static void store_raw(unsigned char* s, int64_t i, int p, double v) {
    if (p == 0) {
        const uint16_t b = mpo_encode_f16(v);
        memcpy(s + 2 * i, &b, 2);
    } else if (p == 1) {
        const float f = (float)v;
        memcpy(s + 4 * i, &f, 4);
    } else {
        memcpy(s + 8 * i, &v, 8);
    }
}
void mpo_convert(int pin, int pout, const void* in, void* out, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
        /* the source MPArray holds set_linear(decoded) state */
        const double v = round_p(load_raw((const unsigned char*)in, i, pin), pin);
        store_raw((unsigned char*)out, i, pout, v);
    }
}

static int promote(int a, int b) { return a >= b ? a : b; }
static int compute_single(int p) { return p != 2; } /* array.hpp:109-111 */

/* ---- linalg::gemm + gemm_kernel (linalg.cpp:316-357, :59-77) ------------ */
int mpo_gemm(int pa, int pb, int pc, int64_t ar, int64_t ac, int64_t br, int64_t bc,
             int64_t cr, int64_t cc, int ta, int tb, double alpha, double beta,
             const double* A, const double* B, double* C) {
    const int64_t m = ta ? ac : ar, k = ta ? ar : ac;
    const int64_t kb = tb ? bc : br, n = tb ? br : bc;
    if (k != kb || cr != m || cc != n) return ST_SHAPE;
    if (pc < promote(pa, pb)) return ST_PREC;
    if (compute_single(pc)) {
        const float al = (float)alpha, be = (float)beta;
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < m; ++i) {
                float acc = 0.0f;
                for (int64_t l = 0; l < k; ++l) {
                    const float x = (float)(ta ? A[i * ar + l] : A[l * ar + i]);
                    const float y = (float)(tb ? B[j + l * br] : B[l + j * br]);
                    acc += x * y;
                }
                const float old = (float)C[j * m + i];
                const float v = al * acc + (be == 0.0f ? 0.0f : be * old);
                C[j * m + i] = round_p((double)v, pc);
            }
    } else {
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < m; ++i) {
                double acc = 0.0;
                for (int64_t l = 0; l < k; ++l) {
                    const double x = ta ? A[i * ar + l] : A[l * ar + i];
                    const double y = tb ? B[j + l * br] : B[l + j * br];
                    acc += x * y;
                }
                const double old = C[j * m + i];
                C[j * m + i] = alpha * acc + (beta == 0.0 ? 0.0 : beta * old);
            }
    }
    return ST_OK;
}

/* ---- crossprod_kernel (linalg.cpp:96-108): out = A^T B, promote(pa,pb) -- */
int mpo_crossprod(int pa, int pb, int64_t m, int64_t na, int64_t mb, int64_t nb,
                  const double* A, const double* B, double* out) {
    if (B == NULL) {
        B = A;
        pb = pa;
        mb = m;
        nb = na;
    }
    if (mb != m) return ST_SHAPE;
    const int po = promote(pa, pb);
    for (int64_t j = 0; j < nb; ++j)
        for (int64_t i = 0; i < na; ++i) {
            if (compute_single(po)) {
                float acc = 0.0f;
                for (int64_t l = 0; l < m; ++l) acc += (float)A[i * m + l] * (float)B[j * m + l];
                out[j * na + i] = round_p((double)acc, po);
            } else {
                double acc = 0.0;
                for (int64_t l = 0; l < m; ++l) acc += A[i * m + l] * B[j * m + l];
                out[j * na + i] = acc;
            }
        }
    return ST_OK;
}

/* ---- chol_kernel (linalg.cpp:110-127): up-looking, reads the upper
 *      triangle, returns upper U with the lower triangle zeroed. ---------- */
int mpo_chol(int p, int64_t n, const double* A, double* U) {
    g_info = -1;
    memcpy(U, A, (size_t)(n * n) * sizeof(double));
    if (compute_single(p)) {
        float* u = (float*)malloc((size_t)(n * n) * sizeof(float));
        if (!u) return ST_NOMEM;
        for (int64_t i = 0; i < n * n; ++i) u[i] = (float)A[i];
        for (int64_t j = 0; j < n; ++j) {
            float* uj = u + j * n;
            for (int64_t i = 0; i < j; ++i) {
                const float* ui = u + i * n;
                float acc = uj[i];
                for (int64_t k = 0; k < i; ++k) acc -= ui[k] * uj[k];
                uj[i] = acc / ui[i];
            }
            float d = uj[j];
            for (int64_t k = 0; k < j; ++k) d -= uj[k] * uj[k];
            if (!(d > 0.0f)) {
                g_info = (int)j;
                free(u);
                return ST_NOT_PD;
            }
            uj[j] = sqrtf(d);
            for (int64_t i = j + 1; i < n; ++i) uj[i] = 0.0f;
        }
        for (int64_t i = 0; i < n * n; ++i) U[i] = round_p((double)u[i], p);
        free(u);
    } else {
        double* u = U;
        for (int64_t j = 0; j < n; ++j) {
            double* uj = u + j * n;
            for (int64_t i = 0; i < j; ++i) {
                const double* ui = u + i * n;
                double acc = uj[i];
                for (int64_t k = 0; k < i; ++k) acc -= ui[k] * uj[k];
                uj[i] = acc / ui[i];
            }
            double d = uj[j];
            for (int64_t k = 0; k < j; ++k) d -= uj[k] * uj[k];
            if (!(d > 0.0)) {
                g_info = (int)j;
                return ST_NOT_PD;
            }
            uj[j] = sqrt(d);
            for (int64_t i = j + 1; i < n; ++i) uj[i] = 0.0;
        }
    }
    return ST_OK;
}

/* ---- tri_solve_kernel (linalg.cpp:130-159), in float or double ---------- */
#define TRI_SOLVE(T)                                                                    \
    static int tri_solve_##T(const T* tri, int64_t n, int upper, int trans, T* b,      \
                             int64_t ncols) {                                           \
        const int eff_lower = (upper == trans);                                         \
        for (int64_t i = 0; i < n; ++i)                                                 \
            if (tri[i * n + i] == (T)0) return ST_SINGULAR;                             \
        for (int64_t c = 0; c < ncols; ++c) {                                           \
            T* x = b + c * n;                                                           \
            if (eff_lower) {                                                            \
                for (int64_t i = 0; i < n; ++i) {                                       \
                    T acc = x[i];                                                       \
                    for (int64_t k = 0; k < i; ++k)                                     \
                        acc -= (trans ? tri[i * n + k] : tri[k * n + i]) * x[k];        \
                    x[i] = acc / tri[i * n + i];                                        \
                }                                                                       \
            } else {                                                                    \
                for (int64_t i = n; i-- > 0;) {                                         \
                    T acc = x[i];                                                       \
                    for (int64_t k = i + 1; k < n; ++k)                                 \
                        acc -= (trans ? tri[i * n + k] : tri[k * n + i]) * x[k];        \
                    x[i] = acc / tri[i * n + i];                                        \
                }                                                                       \
            }                                                                           \
        }                                                                               \
        return ST_OK;                                                                   \
    }
TRI_SOLVE(float)
TRI_SOLVE(double)

/* ---- linalg::trsm (linalg.cpp:498-542): compute in B's precision -------- */
int mpo_trsm(int pa, int pb, int64_t n, int64_t br, int64_t bc, int side_right, int upper,
             int trans, double alpha, const double* A, double* B) {
    (void)pa;
    if (side_right ? bc != n : br != n) return ST_SHAPE;
    const int64_t cnt = br * bc;
    int st;
    if (compute_single(pb)) {
        float* a = (float*)malloc((size_t)(n * n) * sizeof(float));
        float* x = (float*)malloc((size_t)cnt * sizeof(float));
        const float al = (float)alpha;
        for (int64_t i = 0; i < n * n; ++i) a[i] = (float)A[i];
        if (!side_right) {
            for (int64_t i = 0; i < cnt; ++i) x[i] = (float)B[i] * al;
            st = tri_solve_float(a, n, upper, trans, x, bc);
            if (st == ST_OK)
                for (int64_t i = 0; i < cnt; ++i) B[i] = round_p((double)x[i], pb);
        } else {
            for (int64_t j = 0; j < bc; ++j)
                for (int64_t i = 0; i < br; ++i) x[i * bc + j] = (float)B[j * br + i] * al;
            st = tri_solve_float(a, n, upper, !trans, x, br);
            if (st == ST_OK)
                for (int64_t j = 0; j < bc; ++j)
                    for (int64_t i = 0; i < br; ++i) B[j * br + i] = round_p((double)x[i * bc + j], pb);
        }
        free(a);
        free(x);
    } else {
        double* x = (double*)malloc((size_t)cnt * sizeof(double));
        if (!side_right) {
            for (int64_t i = 0; i < cnt; ++i) x[i] = B[i] * alpha;
            st = tri_solve_double(A, n, upper, trans, x, bc);
            if (st == ST_OK) memcpy(B, x, (size_t)cnt * sizeof(double));
        } else {
            for (int64_t j = 0; j < bc; ++j)
                for (int64_t i = 0; i < br; ++i) x[i * bc + j] = B[j * br + i] * alpha;
            st = tri_solve_double(A, n, upper, !trans, x, br);
            if (st == ST_OK)
                for (int64_t j = 0; j < bc; ++j)
                    for (int64_t i = 0; i < br; ++i) B[j * br + i] = x[i * bc + j];
        }
        free(x);
    }
    return st;
}

/* ---- ew_binary / ew_scalar (array.cpp:252-291), reduce (:336-369) ------- */
static float apply_f(int op, float x, float y) {
    return op == 0 ? x + y : op == 1 ? x - y : op == 2 ? x * y : x / y;
}
static double apply_d(int op, double x, double y) {
    return op == 0 ? x + y : op == 1 ? x - y : op == 2 ? x * y : x / y;
}
void mpo_ew_binary(int op, int pa, int pb, int64_t n, const double* A, const double* B,
                   double* out) {
    const int po = promote(pa, pb);
    for (int64_t i = 0; i < n; ++i)
        out[i] = compute_single(po)
                     ? round_p((double)apply_f(op, (float)A[i], (float)B[i]), po)
                     : apply_d(op, A[i], B[i]);
}
void mpo_ew_scalar(int op, int p, int64_t n, const double* A, double s, double* out) {
    const float y = (float)round_p(s, p);
    for (int64_t i = 0; i < n; ++i)
        out[i] = compute_single(p) ? round_p((double)apply_f(op, (float)A[i], y), p)
                                   : apply_d(op, A[i], s);
}
double mpo_reduce(int op, int64_t n, const double* A) {
    if (op == 2 || op == 3) {
        double m = A[0];
        for (int64_t i = 1; i < n; ++i) /* std::min / std::max semantics */
            m = op == 2 ? (A[i] < m ? A[i] : m) : (m < A[i] ? A[i] : m);
        return m;
    }
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += op == 1 ? A[i] * A[i] : A[i];
    return op == 4 ? acc / (double)n : acc;
}

/* ---- Rng (rng.cpp:9-53) -------------------------------------------------- */
static uint64_t splitmix64(uint64_t* x) {
    *x += UINT64_C(0x9E3779B97F4A7C15);
    uint64_t z = *x;
    z = (z ^ (z >> 30)) * UINT64_C(0xBF58476D1CE4E5B9);
    z = (z ^ (z >> 27)) * UINT64_C(0x94D049BB133111EB);
    return z ^ (z >> 31);
}
void mpo_rng_uniform(uint64_t seed, int64_t n, double* out) {
    uint64_t s = seed, st = splitmix64(&s);
    if (st == 0) st = UINT64_C(0x2545F4914F6CDD1D);
    for (int64_t i = 0; i < n; ++i) {
        st ^= st >> 12;
        st ^= st << 25;
        st ^= st >> 27;
        out[i] = (double)((st * UINT64_C(0x2545F4914F6CDD1D)) >> 11) * 0x1p-53;
    }
}

/* ---- MPCRTile right-looking Cholesky (SURVEY.md §8c composition) -------- *
 * tile (i,j) precision prec[j*nt+i]; U_kk = chol(A_kk); A_ik <- trsm(U_kk in
 * p_ik, A_ik, Right, upper); A_ij <- gemm(A_ik->p_ij, A_jk->p_ij, A_ij,
 * {F,T,-1,1}).  Works on a full n x n double copy whose tiles always hold
 * values representable in their tile precision. */
static void tile_get(const double* M, int64_t n, int64_t nb, int64_t ti, int64_t tj,
                     double* t) {
    for (int64_t j = 0; j < nb; ++j)
        memcpy(t + j * nb, M + (tj * nb + j) * n + ti * nb, (size_t)nb * sizeof(double));
}
static void tile_put(double* M, int64_t n, int64_t nb, int64_t ti, int64_t tj,
                     const double* t) {
    for (int64_t j = 0; j < nb; ++j)
        memcpy(M + (tj * nb + j) * n + ti * nb, t + j * nb, (size_t)nb * sizeof(double));
}
static void round_all(double* t, int64_t cnt, int p) {
    for (int64_t i = 0; i < cnt; ++i) t[i] = round_p(t[i], p);
}

int mpo_tile_chol(int64_t n, int64_t nb, const int* prec, const double* A, double* L) {
    g_info = -1;
    if (n % nb) return ST_SHAPE;
    const int64_t nt = n / nb, tt = nb * nb;
    double* u = (double*)malloc((size_t)tt * sizeof(double));
    double* x = (double*)malloc((size_t)tt * sizeof(double));
    double* y = (double*)malloc((size_t)tt * sizeof(double));
    double* c = (double*)malloc((size_t)tt * sizeof(double));
    memcpy(L, A, (size_t)(n * n) * sizeof(double));
    for (int64_t tj = 0; tj < nt; ++tj)
        for (int64_t ti = 0; ti < nt; ++ti) {
            tile_get(L, n, nb, ti, tj, c);
            round_all(c, tt, prec[tj * nt + ti]);
            tile_put(L, n, nb, ti, tj, c);
        }
    int st = ST_OK;
    for (int64_t k = 0; k < nt && st == ST_OK; ++k) {
        const int pk = prec[k * nt + k];
        tile_get(L, n, nb, k, k, c);
        st = mpo_chol(pk, nb, c, u);
        if (st != ST_OK) {
            g_info = (int)(k * nb) + g_info;
            break;
        }
        for (int64_t j = 0; j < nb; ++j) /* L_kk = U_kk^T */
            for (int64_t i = 0; i < nb; ++i) c[j * nb + i] = u[i * nb + j];
        tile_put(L, n, nb, k, k, c);
        for (int64_t i = k + 1; i < nt; ++i) {
            const int pi = prec[k * nt + i];
            memcpy(x, u, (size_t)tt * sizeof(double));
            round_all(x, tt, pi); /* U_kk.converted(p_ik) */
            tile_get(L, n, nb, i, k, y);
            mpo_trsm(pi, pi, nb, nb, nb, 1, 1, 0, 1.0, x, y);
            tile_put(L, n, nb, i, k, y);
        }
        for (int64_t j = k + 1; j < nt; ++j)
            for (int64_t i = j; i < nt; ++i) {
                const int pc = prec[j * nt + i];
                tile_get(L, n, nb, i, k, x);
                round_all(x, tt, pc);
                tile_get(L, n, nb, j, k, y);
                round_all(y, tt, pc);
                tile_get(L, n, nb, i, j, c);
                mpo_gemm(pc, pc, pc, nb, nb, nb, nb, nb, nb, 0, 1, -1.0, 1.0, x, y, c);
                tile_put(L, n, nb, i, j, c);
            }
    }
    if (st == ST_OK) {
        for (int64_t tj = 1; tj < nt; ++tj)
            for (int64_t ti = 0; ti < tj; ++ti) {
                memset(c, 0, (size_t)tt * sizeof(double));
                tile_put(L, n, nb, ti, tj, c);
            }
    }
    free(u);
    free(x);
    free(y);
    free(c);
    return st;
}

/* logdet = 2 sum log L_ii (workloads.cpp:76-80). */
double mpo_logdet_lower(int64_t n, const double* L) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += log(L[i * n + i]);
    return 2.0 * s;
}
