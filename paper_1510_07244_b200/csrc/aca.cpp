// Partially pivoted adaptive cross approximation of many Green matrices,
// host-side, one std::thread per batch slice (clusters are independent).
//
// Restatement of gca.aca (reference pkg/src/gcabem/gca.py:182-245) with the
// same pivot rules: the next row is the largest-magnitude entry of the
// current residual column among unused rows, the next column the largest
// entry of the residual row (ties to the lowest index); stop when
// |u_k| |v_k| <= eps * sqrt(Frobenius estimate) or at the rank cap; a zero
// residual row falls through to the lowest unused row. Elementwise updates
// use the reference's operation order (r -= u_i * v), magnitudes are fabs /
// hypot as numpy's abs, complex division follows numpy's Smith scheme.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <thread>
#include <type_traits>
#include <vector>

#include "gcabem_b200.h"
#include "green_exact.h"
#include "internal.h"

// Compiled twice: as is (baseline x86-64) and from aca_avx2.cpp with -mavx2
// (GCABEM_ACA_AVX2); the baseline unit dispatches at run time. Both builds
// perform the same IEEE operations in the same order (no FMA contraction),
// so results do not depend on the CPU.
#ifdef GCABEM_ACA_AVX2
#include <immintrin.h>
#define GCABEM_ACA_NS aca_avx2
#else
#define GCABEM_ACA_NS aca_base
#endif

namespace GCABEM_ACA_NS {

struct Cx {
    double re, im;
};

inline Cx cmul(Cx a, Cx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
inline Cx csub(Cx a, Cx b) { return {a.re - b.re, a.im - b.im}; }
// numpy CDOUBLE_divide (Smith)
inline Cx cdiv(Cx a, Cx b) {
    const double br = std::fabs(b.re), bi = std::fabs(b.im);
    if (br >= bi) {
        const double rat = b.im / b.re, scl = 1.0 / (b.re + b.im * rat);
        return {(a.re + a.im * rat) * scl, (a.im - a.re * rat) * scl};
    }
    const double rat = b.re / b.im, scl = 1.0 / (b.im + b.re * rat);
    return {(a.re * rat + a.im) * scl, (a.im * rat - a.re) * scl};
}
inline double cabs(Cx a) { return std::hypot(a.re, a.im); }

// Division of many numerators by one divisor: the divisor's part of Smith's
// scheme (branch, rat, scl) once, then per element exactly the operations of
// cdiv(a, b) -- bitwise the per-element division without its two divides.
struct CDivisor {
    bool re_major;
    double rat, scl;
    explicit CDivisor(Cx b) : re_major(std::fabs(b.re) >= std::fabs(b.im)) {
        if (re_major) {
            rat = b.im / b.re;
            scl = 1.0 / (b.re + b.im * rat);
        } else {
            rat = b.re / b.im;
            scl = 1.0 / (b.im + b.re * rat);
        }
    }
    Cx operator()(Cx a) const {
        if (re_major) return {(a.re + a.im * rat) * scl, (a.im - a.re * rat) * scl};
        return {(a.re * rat + a.im) * scl, (a.im * rat - a.re) * scl};
    }
};

template <typename T>
struct Ops;
template <>
struct Ops<double> {
    static double mag(double x) { return std::fabs(x); }
    static double mul(double a, double b) { return a * b; }
    static double sub(double a, double b) { return a - b; }
    static double div(double a, double b) { return a / b; }
    struct Divider {  // real division stays a division (a * (1/b) would round differently)
        double b;
        explicit Divider(double d) : b(d) {}
        double operator()(double a) const { return a / b; }
    };
    static bool zero(double a) { return a == 0.0; }
    static double norm2(double a) { return a * a; }
    static double dotc_re(double a, double b) { return a * b; }  // Re(conj(a) b)
    static double dotc_im(double, double) { return 0.0; }
};
template <>
struct Ops<Cx> {
    static double mag(Cx x) { return cabs(x); }
    static Cx mul(Cx a, Cx b) { return cmul(a, b); }
    static Cx sub(Cx a, Cx b) { return csub(a, b); }
    static Cx div(Cx a, Cx b) { return cdiv(a, b); }
    using Divider = CDivisor;
    static bool zero(Cx a) { return a.re == 0.0 && a.im == 0.0; }
    static double norm2(Cx a) { return a.re * a.re + a.im * a.im; }
    static double dotc_re(Cx a, Cx b) { return a.re * b.re + a.im * b.im; }
    static double dotc_im(Cx a, Cx b) { return a.re * b.im - a.im * b.re; }
};

// sum conj(a_k) b_k over the arrays as doubles, 4 at a time into two 4-lane
// accumulators (alternating) for the products x_e y_e (real part) and
// x_e y_(e^1) (imaginary part: lanes re*im minus im*re), combined in a fixed
// order at the end. The AVX2 build does exactly these IEEE operations with
// vector instructions (no FMA), so both builds agree bitwise. (The
// reference's np.vdot / norm are BLAS reductions with their own association:
// these sums only feed the stopping estimate, see aca_one.)
template <typename T>
Cx dotc(const T *a, const T *b, int64_t n) {
    constexpr int W = std::is_same<T, Cx>::value ? 2 : 1;
    const double *x = reinterpret_cast<const double *>(a);
    const double *y = reinterpret_cast<const double *>(b);
    const int64_t nd = n * W, nv = nd / 4;
    double tr = 0.0, ti = 0.0;
    for (int64_t e = nv * 4; e < nd; e += W) {  // tail: < 4 doubles
        tr += x[e] * y[e];
        if (W == 2) {
            tr += x[e + 1] * y[e + 1];
            ti += x[e] * y[e + 1] - x[e + 1] * y[e];
        }
    }
#ifdef GCABEM_ACA_AVX2
    __m256d r0 = _mm256_setzero_pd(), r1 = r0, i0 = r0, i1 = r0;
    int64_t v = 0;
    for (; v + 2 <= nv; v += 2) {
        const __m256d xa = _mm256_loadu_pd(x + 4 * v), ya = _mm256_loadu_pd(y + 4 * v);
        const __m256d xb = _mm256_loadu_pd(x + 4 * v + 4), yb = _mm256_loadu_pd(y + 4 * v + 4);
        r0 = _mm256_add_pd(r0, _mm256_mul_pd(xa, ya));
        r1 = _mm256_add_pd(r1, _mm256_mul_pd(xb, yb));
        if (W == 2) {
            i0 = _mm256_add_pd(i0, _mm256_mul_pd(xa, _mm256_permute_pd(ya, 0x5)));
            i1 = _mm256_add_pd(i1, _mm256_mul_pd(xb, _mm256_permute_pd(yb, 0x5)));
        }
    }
    if (v < nv) {
        const __m256d xa = _mm256_loadu_pd(x + 4 * v), ya = _mm256_loadu_pd(y + 4 * v);
        r0 = _mm256_add_pd(r0, _mm256_mul_pd(xa, ya));
        if (W == 2) i0 = _mm256_add_pd(i0, _mm256_mul_pd(xa, _mm256_permute_pd(ya, 0x5)));
    }
    alignas(32) double R[2][4], I[2][4];
    _mm256_store_pd(R[0], r0);
    _mm256_store_pd(R[1], r1);
    _mm256_store_pd(I[0], i0);
    _mm256_store_pd(I[1], i1);
#else
    double R[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}}, I[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
    for (int64_t v = 0; v < nv; ++v) {
        const double *xv = x + 4 * v, *yv = y + 4 * v;
        double *rr = R[v & 1], *ii = I[v & 1];
        for (int l = 0; l < 4; ++l) {
            rr[l] += xv[l] * yv[l];
            if (W == 2) ii[l] += xv[l] * yv[l ^ 1];
        }
    }
#endif
    const double re = ((R[0][0] + R[0][1]) + (R[0][2] + R[0][3])) +
                      ((R[1][0] + R[1][1]) + (R[1][2] + R[1][3])) + tr;
    const double im = W == 2 ? ((I[0][0] - I[0][1]) + (I[0][2] - I[0][3])) +
                                   ((I[1][0] - I[1][1]) + (I[1][2] - I[1][3])) + ti
                             : 0.0;
    return {re, im};
}

// x[j] -= s * y[j] (the residual updates and the LU sweeps); the compiler
// vectorises it in the AVX2 build (hand-written intrinsics measured no faster
// on the B200 host)
template <typename T>
inline void mulsub(T *x, T s, const T *y, int64_t n) {
    using O = Ops<T>;
    for (int64_t j = 0; j < n; ++j) x[j] = O::sub(x[j], O::mul(s, y[j]));
}

constexpr int64_t SOLVE_CHUNK = 64;  // right-hand sides per cache-resident pass
constexpr int64_t ACA_TILE = 512;    // column entries per L1-resident update pass

// x[q] <- (...((x[q] - s[0] y_0[q]) - s[1] y_1[q]) ...) - s[cnt-1] y_(cnt-1)[q]
// with y_m = y + m * ys: the updates of cnt mulsub calls in the same order,
// with x held in registers across them (one load and store of x per element
// instead of one per update). Every element sees exactly mulsub's operations,
// so the result is bitwise that of the mulsub sequence in both builds.
template <typename T>
void mulsub_rows(T *x, int64_t n, const T *s, int64_t cnt, const T *y, int64_t ys) {
    using O = Ops<T>;
    int64_t q = 0;
#ifdef GCABEM_ACA_AVX2
    if constexpr (std::is_same<T, Cx>::value) {
        // 2 complex per register: s y = addsub(re(s) y, im(s) swap(y))
        auto step = [](__m256d a, __m256d sr, __m256d si, const double *yp) {
            const __m256d yv = _mm256_loadu_pd(yp);
            const __m256d p = _mm256_addsub_pd(_mm256_mul_pd(sr, yv),
                                               _mm256_mul_pd(si, _mm256_permute_pd(yv, 0x5)));
            return _mm256_sub_pd(a, p);
        };
        for (; q + 8 <= n; q += 8) {
            double *xp = reinterpret_cast<double *>(x + q);
            __m256d a0 = _mm256_loadu_pd(xp), a1 = _mm256_loadu_pd(xp + 4);
            __m256d a2 = _mm256_loadu_pd(xp + 8), a3 = _mm256_loadu_pd(xp + 12);
            for (int64_t m = 0; m < cnt; ++m) {
                const __m256d sr = _mm256_broadcast_sd(&s[m].re);
                const __m256d si = _mm256_broadcast_sd(&s[m].im);
                const double *yp = reinterpret_cast<const double *>(y + m * ys + q);
                a0 = step(a0, sr, si, yp);
                a1 = step(a1, sr, si, yp + 4);
                a2 = step(a2, sr, si, yp + 8);
                a3 = step(a3, sr, si, yp + 12);
            }
            _mm256_storeu_pd(xp, a0);
            _mm256_storeu_pd(xp + 4, a1);
            _mm256_storeu_pd(xp + 8, a2);
            _mm256_storeu_pd(xp + 12, a3);
        }
        for (; q + 2 <= n; q += 2) {
            double *xp = reinterpret_cast<double *>(x + q);
            __m256d a0 = _mm256_loadu_pd(xp);
            for (int64_t m = 0; m < cnt; ++m)
                a0 = step(a0, _mm256_broadcast_sd(&s[m].re), _mm256_broadcast_sd(&s[m].im),
                          reinterpret_cast<const double *>(y + m * ys + q));
            _mm256_storeu_pd(xp, a0);
        }
    } else {
        for (; q + 16 <= n; q += 16) {
            double *xp = reinterpret_cast<double *>(x + q);
            __m256d a0 = _mm256_loadu_pd(xp), a1 = _mm256_loadu_pd(xp + 4);
            __m256d a2 = _mm256_loadu_pd(xp + 8), a3 = _mm256_loadu_pd(xp + 12);
            for (int64_t m = 0; m < cnt; ++m) {
                const __m256d sv = _mm256_broadcast_sd(reinterpret_cast<const double *>(s + m));
                const double *yp = reinterpret_cast<const double *>(y + m * ys + q);
                a0 = _mm256_sub_pd(a0, _mm256_mul_pd(sv, _mm256_loadu_pd(yp)));
                a1 = _mm256_sub_pd(a1, _mm256_mul_pd(sv, _mm256_loadu_pd(yp + 4)));
                a2 = _mm256_sub_pd(a2, _mm256_mul_pd(sv, _mm256_loadu_pd(yp + 8)));
                a3 = _mm256_sub_pd(a3, _mm256_mul_pd(sv, _mm256_loadu_pd(yp + 12)));
            }
            _mm256_storeu_pd(xp, a0);
            _mm256_storeu_pd(xp + 4, a1);
            _mm256_storeu_pd(xp + 8, a2);
            _mm256_storeu_pd(xp + 12, a3);
        }
    }
#endif
    for (; q < n; ++q) {
        T acc = x[q];
        for (int64_t m = 0; m < cnt; ++m) acc = O::sub(acc, O::mul(s[m], y[m * ys + q]));
        x[q] = acc;
    }
}

// np.argmax(np.abs(x)) with masked entries read as 0.0 (first index wins
// ties). Complex magnitudes are hypot as numpy's; a squared-magnitude pass
// first narrows the candidates to those within 1e-12 of the maximum, so
// hypot runs on a handful of entries (the squares carry < 4 ulp error, far
// inside that window).
template <typename T>
int64_t argmax_mag(const T *x, int64_t n, const char *mask, double *best_out) {
    using O = Ops<T>;
    int64_t jp = 0;
    double best = -1.0;
    if constexpr (std::is_same<T, Cx>::value) {
        double smax = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            const double s = (mask && mask[j]) ? 0.0 : O::norm2(x[j]);
            smax = std::max(smax, s);
        }
        const double thr = smax > 1e-290 ? smax * (1.0 - 1e-12) : 0.0;
        for (int64_t j = 0; j < n; ++j) {
            if (mask && mask[j]) {
                if (0.0 > best) {
                    best = 0.0;
                    jp = j;
                }
                continue;
            }
            if (thr > 0.0 && O::norm2(x[j]) < thr) continue;
            const double a = O::mag(x[j]);
            if (a > best) {
                best = a;
                jp = j;
            }
        }
        if (thr > 0.0 && best < 0.0) best = 0.0;
    } else {
        for (int64_t j = 0; j < n; ++j) {
            const double a = (mask && mask[j]) ? 0.0 : O::mag(x[j]);
            if (a > best) {
                best = a;
                jp = j;
            }
        }
    }
    if (best_out) *best_out = best;
    return jp;
}

// Tie window of the ACA decisions. The Green matrix this ACA sees is the
// device's, within a few ulps of the reference's numpy evaluation; a
// decision whose margin is below these bounds could go the other way on the
// reference's bits (exact ties from the sphere's symmetry are the common
// case), so it marks the cluster ambiguous (the caller redoes it on the
// reference's exact arithmetic). Relative to the winning magnitude, and
// absolute relative to the largest entry of the original row/column (the
// residual's rounding scale).
constexpr double TIE_REL = 1e-10;
constexpr double TIE_ABS = 1e-12;
constexpr double STOP_REL = 1e-8;

// another unmasked entry of |x| within delta of best (index jp excluded)?
template <typename T>
bool near_tie(const T *x, int64_t n, const char *mask, int64_t jp, double best, double delta) {
    using O = Ops<T>;
    const double lo = best - delta;
    if (lo <= 0.0) return true;
    const double lo2 = lo * lo * (1.0 - 1e-12);  // squares carry < 4 ulp error
    for (int64_t j = 0; j < n; ++j) {
        if (j == jp || (mask && mask[j])) continue;
        if (O::norm2(x[j]) >= lo2 && O::mag(x[j]) >= lo) return true;
    }
    return false;
}

template <typename T>
double max_mag(const T *x, int64_t n, int64_t stride) {
    using O = Ops<T>;
    double m2 = 0.0;
    for (int64_t j = 0; j < n; ++j) m2 = std::max(m2, O::norm2(x[j * stride]));
    return std::sqrt(m2);
}

// Row / column access of the matrix the ACA works on: a dense row-major
// matrix, or entries evaluated on demand (GreenExact, the tie redo path).
template <typename T>
struct DenseSrc {
    const T *A;
    int64_t nr, nc;
    void row(int64_t i, T *out) const { std::copy(A + i * nc, A + i * nc + nc, out); }
    void col(int64_t j, T *out) const {
        for (int64_t q = 0; q < nr; ++q) out[q] = A[q * nc + j];
    }
};

template <typename T, typename Src>
void aca_core(const Src &src, int64_t nr, int64_t nc, double eps, int64_t cap, int64_t *rows,
              int64_t *cols, int64_t *rank, double *resid, int *ambiguous = nullptr,
              std::vector<T> *orig_cols = nullptr) {
    if (orig_cols) orig_cols->clear();
    using O = Ops<T>;
    bool amb = false;
    std::vector<std::vector<T>> U, W;
    std::vector<char> used(nr, 0);
    std::vector<T> r(nc), c(nr);
    int64_t k = 0, next = 0;
    double est2 = 0.0, res = 0.0;
    while (k < cap) {
        if (next >= nr || used[next]) {
            int64_t f = -1;
            for (int64_t q = 0; q < nr; ++q)
                if (!used[q]) {
                    f = q;
                    break;
                }
            if (f < 0) break;
            next = f;
        }
        const int64_t i = next;
        src.row(i, r.data());
        const double rscale = ambiguous && !amb ? max_mag<T>(r.data(), nc, 1) : 0.0;
        for (size_t m = 0; m < U.size(); ++m) {
            const T ui = U[m][i];
            mulsub<T>(r.data(), ui, W[m].data(), nc);
        }
        double rbest = 0.0;
        const int64_t jp = argmax_mag<T>(r.data(), nc, nullptr, &rbest);
        if (ambiguous && !amb)
            amb = rbest <= TIE_ABS * rscale ||
                  near_tie<T>(r.data(), nc, nullptr, jp, rbest,
                              std::max(TIE_REL * rbest, TIE_ABS * rscale));
        used[i] = 1;
        if (O::zero(r[jp])) {
            next = nr;
            continue;
        }
        std::vector<T> w(nc);
        const T piv = r[jp];
        const typename O::Divider by_piv(piv);
        for (int64_t j = 0; j < nc; ++j) w[j] = by_piv(r[j]);
        src.col(jp, c.data());
        if (orig_cols) orig_cols->insert(orig_cols->end(), c.begin(), c.end());
        const double cscale = ambiguous && !amb ? max_mag<T>(c.data(), nr, 1) : 0.0;
        for (size_t m = 0; m < U.size(); ++m) {
            const T wj = W[m][jp];
            mulsub<T>(c.data(), wj, U[m].data(), nr);
        }
        // norms and the cross terms of the Frobenius estimate: four partial
        // sums (vectorisable; the reference's np.linalg.norm / np.vdot are
        // BLAS reductions with their own association, so no order is "the"
        // reference order here -- only the elementwise residual updates
        // above decide pivots and follow the reference exactly; a stopping
        // test within STOP_REL of its bound is flagged)
        const double nu = std::sqrt(dotc<T>(c.data(), c.data(), nr).re);
        const double nw = std::sqrt(dotc<T>(w.data(), w.data(), nc).re);
        double cross = 0.0;
        for (size_t m = 0; m < U.size(); ++m) {
            const Cx a = dotc<T>(U[m].data(), c.data(), nr);
            const Cx b = dotc<T>(W[m].data(), w.data(), nc);
            cross += a.re * b.re - a.im * b.im;  // Re((u^H c) (w_m^H w))
        }
        U.emplace_back(c.begin(), c.end());
        W.emplace_back(std::move(w));
        rows[k] = i;
        cols[k] = jp;
        ++k;
        est2 = std::max(est2 + nu * nu * nw * nw + 2.0 * cross, 0.0);
        res = nu * nw;
        const double bound = eps * std::sqrt(est2);
        if (ambiguous && !amb) amb = std::fabs(res - bound) <= STOP_REL * bound;
        if (res <= bound) break;
        double mb = 0.0;
        const int64_t nb = argmax_mag<T>(c.data(), nr, used.data(), &mb);
        if (ambiguous && !amb && k < cap)
            amb = mb <= TIE_ABS * cscale ||
                  near_tie<T>(c.data(), nr, used.data(), nb, mb,
                              std::max(TIE_REL * mb, TIE_ABS * cscale));
        next = mb == 0.0 ? nr : nb;
    }
    *rank = k;
    *resid = res;
    if (ambiguous) *ambiguous = amb ? 1 : 0;
}

template <typename T>
void aca_one(const T *A, int64_t nr, int64_t nc, double eps, int64_t cap, int64_t *rows,
             int64_t *cols, int64_t *rank, double *resid, int *ambiguous = nullptr,
             std::vector<T> *orig_cols = nullptr) {
    aca_core<T>(DenseSrc<T>{A, nr, nc}, nr, nc, eps, cap, rows, cols, rank, resid, ambiguous,
                orig_cols);
}

// ---------------------------------------------------------------------------
// GCA operator of one cluster (reference gca.py:248-282): pivot-block
// condition check (np.linalg.cond, 2-norm), V = A[:, cols] inv(B) by LU with
// partial pivoting of B^T (numpy solve = LAPACK gesv on B^T, pivot choice by
// |re| + |im| as izamax), two refinement sweeps with the reference's early
// exit. V parity is within roundoff x cond(B) of LAPACK, not bitwise.

inline Cx cadd(Cx a, Cx b) { return {a.re + b.re, a.im + b.im}; }
inline double abs1(double x) { return std::fabs(x); }
inline double abs1(Cx x) { return std::fabs(x.re) + std::fabs(x.im); }
inline double add_(double a, double b) { return a + b; }
inline Cx add_(Cx a, Cx b) { return cadd(a, b); }
template <typename T>
T one();
template <>
double one<double>() { return 1.0; }
template <>
Cx one<Cx>() { return Cx{1.0, 0.0}; }

// 2-norm condition number by one-sided (Hestenes) Jacobi SVD of the r x r
// row-major block: rotate column pairs until mutually orthogonal; the
// singular values are the final column norms (relative accuracy).
template <typename T>
double cond2(const T *B, int64_t r) {
    using O = Ops<T>;
    // column-major copy
    std::vector<T> a((size_t)(r * r));
    for (int64_t i = 0; i < r; ++i)
        for (int64_t j = 0; j < r; ++j) a[(size_t)(j * r + i)] = B[i * r + j];
    // rounding in the pair inner products is ~eps sqrt(r) relative: a
    // tighter stop would never be met
    const double tol = 4.0 * 2.220446049250313e-16 * (double)std::max<int64_t>(r, 4);
    for (int sweep = 0; sweep < 40; ++sweep) {
        bool rotated = false;
        for (int64_t p = 0; p < r - 1; ++p) {
            T *ap = a.data() + p * r;
            for (int64_t q = p + 1; q < r; ++q) {
                T *aq = a.data() + q * r;
                double alpha = 0.0, beta = 0.0, gr = 0.0, gi = 0.0;
                for (int64_t i = 0; i < r; ++i) {
                    alpha += O::norm2(ap[i]);
                    beta += O::norm2(aq[i]);
                    gr += O::dotc_re(ap[i], aq[i]);
                    gi += O::dotc_im(ap[i], aq[i]);
                }
                const double g = std::hypot(gr, gi);
                if (g == 0.0 || g <= tol * std::sqrt(alpha * beta)) continue;
                rotated = true;
                // a_q <- e^{-i phi} a_q makes the pair's inner product real
                // (= g); then a real rotation zeroes it.
                const double zeta = (beta - alpha) / (2.0 * g);
                const double t = (zeta >= 0.0 ? 1.0 : -1.0) /
                                 (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
                const double pr = gr / g, pi = gi / g;  // e^{i phi}
                for (int64_t i = 0; i < r; ++i) {
                    T x = ap[i], y = aq[i];
                    if constexpr (std::is_same<T, Cx>::value) {
                        y = Cx{y.re * pr + y.im * pi, y.im * pr - y.re * pi};  // e^{-i phi} y
                        ap[i] = Cx{c * x.re - s * y.re, c * x.im - s * y.im};
                        aq[i] = Cx{s * x.re + c * y.re, s * x.im + c * y.im};
                    } else {
                        y = y * pr;
                        ap[i] = c * x - s * y;
                        aq[i] = s * x + c * y;
                    }
                }
            }
        }
        if (!rotated) break;
    }
    double smax = 0.0, smin = HUGE_VAL;
    for (int64_t j = 0; j < r; ++j) {
        double n2 = 0.0;
        for (int64_t i = 0; i < r; ++i) n2 += O::norm2(a[(size_t)(j * r + i)]);
        const double sv = std::sqrt(n2);
        smax = std::max(smax, sv);
        smin = std::min(smin, sv);
    }
    return smin > 0.0 ? smax / smin : HUGE_VAL;
}

// LU with partial pivoting of M (r x r, row-major) and multi-RHS solves on
// row-major (r x n) right-hand sides (inner loops run along n: contiguous).

template <typename T>
struct LU {
    int64_t r = 0;
    std::vector<T> m;
    std::vector<int64_t> piv;
    bool factor(const T *M, int64_t n) {
        using O = Ops<T>;
        r = n;
        m.assign(M, M + n * n);
        piv.resize(n);
        for (int64_t k = 0; k < n; ++k) {
            int64_t p = k;
            double best = abs1(m[k * n + k]);
            for (int64_t i = k + 1; i < n; ++i) {
                const double v = abs1(m[i * n + k]);
                if (v > best) {
                    best = v;
                    p = i;
                }
            }
            piv[k] = p;
            if (best == 0.0) return false;
            if (p != k)
                for (int64_t j = 0; j < n; ++j) std::swap(m[k * n + j], m[p * n + j]);
            const typename O::Divider by_d(m[k * n + k]);
            for (int64_t i = k + 1; i < n; ++i) {
                const T l = by_d(m[i * n + k]);
                m[i * n + k] = l;
                for (int64_t j = k + 1; j < n; ++j)
                    m[i * n + j] = O::sub(m[i * n + j], O::mul(l, m[k * n + j]));
            }
        }
        return true;
    }
    // X (r x n, row-major) <- M^-1 X
    void solve(T *X, int64_t n) const {
        for (int64_t q0 = 0; q0 < n; q0 += SOLVE_CHUNK)
            solve_cols(X, n, q0, std::min(SOLVE_CHUNK, n - q0));
    }
    // columns [q0, q0 + nq) of X (row stride ld): every column is an
    // independent right-hand side, so a chunk small enough to stay in L1/L2
    // performs exactly the per-column operations of the whole solve
    void solve_cols(T *X, int64_t ld, int64_t q0, int64_t nq) const {
        using O = Ops<T>;
        X += q0;
        for (int64_t k = 0; k < r; ++k)
            if (piv[k] != k)
                for (int64_t q = 0; q < nq; ++q) std::swap(X[k * ld + q], X[piv[k] * ld + q]);
        for (int64_t i = 1; i < r; ++i) mulsub_rows<T>(X + i * ld, nq, &m[i * r], i, X, ld);
        for (int64_t i = r - 1; i >= 0; --i) {
            T *xi = X + i * ld;
            mulsub_rows<T>(xi, nq, &m[i * r + i + 1], r - 1 - i, X + (i + 1) * ld, ld);
            const typename O::Divider by_d(m[i * r + i]);
            for (int64_t q = 0; q < nq; ++q) xi[q] = by_d(xi[q]);
        }
    }
};

// np.linalg.cond(B) <= 1e14 (2-norm), decided from the Frobenius condition
// kF = |B|_F |B^-1|_F, which brackets it: kF / r <= cond2 <= kF. Only in
// the ambiguous window does the exact Jacobi SVD run.
template <typename T>
bool cond_ok(const T *B, const LU<T> &luT, int64_t r) {
    using O = Ops<T>;
    std::vector<T> Y((size_t)(r * r), T());
    for (int64_t i = 0; i < r; ++i) Y[i * r + i] = O::div(one<T>(), one<T>());
    luT.solve(Y.data(), r);  // (B^T)^-1, same Frobenius norm as B^-1
    double fb = 0.0, fi = 0.0;
    for (int64_t e = 0; e < r * r; ++e) {
        fb += O::norm2(B[e]);
        fi += O::norm2(Y[e]);
    }
    const double kf = std::sqrt(fb) * std::sqrt(fi);
    if (!(kf == kf)) return false;
    if (kf <= 0.5e14) return true;
    if (kf >= 2e14 * (double)r) return false;
    return cond2<T>(B, r) <= 1e14;
}

// V = A[:, cols] B^-1 for ACA pivots (rows, rank k) given the pivot columns
// Acol[b * nr + q] = A[q, cols[b]]: 0, or 2 when the pivot block is singular
// or its condition number is above 1e14
template <typename T>
int solve_one(const T *Acol, int64_t nr, int64_t k, const int64_t *rows,
              std::vector<int64_t> &rows_out, std::vector<double> &V_out) {
    using O = Ops<T>;
    // pivot block B[a][b] = A[rows[a], cols[b]], and M = B^T
    std::vector<T> B((size_t)(k * k)), M((size_t)(k * k));
    for (int64_t a = 0; a < k; ++a)
        for (int64_t b = 0; b < k; ++b) {
            B[a * k + b] = Acol[b * nr + rows[a]];
            M[b * k + a] = B[a * k + b];
        }
    LU<T> lu;
    if (!lu.factor(M.data(), k)) return 2;  // exactly singular: cond = inf
    if (!cond_ok<T>(B.data(), lu, k)) return 2;
    // X = V^T (k x nr) solves M X = A_cols^T, in chunks of SOLVE_CHUNK
    // columns stored chunk-major (chunk c, row b at (c k + b) SOLVE_CHUNK):
    // every chunk is a contiguous, cache-resident block, and each column
    // sees the operations of whole-matrix passes (columns are independent)
    constexpr int64_t QB = SOLVE_CHUNK;
    const int64_t nch = (nr + QB - 1) / QB;
    std::vector<T> RHS((size_t)(nch * k * QB)), X((size_t)(nch * k * QB)),
        R((size_t)(k * QB));
    double amax = 0.0;
    for (int64_t b = 0; b < k; ++b)
        for (int64_t q = 0; q < nr; ++q) {
            const T v = Acol[b * nr + q];
            RHS[((q / QB) * k + b) * QB + q % QB] = v;
            amax = std::max(amax, O::mag(v));
        }
    X = RHS;
    const double lim = 1e-15 * std::max(amax, 1.0);
    // R = RHS - M X on one chunk (R^T = A_cols^T - B^T V^T), its max |.|
    auto residual = [&](int64_t ch, int64_t nq) {
        const T *xc = X.data() + ch * k * QB, *hc = RHS.data() + ch * k * QB;
        double rmax = 0.0;
        for (int64_t b = 0; b < k; ++b) {
            T *rb = R.data() + b * QB;
            std::copy(hc + b * QB, hc + b * QB + nq, rb);
            mulsub_rows<T>(rb, nq, &M[b * k], k, xc, QB);
            for (int64_t q = 0; q < nq; ++q) rmax = std::max(rmax, O::mag(rb[q]));
        }
        return rmax;
    };
    std::vector<double> chmax((size_t)nch);
    double rmax = 0.0;
    for (int64_t ch = 0; ch < nch; ++ch) {
        const int64_t nq = std::min(QB, nr - ch * QB);
        lu.solve_cols(X.data() + ch * k * QB, QB, 0, nq);
        rmax = std::max(rmax, residual(ch, nq));
    }
    for (int sweep = 0; sweep < 2 && rmax > lim; ++sweep) {
        // X += M^-1 (RHS - M X), then (first sweep only) the new residual
        const bool last = sweep == 1;
        rmax = 0.0;
        for (int64_t ch = 0; ch < nch; ++ch) {
            const int64_t nq = std::min(QB, nr - ch * QB);
            residual(ch, nq);
            lu.solve_cols(R.data(), QB, 0, nq);
            T *xc = X.data() + ch * k * QB;
            for (int64_t b = 0; b < k; ++b)
                for (int64_t q = 0; q < nq; ++q)
                    xc[b * QB + q] = add_(xc[b * QB + q], R[b * QB + q]);
            if (!last) rmax = std::max(rmax, residual(ch, nq));
        }
    }
    rows_out.assign(rows, rows + k);
    const int w = std::is_same<T, Cx>::value ? 2 : 1;
    V_out.resize((size_t)(nr * k * w));
    T *V = reinterpret_cast<T *>(V_out.data());
    for (int64_t ch = 0; ch < nch; ++ch) {
        const int64_t q0 = ch * QB, nq = std::min(QB, nr - q0);
        const T *xc = X.data() + ch * k * QB;
        for (int64_t q = 0; q < nq; ++q)
            for (int64_t b = 0; b < k; ++b) V[(q0 + q) * k + b] = xc[b * QB + q];
    }
    return 0;
}

// The whole operator: ACA at eps (or the given first-attempt pivots), the
// solve, and one retry at eps / 10 when the pivot block is rejected
template <typename T>
int operator_one(const T *A, int64_t nr, int64_t nc, double eps, std::vector<int64_t> &rows_out,
                 std::vector<double> &V_out, int *ambiguous = nullptr) {
    const int64_t cap = std::min(nr, nc);
    std::vector<int64_t> rows(cap), cols(cap);
    std::vector<T> acol;  // the pivot columns A[:, cols[b]] the ACA fetched
    for (int attempt = 0; attempt < 2; ++attempt, eps *= 0.1) {
        int64_t k = 0;
        const int64_t *r = rows.data();
        double resid = 0.0;
        int amb = 0;
        aca_one<T>(A, nr, nc, eps, cap, rows.data(), cols.data(), &k, &resid,
                   ambiguous ? &amb : nullptr, &acol);
        if (ambiguous && amb) *ambiguous = 1;
        if (k == 0) return 1;
        if (solve_one<T>(acol.data(), nr, k, r, rows_out, V_out) == 0) return 0;
    }
    return 2;
}

// On-demand exact entries (GreenExact); columns are kept for the solve
template <typename T>
struct ExactSrc {
    const gcabem::GreenExact *g;
    int64_t nr, nc;
    mutable std::vector<std::vector<T>> cols;  // by column index, filled on demand
    static T make(double re, double im) {
        if constexpr (std::is_same<T, Cx>::value)
            return Cx{re, im};
        else
            return re;
    }
    void row(int64_t i, T *out) const {
        for (int64_t j = 0; j < nc; ++j) {
            double re, im;
            g->entry(i, j, re, im);
            out[j] = make(re, im);
        }
    }
    const std::vector<T> &column(int64_t j) const {
        if (cols.empty()) cols.resize(nc);
        std::vector<T> &c = cols[j];
        if (c.empty()) {
            c.resize(nr);
            for (int64_t q = 0; q < nr; ++q) {
                double re, im;
                g->entry(q, j, re, im);
                c[q] = make(re, im);
            }
        }
        return c;
    }
    void col(int64_t j, T *out) const {
        const std::vector<T> &c = column(j);
        std::copy(c.begin(), c.end(), out);
    }
};

template <typename T>
int operator_exact(const gcabem::GreenExact &g, double eps, std::vector<int64_t> &rows_out,
                   std::vector<double> &V_out) {
    const int64_t nr = g.nr, nc = g.nsrc(), cap = std::min(nr, nc);
    ExactSrc<T> src{&g, nr, nc, {}};
    std::vector<int64_t> rows(cap), cols(cap);
    std::vector<T> acol;
    for (int attempt = 0; attempt < 2; ++attempt, eps *= 0.1) {
        int64_t k = 0;
        double resid = 0.0;
        aca_core<T>(src, nr, nc, eps, cap, rows.data(), cols.data(), &k, &resid, nullptr,
                    &acol);
        if (k == 0) return 1;
        if (solve_one<T>(acol.data(), nr, k, rows.data(), rows_out, V_out) == 0) return 0;
    }
    return 2;
}

// entry points of this build
int exact_entry(bool is_complex, const gcabem::GreenExact &g, double epsilon,
                std::vector<int64_t> &rows, std::vector<double> &V) {
    return is_complex ? operator_exact<Cx>(g, epsilon, rows, V)
                      : operator_exact<double>(g, epsilon, rows, V);
}

void aca_entry(bool is_complex, const double *A, int64_t nr, int64_t nc, double eps, int64_t cap,
               int64_t *rows, int64_t *cols, int64_t *rank, double *resid) {
    if (is_complex)
        aca_one<Cx>(reinterpret_cast<const Cx *>(A), nr, nc, eps, cap, rows, cols, rank, resid);
    else
        aca_one<double>(A, nr, nc, eps, cap, rows, cols, rank, resid);
}

int operator_entry(bool is_complex, const double *A, int64_t nr, int64_t nc, double epsilon,
                   std::vector<int64_t> &rows, std::vector<double> &V, int *ambiguous) {
    if (is_complex)
        return operator_one<Cx>(reinterpret_cast<const Cx *>(A), nr, nc, epsilon, rows, V,
                                ambiguous);
    return operator_one<double>(A, nr, nc, epsilon, rows, V, ambiguous);
}

}  // namespace GCABEM_ACA_NS

#ifndef GCABEM_ACA_AVX2
namespace aca_avx2 {
void aca_entry(bool is_complex, const double *A, int64_t nr, int64_t nc, double eps, int64_t cap,
               int64_t *rows, int64_t *cols, int64_t *rank, double *resid);
int operator_entry(bool is_complex, const double *A, int64_t nr, int64_t nc, double epsilon,
                   std::vector<int64_t> &rows, std::vector<double> &V, int *ambiguous);
int exact_entry(bool is_complex, const gcabem::GreenExact &g, double epsilon,
                std::vector<int64_t> &rows, std::vector<double> &V);
}  // namespace aca_avx2

namespace {
// GCABEM_ACA_BASELINE=1 forces the baseline build (tests: both builds agree bitwise)
bool use_avx2() {
    static const bool yes =
        __builtin_cpu_supports("avx2") && std::getenv("GCABEM_ACA_BASELINE") == nullptr;
    return yes;
}
void aca_dispatch(bool is_complex, const double *A, int64_t nr, int64_t nc, double eps,
                  int64_t cap, int64_t *rows, int64_t *cols, int64_t *rank, double *resid) {
    if (use_avx2())
        aca_avx2::aca_entry(is_complex, A, nr, nc, eps, cap, rows, cols, rank, resid);
    else
        aca_base::aca_entry(is_complex, A, nr, nc, eps, cap, rows, cols, rank, resid);
}
}  // namespace

extern "C" int gcabem_aca_batch(int is_complex, int64_t ncl, const int64_t *rows_at,
                                int64_t ncols, const double *A, double epsilon, int64_t max_rank,
                                int nthreads, int64_t *out_rank, int64_t *out_rows,
                                int64_t *out_cols, double *out_resid) {
    if (ncl < 0 || ncols <= 0 || !(epsilon > 0.0))
        return gcabem_internal_error(GCABEM_ERR_ARG, "aca: bad sizes or epsilon");
    if (nthreads <= 0) nthreads = (int)std::max(1u, std::thread::hardware_concurrency());
    std::atomic<int64_t> next{0};
    auto work = [&]() {
        for (;;) {
            const int64_t c = next.fetch_add(1);
            if (c >= ncl) return;
            const int64_t r0 = rows_at[c], nr = rows_at[c + 1] - r0;
            int64_t cap = std::min(nr, ncols);
            if (max_rank > 0) cap = std::min(cap, max_rank);
            const int64_t w = is_complex ? 2 : 1;
            aca_dispatch(is_complex != 0, A + r0 * ncols * w, nr, ncols, epsilon, cap,
                         out_rows + r0, out_cols + r0, out_rank + c, out_resid + c);
        }
    };
    std::vector<std::thread> th;
    const int nt = (int)std::min<int64_t>(nthreads, std::max<int64_t>(ncl, 1));
    for (int t = 1; t < nt; ++t) th.emplace_back(work);
    work();
    for (auto &t : th) t.join();
    return GCABEM_OK;
}

namespace gcabem {
int gca_operator(bool is_complex, const double *A, int64_t nr, int64_t nc, double epsilon,
                 std::vector<int64_t> &rows, std::vector<double> &V, int *ambiguous) {
    if (use_avx2())
        return aca_avx2::operator_entry(is_complex, A, nr, nc, epsilon, rows, V, ambiguous);
    return aca_base::operator_entry(is_complex, A, nr, nc, epsilon, rows, V, ambiguous);
}
int gca_operator_exact(bool is_complex, const GreenExact &g, double epsilon,
                       std::vector<int64_t> &rows, std::vector<double> &V) {
    if (use_avx2()) return aca_avx2::exact_entry(is_complex, g, epsilon, rows, V);
    return aca_base::exact_entry(is_complex, g, epsilon, rows, V);
}
int64_t gca_aca(bool is_complex, const double *A, int64_t nr, int64_t nc, double epsilon,
                int64_t *rows, int64_t *cols) {
    int64_t k = 0;
    double resid = 0.0;
    aca_dispatch(is_complex, A, nr, nc, epsilon, std::min(nr, nc), rows, cols, &k, &resid);
    return k;
}
}  // namespace gcabem

// Host-exact Green matrix of one cluster (tests: bitwise against the numpy
// restatement gca.green_matrix_exact and the reference's golden matrices)
// and the exact-path operator of that cluster. charts: nt x 16 doubles as
// the device Chart layout is built by gcabem_mesh_create; here from arrays.
namespace {
std::vector<gcabem::Chart> host_charts(int64_t nv, const double *V, int64_t nt, const int64_t *T,
                                       const double *gram) {
    std::vector<gcabem::Chart> ch(nt);
    for (int64_t t = 0; t < nt; ++t) {
        const int64_t i0 = T[3 * t], i1 = T[3 * t + 1], i2 = T[3 * t + 2];
        for (int k = 0; k < 3; ++k) {
            ch[t].o[k] = V[3 * i0 + k];
            ch[t].e1[k] = V[3 * i1 + k] - V[3 * i0 + k];
            ch[t].e2[k] = V[3 * i2 + k] - V[3 * i1 + k];
            ch[t].n[k] = 0.0;
        }
        ch[t].gram = gram[t];
    }
    (void)nv;
    return ch;
}
gcabem::GreenBox enlarged_box(const double *lo, const double *hi, double delta, double scene) {
    gcabem::GreenBox b;
    double ext = hi[0] - lo[0];
    ext = std::max(ext, hi[1] - lo[1]);
    ext = std::max(ext, hi[2] - lo[2]);
    const double hmax = 0.5 * std::max(ext, 1e-8 * scene);
    for (int k = 0; k < 3; ++k) {
        b.center[k] = 0.5 * (lo[k] + hi[k]);
        b.half[k] = 0.5 * (hi[k] - lo[k]) + delta * hmax;
    }
    return b;
}
}  // namespace

extern "C" int gcabem_green_exact(int equation, double kappa, int64_t nv, const double *V,
                                  int64_t nt, const int64_t *T, const double *gram, int64_t nr,
                                  const int64_t *panels, const double *box_lo,
                                  const double *box_hi, double delta, int m,
                                  const double *gauss_pts, const double *gauss_wts,
                                  double scene_diameter, int64_t nduffy, const double *duffy,
                                  double epsilon, double *A, int64_t *rank, int64_t *rows,
                                  double *Vop) {
    if (!V || !T || !gram || !panels || nr <= 0 || m < 1 || nduffy < 1 ||
        !(equation == 0 || equation == 1))
        return gcabem_internal_error(GCABEM_ERR_ARG, "green_exact: bad arguments");
    const auto charts = host_charts(nv, V, nt, T, gram);
    std::vector<int32_t> pan(nr);
    for (int64_t p = 0; p < nr; ++p) {
        if (panels[p] < 0 || panels[p] >= nt)
            return gcabem_internal_error(GCABEM_ERR_ARG, "green_exact: panel out of range");
        pan[p] = (int32_t)panels[p];
    }
    gcabem::GreenExact g;
    g.charts = charts.data();
    g.panels = pan.data();
    g.nr = nr;
    g.equation = equation;
    g.kappa = kappa;
    g.duffy = duffy;
    g.nq = (int)nduffy;
    g.m = m;
    g.sources(enlarged_box(box_lo, box_hi, delta, scene_diameter), gauss_pts, gauss_wts);
    const int64_t nc = g.nsrc();
    if (A)
        for (int64_t p = 0; p < nr; ++p)
            for (int64_t s = 0; s < nc; ++s) {
                double re, im;
                g.entry(p, s, re, im);
                if (equation == 0) {
                    A[p * nc + s] = re;
                } else {
                    A[2 * (p * nc + s)] = re;
                    A[2 * (p * nc + s) + 1] = im;
                }
            }
    if (rank && rows && Vop) {
        std::vector<int64_t> r;
        std::vector<double> v;
        const int rc = gcabem::gca_operator_exact(equation == 1, g, epsilon, r, v);
        if (rc == 1) return gcabem_internal_error(GCABEM_ERR_GCA, "zero Green matrix");
        if (rc == 2)
            return gcabem_internal_error(GCABEM_ERR_GCA,
                                         "singular ACA pivot block (condition above 1e+14)");
        *rank = (int64_t)r.size();
        std::copy(r.begin(), r.end(), rows);
        std::copy(v.begin(), v.end(), Vop);
    }
    return GCABEM_OK;
}

// Host entry for one matrix (tests, gca._operator_from_green): rows and V
// sized for the rank cap min(nr, nc).
extern "C" int gcabem_gca_operator(int is_complex, const double *A, int64_t nr, int64_t nc,
                                   double epsilon, int64_t *rank, int64_t *rows, double *V) {
    if (!A || !rank || !rows || !V || nr <= 0 || nc <= 0 || !(epsilon > 0.0))
        return gcabem_internal_error(GCABEM_ERR_ARG, "gca_operator: bad arguments");
    std::vector<int64_t> r;
    std::vector<double> v;
    const int rc = gcabem::gca_operator(is_complex != 0, A, nr, nc, epsilon, r, v);
    if (rc == 1) return gcabem_internal_error(GCABEM_ERR_GCA, "zero Green matrix");
    if (rc == 2)
        return gcabem_internal_error(GCABEM_ERR_GCA,
                                     "singular ACA pivot block (condition above 1e+14)");
    *rank = (int64_t)r.size();
    std::copy(r.begin(), r.end(), rows);
    std::copy(v.begin(), v.end(), V);
    return GCABEM_OK;
}

#endif  // !GCABEM_ACA_AVX2
