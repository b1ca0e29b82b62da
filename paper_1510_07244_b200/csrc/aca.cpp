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
#include <thread>
#include <vector>

#include "gcabem_b200.h"

int gcabem_internal_error(int code, const char *msg);  // api.cu

namespace {

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

template <typename T>
struct Ops;
template <>
struct Ops<double> {
    static double mag(double x) { return std::fabs(x); }
    static double mul(double a, double b) { return a * b; }
    static double sub(double a, double b) { return a - b; }
    static double div(double a, double b) { return a / b; }
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
    static bool zero(Cx a) { return a.re == 0.0 && a.im == 0.0; }
    static double norm2(Cx a) { return a.re * a.re + a.im * a.im; }
    static double dotc_re(Cx a, Cx b) { return a.re * b.re + a.im * b.im; }
    static double dotc_im(Cx a, Cx b) { return a.re * b.im - a.im * b.re; }
};

template <typename T>
void aca_one(const T *A, int64_t nr, int64_t nc, double eps, int64_t cap, int64_t *rows,
             int64_t *cols, int64_t *rank, double *resid) {
    using O = Ops<T>;
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
        for (int64_t j = 0; j < nc; ++j) r[j] = A[i * nc + j];
        for (size_t m = 0; m < U.size(); ++m) {
            const T ui = U[m][i];
            for (int64_t j = 0; j < nc; ++j) r[j] = O::sub(r[j], O::mul(ui, W[m][j]));
        }
        int64_t jp = 0;
        double best = -1.0;
        for (int64_t j = 0; j < nc; ++j) {
            const double a = O::mag(r[j]);
            if (a > best) {
                best = a;
                jp = j;
            }
        }
        used[i] = 1;
        if (O::zero(r[jp])) {
            next = nr;
            continue;
        }
        std::vector<T> w(nc);
        const T piv = r[jp];
        for (int64_t j = 0; j < nc; ++j) w[j] = O::div(r[j], piv);
        for (int64_t q = 0; q < nr; ++q) c[q] = A[q * nc + jp];
        for (size_t m = 0; m < U.size(); ++m) {
            const T wj = W[m][jp];
            for (int64_t q = 0; q < nr; ++q) c[q] = O::sub(c[q], O::mul(wj, U[m][q]));
        }
        double nu = 0.0, nw = 0.0;
        for (int64_t q = 0; q < nr; ++q) nu += O::norm2(c[q]);
        for (int64_t j = 0; j < nc; ++j) nw += O::norm2(w[j]);
        nu = std::sqrt(nu);
        nw = std::sqrt(nw);
        double cross = 0.0;
        for (size_t m = 0; m < U.size(); ++m) {
            double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
            for (int64_t q = 0; q < nr; ++q) {
                ar += O::dotc_re(U[m][q], c[q]);
                ai += O::dotc_im(U[m][q], c[q]);
            }
            for (int64_t j = 0; j < nc; ++j) {
                br += O::dotc_re(W[m][j], w[j]);
                bi += O::dotc_im(W[m][j], w[j]);
            }
            cross += ar * br - ai * bi;  // Re((u^H c) (w_m^H w))
        }
        U.emplace_back(c.begin(), c.end());
        W.emplace_back(std::move(w));
        rows[k] = i;
        cols[k] = jp;
        ++k;
        est2 = std::max(est2 + nu * nu * nw * nw + 2.0 * cross, 0.0);
        res = nu * nw;
        if (res <= eps * std::sqrt(est2)) break;
        int64_t nb = 0;
        double mb = -1.0;
        for (int64_t q = 0; q < nr; ++q) {
            const double a = used[q] ? 0.0 : O::mag(c[q]);
            if (a > mb) {
                mb = a;
                nb = q;
            }
        }
        next = mb == 0.0 ? nr : nb;
    }
    *rank = k;
    *resid = res;
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
            if (is_complex)
                aca_one<Cx>(reinterpret_cast<const Cx *>(A) + r0 * ncols, nr, ncols, epsilon, cap,
                            out_rows + r0, out_cols + r0, out_rank + c, out_resid + c);
            else
                aca_one<double>(A + r0 * ncols, nr, ncols, epsilon, cap, out_rows + r0,
                                out_cols + r0, out_rank + c, out_resid + c);
        }
    };
    std::vector<std::thread> th;
    const int nt = (int)std::min<int64_t>(nthreads, std::max<int64_t>(ncl, 1));
    for (int t = 1; t < nt; ++t) th.emplace_back(work);
    work();
    for (auto &t : th) t.join();
    return GCABEM_OK;
}
