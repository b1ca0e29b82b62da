/*
 * ORACLE — test infrastructure only. Never linked into the product path.
 *
 * Plain-C restatement of the reference's fused pair-quadrature loop
 * (reference: pkg/src/gcabem/pairquad.py:27-92, the numba `_pair_loop.run`
 * and its four point kernels :59-84), written so that every floating-point
 * operation happens in the same order and with the same rounding as the
 * numba/LLVM build of the reference (no FMA contraction, IEEE sqrt/div,
 * glibc cos/sin/exp). numba types `float * complex` by promoting the float
 * to complex(x, 0.0) and multiplying with (ac-bd, ad+bc); we do the same,
 * zero products included, so non-finite patterns match too.
 *
 * Parity is PINNED: tests/test_oracle.py checks this file bit-for-bit
 * against tests/golden/pair_values_L3.npz (outputs of the unmodified
 * reference) and against the reference GCAMatrix checksums in
 * tests/golden/golden.json.
 *
 * Also provides the index-based batch (scheduler.py:235-261 batch backend:
 * mesh.chart_arrays gather :207-222 + pair_values) with OpenMP threads over
 * pairs — the CPU baseline timed by bench.py (`cpu_baseline`, kind "port").
 *
 * Build: oracle/Makefile  (gcc -O2 -ffp-contract=off -fopenmp -shared)
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct { double re, im; } cplx;

/* numba complex_mul_impl: (a+bi)(c+di) = (ac-bd) + (ad+bc)i */
static inline cplx cmul(cplx x, cplx y) {
    double ac = x.re * y.re, bd = x.im * y.im;
    double ad = x.re * y.im, bc = x.im * y.re;
    cplx z = {ac - bd, ad + bc};
    return z;
}
static inline cplx creal_(double v) { cplx z = {v, 0.0}; return z; }

/* numba cmathimpl.exp_impl, all branches (numba/cpython/cmathimpl.py) */
static cplx cexp_numba(cplx z) {
    double x = z.re, y = z.im;
    cplx out;
    if (isfinite(x)) {
        if (isfinite(y)) {
            double c = cos(y), s = sin(y), r = exp(x);
            out.re = r * c; out.im = r * s;
        } else { out.re = NAN; out.im = NAN; }
    } else if (isnan(x)) {
        if (y != 0.0) { out.re = x; out.im = x; } else { out.re = x; out.im = y; }
    } else if (x > 0.0) {
        if (isfinite(y)) {
            double re = cos(y), im = sin(y);
            if (re != 0) re *= x;
            if (im != 0) im *= x;
            out.re = re; out.im = im;
        } else { out.re = x; out.im = NAN; }
    } else {
        if (isfinite(y)) {
            double r = exp(x), c = cos(y), s = sin(y);
            out.re = r * c; out.im = r * s;
        } else { out.re = 0.0; out.im = 0.0; }
    }
    return out;
}

static const double INV_4PI = 1.0 / (4.0 * 3.14159265358979323846);

/* pairquad.py:59-62 */
static inline cplx k_lslp(double d0, double d1, double d2, double n0, double n1, double n2,
                          double kappa) {
    (void)n0; (void)n1; (void)n2; (void)kappa;
    double r = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
    return creal_(INV_4PI / r);
}
/* pairquad.py:65-70 */
static inline cplx k_ldlp(double d0, double d1, double d2, double n0, double n1, double n2,
                          double kappa) {
    (void)kappa;
    double r2 = d0 * d0 + d1 * d1 + d2 * d2;
    double r = sqrt(r2);
    double dn = d0 * n0 + d1 * n1 + d2 * n2;
    return creal_(INV_4PI * dn / (r2 * r));
}
/* 1j * v with v promoted to complex(v, 0) */
static inline cplx times_i(double v) {
    cplx j = {0.0, 1.0};
    return cmul(j, creal_(v));
}
/* pairquad.py:73-76 */
static inline cplx k_hslp(double d0, double d1, double d2, double n0, double n1, double n2,
                          double kappa) {
    (void)n0; (void)n1; (void)n2;
    double r = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
    cplx e = cexp_numba(times_i(kappa * r));
    return cmul(e, creal_(1.0 / r));
}
/* pairquad.py:79-84 */
static inline cplx k_hdlp(double d0, double d1, double d2, double n0, double n1, double n2,
                          double kappa) {
    double r2 = d0 * d0 + d1 * d1 + d2 * d2;
    double r = sqrt(r2);
    double dn = d0 * n0 + d1 * n1 + d2 * n2;
    cplx e = cexp_numba(times_i(kappa * r));
    cplx ik = times_i(kappa * r);
    cplx t = {1.0 - ik.re, 0.0 - ik.im};  /* float - complex: (1,0) - z */
    return cmul(cmul(e, t), creal_(dn / (r2 * r)));
}

typedef cplx (*point_fn)(double, double, double, double, double, double, double);

static point_fn select_kernel(int equation, int layer) {
    if (equation == 0) return layer == 0 ? k_lslp : k_ldlp;
    return layer == 0 ? k_hslp : k_hdlp;
}

/* pairquad.py:31-51, one pair. Arrays are (n,3) C-order; index i. */
static inline void one_pair(point_fn kp, int64_t i,
                            const double *ox, const double *e1x, const double *e2x,
                            const double *gx,
                            const double *oy, const double *e1y, const double *e2y,
                            const double *gy, const double *ny, double kappa,
                            int64_t nq, const double *xs, const double *ys, const double *w,
                            double *out) {
    cplx acc = {0.0, 0.0};
    const double *a = ox + 3 * i, *b = e1x + 3 * i, *c = e2x + 3 * i;
    const double *p = oy + 3 * i, *q = e1y + 3 * i, *r = e2y + 3 * i;
    double n0 = ny ? ny[3 * i] : 0.0, n1 = ny ? ny[3 * i + 1] : 0.0,
           n2 = ny ? ny[3 * i + 2] : 0.0;
    for (int64_t k = 0; k < nq; ++k) {
        double s = xs[2 * k], t = xs[2 * k + 1];
        double x0 = a[0] + s * b[0] + t * c[0];
        double x1 = a[1] + s * b[1] + t * c[1];
        double x2 = a[2] + s * b[2] + t * c[2];
        s = ys[2 * k]; t = ys[2 * k + 1];
        double y0 = p[0] + s * q[0] + t * r[0];
        double y1 = p[1] + s * q[1] + t * r[1];
        double y2 = p[2] + s * q[2] + t * r[2];
        cplx v = cmul(creal_(w[k]), kp(x0 - y0, x1 - y1, x2 - y2, n0, n1, n2, kappa));
        acc.re = acc.re + v.re;
        acc.im = acc.im + v.im;
    }
    cplx val = cmul(acc, creal_(gx[i]));
    val = cmul(val, creal_(gy[i]));
    out[2 * i] = val.re;
    out[2 * i + 1] = val.im;
}

/* Same contract as pair_values (pairquad.py:95-112); out is interleaved
 * complex128 (n,). ny may be NULL (zeros, as pair_values substitutes). */
int oracle_pair_values(int equation, int layer, double kappa, int64_t n,
                       const double *ox, const double *e1x, const double *e2x, const double *gx,
                       const double *oy, const double *e1y, const double *e2y, const double *gy,
                       const double *ny, int64_t nq, const double *xs, const double *ys,
                       const double *w, double *out, int nthreads) {
    point_fn kp = select_kernel(equation, layer);
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads)
#endif
    for (int64_t i = 0; i < n; ++i)
        one_pair(kp, i, ox, e1x, e2x, gx, oy, e1y, e2y, gy, ny, kappa, nq, xs, ys, w, out);
    (void)nthreads;
    return 0;
}

/* chart of one triangle with a vertex permutation (mesh.py:207-222):
 * v0 = V[idx[p0]], e1 = V[idx[p1]] - v0, e2 = V[idx[p2]] - V[idx[p1]] */
static inline void chart_of(const double *V, const int64_t *T, int64_t tri, const int64_t *perm,
                            double *o, double *e1, double *e2) {
    int64_t i0 = T[3 * tri + (perm ? perm[0] : 0)];
    int64_t i1 = T[3 * tri + (perm ? perm[1] : 1)];
    int64_t i2 = T[3 * tri + (perm ? perm[2] : 2)];
    for (int k = 0; k < 3; ++k) {
        o[k] = V[3 * i0 + k];
        e1[k] = V[3 * i1 + k] - o[k];
        e2[k] = V[3 * i2 + k] - V[3 * i1 + k];
    }
}

/* Index-based batch (scheduler.py:257-261 batch backend): the gather of
 * chart_arrays plus the fused loop, per pair, with OpenMP over pairs.
 * perm_x/perm_y (n,3) int64 may be NULL (identity). normals (nt,3) used
 * only for the double layer, taken at tri_y. */
int oracle_batch_quadrature(int equation, int layer, double kappa,
                            const double *V, const int64_t *T, const double *normals,
                            const double *gram, int64_t n, const int64_t *tri_x,
                            const int64_t *tri_y, const int64_t *perm_x, const int64_t *perm_y,
                            int64_t nq, const double *xs, const double *ys, const double *w,
                            double *out, int nthreads) {
    point_fn kp = select_kernel(equation, layer);
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads)
#endif
    for (int64_t i = 0; i < n; ++i) {
        double ox[3], e1x[3], e2x[3], oy[3], e1y[3], e2y[3], ny[3] = {0.0, 0.0, 0.0};
        chart_of(V, T, tri_x[i], perm_x ? perm_x + 3 * i : NULL, ox, e1x, e2x);
        chart_of(V, T, tri_y[i], perm_y ? perm_y + 3 * i : NULL, oy, e1y, e2y);
        if (layer == 1) memcpy(ny, normals + 3 * tri_y[i], sizeof ny);
        double gx = gram[tri_x[i]], gy = gram[tri_y[i]];
        double res[2];
        one_pair(kp, 0, ox, e1x, e2x, &gx, oy, e1y, e2y, &gy, ny, kappa, nq, xs, ys, w, res);
        out[2 * i] = res[0];
        out[2 * i + 1] = res[1];
    }
    (void)nthreads;
    return 0;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
