/*
 * ORACLE — test infrastructure only. Never linked into the product path.
 *
 * High-precision (IEEE binary128, libquadmath) evaluation of the SAME
 * discrete quadrature the reference computes in pairquad.py:27-84 for the
 * batch backend (scheduler.py:257-261): identical double-precision inputs
 * (the reference's chart arrays of mesh.chart_arrays, mesh.py:207-222:
 * v0 = V[idx[p0]], e1 = V[idx[p1]] - v0, e2 = V[idx[p2]] - V[idx[p1]], all
 * rounded to double exactly as the reference rounds them; gramians and
 * normals as stored; the double-precision rule points and weights), but
 * every operation after the chart gather carried out in 113-bit arithmetic.
 * The result is the "exact" value of the reference's discrete rule on its
 * own inputs, to ~1e-30 relative.
 *
 * Purpose: SURVEY §8(a) P2 says entries that are roundoff in the reference
 * may be compared on their leaf-block scale. tests/test_p2_evidence.py uses
 * this file to MEASURE that claim instead of asserting it: where the device
 * and the reference differ by more than 1e-12 relative, the device must be
 * within 1e-12 of this value and the reference's own error must account for
 * the difference.
 */
#include <quadmath.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef __float128 q;

static const q INV_4PI_Q = 0.0795774715459476678844418816862571810Q;

static inline void chart_of(const double *V, const int64_t *T, int64_t tri, const int64_t *perm,
                            double *o, double *e1, double *e2) {
    int64_t i0 = T[3 * tri + (perm ? perm[0] : 0)];
    int64_t i1 = T[3 * tri + (perm ? perm[1] : 1)];
    int64_t i2 = T[3 * tri + (perm ? perm[2] : 2)];
    for (int k = 0; k < 3; ++k) {
        o[k] = V[3 * i0 + k];
        e1[k] = V[3 * i1 + k] - o[k];          /* rounded to double, as the reference */
        e2[k] = V[3 * i2 + k] - V[3 * i1 + k];
    }
}

/* out (n,) interleaved complex; same arguments as oracle_batch_quadrature */
int oracle_batch_quadrature_hp(int equation, int layer, double kappa,
                               const double *V, const int64_t *T, const double *normals,
                               const double *gram, int64_t n, const int64_t *tri_x,
                               const int64_t *tri_y, const int64_t *perm_x,
                               const int64_t *perm_y, int64_t nq, const double *xs,
                               const double *ys, const double *w, double *out, int nthreads) {
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads)
#endif
    for (int64_t i = 0; i < n; ++i) {
        double ox[3], e1x[3], e2x[3], oy[3], e1y[3], e2y[3];
        chart_of(V, T, tri_x[i], perm_x ? perm_x + 3 * i : NULL, ox, e1x, e2x);
        chart_of(V, T, tri_y[i], perm_y ? perm_y + 3 * i : NULL, oy, e1y, e2y);
        q nrm[3] = {0, 0, 0};
        if (layer == 1)
            for (int k = 0; k < 3; ++k) nrm[k] = normals[3 * tri_y[i] + k];
        q re = 0, im = 0, kap = kappa;
        for (int64_t p = 0; p < nq; ++p) {
            q s = xs[2 * p], t = xs[2 * p + 1], u = ys[2 * p], v = ys[2 * p + 1];
            q d[3];
            for (int k = 0; k < 3; ++k)
                d[k] = ((q)ox[k] + s * e1x[k] + t * e2x[k]) - ((q)oy[k] + u * e1y[k] + v * e2y[k]);
            q r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
            q r = sqrtq(r2);
            q kr, kim;
            if (equation == 0) {
                kr = layer == 0 ? INV_4PI_Q / r
                                : INV_4PI_Q * (d[0] * nrm[0] + d[1] * nrm[1] + d[2] * nrm[2])
                                      / (r2 * r);
                kim = 0;
            } else {
                q c = cosq(kap * r), sn = sinq(kap * r);
                if (layer == 0) {
                    kr = c / r;
                    kim = sn / r;
                } else {
                    /* e^{i k r} (1 - i k r) dn / r^3 */
                    q f = (d[0] * nrm[0] + d[1] * nrm[1] + d[2] * nrm[2]) / (r2 * r);
                    kr = (c + sn * kap * r) * f;
                    kim = (sn - c * kap * r) * f;
                }
            }
            re += (q)w[p] * kr;
            im += (q)w[p] * kim;
        }
        q g = (q)gram[tri_x[i]] * (q)gram[tri_y[i]];
        out[2 * i] = (double)(re * g);
        out[2 * i + 1] = (double)(im * g);
    }
    (void)nthreads;
    return 0;
}
