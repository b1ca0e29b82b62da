// Host evaluation of single Green-matrix entries in the REFERENCE's numpy
// arithmetic (gca.py:136-179 with kernels.py:46-64 and gca.py:83-133), so
// the bits equal the reference's. Used only where the device's Green matrix
// (a few ulps away) leaves an ACA decision inside the tie window: the
// cluster's ACA is then redone on entries from here, evaluated on demand
// (the rows and columns the ACA touches, not the whole matrix).
//
// Operation order, element by element (no FMA: -ffp-contract=off):
//   X    = (v0 + p0*e1) + p1*e2                 (broadcast expression)
//   d    = X - source
//   r2   = (d0*d0 + d1*d1) + d2*d2, r = sqrt(r2)
//   Laplace   mono  1/(4 pi) / r
//             dip   (1/(4 pi) * dn) / (r2*r),    dn = (d0*n0 + d1*n1) + d2*n2
//   Helmholtz phase = exp(i kr) = (cos kr, sin kr) (libm, as numpy's cexp)
//             mono  phase / r, dip ((phase * (1 - i kr)) * dn) / (r2*r), with
//                   numpy's complex promotion of every real operand and its
//                   division (rat = 0/b, scl = 1/(b + 0*rat))
//   einsum("q,pqs->ps") = sequential sum over q from 0 of (w_q*K_q)
//   then * gram, then * source weight (complex x real promoted).
// tests/test_host.py checks every entry bitwise against the numpy
// restatement gca.green_matrix_exact and the reference's golden matrices.
#pragma once
#include <cmath>
#include <cstdint>
#include <vector>

#include "gcabem_common.cuh"

namespace gcabem {

struct GreenExact {
    const Chart *charts = nullptr;    // host charts (mesh.chart_arrays, identity perm)
    const int32_t *panels = nullptr;  // the cluster's panels, cluster order
    int64_t nr = 0;
    int equation = 0;
    double kappa = 0.0;
    const double *duffy = nullptr;  // nq x {p0, p1, w}
    int nq = 0;
    int m = 0;
    // per geometric source point g (6 m^2): coordinates, normal, weight
    std::vector<double> sp, sn, sw;

    int64_t nsrc() const { return 12 * (int64_t)m * m; }

    // green_sources (gca.py:83-133) from the enlarged box, in its op order
    void sources(const GreenBox &bx, const double *gauss_pts, const double *gauss_wts) {
        const int ng = 6 * m * m;
        sp.assign(3 * ng, 0.0);
        sn.assign(3 * ng, 0.0);
        sw.assign(ng, 0.0);
        for (int g = 0; g < ng; ++g) {
            const int face = g / (m * m), idx = g - face * m * m;
            const int ui = idx / m, vi = idx - ui * m;
            const int axis = face >> 1;
            const int a1 = (axis + 1) % 3, a2 = (axis + 2) % 3;
            const double sgn = (face & 1) ? 1.0 : -1.0;
            const double h1 = bx.half[a1], h2 = bx.half[a2];
            const double u = -h1 + (2.0 * h1) * gauss_pts[ui];
            const double v = -h2 + (2.0 * h2) * gauss_pts[vi];
            sp[3 * g + axis] = bx.center[axis] + sgn * bx.half[axis];
            sp[3 * g + a1] = bx.center[a1] + u;
            sp[3 * g + a2] = bx.center[a2] + v;
            sn[3 * g + axis] = sgn;
            sw[g] = (gauss_wts[ui] * gauss_wts[vi]) * ((4.0 * h1) * h2);
        }
    }

    // entry (p, s) of the (|t| x 12 m^2) matrix; im = 0 for Laplace
    void entry(int64_t p, int64_t s, double &re, double &im) const {
        constexpr double INV_4PI = 1.0 / (4.0 * 3.14159265358979323846);
        const Chart &ch = charts[panels[p]];
        const int64_t g = s >> 1;
        const bool dip = (s & 1) != 0;
        const double *S = &sp[3 * g], *N = &sn[3 * g];
        double ar = 0.0, ai = 0.0;
        for (int q = 0; q < nq; ++q) {
            const double p0 = duffy[3 * q], p1 = duffy[3 * q + 1], w = duffy[3 * q + 2];
            double d[3];
            for (int k = 0; k < 3; ++k) {
                const double a = ch.o[k] + p0 * ch.e1[k];
                const double X = a + p1 * ch.e2[k];
                d[k] = X - S[k];
            }
            const double r2 = (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2];
            const double r = std::sqrt(r2);
            double kr, ki;
            if (equation == 0) {
                if (!dip) {
                    kr = INV_4PI / r;
                } else {
                    const double dn = (d[0] * N[0] + d[1] * N[1]) + d[2] * N[2];
                    kr = (INV_4PI * dn) / (r2 * r);
                }
                ar = ar + w * kr;
                continue;
            }
            const double x = kappa * r;
            const double c = std::cos(x), sn_ = std::sin(x);
            if (!dip) {
                // (c, s) / (r, 0)
                const double rat = 0.0 / r, scl = 1.0 / (r + 0.0 * rat);
                kr = (c + sn_ * rat) * scl;
                ki = (sn_ - c * rat) * scl;
            } else {
                const double dn = (d[0] * N[0] + d[1] * N[1]) + d[2] * N[2];
                // t = 1j * x = (0, 1) (x, 0); u = (1, 0) - t
                const double tr = 0.0 * x - 1.0 * 0.0, ti = 0.0 * 0.0 + 1.0 * x;
                const double ur = 1.0 - tr, ui = 0.0 - ti;
                // phase * u
                const double pr = c * ur - sn_ * ui, pi = c * ui + sn_ * ur;
                // * (dn, 0)
                const double qr = pr * dn - pi * 0.0, qi = pr * 0.0 + pi * dn;
                // / (r2 r, 0)
                const double r3 = r2 * r;
                const double rat = 0.0 / r3, scl = 1.0 / (r3 + 0.0 * rat);
                kr = (qr + qi * rat) * scl;
                ki = (qi - qr * rat) * scl;
            }
            // (w, 0) * (kr, ki)
            ar = ar + (w * kr - 0.0 * ki);
            ai = ai + (w * ki + 0.0 * kr);
        }
        const double gram = ch.gram, ws = sw[g];
        if (equation == 0) {
            re = (ar * gram) * ws;
            im = 0.0;
            return;
        }
        const double br = ar * gram - ai * 0.0, bi = ar * 0.0 + ai * gram;
        re = br * ws - bi * 0.0;
        im = br * 0.0 + bi * ws;
    }
};

}  // namespace gcabem
