// Disjoint-rule pair quadrature (reference pairquad.py:27-92 over
// quadrature.py:108's factored Duffy rule): constant-memory rule tables,
// the expanded/direct evaluation forms and disjoint_kernel<N, KIND>.
// Instantiated per order range in disjoint_o*.cu (parallel compilation).
#pragma once
#include "device_math.cuh"

namespace gcabem {

// ---------------------------------------------------------------------------
// disjoint rule, factored: x = (a, a b), y = (c, c d), w = (wa wb a)(wc wd c)

static __constant__ double c_gauss[MAX_ORDER + 1][MAX_ORDER];  // 1D Gauss points on [0,1]
__host__ __device__ constexpr int duffy_offset(int n) { return (n - 1) * n * (2 * n - 1) / 6; }
constexpr int DUFFY_TOTAL = duffy_offset(MAX_ORDER + 1);
static __constant__ double c_duffy_t[DUFFY_TOTAL];  // t = a*b   (s = a = c_gauss[n][p / n])
static __constant__ double c_duffy_w[DUFFY_TOTAL];  // (wa*wb)*a  == duffy_panel_rule weights

// every translation unit that includes this header owns a copy of the
// tables (static __constant__); its upload_tables() fills that copy
static cudaError_t upload_tables(int n, const double *g, const double *gw) {
    double t[MAX_ORDER * MAX_ORDER], w[MAX_ORDER * MAX_ORDER];
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
            t[a * n + b] = g[a] * g[b];             // quadrature.py:95 a*b
            w[a * n + b] = (gw[a] * gw[b]) * g[a];  // quadrature.py:96
        }
    cudaError_t e = cudaMemcpyToSymbol(c_gauss, g, sizeof(double) * n,
                                       sizeof(double) * MAX_ORDER * n);
    if (e != cudaSuccess) return e;
    e = cudaMemcpyToSymbol(c_duffy_t, t, sizeof(double) * n * n,
                           sizeof(double) * duffy_offset(n));
    if (e != cudaSuccess) return e;
    return cudaMemcpyToSymbol(c_duffy_w, w, sizeof(double) * n * n,
                              sizeof(double) * duffy_offset(n));
}

// Two evaluation forms for the disjoint rule x = (a, ab), y = (c, cd):
//
//  direct    d_pq = xo_p - g_c u_d  (3 DFMA), r^2 = |d|^2 (3)
//  expanded  r^2 = |xo_p|^2 - 2 g_c (xo_p . u_d) + g_c^2 |u_d|^2
//            = fma(g_c, fma(g_c, |u_d|^2, -2 xo.u_d), |xo|^2)   (2 DFMA)
//
// with xo_p = (ox - oy) + a e1x + ab e2x and u_d = e1y + g_d e2y. The expanded
// form cancels when the pair is close: its rounding error is below
// eps * S^2 / r_min^2 with S = |ox-oy| + |e1x| + |e2x| + |e1y| + |e2y| and
// r_min a lower bound of the pair distance (bounding spheres). Pairs with
// S^2 <= EXPANDED_MAX_RATIO * r_min^2 (error < 2.3e-13, measured < 3e-15)
// take it; the rest (about 1% of near-field pairs) the direct form.
#ifndef GCABEM_EXPANDED_MAX_RATIO
#define GCABEM_EXPANDED_MAX_RATIO 1024.0
#endif
constexpr double EXPANDED_MAX_RATIO = GCABEM_EXPANDED_MAX_RATIO;
// fused pair kinds roll the outer y loop from this order on (see below)
#ifndef GCABEM_ROLL_OUTER_N
#define GCABEM_ROLL_OUTER_N 6
#endif

// accumulator slots a kind uses (in[] / acc[] of 6): {re, im} of the single
// layer or of a single kind's operator, then the pair kinds' double layer,
// then (MIR) the transposed pair's double layer (see accumulate_mirror)
__host__ __device__ constexpr bool slot_used(int kind, bool mir, int k) {
    return k == 0 ? true
         : k == 1 ? kind_helm(kind)
         : k == 2 ? (kind_pair(kind) || (mir && (kind == L_DLP || kind == H_DLP)))
         : k == 3 ? (kind == H_PAIR || (mir && kind == H_DLP))
         : k == 4 ? (mir && kind_pair(kind))
         : k == 5 ? (mir && kind == H_PAIR) : false;
}

template <int KIND, bool MIR, int PH>
__device__ __forceinline__ void accumulate_any(double r2, double dn, double dnm, double w,
                                               double kappa, double phi0, double in[6]) {
    if constexpr (MIR)
        accumulate_mirror<KIND, PH>(r2, dn, dnm, w, kappa, phi0, in);
    else
        accumulate<KIND, PH>(r2, dn, w, kappa, phi0, in);
}




// MIR: also the transposed pair (j, i) (ROLE_PRIMARY / ROLE_SELF blocks): its
// double layer needs d . n_x, n_x the x panel's normal (nx); dnm = -d . n_x =
// gc u_d . n_x - xo . n_x, formed like dn from per-y (unm) and per-x (xonm) parts
template <int N, int KIND, int PH, bool MIR = false>
__device__ __forceinline__ void disjoint_expanded(const double dO[3], const double e1x[3],
                                                  const double e2x[3], const double e1y[3],
                                                  const double e2y[3], const double n[3],
                                                  double kappa, double phi0, double acc[6],
                                                  const double *nx = nullptr) {
    constexpr bool DL = kind_normal(KIND);
    constexpr bool DM = MIR && DL;   // the transposed pair's double layer
    double uu[N], un[N], unm[N];
#pragma unroll
    for (int d = 0; d < N; ++d) {
        const double gd = c_gauss[N][d];
        const double ux = fma(gd, e2y[0], e1y[0]);
        const double uy = fma(gd, e2y[1], e1y[1]);
        const double uz = fma(gd, e2y[2], e1y[2]);
        uu[d] = fma(ux, ux, fma(uy, uy, uz * uz));
        un[d] = DL ? fma(ux, n[0], fma(uy, n[1], uz * n[2])) : 0.0;
        unm[d] = DM ? fma(ux, nx[0], fma(uy, nx[1], uz * nx[2])) : 0.0;
    }
    // x-side quantities as polynomials in the x point (s, t) = (a, a b):
    //   |xo|^2     = Q0 + s (2 P1 + s Q11) + t (2 P2 + 2 s Q12 + t Q22)
    //   -2 xo.e1y  = A0 + s A1 + t A2,  -2 xo.e2y = B0 + s B1 + t B2
    //   xo.n_y     = N0 + s N1 + t N2
    // with xo = dO + s e1x + t e2x; the s parts once per a, 5 FMA per x point
    auto dot = [](const double *u, const double *v) { return fma(u[0], v[0], fma(u[1], v[1], u[2] * v[2])); };
    const double Q0 = dot(dO, dO), P1 = 2.0 * dot(dO, e1x), P2 = 2.0 * dot(dO, e2x);
    const double Q11 = dot(e1x, e1x), Q12 = 2.0 * dot(e1x, e2x), Q22 = dot(e2x, e2x);
    const double A0 = -2.0 * dot(dO, e1y), A1 = -2.0 * dot(e1x, e1y), A2 = -2.0 * dot(e2x, e1y);
    const double B0 = -2.0 * dot(dO, e2y), B1 = -2.0 * dot(e1x, e2y), B2 = -2.0 * dot(e2x, e2y);
    const double N0 = DL ? dot(dO, n) : 0.0, N1 = DL ? dot(e1x, n) : 0.0,
                 N2 = DL ? dot(e2x, n) : 0.0;
    // xo . n_x (MIR): dO . n_x + s e1x . n_x + t e2x . n_x
    const double M0 = DM ? dot(dO, nx) : 0.0, M1 = DM ? dot(e1x, nx) : 0.0,
                 M2 = DM ? dot(e2x, nx) : 0.0;

#pragma unroll 1
    for (int ia = 0; ia < N; ++ia) {
        const double s = c_gauss[N][ia];
        const double xs = fma(s, fma(s, Q11, P1), Q0);
        const double vs = fma(s, Q12, P2);
        const double as = fma(s, A1, A0);
        const double bs = fma(s, B1, B0);
        const double ns = DL ? fma(s, N1, N0) : 0.0;
        const double ms = DM ? fma(s, M1, M0) : 0.0;
#pragma unroll 1
        for (int ib = 0; ib < N; ++ib) {
            const int p = ia * N + ib;
            const double t = c_duffy_t[duffy_offset(N) + p];
            const double wx = c_duffy_w[duffy_offset(N) + p];
            const double xx = fma(t, fma(t, Q22, vs), xs);
            const double xon = DL ? fma(t, N2, ns) : 0.0;
            const double xonm = DM ? fma(t, M2, ms) : 0.0;
            const double a2 = fma(t, A2, as);
            const double b2 = fma(t, B2, bs);
            double in[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            // fused pair kinds at orders >= 6 roll the outer y loop (the fully
            // unrolled N^2 body spills their two layers of state)
            constexpr int OUTER = (kind_pair(KIND) && N >= GCABEM_ROLL_OUTER_N) ? 1 : N;
#pragma unroll OUTER
            for (int d = 0; d < N; ++d) {
                const double m2b = fma(c_gauss[N][d], b2, a2);
#pragma unroll
                for (int c = 0; c < N; ++c) {
                    const double gc = c_gauss[N][c];
                    const double wy = c_duffy_w[duffy_offset(N) + c * N + d];
                    const double r2 = fma(gc, fma(gc, uu[d], m2b), xx);
                    const double dn = DL ? fma(-gc, un[d], xon) : 0.0;
                    const double dnm = DM ? fma(gc, unm[d], -xonm) : 0.0;
                    accumulate_any<KIND, MIR, PH>(r2, dn, dnm, wy, kappa, phi0, in);
                }
            }
#pragma unroll
            for (int k = 0; k < 6; ++k)
                if (slot_used(KIND, MIR, k)) acc[k] = fma(wx, in[k], acc[k]);
        }
    }
}

template <int N, int KIND, int PH, bool MIR = false>
__device__ __forceinline__ void disjoint_direct(const double dO[3], const double e1x[3],
                                                const double e2x[3], const double e1y[3],
                                                const double e2y[3], const double n[3],
                                                double kappa, double phi0, double acc[6],
                                                const double *nx = nullptr) {
    constexpr bool DL = kind_normal(KIND);
    constexpr bool DM = MIR && DL;
    double ux[N], uy[N], uz[N], un[N], unm[N];
#pragma unroll
    for (int d = 0; d < N; ++d) {
        const double gd = c_gauss[N][d];
        ux[d] = fma(gd, e2y[0], e1y[0]);
        uy[d] = fma(gd, e2y[1], e1y[1]);
        uz[d] = fma(gd, e2y[2], e1y[2]);
        un[d] = DL ? fma(ux[d], n[0], fma(uy[d], n[1], uz[d] * n[2])) : 0.0;
        unm[d] = DM ? fma(ux[d], nx[0], fma(uy[d], nx[1], uz[d] * nx[2])) : 0.0;
    }
#pragma unroll 1
    for (int p = 0; p < N * N; ++p) {
        const double s = c_gauss[N][p / N];
        const double t = c_duffy_t[duffy_offset(N) + p];
        const double wx = c_duffy_w[duffy_offset(N) + p];
        const double xo0 = fma(t, e2x[0], fma(s, e1x[0], dO[0]));
        const double xo1 = fma(t, e2x[1], fma(s, e1x[1], dO[1]));
        const double xo2 = fma(t, e2x[2], fma(s, e1x[2], dO[2]));
        const double xon = DL ? fma(xo0, n[0], fma(xo1, n[1], xo2 * n[2])) : 0.0;
        const double xonm = DM ? fma(xo0, nx[0], fma(xo1, nx[1], xo2 * nx[2])) : 0.0;
        double in[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        constexpr int OUTER = (kind_pair(KIND) && N >= GCABEM_ROLL_OUTER_N) ? 1 : N;  // see disjoint_expanded
#pragma unroll OUTER
        for (int c = 0; c < N; ++c) {
            const double gc = c_gauss[N][c];
#pragma unroll
            for (int d = 0; d < N; ++d) {
                const double wy = c_duffy_w[duffy_offset(N) + c * N + d];
                const double dx = fma(-gc, ux[d], xo0);
                const double dy = fma(-gc, uy[d], xo1);
                const double dz = fma(-gc, uz[d], xo2);
                const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
                const double dn = DL ? fma(-gc, un[d], xon) : 0.0;
                const double dnm = DM ? fma(gc, unm[d], -xonm) : 0.0;
                accumulate_any<KIND, MIR, PH>(r2, dn, dnm, wy, kappa, phi0, in);
            }
        }
#pragma unroll
        for (int k = 0; k < 6; ++k)
            if (slot_used(KIND, MIR, k)) acc[k] = fma(wx, in[k], acc[k]);
    }
}

// One thread = one panel pair of one WorkBlock; a task = DISJOINT_TPB
// consecutive (row-major) pairs of one block. Rule constants are
// compile-time offsets into constant memory (DFMA operands), so the inner
// N^2 loop issues no loads. Pairs that share a vertex are written as 0: the
// singular pass of the same plan overwrites every one of them (the overwrite
// protocol, scheduler.py:9-12), so their disjoint-rule value (non-finite for
// identical pairs) is never observable.
// resident CTAs per SM the register allocation must allow, per kind:
// L-SLP 7 (72 registers), L-DLP 6 (80), Helmholtz 5 (<= 102); measured on the B200 against
// the compiler's choice (96 / 128 registers): +1% (C2 L-DLP) and +10% (C3
// H-DLP) from the extra warps hiding the FP64 dependency latency, despite a
// few spilled bytes in the cold full-sincos tier (orders above 7 keep the
// compiler's choice: they would spill heavily); the fused pair kinds carry two
// layers of accumulators and get fewer CTAs at the higher orders.
// pair kinds at orders <= 4: L_PAIR 4 (124 registers; 5 measured 1-2% slower at
// C2), H_PAIR 5 (96 registers, a few spilled bytes in the cold full-sincos
// tier; 4 and 6 measured 1.6% and 3% slower at C3, re-checked with the v11
// point kernels)
// threads per CTA of the disjoint kernels: a task's DISJOINT_TPB pairs may run
// as CTA_SPLIT CTAs (the resident-CTA counts below are per 128 threads and
// scale with the CTA size); with one-warp tasks the split is 1
#ifndef GCABEM_DISJOINT_CTA
#define GCABEM_DISJOINT_CTA 32
#endif
constexpr int DISJOINT_CTA = GCABEM_DISJOINT_CTA;
constexpr int CTA_SPLIT = DISJOINT_TPB / DISJOINT_CTA;
constexpr int CTA_SCALE = 128 / DISJOINT_CTA;   // resident CTAs per "128-thread CTA" below
static_assert(DISJOINT_TPB % DISJOINT_CTA == 0 && DISJOINT_CTA % 32 == 0, "whole warps");

#ifndef GCABEM_HPAIR_MINB
#define GCABEM_HPAIR_MINB 5
#endif
constexpr int disjoint_minb(int n, int kind) {
    return n > 7 ? 1                                     // would spill heavily
           : kind == L_SLP ? 7 : kind == L_DLP ? 6 : kind <= H_DLP ? 5
           : n <= 4 ? (kind == L_PAIR ? 4 : GCABEM_HPAIR_MINB)
           : n <= 6 ? 3 : 2;                             // pair kinds: 2 layers of state
}

// mirrored kernels (MIR) carry a third accumulator pair (the transposed
// double layer): one CTA fewer per SM than the plain kernel of the kind
#ifndef GCABEM_MIR_MINB_LPAIR
#define GCABEM_MIR_MINB_LPAIR 3
#endif
#ifndef GCABEM_MIR_MINB_HPAIR
#define GCABEM_MIR_MINB_HPAIR 4
#endif
constexpr int disjoint_minb_mir(int n, int kind) {
    return n > 7 ? 1 : kind == L_SLP ? 7 : kind == H_SLP ? 5
           : kind == L_DLP ? 5 : kind == H_DLP ? 4
           : n <= 4 ? (kind == L_PAIR ? GCABEM_MIR_MINB_LPAIR : GCABEM_MIR_MINB_HPAIR)
           : n <= 6 ? 3 : 2;
}

template <int N, int KIND, bool MIR>
__global__ void __launch_bounds__(DISJOINT_CTA, (MIR ? disjoint_minb_mir(N, KIND)
                                                     : disjoint_minb(N, KIND)) * CTA_SCALE)
disjoint_kernel(const Chart *__restrict__ charts, const int32_t *__restrict__ T,
                const TaskDesc *__restrict__ tasks, const int32_t *__restrict__ panels, double2 *__restrict__ payload,
                double2 *__restrict__ payload2, double kappa) {
    // CTA_SPLIT CTAs of DISJOINT_CTA threads per task of DISJOINT_TPB pairs
    const TaskDesc &td = tasks[blockIdx.x / CTA_SPLIT];
    const BlockDesc b = td.b;
    const int k = td.k0 + (int)(blockIdx.x % CTA_SPLIT) * DISJOINT_CTA + threadIdx.x;
    // no early exit before the warp votes below: every lane of the CTA's
    // full warp(s) reaches them
    bool inb = k < b.nr * b.nc;
    const int i = inb ? k / b.nc : 0;
    const int j = inb ? k - i * b.nc : 0;
    // ROLE_SELF (diagonal leaf): the strict lower triangle is written by the
    // upper one (the diagonal holds identical pairs: shared, written 0)
    if (MIR && b.role == ROLE_SELF && i + b.dr > j) inb = false;
    const int tx = panels[b.rows_at + i], ty = panels[b.cols_at + j];
    const int64_t pos = b.base + (int64_t)i * b.ld + j;
    double2 *dst = payload + pos;
    double2 *dst2 = kind_pair(KIND) ? payload2 + pos : nullptr;
    // the transposed pair's entry (MIR): mirror leaf, row j, column i
    const int64_t mpos = MIR ? b.mbase + (int64_t)j * b.mld + i : 0;
    double2 *mdst = MIR ? payload + mpos : nullptr;
    double2 *mdst2 = MIR && kind_pair(KIND) ? payload2 + mpos : nullptr;
    bool shared;
    {
        const int a0 = T[3 * tx], a1 = T[3 * tx + 1], a2 = T[3 * tx + 2];
        const int b0 = T[3 * ty], b1 = T[3 * ty + 1], b2 = T[3 * ty + 2];
        shared = a0 == b0 || a0 == b1 || a0 == b2 || a1 == b0 || a1 == b1 || a1 == b2 ||
                 a2 == b0 || a2 == b1 || a2 == b2;
    }
    const bool active = inb && !shared;
    const Chart *cx = charts + tx;
    const Chart *cy = charts + ty;
    double dO[3], e1x[3], e2x[3], e1y[3], e2y[3], n[3] = {0.0, 0.0, 0.0},
           nx[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        dO[c] = cx->o[c] - cy->o[c];
        e1x[c] = cx->e1[c];
        e2x[c] = cx->e2[c];
        e1y[c] = cy->e1[c];
        e2y[c] = cy->e2[c];
        if (kind_normal(KIND)) n[c] = cy->n[c];
        if (MIR && kind_normal(KIND)) nx[c] = cx->n[c];
    }
    const double gx = cx->gram, gy = cy->gram;
    const double rx = cx->radius, ry = cy->radius;
    // centroid difference: dO + (2 e1x + e2x)/3 - (2 e1y + e2y)/3
    double dc[3];
#pragma unroll
    for (int c = 0; c < 3; ++c)
        dc[c] = fma(1.0 / 3.0, (2.0 * e1x[c] + e2x[c]) - (2.0 * e1y[c] + e2y[c]), dO[c]);
    const double dcen = norm3(dc[0], dc[1], dc[2]);
    const double rmin = dcen - rx - ry;
    const double S = norm3(dO[0], dO[1], dO[2]) + cx->enorm + cy->enorm;
    double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    // evaluation form and phase tier are chosen per WARP (votes over the
    // active lanes): a lane that needs the direct form or a longer phase
    // polynomial takes its whole warp along instead of splitting it into
    // serialised branches
    const bool expanded =
        __all_sync(0xffffffffu, !active || (rmin > 0.0 && S * S <= EXPANDED_MAX_RATIO * rmin * rmin));
    constexpr bool HELM = kind_helm(KIND);
    // Helmholtz phase about the centroid distance: |kappa r - kappa D| <= kappa (rx + ry)
    const double phi0 = HELM ? kappa * dcen : 0.0;
    const double dmax = HELM && active ? kappa * (rx + ry) : 0.0;
    // kappa = 0 takes the full-sincos tier (unscaled geometry, see below)
    const bool tiny = HELM && kappa > 0.0 && __all_sync(0xffffffffu, dmax <= TINY_PHASE_MAX);
    const bool smallp = HELM && kappa > 0.0 && __all_sync(0xffffffffu, dmax <= SMALL_PHASE_MAX);
    if (!active) {
        if (inb) {
            *dst = make_double2(0.0, 0.0);
            if (kind_pair(KIND)) *dst2 = make_double2(0.0, 0.0);
            if (MIR) {
                *mdst = make_double2(0.0, 0.0);
                if (kind_pair(KIND)) *mdst2 = make_double2(0.0, 0.0);
            }
        }
        return;
    }
    if constexpr (HELM) {
        if (tiny || smallp) {
            // geometry in units of 1/kappa: kappa r = r2' y' with no product
            // by kappa per point (the point kernels get kappa = 1); the sums
            // come out as S / kappa (single layer) and D / kappa^2 (double)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                dO[c] *= kappa;
                e1x[c] *= kappa;
                e2x[c] *= kappa;
                e1y[c] *= kappa;
                e2y[c] *= kappa;
            }
            if (tiny) {
                if (expanded)
                    disjoint_expanded<N, KIND, 2, MIR>(dO, e1x, e2x, e1y, e2y, n, 1.0, phi0, acc, nx);
                else
                    disjoint_direct<N, KIND, 2, MIR>(dO, e1x, e2x, e1y, e2y, n, 1.0, phi0, acc, nx);
            } else {
                if (expanded)
                    disjoint_expanded<N, KIND, 1, MIR>(dO, e1x, e2x, e1y, e2y, n, 1.0, phi0, acc, nx);
                else
                    disjoint_direct<N, KIND, 1, MIR>(dO, e1x, e2x, e1y, e2y, n, 1.0, phi0, acc, nx);
            }
            rotate_acc<KIND, MIR>(phi0, acc);
            unscale_acc<KIND, MIR>(kappa, acc);
        } else {
            if (expanded)
                disjoint_expanded<N, KIND, 0, MIR>(dO, e1x, e2x, e1y, e2y, n, kappa, 0.0, acc, nx);
            else
                disjoint_direct<N, KIND, 0, MIR>(dO, e1x, e2x, e1y, e2y, n, kappa, 0.0, acc, nx);
        }
    } else {
        if (expanded)
            disjoint_expanded<N, KIND, 0, MIR>(dO, e1x, e2x, e1y, e2y, n, kappa, 0.0, acc, nx);
        else
            disjoint_direct<N, KIND, 0, MIR>(dO, e1x, e2x, e1y, e2y, n, kappa, 0.0, acc, nx);
    }
    if constexpr (MIR)
        finish_acc_mirror<KIND>(acc, gx, gy, dst, dst2, mdst, mdst2);
    else
        finish_acc<KIND>(acc, gx, gy, dst, dst2);
}

template <int N, bool MIR>
static cudaError_t launch_disjoint_nm(int kind, const Chart *charts, const int32_t *T,
                                      const TaskDesc *tasks, int64_t ntasks,
                                      const int32_t *panels, double2 *payload, double2 *payload2,
                                      double kappa, cudaStream_t s) {
    const dim3 grid((unsigned)(ntasks * CTA_SPLIT)), block(DISJOINT_CTA);
    switch (kind) {
        case L_SLP: disjoint_kernel<N, L_SLP, MIR><<<grid, block, 0, s>>>(charts, T, tasks, panels, payload, payload2, kappa); break;
        case L_DLP: disjoint_kernel<N, L_DLP, MIR><<<grid, block, 0, s>>>(charts, T, tasks, panels, payload, payload2, kappa); break;
        case H_SLP: disjoint_kernel<N, H_SLP, MIR><<<grid, block, 0, s>>>(charts, T, tasks, panels, payload, payload2, kappa); break;
        case H_DLP: disjoint_kernel<N, H_DLP, MIR><<<grid, block, 0, s>>>(charts, T, tasks, panels, payload, payload2, kappa); break;
        case L_PAIR: disjoint_kernel<N, L_PAIR, MIR><<<grid, block, 0, s>>>(charts, T, tasks, panels, payload, payload2, kappa); break;
        default:    disjoint_kernel<N, H_PAIR, MIR><<<grid, block, 0, s>>>(charts, T, tasks, panels, payload, payload2, kappa); break;
    }
    return cudaGetLastError();
}

// kind >= MIRRORED: the mirrored kernel (orders <= MAX_MIRROR_ORDER)
template <int N>
static cudaError_t launch_disjoint_n(int kind, const Chart *charts, const int32_t *T,
                                     const TaskDesc *tasks, int64_t ntasks,
                                     const int32_t *panels, double2 *payload, double2 *payload2,
                                     double kappa, cudaStream_t s) {
    if (kind >= MIRRORED) {
        if constexpr (N <= MAX_MIRROR_ORDER)
            return launch_disjoint_nm<N, true>(kind - MIRRORED, charts, T, tasks, ntasks,
                                               panels, payload, payload2, kappa, s);
        else
            return cudaErrorInvalidValue;
    }
    return launch_disjoint_nm<N, false>(kind, charts, T, tasks, ntasks, panels, payload,
                                        payload2, kappa, s);
}

}  // namespace gcabem
