// Piecewise-linear (P1) near-field assembly with a deterministic scatter-add
// (BASELINE config 4). The reference assembles P0 matrices
// only; its per-pair API integrate_pair(..., basis_x, basis_y)
// (quadrature.py:223-271) defines the P1 local matrix of a triangle pair:
//
//   M[a][b] = g_x g_y sum_q w_q lambda_a(x_q) k(Phi_x(x_q), Phi_y(y_q)) lambda_b(y_q)
//
// with the chart barycentrics lambda = (1 - s, s - t, t) of
// Phi(s, t) = v0 + s (v1 - v0) + t (v2 - v1). Kernels here compute M for every
// near-field pair (the dense leaves of the block tree), store it in the
// triangles' STORED vertex order (singular pairs are evaluated on permuted
// charts and written back through their permutations), and the global
// vertex-vertex near-field matrix is then gathered in a fixed order:
//
//   plan (once per layout): key(c) = (vertex_x, vertex_y) of every local
//        entry c = 9 p + 3 a + b, stable radix sort (CUB) -> unique keys
//        (CSR pattern) and, per nonzero, its contributions in ascending c;
//   assemble: local matrices (sm_100a kernels), then one thread per nonzero
//        sums its contributions in that order -- bitwise reproducible, no
//        atomics.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>

#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "disjoint.cuh"
#include "internal.h"

using namespace gcabem;

namespace {

// kernel value k(d) (no quadrature weight) for the P1 accumulations
template <int KIND, int PH>
__device__ __forceinline__ void point_value(double r2, double dn, double kappa, double phi0,
                                            double &re, double &im) {
    re = 0.0;
    im = 0.0;
    point_accumulate<KIND, PH>(r2, dn, 1.0, kappa, phi0, re, im);
}

// --- disjoint rule, factored (x = (a, ab), y = (c, cd)), direct form -------
// (the expanded r^2 form of disjoint_kernel measured slower here: with 18
// accumulators the kernel is register-bound, 254 vs 242 registers)
template <int N, int KIND, int PH>
__device__ __forceinline__ void p1_disjoint_pair(const double dO[3], const double e1x[3],
                                                 const double e2x[3], const double e1y[3],
                                                 const double e2y[3], const double n[3],
                                                 double kappa, double phi0, double acc[9][2]) {
    constexpr bool DL = (KIND == L_DLP || KIND == H_DLP);
    constexpr bool CPLX = (KIND == H_SLP || KIND == H_DLP);
    double ux[N], uy[N], uz[N], un[N];
#pragma unroll
    for (int d = 0; d < N; ++d) {
        const double gd = c_gauss[N][d];
        ux[d] = fma(gd, e2y[0], e1y[0]);
        uy[d] = fma(gd, e2y[1], e1y[1]);
        uz[d] = fma(gd, e2y[2], e1y[2]);
        un[d] = DL ? fma(ux[d], n[0], fma(uy[d], n[1], uz[d] * n[2])) : 0.0;
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
        double in[3][2] = {{0, 0}, {0, 0}, {0, 0}};
#pragma unroll
        for (int c = 0; c < N; ++c) {
            const double gc = c_gauss[N][c];
#pragma unroll
            for (int d = 0; d < N; ++d) {
                const double wy = c_duffy_w[duffy_offset(N) + c * N + d];
                const double ty = c_duffy_t[duffy_offset(N) + c * N + d];  // = gc gd
                const double dx = fma(-gc, ux[d], xo0);
                const double dy = fma(-gc, uy[d], xo1);
                const double dz = fma(-gc, uz[d], xo2);
                const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
                const double dn = DL ? fma(-gc, un[d], xon) : 0.0;
                double kr, ki;
                point_value<KIND, PH>(r2, dn, kappa, phi0, kr, ki);
                // lambda(y) = (1 - c, c - cd, cd): compile-time weights
                const double l0 = wy * (1.0 - gc), l1 = wy * (gc - ty), l2 = wy * ty;
                in[0][0] = fma(l0, kr, in[0][0]);
                in[1][0] = fma(l1, kr, in[1][0]);
                in[2][0] = fma(l2, kr, in[2][0]);
                if (CPLX) {
                    in[0][1] = fma(l0, ki, in[0][1]);
                    in[1][1] = fma(l1, ki, in[1][1]);
                    in[2][1] = fma(l2, ki, in[2][1]);
                }
            }
        }
        const double lx[3] = {wx * (1.0 - s), wx * (s - t), wx * t};
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                acc[3 * a + b][0] = fma(lx[a], in[b][0], acc[3 * a + b][0]);
                if (CPLX) acc[3 * a + b][1] = fma(lx[a], in[b][1], acc[3 * a + b][1]);
            }
    }
}

// geometry in units of 1/kappa (Helmholtz tiers with kappa > 0, as
// disjoint_kernel): the point kernels get kappa = 1, the sums come out as
// S / kappa (single layer) and D / kappa^2 (double layer)
__device__ __forceinline__ void scale_geometry(double kappa, double dO[3], double e1x[3],
                                               double e2x[3], double e1y[3], double e2y[3]) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        dO[c] *= kappa;
        e1x[c] *= kappa;
        e2x[c] *= kappa;
        e1y[c] *= kappa;
        e2y[c] *= kappa;
    }
}

template <int KIND>
__device__ __forceinline__ void p1_unscale(double kappa, double acc[9][2]) {
    const double f = KIND == H_DLP ? kappa * kappa : kappa;
#pragma unroll
    for (int e = 0; e < 9; ++e) {
        acc[e][0] *= f;
        acc[e][1] *= f;
    }
}

template <int KIND>
// entry e of the pair whose entries start at base9 = 9 x (payload index) goes
// to local[pos[base9 + e]] (the scatter plan's sorted position: the
// gather-sum then reads each nonzero's contributions contiguously), or to
// local[base9 + e] without a plan (pos null: index batches)
__device__ __forceinline__ void p1_finish(double acc[9][2], double gx, double gy, bool helm_rot,
                                          double phi0, const uint8_t *px, const uint8_t *py,
                                          double2 *local, const int32_t *pos, int64_t base9) {
    const double g = gx * gy;
    const double scale = (KIND == L_SLP || KIND == L_DLP) ? INV_4PI : 1.0;
    double sn = 0.0, cs = 1.0;
    if (helm_rot) sincos_fast(phi0, sn, cs);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            double re = acc[3 * a + b][0], im = acc[3 * a + b][1];
            if (helm_rot) {  // (re + i im) e^{i phi0}
                const double r = re * cs - im * sn;
                im = fma(re, sn, im * cs);
                re = r;
            }
            if (KIND == L_SLP || KIND == L_DLP) im = 0.0;
            const int64_t e = base9 + 3 * px[a] + py[b];
            local[pos ? (int64_t)pos[e] : e] = make_double2((re * scale) * g, im * g);
        }
}

// unconstrained registers (242, 8 warps/SM): measured faster on the B200 than
// 12 warps/SM with the y loop rolled (34.2 vs 30.6 ms at C4) -- ILP wins here
#ifndef GCABEM_P1_MINB
#define GCABEM_P1_MINB 1
#endif
template <int N, int KIND>
__global__ void __launch_bounds__(DISJOINT_TPB, GCABEM_P1_MINB)
p1_disjoint_kernel(const Chart *__restrict__ charts, const int32_t *__restrict__ T,
                   const TaskDesc *__restrict__ tasks,
                   const int32_t *__restrict__ panels, double2 *__restrict__ local,
                   const int32_t *__restrict__ pos, double kappa) {
    const TaskDesc &td = tasks[blockIdx.x];   // block descriptor + first pair
    const BlockDesc b = td.b;
    const int k = td.k0 + threadIdx.x;
    const bool inb = k < b.nr * b.nc;
    const int i = inb ? k / b.nc : 0;
    const int j = inb ? k - i * b.nc : 0;
    const int tx = panels[b.rows_at + i], ty = panels[b.cols_at + j];
    const int64_t base9 = 9 * (b.base + (int64_t)i * b.ld + j);
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
    double dO[3], e1x[3], e2x[3], e1y[3], e2y[3], n[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        dO[c] = cx->o[c] - cy->o[c];
        e1x[c] = cx->e1[c];
        e2x[c] = cx->e2[c];
        e1y[c] = cy->e1[c];
        e2y[c] = cy->e2[c];
        if (KIND == L_DLP || KIND == H_DLP) n[c] = cy->n[c];
    }
    double dc[3];
#pragma unroll
    for (int c = 0; c < 3; ++c)
        dc[c] = fma(1.0 / 3.0, (2.0 * e1x[c] + e2x[c]) - (2.0 * e1y[c] + e2y[c]), dO[c]);
    constexpr bool HELM = (KIND == H_SLP || KIND == H_DLP);
    const double phi0 = HELM ? kappa * norm3(dc[0], dc[1], dc[2]) : 0.0;
    const double dmax = HELM && active ? kappa * (cx->radius + cy->radius) : 0.0;
    // kappa = 0 takes the full-sincos tier (unscaled geometry)
    const bool tiny = kappa > 0.0 && __all_sync(0xffffffffu, dmax <= TINY_PHASE_MAX);
    const bool smallp = kappa > 0.0 && __all_sync(0xffffffffu, dmax <= SMALL_PHASE_MAX);
    if (!active) {
        // singular pairs are overwritten by the singular pass; keep them 0
        if (inb)
            for (int e = 0; e < 9; ++e)
                local[pos ? (int64_t)pos[base9 + e] : base9 + e] = make_double2(0.0, 0.0);
        return;
    }
    double acc[9][2];
#pragma unroll
    for (int e = 0; e < 9; ++e) acc[e][0] = acc[e][1] = 0.0;
    bool rot = false;
    if constexpr (HELM) {
        const int ph = tiny ? 2 : (smallp ? 1 : 0);
        rot = ph > 0;
        if (ph > 0) {
            scale_geometry(kappa, dO, e1x, e2x, e1y, e2y);
            if (ph == 2)
                p1_disjoint_pair<N, KIND, 2>(dO, e1x, e2x, e1y, e2y, n, 1.0, phi0, acc);
            else
                p1_disjoint_pair<N, KIND, 1>(dO, e1x, e2x, e1y, e2y, n, 1.0, phi0, acc);
            p1_unscale<KIND>(kappa, acc);
        } else {
            p1_disjoint_pair<N, KIND, 0>(dO, e1x, e2x, e1y, e2y, n, kappa, 0.0, acc);
        }
    } else {
        p1_disjoint_pair<N, KIND, 0>(dO, e1x, e2x, e1y, e2y, n, kappa, 0.0, acc);
    }
    const uint8_t id[3] = {0, 1, 2};
    p1_finish<KIND>(acc, cx->gram, cy->gram, rot, phi0, id, id, local, pos, base9);
}

// --- generic rule (singular items, index batches) ---------------------------
// the singular-rule point loop of one pair (rule staged through shared
// memory in chunks; every thread walks the same points)
template <int KIND, int PH>
__device__ __forceinline__ void p1_generic_rule(bool valid, const double dO[3],
                                                const double e1x[3], const double e2x[3],
                                                const double e1y[3], const double e2y[3],
                                                const double ny[3], const double *__restrict__ rule,
                                                int64_t q, double kappa, double phi0,
                                                double acc[9][2]) {
    __shared__ double sr[RULE_CHUNK * 5];
    for (int64_t base = 0; base < q; base += RULE_CHUNK) {
        const int cnt = (int)min((int64_t)RULE_CHUNK, q - base);
        __syncthreads();
        for (int e = threadIdx.x; e < cnt * 5; e += blockDim.x) sr[e] = rule[base * 5 + e];
        __syncthreads();
        if (!valid) continue;
        for (int k = 0; k < cnt; ++k) {
            const double xs = sr[5 * k], xt = sr[5 * k + 1];
            const double ys = sr[5 * k + 2], yt = sr[5 * k + 3], w = sr[5 * k + 4];
            double d[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double xp = fma(xt, e2x[c], fma(xs, e1x[c], dO[c]));
                d[c] = fma(-yt, e2y[c], fma(-ys, e1y[c], xp));
            }
            const double r2 = fma(d[0], d[0], fma(d[1], d[1], d[2] * d[2]));
            double dn = 0.0;
            if (KIND == L_DLP || KIND == H_DLP)
                dn = fma(d[0], ny[0], fma(d[1], ny[1], d[2] * ny[2]));
            double kr, ki;
            point_value<KIND, PH>(r2, dn, kappa, phi0, kr, ki);
            const double lx[3] = {1.0 - xs, xs - xt, xt};
            const double ly[3] = {w * (1.0 - ys), w * (ys - yt), w * yt};
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                const double ur = ly[b] * kr, ui = ly[b] * ki;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    acc[3 * a + b][0] = fma(lx[a], ur, acc[3 * a + b][0]);
                    if (KIND == H_SLP || KIND == H_DLP)
                        acc[3 * a + b][1] = fma(lx[a], ui, acc[3 * a + b][1]);
                }
            }
        }
    }
}

template <int KIND>
__global__ void __launch_bounds__(GENERIC_TPB)
p1_generic_kernel(const double *__restrict__ V, const int32_t *__restrict__ T,
                  const Chart *__restrict__ charts, const SingItem *__restrict__ items, int64_t n,
                  const double *__restrict__ rule, int64_t q, double2 *__restrict__ local,
                  const int32_t *__restrict__ pos, double kappa) {
    const int64_t idx = (int64_t)blockIdx.x * GENERIC_TPB + threadIdx.x;
    const bool valid = idx < n;
    double dO[3] = {0, 0, 0}, e1x[3] = {0, 0, 0}, e2x[3] = {0, 0, 0};
    double e1y[3] = {0, 0, 0}, e2y[3] = {0, 0, 0}, ny[3] = {0, 0, 0};
    double gx = 0.0, gy = 0.0;
    SingItem it;
    if (valid) {
        it = items[idx];
        const int32_t *tx = T + 3 * (int64_t)it.tri_x, *ty = T + 3 * (int64_t)it.tri_y;
        const double *x0 = V + 3 * (int64_t)tx[it.px[0]], *x1 = V + 3 * (int64_t)tx[it.px[1]],
                     *x2 = V + 3 * (int64_t)tx[it.px[2]];
        const double *y0 = V + 3 * (int64_t)ty[it.py[0]], *y1 = V + 3 * (int64_t)ty[it.py[1]],
                     *y2 = V + 3 * (int64_t)ty[it.py[2]];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            dO[c] = x0[c] - y0[c];
            e1x[c] = x1[c] - x0[c];
            e2x[c] = x2[c] - x1[c];
            e1y[c] = y1[c] - y0[c];
            e2y[c] = y2[c] - y1[c];
            ny[c] = charts[it.tri_y].n[c];
        }
        gx = charts[it.tri_x].gram;
        gy = charts[it.tri_y].gram;
    }
    double acc[9][2];
#pragma unroll
    for (int e = 0; e < 9; ++e) acc[e][0] = acc[e][1] = 0.0;
    // Helmholtz phase about the centroid distance, tier CTA-uniform (the
    // rule loop stages shared memory with __syncthreads), as generic_kernel
    constexpr bool HELM = (KIND == H_SLP || KIND == H_DLP);
    double phi0 = 0.0;
    int tier = 0;
    if constexpr (HELM) {
        double dc[3];
#pragma unroll
        for (int c = 0; c < 3; ++c)
            dc[c] = fma(1.0 / 3.0, (2.0 * e1x[c] + e2x[c]) - (2.0 * e1y[c] + e2y[c]), dO[c]);
        phi0 = kappa * norm3(dc[0], dc[1], dc[2]);
        const double rsum = valid ? charts[it.tri_x].radius + charts[it.tri_y].radius : 0.0;
        if (kappa > 0.0 && __syncthreads_and(!valid || kappa * rsum <= TINY_PHASE_MAX))
            tier = 2;
        else if (kappa > 0.0 && __syncthreads_and(!valid || kappa * rsum <= SMALL_PHASE_MAX))
            tier = 1;
    }
    if (tier > 0) {
        scale_geometry(kappa, dO, e1x, e2x, e1y, e2y);
        if (tier == 2)
            p1_generic_rule<KIND, 2>(valid, dO, e1x, e2x, e1y, e2y, ny, rule, q, 1.0, phi0, acc);
        else
            p1_generic_rule<KIND, 1>(valid, dO, e1x, e2x, e1y, e2y, ny, rule, q, 1.0, phi0, acc);
        p1_unscale<KIND>(kappa, acc);
    } else {
        p1_generic_rule<KIND, 0>(valid, dO, e1x, e2x, e1y, e2y, ny, rule, q, kappa, 0.0, acc);
    }
    if (valid) p1_finish<KIND>(acc, gx, gy, tier > 0, phi0, it.px, it.py, local, pos, 9 * it.out);
}

// --- scatter plan and gather-sum --------------------------------------------
// keys of the 9 local entries of every pair (vertex_x * nv + vertex_y), in
// the triangles' stored vertex order (the order the local matrices use)
__global__ void __launch_bounds__(DISJOINT_TPB)
p1_keys_kernel(const int32_t *__restrict__ T, const BlockDesc *__restrict__ blocks,
               const int2 *__restrict__ tasks, const int32_t *__restrict__ panels, int64_t nv,
               uint64_t *__restrict__ keys, int32_t *__restrict__ vals) {
    const int2 task = tasks[blockIdx.x];
    const BlockDesc b = blocks[task.x];
    const int k = task.y + threadIdx.x;
    if (k >= b.nr * b.nc) return;
    const int i = k / b.nc, j = k - i * b.nc;
    const int tx = panels[b.rows_at + i], ty = panels[b.cols_at + j];
    const int64_t p = b.base + (int64_t)i * b.ld + j;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            keys[9 * p + 3 * a + c] = (uint64_t)T[3 * tx + a] * (uint64_t)nv + T[3 * ty + c];
            vals[9 * p + 3 * a + c] = (int32_t)(9 * p + 3 * a + c);
        }
}

__global__ void rowptr_kernel(const uint64_t *__restrict__ ukeys, int64_t nnz, int64_t nv,
                              int64_t *__restrict__ row_ptr, int32_t *__restrict__ col) {
    const int64_t r = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (r <= nv) {  // row_ptr[r] = first unique key >= r * nv
        const uint64_t target = (uint64_t)r * (uint64_t)nv;
        int64_t lo = 0, hi = nnz;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (ukeys[mid] < target) lo = mid + 1; else hi = mid;
        }
        row_ptr[r] = lo;
    }
    if (r < nnz) col[r] = (int32_t)(ukeys[r] % (uint64_t)nv);
}

// nonzero e = the sum of its contributions, stored contiguously in sorted
// order (local[seg[e] .. seg[e + 1])), in that order: deterministic
__global__ void gather_sum_kernel(const int64_t *__restrict__ seg, int64_t nnz,
                                  const double2 *__restrict__ local, double2 *__restrict__ out) {
    const int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (e >= nnz) return;
    double re = 0.0, im = 0.0;
    for (int64_t q = seg[e]; q < seg[e + 1]; ++q) {
        const double2 v = local[q];
        re += v.x;
        im += v.y;
    }
    out[e] = make_double2(re, im);
}

// pos[src[q]] = q: the sorted position of each (pair, entry)
__global__ void invert_perm_kernel(const int32_t *__restrict__ src, int64_t n,
                                   int32_t *__restrict__ pos) {
    const int64_t q = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (q < n) pos[src[q]] = (int32_t)q;
}

// local entries back in pair order (the download of the local matrices)
__global__ void unsort_kernel(const double2 *__restrict__ local, const int32_t *__restrict__ pos,
                              int64_t n, double2 *__restrict__ out) {
    const int64_t k = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (k < n) out[k] = local[pos[k]];
}

template <int N>
cudaError_t launch_p1_disjoint_n(int kind, const Chart *charts, const int32_t *T,
                                 const TaskDesc *tasks, int64_t ntasks,
                                 const int32_t *panels, double2 *local, const int32_t *pos,
                                 double kappa, cudaStream_t s) {
    const dim3 grid((unsigned)ntasks), block(DISJOINT_TPB);
    switch (kind) {
        case L_SLP: p1_disjoint_kernel<N, L_SLP><<<grid, block, 0, s>>>(charts, T, tasks, panels, local, pos, kappa); break;
        case L_DLP: p1_disjoint_kernel<N, L_DLP><<<grid, block, 0, s>>>(charts, T, tasks, panels, local, pos, kappa); break;
        case H_SLP: p1_disjoint_kernel<N, H_SLP><<<grid, block, 0, s>>>(charts, T, tasks, panels, local, pos, kappa); break;
        default:    p1_disjoint_kernel<N, H_DLP><<<grid, block, 0, s>>>(charts, T, tasks, panels, local, pos, kappa); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_p1_disjoint(int kind, int order, const Chart *charts, const int32_t *T,
                               const TaskDesc *tasks, int64_t ntasks,
                               const int32_t *panels, double2 *local, const int32_t *pos,
                               double kappa, cudaStream_t s) {
    if (ntasks <= 0) return cudaSuccess;
    switch (order) {
        case 1: return launch_p1_disjoint_n<1>(kind, charts, T, tasks, ntasks, panels, local, pos, kappa, s);
        case 2: return launch_p1_disjoint_n<2>(kind, charts, T, tasks, ntasks, panels, local, pos, kappa, s);
        case 3: return launch_p1_disjoint_n<3>(kind, charts, T, tasks, ntasks, panels, local, pos, kappa, s);
        case 4: return launch_p1_disjoint_n<4>(kind, charts, T, tasks, ntasks, panels, local, pos, kappa, s);
        case 5: return launch_p1_disjoint_n<5>(kind, charts, T, tasks, ntasks, panels, local, pos, kappa, s);
        case 6: return launch_p1_disjoint_n<6>(kind, charts, T, tasks, ntasks, panels, local, pos, kappa, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_p1_generic(int kind, const double *V, const int32_t *T, const Chart *charts,
                              const SingItem *items, int64_t n, const double *rule, int64_t q,
                              double2 *local, const int32_t *pos, double kappa, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const dim3 grid((unsigned)((n + GENERIC_TPB - 1) / GENERIC_TPB)), block(GENERIC_TPB);
    switch (kind) {
        case L_SLP: p1_generic_kernel<L_SLP><<<grid, block, 0, s>>>(V, T, charts, items, n, rule, q, local, pos, kappa); break;
        case L_DLP: p1_generic_kernel<L_DLP><<<grid, block, 0, s>>>(V, T, charts, items, n, rule, q, local, pos, kappa); break;
        case H_SLP: p1_generic_kernel<H_SLP><<<grid, block, 0, s>>>(V, T, charts, items, n, rule, q, local, pos, kappa); break;
        default:    p1_generic_kernel<H_DLP><<<grid, block, 0, s>>>(V, T, charts, items, n, rule, q, local, pos, kappa); break;
    }
    return cudaGetLastError();
}

std::mutex g_p1_rule_mutex;
std::set<std::pair<int, int>> g_p1_rules;

cudaError_t ensure_p1_rule(int device, int order, const double *g, const double *gw) {
    std::lock_guard<std::mutex> lock(g_p1_rule_mutex);
    if (g_p1_rules.count({device, order})) return cudaSuccess;
    cudaError_t e = upload_tables(order, g, gw);  // this unit's constant tables
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e == cudaSuccess) g_p1_rules.insert({device, order});
    return e;
}

}  // namespace

struct gcabem_p1_s {
    gcabem_layout_t L = nullptr;
    int kind = 0, order = 0;
    double kappa = 0.0;
    cudaStream_t stream = nullptr;
    DevBuf<double> srule[3];
    int64_t sq[3] = {0, 0, 0};
    PoolBuf<double2> local;       // 9 per pair
    DevBuf<int64_t> row_ptr, seg; // CSR rows (nv + 1), contribution segments (nnz + 1)
    DevBuf<int32_t> col;          // CSR columns (nnz)
    DevBuf<int32_t> pos;          // sorted position of each (pair, entry) (9 P)
    DevBuf<double2> values;       // nnz
    int64_t nv = 0, nnz = 0;
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
};

extern "C" {

int gcabem_p1_create(gcabem_layout_t L, int equation, int layer, double kappa, int disjoint_n,
                     const double *gauss_pts, const double *gauss_wts, const int64_t *sq,
                     const double *const *srule, gcabem_p1_t *out) {
    if (!L || !out) return gcabem_internal_error(GCABEM_ERR_ARG, "null argument");
    *out = nullptr;
    if (!(equation == 0 || equation == 1) || !(layer == 0 || layer == 1) ||
        (equation == 1 && kappa < 0.0))
        return gcabem_internal_error(GCABEM_ERR_ARG, "bad kernel specification");
    if (disjoint_n < 1 || disjoint_n > 6)
        return gcabem_internal_error(GCABEM_ERR_ARG, "P1 disjoint order outside [1, 6]");
    gcabem_mesh_t mesh = L->mesh;
    const int64_t P = L->payload_len;
    if (9 * P >= (int64_t(1) << 31))
        return gcabem_internal_error(GCABEM_ERR_ARG, "P1 near field too large for one plan");
    Trace tr("p1_create");
    auto *p = new gcabem_p1_s();
    p->L = L;
    ++L->refs;
    p->kind = kind_of(equation, layer);
    p->order = disjoint_n;
    p->kappa = kappa;
    p->nv = mesh->nv;
    cudaError_t e = cudaSetDevice(mesh->device);
    if (e == cudaSuccess) e = ensure_p1_rule(mesh->device, disjoint_n, gauss_pts, gauss_wts);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking);
    cudaStream_t s = p->stream;
    for (int c = 0; c < 3 && e == cudaSuccess; ++c) {
        p->sq[c] = sq ? sq[c] : 0;
        if (L->case_at[c + 1] > L->case_at[c]) {
            if (p->sq[c] <= 0) {
                delete p;
                return gcabem_internal_error(GCABEM_ERR_ARG, "singular items without a rule");
            }
            e = p->srule[c].upload(srule[c], 5 * p->sq[c], s);
        }
    }
    for (int k = 0; k < 3 && e == cudaSuccess; ++k) e = cudaEventCreate(&p->ev[k]);
    if (e == cudaSuccess) e = pool_init(mesh->device);
    if (e == cudaSuccess) e = p->local.alloc(9 * P, s);
    tr.mark("rules+local");
    // scatter plan: sort the 9 P entry keys, run-length encode, row pointers
    const int64_t E = 9 * P;
    // plan temporaries from the device pool (stream-ordered: tens of GB at C4,
    // whose cudaMalloc/cudaFree would each synchronise the device)
    PoolBuf<uint64_t> keys, keys_out, ukeys;
    PoolBuf<int32_t> vals, counts;
    PoolBuf<int64_t> d_nnz;
    PoolBuf<char> tmp;
    int end_bit = 1;
    while (end_bit < 64 && ((uint64_t)1 << end_bit) < (uint64_t)mesh->nv * (uint64_t)mesh->nv)
        ++end_bit;
    if (e == cudaSuccess) e = keys.alloc(std::max<int64_t>(E, 1), s);
    if (e == cudaSuccess) e = keys_out.alloc(std::max<int64_t>(E, 1), s);
    if (e == cudaSuccess) e = vals.alloc(std::max<int64_t>(E, 1), s);
    PoolBuf<int32_t> src;   // sorted contributions: inverted into p->pos below
    if (e == cudaSuccess) e = src.alloc(std::max<int64_t>(E, 1), s);
    if (e == cudaSuccess && L->ntasks > 0) {
        p1_keys_kernel<<<(unsigned)L->ntasks, DISJOINT_TPB, 0, s>>>(
            mesh->T.p, L->blocks.p, L->tasks.p, L->panels.p, mesh->nv, keys.p, vals.p);
        e = cudaGetLastError();
    }
    size_t tb = 0, tb2 = 0, tb3 = 0;
    if (e == cudaSuccess)
        e = cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, keys_out.p, vals.p, src.p,
                                            (int)E, 0, end_bit, s);
    if (e == cudaSuccess) e = ukeys.alloc(std::max<int64_t>(E, 1), s);
    if (e == cudaSuccess) e = counts.alloc(E + 1, s);
    if (e == cudaSuccess) e = d_nnz.alloc(1, s);
    if (e == cudaSuccess)
        e = cub::DeviceRunLengthEncode::Encode(nullptr, tb2, keys_out.p, ukeys.p, counts.p,
                                               d_nnz.p, (int)E, s);
    if (e == cudaSuccess) e = p->seg.alloc(E + 1);
    if (e == cudaSuccess)
        e = cub::DeviceScan::ExclusiveSum(nullptr, tb3, counts.p, p->seg.p, (int)E + 1, s);
    if (e == cudaSuccess) e = tmp.alloc(std::max(tb, std::max(tb2, tb3)), s);
    if (e == cudaSuccess && E > 0)
        e = cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.p, keys_out.p, vals.p, src.p,
                                            (int)E, 0, end_bit, s);
    if (e == cudaSuccess && E > 0)
        e = cub::DeviceRunLengthEncode::Encode(tmp.p, tb2, keys_out.p, ukeys.p, counts.p,
                                               d_nnz.p, (int)E, s);
    int64_t nnz = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&nnz, d_nnz.p, 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    tr.mark("sort+rle");
    if (E == 0) nnz = 0;
    // segment offsets: exclusive scan of the run lengths (nnz + 1 entries;
    // counts[nnz] is zeroed first so the last offset is the total)
    if (e == cudaSuccess) e = cudaMemsetAsync(counts.p + nnz, 0, sizeof(int32_t), s);
    if (e == cudaSuccess)
        e = cub::DeviceScan::ExclusiveSum(tmp.p, tb3, counts.p, p->seg.p, (int)nnz + 1, s);
    p->nnz = nnz;
    if (e == cudaSuccess) e = p->row_ptr.alloc(p->nv + 1);
    if (e == cudaSuccess) e = p->col.alloc(std::max<int64_t>(nnz, 1));
    if (e == cudaSuccess) e = p->values.alloc(std::max<int64_t>(nnz, 1));
    if (e == cudaSuccess) {
        const int64_t n = std::max<int64_t>(nnz, p->nv + 1);
        rowptr_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ukeys.p, nnz, p->nv,
                                                                   p->row_ptr.p, p->col.p);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = p->pos.alloc(std::max<int64_t>(E, 1));
    if (e == cudaSuccess && E > 0) {
        invert_perm_kernel<<<(unsigned)((E + 255) / 256), 256, 0, s>>>(src.p, E, p->pos.p);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    tr.mark("csr");
    if (e != cudaSuccess) {
        gcabem_p1_destroy(p);
        return gcabem_internal_error(GCABEM_ERR_CUDA,
                                     (std::string("p1_create: ") + cudaGetErrorString(e)).c_str());
    }
    *out = p;
    return GCABEM_OK;
}

int gcabem_p1_execute(gcabem_p1_t p) {
    if (!p) return gcabem_internal_error(GCABEM_ERR_ARG, "null plan");
    gcabem_layout_t L = p->L;
    gcabem_mesh_t m = L->mesh;
    cudaStream_t s = p->stream;
    cudaError_t e = cudaSetDevice(m->device);
    if (e == cudaSuccess) e = cudaEventRecord(p->ev[0], s);
    if (e == cudaSuccess)
        e = launch_p1_disjoint(p->kind, p->order, m->charts.p, m->T.p, L->tdesc.p,
                               L->ntasks, L->panels.p, p->local.p, p->pos.p, p->kappa, s);
    for (int c = 0; c < 3 && e == cudaSuccess; ++c) {
        const int64_t n = L->case_at[c + 1] - L->case_at[c];
        if (n > 0)
            e = launch_p1_generic(p->kind, m->V.p, m->T.p, m->charts.p, L->items.p + L->case_at[c],
                                  n, p->srule[c].p, p->sq[c], p->local.p, p->pos.p, p->kappa,
                                  s);
    }
    if (e == cudaSuccess) e = cudaEventRecord(p->ev[1], s);
    if (e == cudaSuccess && p->nnz > 0) {
        gather_sum_kernel<<<(unsigned)((p->nnz + 255) / 256), 256, 0, s>>>(
            p->seg.p, p->nnz, p->local.p, p->values.p);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaEventRecord(p->ev[2], s);
    if (e != cudaSuccess)
        return gcabem_internal_error(GCABEM_ERR_CUDA,
                                     (std::string("p1_execute: ") + cudaGetErrorString(e)).c_str());
    return GCABEM_OK;
}

int gcabem_p1_info(gcabem_p1_t p, int64_t *info4, float *ms2) {
    if (!p || !info4) return gcabem_internal_error(GCABEM_ERR_ARG, "null argument");
    info4[0] = p->nv;
    info4[1] = p->nnz;
    info4[2] = p->L->payload_len;
    info4[3] = p->L->case_at[3];
    if (ms2) {
        cudaSetDevice(p->L->mesh->device);
        if (cudaEventSynchronize(p->ev[2]) != cudaSuccess ||
            cudaEventElapsedTime(&ms2[0], p->ev[0], p->ev[1]) != cudaSuccess ||
            cudaEventElapsedTime(&ms2[1], p->ev[1], p->ev[2]) != cudaSuccess)
            ms2[0] = ms2[1] = -1.0f;
    }
    return GCABEM_OK;
}

int gcabem_p1_download(gcabem_p1_t p, int64_t *row_ptr, int32_t *col, double *values,
                       double *local) {
    if (!p) return gcabem_internal_error(GCABEM_ERR_ARG, "null plan");
    cudaStream_t s = p->stream;
    cudaError_t e = cudaSetDevice(p->L->mesh->device);
    if (e == cudaSuccess && row_ptr)
        e = cudaMemcpyAsync(row_ptr, p->row_ptr.p, 8 * (p->nv + 1), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && col && p->nnz)
        e = cudaMemcpyAsync(col, p->col.p, 4 * p->nnz, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && values && p->nnz)
        e = cudaMemcpyAsync(values, p->values.p, 16 * p->nnz, cudaMemcpyDeviceToHost, s);
    PoolBuf<double2> unsorted;   // the local matrices in pair order
    const int64_t E = 9 * p->L->payload_len;
    if (e == cudaSuccess && local && E) e = unsorted.alloc(E, s);
    if (e == cudaSuccess && local && E) {
        unsort_kernel<<<(unsigned)((E + 255) / 256), 256, 0, s>>>(p->local.p, p->pos.p, E,
                                                                 unsorted.p);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess && local && E)
        e = cudaMemcpyAsync(local, unsorted.p, 16 * E, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess)
        return gcabem_internal_error(GCABEM_ERR_CUDA,
                                     (std::string("p1_download: ") + cudaGetErrorString(e)).c_str());
    return GCABEM_OK;
}

int gcabem_p1_destroy(gcabem_p1_t p) {
    if (!p) return GCABEM_OK;
    cudaSetDevice(p->L->mesh->device);
    if (p->stream) cudaStreamSynchronize(p->stream);
    for (auto &e : p->ev)
        if (e) cudaEventDestroy(e);
    cudaStream_t s = p->stream;
    gcabem_layout_t L = p->L;
    delete p;
    if (s) cudaStreamDestroy(s);
    gcabem_layout_release(L);
    return GCABEM_OK;
}

// Index-based P1 local matrices for caller-supplied pairs and rule (tests,
// the reference's per-pair integrate_pair with P1 bases): out is n x 9
// complex128 in the triangles' stored vertex order.
int gcabem_p1_batch(gcabem_mesh_t mesh, int equation, int layer, double kappa, int64_t n,
                    const int64_t *tri_x, const int64_t *tri_y, const uint8_t *perm_x,
                    const uint8_t *perm_y, int64_t nq, const double *xs, const double *ys,
                    const double *w, double *out) {
    if (!mesh || (n > 0 && (!tri_x || !tri_y || !out)))
        return gcabem_internal_error(GCABEM_ERR_ARG, "null argument");
    if (n == 0) return GCABEM_OK;
    std::vector<SingItem> items(n);
    for (int64_t i = 0; i < n; ++i) {
        if (tri_x[i] < 0 || tri_x[i] >= mesh->nt || tri_y[i] < 0 || tri_y[i] >= mesh->nt)
            return gcabem_internal_error(GCABEM_ERR_ARG, "triangle index out of range");
        SingItem &it = items[i];
        it.out = i;
        it.tri_x = (int32_t)tri_x[i];
        it.tri_y = (int32_t)tri_y[i];
        for (int k = 0; k < 3; ++k) {
            it.px[k] = perm_x ? perm_x[3 * i + k] : (uint8_t)k;
            it.py[k] = perm_y ? perm_y[3 * i + k] : (uint8_t)k;
            if (it.px[k] > 2 || it.py[k] > 2)
                return gcabem_internal_error(GCABEM_ERR_ARG, "bad permutation");
        }
        it.pad[0] = it.pad[1] = 0;
    }
    std::vector<double> rule(5 * nq);
    for (int64_t k = 0; k < nq; ++k) {
        rule[5 * k] = xs[2 * k];
        rule[5 * k + 1] = xs[2 * k + 1];
        rule[5 * k + 2] = ys[2 * k];
        rule[5 * k + 3] = ys[2 * k + 1];
        rule[5 * k + 4] = w[k];
    }
    cudaStream_t s = mesh->stream;
    DevBuf<SingItem> di;
    DevBuf<double> dr;
    DevBuf<double2> dout;
    cudaError_t e = cudaSetDevice(mesh->device);
    if (e == cudaSuccess) e = di.upload(items.data(), n, s);
    if (e == cudaSuccess) e = dr.upload(rule.data(), rule.size(), s);
    if (e == cudaSuccess) e = dout.alloc(9 * n);
    if (e == cudaSuccess)
        e = launch_p1_generic(kind_of(equation, layer), mesh->V.p, mesh->T.p, mesh->charts.p, di.p,
                              n, dr.p, nq, dout.p, nullptr, kappa, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(out, dout.p, 16 * 9 * n, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess)
        return gcabem_internal_error(GCABEM_ERR_CUDA,
                                     (std::string("p1_batch: ") + cudaGetErrorString(e)).c_str());
    return GCABEM_OK;
}

}  // extern "C"
