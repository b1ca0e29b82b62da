// Device-resident compressed operator and its matrix-vector product
// (reference h2.matvec, pkg/src/gcabem/h2.py:49-71):
//
//   y = sum over block-tree leaves (t, s):
//         dense       y[t] += P x[s]
//         admissible  y[t] += V_t (P (V_s^T x[s]))      (W_s = conj(V_s))
//
// in the permuted (cluster) index space, x and y permuted by the column /
// row tree. Every stage is a gather with a FIXED summation order, so the
// product is bitwise reproducible run to run (no atomics):
//
//   1 xp = x[col_perm]
//   2 xs_s = V_s^T xp[s]                 per column operator (once, not per leaf)
//   3 c_l  = P_l xp[s]   (dense)         per leaf row
//     w_l  = P_l xs_s    (admissible)
//   4 z_t  = sum_l w_l                   per row operator, leaves in preorder
//   5 u_t  = V_t z_t                     per row operator row
//   6 yp_i = sum of c_l[i - t0] and u_t[i - t0] over the leaves / operators
//            covering i, in a fixed (host-built CSR) order
//   7 y[row_perm] = yp
//
// HBM traffic per product: the payload once, the bases twice, O(n) vectors.
#include <algorithm>
#include <string>
#include <vector>

#include "internal.h"

using namespace gcabem;

namespace {

constexpr int MV_TPB = 128;

__global__ void gather_kernel(const double2 *__restrict__ x, const int32_t *__restrict__ perm,
                              int64_t n, double2 *__restrict__ xp) {
    const int64_t i = (int64_t)blockIdx.x * MV_TPB + threadIdx.x;
    if (i < n) xp[i] = x[perm[i]];
}

__global__ void scatter_kernel(const double2 *__restrict__ yp, const int32_t *__restrict__ perm,
                               int64_t n, double2 *__restrict__ y) {
    const int64_t i = (int64_t)blockIdx.x * MV_TPB + threadIdx.x;
    if (i < n) y[perm[i]] = yp[i];
}

__device__ __forceinline__ double2 cmac(double2 acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
    acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
    return acc;
}

// xs = M^T v (M row-major nrows x width, width <= TM_MAX), split into
// tasks of TM_ROWS rows: warp w of the task's CTA takes rows w, w + 4, ...;
// lane l owns components l, l + 32, ... (a row read is coalesced); the
// warps' partials are added in warp order into the task's partial vector,
// and treduce_kernel sums the tasks of an item in task order -- fixed
// association, deterministic, and a large cluster spreads over many CTAs.
constexpr int TM_MAX = 128;
constexpr int TM_ROWS = 128;
__global__ void __launch_bounds__(MV_TPB)
tmatvec_kernel(const int64_t *__restrict__ task_item, const int32_t *__restrict__ task_r0,
               int64_t ntasks, const int64_t *__restrict__ m_at,
               const int32_t *__restrict__ nrows, const int32_t *__restrict__ width,
               const int64_t *__restrict__ v_at, const int64_t *__restrict__ part_at,
               const double2 *__restrict__ M, const double2 *__restrict__ v,
               double2 *__restrict__ part) {
    __shared__ double2 sp[MV_TPB / 32][TM_MAX];
    const int64_t t = blockIdx.x;
    if (t >= ntasks) return;
    const int64_t it = task_item[t];
    const int w = width[it], n = nrows[it];
    const int r0 = task_r0[t], r1 = min(n, r0 + TM_ROWS);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double2 *Mi = M + m_at[it];
    const double2 *vi = v + v_at[it];
    double2 acc[TM_MAX / 32];
#pragma unroll
    for (int q = 0; q < TM_MAX / 32; ++q) acc[q] = make_double2(0.0, 0.0);
    for (int i = r0 + warp; i < r1; i += MV_TPB / 32) {
        const double2 x = vi[i];
#pragma unroll
        for (int q = 0; q < TM_MAX / 32; ++q)
            if (lane + 32 * q < w) acc[q] = cmac(acc[q], Mi[(int64_t)i * w + lane + 32 * q], x);
    }
#pragma unroll
    for (int q = 0; q < TM_MAX / 32; ++q) sp[warp][lane + 32 * q] = acc[q];
    __syncthreads();
    for (int k = threadIdx.x; k < w; k += MV_TPB) {
        double2 s = sp[0][k];
#pragma unroll
        for (int q = 1; q < MV_TPB / 32; ++q) {
            s.x += sp[q][k].x;
            s.y += sp[q][k].y;
        }
        part[part_at[t] + k] = s;
    }
}

// out[out_at[it] + k] = sum over the item's tasks (in order) of their partials
__global__ void treduce_kernel(const int64_t *__restrict__ item_task_at,
                               const int64_t *__restrict__ part_at,
                               const int32_t *__restrict__ width,
                               const int64_t *__restrict__ out_at, const int64_t *__restrict__ ek_at,
                               int64_t nitems, int64_t nk, const double2 *__restrict__ part,
                               double2 *__restrict__ out) {
    const int64_t e = (int64_t)blockIdx.x * MV_TPB + threadIdx.x;
    if (e >= nk) return;
    // item of component e: binary search in ek_at (prefix of widths)
    int64_t lo = 0, hi = nitems;
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (ek_at[mid] <= e) lo = mid; else hi = mid;
    }
    const int64_t it = lo;
    const int k = (int)(e - ek_at[it]);
    double2 s = make_double2(0.0, 0.0);
    for (int64_t t = item_task_at[it]; t < item_task_at[it + 1]; ++t) {
        const double2 p = part[part_at[t] + k];
        s.x += p.x;
        s.y += p.y;
    }
    out[out_at[it] + k] = s;
}

// out[out_at[it] + r] = sum_j M[r, j] v[v_at + j] (M row-major rows x cols):
// RPG lanes per row over the flattened rows of the batch (tasks are rows, in
// item order): lane g of a row group reads columns g, g + RPG, ..., so one
// load instruction covers 32 / RPG rows x RPG consecutive elements (full
// 128 B segments), then a fixed butterfly over the group -- deterministic.
constexpr int RPG = 8;
__global__ void __launch_bounds__(MV_TPB)
matvec_kernel(const int64_t *__restrict__ task_item, const int32_t *__restrict__ task_r0,
              int64_t ntasks, const int64_t *__restrict__ m_at, const int32_t *__restrict__ rows,
              const int32_t *__restrict__ cols, const int64_t *__restrict__ v_at,
              const int64_t *__restrict__ out_at, const double2 *__restrict__ M,
              const double2 *__restrict__ v, double2 *__restrict__ out) {
    const int64_t gt = (int64_t)blockIdx.x * MV_TPB + threadIdx.x;
    const int64_t t = gt / RPG;
    const int g = (int)(gt % RPG);
    const bool live = t < ntasks;
    double2 acc = make_double2(0.0, 0.0);
    int64_t it = 0;
    int r = 0;
    if (live) {
        it = task_item[t];
        r = task_r0[t];
        const int nc = cols[it];
        const double2 *Mr = M + m_at[it] + (int64_t)r * nc;
        const double2 *vv = v + v_at[it];
        for (int j = g; j < nc; j += RPG) acc = cmac(acc, Mr[j], vv[j]);
    }
#pragma unroll
    for (int o = RPG / 2; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if (live && g == 0) out[out_at[it] + r] = acc;
}

// CSR gather-sum: out[i] = sum_{p in [at[i], at[i+1])} src[idx[p]] (in order)
__global__ void csr_sum_kernel(const int64_t *__restrict__ at, const int64_t *__restrict__ idx,
                               int64_t n, const double2 *__restrict__ src,
                               double2 *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * MV_TPB + threadIdx.x;
    if (i >= n) return;
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t p = at[i]; p < at[i + 1]; ++p) {
        const double2 v = src[idx[p]];
        acc.x += v.x;
        acc.y += v.y;
    }
    out[i] = acc;
}

// A batch of small products described on the host: items with matrix offset,
// shape, input offset, output offset; tasks of MV_TPB rows (or components).
struct Batch {
    std::vector<int64_t> m_at, v_at, out_at;
    std::vector<int32_t> rows, cols;
    std::vector<int64_t> task_item;
    std::vector<int32_t> task_r0;
    DevBuf<int64_t> d_m_at, d_v_at, d_out_at, d_task_item;
    DevBuf<int32_t> d_rows, d_cols, d_task_r0;
    // tasks_over rows (or 1 task per item when step <= 0), `step` per task
    void add(int64_t m, int32_t r, int32_t c, int64_t v, int64_t o, int32_t tasks_over,
             int32_t step) {
        const int64_t it = (int64_t)m_at.size();
        m_at.push_back(m);
        rows.push_back(r);
        cols.push_back(c);
        v_at.push_back(v);
        out_at.push_back(o);
        if (step <= 0) {
            task_item.push_back(it);
            task_r0.push_back(0);
            return;
        }
        for (int32_t r0 = 0; r0 < tasks_over; r0 += step) {
            task_item.push_back(it);
            task_r0.push_back(r0);
        }
    }
    cudaError_t upload(cudaStream_t s) {
        cudaError_t e = d_m_at.upload(m_at.data(), m_at.size(), s);
        if (e == cudaSuccess) e = d_v_at.upload(v_at.data(), v_at.size(), s);
        if (e == cudaSuccess) e = d_out_at.upload(out_at.data(), out_at.size(), s);
        if (e == cudaSuccess) e = d_rows.upload(rows.data(), rows.size(), s);
        if (e == cudaSuccess) e = d_cols.upload(cols.data(), cols.size(), s);
        if (e == cudaSuccess) e = d_task_item.upload(task_item.data(), task_item.size(), s);
        if (e == cudaSuccess) e = d_task_r0.upload(task_r0.data(), task_r0.size(), s);
        return e;
    }
    int64_t ntasks() const { return (int64_t)task_item.size(); }
};

}  // namespace

struct gcabem_h2_s {
    int device = 0;
    int64_t nrows = 0, ncols = 0;
    cudaStream_t stream = nullptr;
    DevBuf<double2> payload, V, xh, xp, xs, yp, cbuf, wbuf, zbuf;
    DevBuf<int32_t> row_perm, col_perm;
    DevBuf<int64_t> z_at, z_idx, y_at, y_idx;
    Batch colop;   // xs_s = V_s^T xp[s]            (tmatvec, TM_ROWS-row tasks)
    DevBuf<int64_t> d_part_at, d_item_task_at, d_ek_at;
    DevBuf<double2> part;
    int64_t nk = 0;
    Batch leafmv;  // dense leaves: c = P xp[s]      (matvec)
    Batch coup;    // admissible leaves: w = P xs_s  (matvec)
    Batch rowop;   // u_t = V_t z_t                  (matvec)
    int64_t nrowops = 0, nz = 0;
    double bytes_per_product = 0.0;
};

extern "C" {

int gcabem_h2_create(int device, int64_t nrows, int64_t ncols, const int64_t *row_perm,
                     const int64_t *col_perm, int64_t nleaves, const int64_t *leaf_desc,
                     const int64_t *leaf_base, int64_t payload_len, const double *payload,
                     int64_t nrowops, const int64_t *rowop_desc, int64_t ncolops,
                     const int64_t *colop_desc, int64_t v_len, const double *V,
                     gcabem_h2_t *out) {
    if (!out || nrows <= 0 || ncols <= 0 || nleaves < 0 || nrowops < 0 || ncolops < 0)
        return gcabem_internal_error(GCABEM_ERR_ARG, "h2_create: bad arguments");
    *out = nullptr;
    auto fail = [](const std::string &m) { return gcabem_internal_error(GCABEM_ERR_ARG, m.c_str()); };
    // operator descriptors {start, size, rank, v_offset}; leaf descriptors
    // {row_start, row_size, col_start, col_size, dense, row_op, col_op}
    for (int64_t o = 0; o < nrowops + ncolops; ++o) {
        const int64_t *d = o < nrowops ? rowop_desc + 4 * o : colop_desc + 4 * (o - nrowops);
        const int64_t lim = o < nrowops ? nrows : ncols;
        if (d[0] < 0 || d[1] < 1 || d[0] + d[1] > lim || d[2] < 1 || d[3] < 0 ||
            d[3] + d[1] * d[2] > v_len)
            return fail("h2_create: operator descriptor out of bounds");
    }
    auto *H = new gcabem_h2_s();
    H->device = device;
    H->nrows = nrows;
    H->ncols = ncols;
    H->nrowops = nrowops;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&H->stream, cudaStreamNonBlocking);
    cudaStream_t s = H->stream;
    // column operators: xs offsets
    std::vector<int64_t> xs_at(ncolops + 1, 0);
    for (int64_t o = 0; o < ncolops; ++o) {
        const int64_t *d = colop_desc + 4 * o;
        xs_at[o + 1] = xs_at[o] + d[2];
        if (d[2] > TM_MAX) {
            delete H;
            return fail("h2_create: rank above 128");
        }
        H->colop.add(d[3], (int32_t)d[1], (int32_t)d[2], d[0], xs_at[o], (int32_t)d[1], TM_ROWS);
    }
    // leaves: dense rows into cbuf, admissible rows into wbuf
    std::vector<int64_t> c_at(nleaves, -1), w_at(nleaves, -1);
    int64_t nc_total = 0, nw_total = 0;
    std::vector<std::vector<int64_t>> row_leaves(nrowops);  // admissible leaves per row op
    for (int64_t l = 0; l < nleaves; ++l) {
        const int64_t *d = leaf_desc + 7 * l;
        const int64_t r0 = d[0], nr = d[1], c0 = d[2], ncl = d[3], dense = d[4];
        if (r0 < 0 || nr < 1 || r0 + nr > nrows || c0 < 0 || ncl < 1 || c0 + ncl > ncols) {
            delete H;
            return fail("h2_create: leaf cluster range out of bounds");
        }
        if (dense) {
            if (leaf_base[l] < 0 || leaf_base[l] + nr * ncl > payload_len) {
                delete H;
                return fail("h2_create: dense leaf payload out of bounds");
            }
            c_at[l] = nc_total;
            H->leafmv.add(leaf_base[l], (int32_t)nr, (int32_t)ncl, c0, nc_total, (int32_t)nr,
                          1);
            nc_total += nr;
        } else {
            const int64_t ro = d[5], co = d[6];
            if (ro < 0 || ro >= nrowops || co < 0 || co >= ncolops) {
                delete H;
                return fail("h2_create: admissible leaf without operators");
            }
            const int64_t kr = rowop_desc[4 * ro + 2], kc = colop_desc[4 * co + 2];
            if (leaf_base[l] < 0 || leaf_base[l] + kr * kc > payload_len) {
                delete H;
                return fail("h2_create: coupling payload out of bounds");
            }
            w_at[l] = nw_total;
            // input: xs of the column operator; offset is into xs, flagged by
            // a separate batch pointer below (the leaf batch reads xp for
            // dense rows and xs for coupling rows: two launches)
            row_leaves[ro].push_back(l);
            nw_total += kr;
        }
    }
    // admissible leaves as their own batch over xs
    Batch &coup = H->coup;
    for (int64_t l = 0; l < nleaves; ++l) {
        if (w_at[l] < 0) continue;
        const int64_t *d = leaf_desc + 7 * l;
        const int64_t ro = d[5], co = d[6];
        const int64_t kr = rowop_desc[4 * ro + 2], kc = colop_desc[4 * co + 2];
        coup.add(leaf_base[l], (int32_t)kr, (int32_t)kc, xs_at[co], w_at[l], (int32_t)kr,
                 1);
    }
    // row operators: z_t = sum of w over its leaves (preorder), u_t = V_t z_t
    std::vector<int64_t> z_at_h(1, 0), z_idx_h, zoff(nrowops + 1, 0);
    for (int64_t o = 0; o < nrowops; ++o) {
        const int64_t k = rowop_desc[4 * o + 2];
        zoff[o + 1] = zoff[o] + k;
        for (int64_t a = 0; a < k; ++a) {
            for (int64_t l : row_leaves[o]) z_idx_h.push_back(w_at[l] + a);
            z_at_h.push_back((int64_t)z_idx_h.size());
        }
    }
    H->nz = zoff[nrowops];
    std::vector<int64_t> u_at(nrowops);
    int64_t nu_total = 0;
    for (int64_t o = 0; o < nrowops; ++o) {
        const int64_t *d = rowop_desc + 4 * o;
        u_at[o] = nu_total;
        H->rowop.add(d[3], (int32_t)d[1], (int32_t)d[2], zoff[o], nc_total + nu_total,
                     (int32_t)d[1], 1);
        nu_total += d[1];
    }
    // output CSR over permuted rows: dense leaf rows (preorder), then row
    // operators (operator order); both write into one contribution buffer
    // [c (dense rows) | u (operator rows)]
    std::vector<std::vector<int64_t>> cover(nrows);
    for (int64_t l = 0; l < nleaves; ++l) {
        if (c_at[l] < 0) continue;
        const int64_t *d = leaf_desc + 7 * l;
        for (int64_t i = 0; i < d[1]; ++i) cover[d[0] + i].push_back(c_at[l] + i);
    }
    for (int64_t o = 0; o < nrowops; ++o) {
        const int64_t *d = rowop_desc + 4 * o;
        if (row_leaves[o].empty()) continue;
        for (int64_t i = 0; i < d[1]; ++i) cover[d[0] + i].push_back(nc_total + u_at[o] + i);
    }
    std::vector<int64_t> y_at_h(nrows + 1, 0), y_idx_h;
    for (int64_t i = 0; i < nrows; ++i) {
        y_idx_h.insert(y_idx_h.end(), cover[i].begin(), cover[i].end());
        y_at_h[i + 1] = (int64_t)y_idx_h.size();
    }
    std::vector<int32_t> rp(nrows), cp(ncols);
    for (int64_t i = 0; i < nrows; ++i) rp[i] = (int32_t)row_perm[i];
    for (int64_t i = 0; i < ncols; ++i) cp[i] = (int32_t)col_perm[i];
    // device state
    if (e == cudaSuccess)
        e = H->payload.upload(reinterpret_cast<const double2 *>(payload), payload_len, s);
    if (e == cudaSuccess) e = H->V.upload(reinterpret_cast<const double2 *>(V), v_len, s);
    if (e == cudaSuccess) e = H->row_perm.upload(rp.data(), rp.size(), s);
    if (e == cudaSuccess) e = H->col_perm.upload(cp.data(), cp.size(), s);
    if (e == cudaSuccess) e = H->xh.alloc(ncols);
    if (e == cudaSuccess) e = H->xp.alloc(ncols);
    if (e == cudaSuccess) e = H->xs.alloc(std::max<int64_t>(xs_at[ncolops], 1));
    if (e == cudaSuccess) e = H->yp.alloc(nrows);
    if (e == cudaSuccess) e = H->cbuf.alloc(std::max<int64_t>(nc_total + nu_total, 1));
    if (e == cudaSuccess) e = H->wbuf.alloc(std::max<int64_t>(nw_total, 1));
    if (e == cudaSuccess) e = H->zbuf.alloc(std::max<int64_t>(H->nz, 1));
    if (e == cudaSuccess) e = H->z_at.upload(z_at_h.data(), z_at_h.size(), s);
    if (e == cudaSuccess) e = H->z_idx.upload(z_idx_h.data(), std::max<size_t>(z_idx_h.size(), 1), s);
    if (e == cudaSuccess) e = H->y_at.upload(y_at_h.data(), y_at_h.size(), s);
    if (e == cudaSuccess) e = H->y_idx.upload(y_idx_h.data(), std::max<size_t>(y_idx_h.size(), 1), s);
    if (e == cudaSuccess) e = H->colop.upload(s);
    {   // partial-sum layout of the chunked transposed products
        const Batch &b = H->colop;
        std::vector<int64_t> part_at(b.task_item.size() + 1, 0), item_task_at(ncolops + 1, 0);
        for (size_t t = 0; t < b.task_item.size(); ++t) {
            part_at[t + 1] = part_at[t] + b.cols[b.task_item[t]];
            item_task_at[b.task_item[t] + 1] = (int64_t)t + 1;
        }
        for (int64_t o = 0; o < ncolops; ++o)
            item_task_at[o + 1] = std::max(item_task_at[o + 1], item_task_at[o]);
        H->nk = xs_at[ncolops];
        if (e == cudaSuccess) e = H->d_part_at.upload(part_at.data(), part_at.size(), s);
        if (e == cudaSuccess) e = H->d_item_task_at.upload(item_task_at.data(), item_task_at.size(), s);
        if (e == cudaSuccess) e = H->d_ek_at.upload(xs_at.data(), xs_at.size(), s);
        if (e == cudaSuccess) e = H->part.alloc(std::max<int64_t>(part_at.back(), 1));
    }
    if (e == cudaSuccess) e = H->leafmv.upload(s);
    if (e == cudaSuccess) e = H->rowop.upload(s);
    if (e == cudaSuccess) e = coup.upload(s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        delete H;
        return gcabem_internal_error(GCABEM_ERR_CUDA,
                                     (std::string("h2_create: ") + cudaGetErrorString(e)).c_str());
    }
    H->bytes_per_product = 16.0 * (double)(payload_len + 2 * v_len + 4 * (nrows + ncols));
    *out = H;
    return GCABEM_OK;
}

namespace {
cudaError_t run_matvec(gcabem_h2_s *H, Batch &b, const double2 *M, const double2 *v,
                       double2 *out, bool transposed) {
    const int64_t nt = b.ntasks();
    if (nt == 0) return cudaSuccess;
    if (transposed) {
        tmatvec_kernel<<<(unsigned)nt, MV_TPB, 0, H->stream>>>(
            b.d_task_item.p, b.d_task_r0.p, nt, b.d_m_at.p, b.d_rows.p, b.d_cols.p, b.d_v_at.p,
            H->d_part_at.p, M, v, H->part.p);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess || H->nk == 0) return e;
        treduce_kernel<<<(unsigned)((H->nk + MV_TPB - 1) / MV_TPB), MV_TPB, 0, H->stream>>>(
            H->d_item_task_at.p, H->d_part_at.p, b.d_cols.p, b.d_out_at.p, H->d_ek_at.p,
            (int64_t)b.m_at.size(), H->nk, H->part.p, out);
    } else
        matvec_kernel<<<(unsigned)((nt * RPG + MV_TPB - 1) / MV_TPB), MV_TPB, 0, H->stream>>>(
            b.d_task_item.p, b.d_task_r0.p, nt, b.d_m_at.p, b.d_rows.p, b.d_cols.p, b.d_v_at.p,
            b.d_out_at.p, M, v, out);
    return cudaGetLastError();
}
}  // namespace

int gcabem_h2_matvec(gcabem_h2_t H, const double *x, double *y, float *device_ms) {
    if (!H || !x || !y) return gcabem_internal_error(GCABEM_ERR_ARG, "h2_matvec: null argument");
    cudaStream_t s = H->stream;
    const unsigned gx = (unsigned)((H->ncols + MV_TPB - 1) / MV_TPB);
    const unsigned gy = (unsigned)((H->nrows + MV_TPB - 1) / MV_TPB);
    cudaEvent_t ev[2] = {nullptr, nullptr};
    cudaError_t e = cudaSetDevice(H->device);
    for (int k = 0; k < 2 && e == cudaSuccess; ++k) e = cudaEventCreate(&ev[k]);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(H->xh.p, x, 16 * H->ncols, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaEventRecord(ev[0], s);
    if (e == cudaSuccess) {
        gather_kernel<<<gx, MV_TPB, 0, s>>>(H->xh.p, H->col_perm.p, H->ncols, H->xp.p);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = run_matvec(H, H->colop, H->V.p, H->xp.p, H->xs.p, true);
    if (e == cudaSuccess) e = run_matvec(H, H->leafmv, H->payload.p, H->xp.p, H->cbuf.p, false);
    if (e == cudaSuccess) e = run_matvec(H, H->coup, H->payload.p, H->xs.p, H->wbuf.p, false);
    if (e == cudaSuccess && H->nz > 0) {
        csr_sum_kernel<<<(unsigned)((H->nz + MV_TPB - 1) / MV_TPB), MV_TPB, 0, s>>>(
            H->z_at.p, H->z_idx.p, H->nz, H->wbuf.p, H->zbuf.p);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = run_matvec(H, H->rowop, H->V.p, H->zbuf.p, H->cbuf.p, false);
    if (e == cudaSuccess) {
        csr_sum_kernel<<<gy, MV_TPB, 0, s>>>(H->y_at.p, H->y_idx.p, H->nrows, H->cbuf.p, H->yp.p);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
        scatter_kernel<<<gy, MV_TPB, 0, s>>>(H->yp.p, H->row_perm.p, H->nrows, H->xh.p);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaEventRecord(ev[1], s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(y, H->xh.p, 16 * H->nrows, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess && device_ms) e = cudaEventElapsedTime(device_ms, ev[0], ev[1]);
    for (auto &v : ev)
        if (v) cudaEventDestroy(v);
    if (e != cudaSuccess)
        return gcabem_internal_error(GCABEM_ERR_CUDA,
                                     (std::string("h2_matvec: ") + cudaGetErrorString(e)).c_str());
    return GCABEM_OK;
}

int gcabem_h2_info(gcabem_h2_t H, double *bytes_per_product) {
    if (!H || !bytes_per_product) return gcabem_internal_error(GCABEM_ERR_ARG, "null argument");
    *bytes_per_product = H->bytes_per_product;
    return GCABEM_OK;
}

int gcabem_h2_free(gcabem_h2_t H) {
    if (!H) return GCABEM_OK;
    cudaSetDevice(H->device);
    if (H->stream) cudaStreamSynchronize(H->stream);
    cudaStream_t s = H->stream;
    delete H;
    if (s) cudaStreamDestroy(s);
    return GCABEM_OK;
}

}  // extern "C"
