// Cluster tree and block tree construction (host, native), bit-exact with
// the reference (pkg/src/gcabem/cluster.py:87-152):
//  * geometric bisection: box of the node's triangles, split along the
//    longest axis (first maximum) at the median of the midpoints, order by
//    (midpoint coordinate, panel index), preorder node numbering;
//  * block tree: admissible <=> max(diam_t, diam_s) <= eta * dist(t, s);
//    else dense if both are leaves; else recurse over the children
//    (a leaf cluster stands in for itself), preorder numbering.
// dist uses the 3-term sum-of-squares variant that reproduces the host's
// np.linalg.norm bit for bit (selected by the Python side's self-test);
// diameters are passed in precomputed by numpy itself.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <map>
#include <thread>
#include <vector>

#include "gcabem_b200.h"

int gcabem_internal_error(int code, const char *msg);  // api.cu

namespace {

// Preorder bisection tree. The node count of a subtree depends only on its
// panel count, so every subtree's node and panel offsets are known before it
// is built: the two halves of a large node are built concurrently into
// preallocated arrays. A node only needs its halves as SETS (each child
// re-sorts by its own axis), so the split is an nth_element on the
// reference's key (midpoint coordinate, panel index); a half that becomes a
// leaf keeps the parent's sorted order (the leaf's panel order), so it is
// fully sorted.
struct CTree {
    const double *tlo, *thi, *mid;
    int64_t leaf;
    std::vector<int64_t> start, size, c0, c1, perm, idx;
    std::vector<double> lo, hi;
    std::map<int64_t, int64_t> memo;

    int64_t count(int64_t n) {
        if (n <= leaf) return 1;
        auto it = memo.find(n);
        if (it != memo.end()) return it->second;
        const int64_t c = 1 + count(n / 2) + count(n - n / 2);
        memo[n] = c;
        return c;
    }
    // node ids: the counts of every size that occurs, computed up front
    // (the concurrent builds only read the memo)
    void prime(int64_t n) {
        if (n <= leaf || memo.count(n)) return;
        prime(n / 2);
        prime(n - n / 2);
        count(n);
    }
    int64_t cnt(int64_t n) const {
        if (n <= leaf) return 1;
        return memo.at(n);
    }

    void build(int64_t me, int64_t a, int64_t b, int depth) {
        start[me] = a;
        size[me] = b - a;
        double l[3] = {tlo[3 * idx[a]], tlo[3 * idx[a] + 1], tlo[3 * idx[a] + 2]};
        double h[3] = {thi[3 * idx[a]], thi[3 * idx[a] + 1], thi[3 * idx[a] + 2]};
        for (int64_t k = a + 1; k < b; ++k)
            for (int q = 0; q < 3; ++q) {
                l[q] = std::min(l[q], tlo[3 * idx[k] + q]);
                h[q] = std::max(h[q], thi[3 * idx[k] + q]);
            }
        for (int q = 0; q < 3; ++q) {
            lo[3 * me + q] = l[q];
            hi[3 * me + q] = h[q];
        }
        if (b - a <= leaf) {
            for (int64_t k = a; k < b; ++k) perm[k] = idx[k];
            return;
        }
        int axis = 0;
        double ext = h[0] - l[0];
        for (int q = 1; q < 3; ++q)
            if (h[q] - l[q] > ext) {
                ext = h[q] - l[q];
                axis = q;
            }
        auto less = [&](int64_t u, int64_t v) {
            const double mu = mid[3 * u + axis], mv = mid[3 * v + axis];
            return mu < mv || (mu == mv && u < v);
        };
        const int64_t half = (b - a) / 2;
        std::nth_element(idx.begin() + a, idx.begin() + a + half, idx.begin() + b, less);
        if (half <= leaf) std::sort(idx.begin() + a, idx.begin() + a + half, less);
        if (b - a - half <= leaf) std::sort(idx.begin() + a + half, idx.begin() + b, less);
        const int64_t left = me + 1, right = me + 1 + cnt(half);
        c0[me] = left;
        c1[me] = right;
        if (depth < 3 && b - a > 4096) {
            std::thread th([&, left, a, half, depth] { build(left, a, a + half, depth + 1); });
            build(right, a + half, b, depth + 1);
            th.join();
        } else {
            build(left, a, a + half, depth + 1);
            build(right, a + half, b, depth + 1);
        }
    }
};

inline double norm3(const double g[3], int variant) {
    const double x = g[0], y = g[1], z = g[2];
    switch (variant) {
        case 1: return std::sqrt(std::fma(z, z, std::fma(y, y, x * x)));
        case 2: return std::sqrt(std::fma(x, x, std::fma(y, y, z * z)));
        case 3: return std::sqrt(x * x + (y * y + z * z));
        default: return std::sqrt((x * x + y * y) + z * z);
    }
}

struct BTree {
    const int64_t *rc0, *rc1, *cc0, *cc1;
    const double *rlo, *rhi, *clo, *chi, *rdiam, *cdiam;
    double eta;
    int variant;
    std::vector<int64_t> row, col, kind, first, nkids, kids;  // kind: 0 adm, 1 dense, 2 split

    bool admissible(int64_t t, int64_t s) const {
        double g[3];
        bool touch = true;
        for (int q = 0; q < 3; ++q) {
            const double a = rlo[3 * t + q] - chi[3 * s + q];
            const double b = clo[3 * s + q] - rhi[3 * t + q];
            g[q] = std::max(0.0, std::max(a, b));
            touch = touch && rlo[3 * t + q] <= chi[3 * s + q] && clo[3 * s + q] <= rhi[3 * t + q];
        }
        if (touch) return false;  // dist == 0 and diam > 0
        const double diam = std::max(rdiam[t], cdiam[s]);
        return diam <= eta * norm3(g, variant);
    }

    int64_t build(int64_t t, int64_t s) {
        const int64_t me = (int64_t)row.size();
        row.push_back(t);
        col.push_back(s);
        kind.push_back(0);
        first.push_back(0);
        nkids.push_back(0);
        const bool tleaf = rc0[t] < 0, sleaf = cc0[s] < 0;
        if (admissible(t, s)) {
            kind[me] = 0;
        } else if (tleaf && sleaf) {
            kind[me] = 1;
        } else {
            kind[me] = 2;
            int64_t tk[2], sk[2];
            int nt = 0, ns = 0;
            if (tleaf) tk[nt++] = t; else { tk[nt++] = rc0[t]; tk[nt++] = rc1[t]; }
            if (sleaf) sk[ns++] = s; else { sk[ns++] = cc0[s]; sk[ns++] = cc1[s]; }
            int64_t mine[4];
            int nm = 0;
            for (int a = 0; a < nt; ++a)
                for (int b = 0; b < ns; ++b) mine[nm++] = build(tk[a], sk[b]);
            first[me] = (int64_t)kids.size();
            nkids[me] = nm;
            kids.insert(kids.end(), mine, mine + nm);
        }
        return me;
    }
};

struct TreeResult {
    std::vector<int64_t> a, b, c, d, e, f;
    std::vector<double> lo, hi;
};

}  // namespace

struct gcabem_tree_s : TreeResult {};

extern "C" {

// Cluster tree. Output arrays fetched with gcabem_tree_fetch:
// {start, size, child0, child1, perm} (int64) and {lo, hi} (n x 3).
int gcabem_cluster_tree(int64_t nt, const double *tri_lo, const double *tri_hi,
                        const double *mid, int64_t leaf_size, gcabem_tree_t *out) {
    if (!out || nt <= 0 || leaf_size < 1)
        return gcabem_internal_error(GCABEM_ERR_ARG, "cluster tree: bad arguments");
    CTree t;
    t.tlo = tri_lo;
    t.thi = tri_hi;
    t.mid = mid;
    t.leaf = leaf_size;
    t.prime(nt);
    const int64_t nn = t.cnt(nt);
    t.start.assign(nn, 0);
    t.size.assign(nn, 0);
    t.c0.assign(nn, -1);
    t.c1.assign(nn, -1);
    t.lo.assign(3 * nn, 0.0);
    t.hi.assign(3 * nn, 0.0);
    t.perm.assign(nt, 0);
    t.idx.resize(nt);
    for (int64_t k = 0; k < nt; ++k) t.idx[k] = k;
    t.build(0, 0, nt, 0);
    auto *r = new gcabem_tree_s();
    r->a = std::move(t.start);
    r->b = std::move(t.size);
    r->c = std::move(t.c0);
    r->d = std::move(t.c1);
    r->e = std::move(t.perm);
    r->lo = std::move(t.lo);
    r->hi = std::move(t.hi);
    *out = r;
    return GCABEM_OK;
}

// The same from the mesh arrays: per-triangle bounds (min/max of the
// corners, mesh.py:70-73) and midpoints ((v0 + v1 + v2) / 3, mesh.py:65-68,
// the same IEEE operations) formed here.
int gcabem_cluster_tree_mesh(int64_t nt, const int64_t *T, const double *V, int64_t leaf_size,
                             gcabem_tree_t *out) {
    if (!T || !V || nt <= 0)
        return gcabem_internal_error(GCABEM_ERR_ARG, "cluster tree: bad arguments");
    std::vector<double> lo(3 * nt), hi(3 * nt), mid(3 * nt);
    for (int64_t k = 0; k < nt; ++k) {
        const double *a = V + 3 * T[3 * k], *b = V + 3 * T[3 * k + 1], *c = V + 3 * T[3 * k + 2];
        for (int q = 0; q < 3; ++q) {
            lo[3 * k + q] = std::min(std::min(a[q], b[q]), c[q]);
            hi[3 * k + q] = std::max(std::max(a[q], b[q]), c[q]);
            mid[3 * k + q] = ((a[q] + b[q]) + c[q]) / 3.0;
        }
    }
    return gcabem_cluster_tree(nt, lo.data(), hi.data(), mid.data(), leaf_size, out);
}

// Block tree over (row tree, col tree). Output arrays:
// {row, col, kind (0 admissible, 1 dense, 2 split), first child slot,
//  number of children, children} (int64).
int gcabem_block_tree(int64_t nrow, const int64_t *row_c0, const int64_t *row_c1,
                      const double *row_lo, const double *row_hi, const double *row_diam,
                      int64_t ncol, const int64_t *col_c0, const int64_t *col_c1,
                      const double *col_lo, const double *col_hi, const double *col_diam,
                      double eta, int norm_variant, gcabem_tree_t *out) {
    if (!out || nrow <= 0 || ncol <= 0)
        return gcabem_internal_error(GCABEM_ERR_ARG, "block tree: bad arguments");
    BTree t{row_c0, row_c1, col_c0, col_c1, row_lo, row_hi, col_lo, col_hi, row_diam, col_diam,
            eta, norm_variant, {}, {}, {}, {}, {}, {}};
    const size_t guess = (size_t)(64 * std::max(nrow, ncol));
    for (auto *v : {&t.row, &t.col, &t.kind, &t.first, &t.nkids, &t.kids}) v->reserve(guess);
    t.build(0, 0);
    auto *r = new gcabem_tree_s();
    r->a = std::move(t.row);
    r->b = std::move(t.col);
    r->c = std::move(t.kind);
    r->d = std::move(t.first);
    r->e = std::move(t.nkids);
    r->f = std::move(t.kids);
    *out = r;
    return GCABEM_OK;
}

// norm variant probe: writes norm3(v_k, variant) for n vectors
int gcabem_norm3(int64_t n, const double *v, int variant, double *out) {
    for (int64_t k = 0; k < n; ++k) out[k] = norm3(v + 3 * k, variant);
    return GCABEM_OK;
}

// sizes[8]: lengths of a, b, c, d, e, f, lo, hi
int gcabem_tree_sizes(gcabem_tree_t t, int64_t *sizes) {
    if (!t || !sizes) return GCABEM_ERR_ARG;
    sizes[0] = (int64_t)t->a.size();
    sizes[1] = (int64_t)t->b.size();
    sizes[2] = (int64_t)t->c.size();
    sizes[3] = (int64_t)t->d.size();
    sizes[4] = (int64_t)t->e.size();
    sizes[5] = (int64_t)t->f.size();
    sizes[6] = (int64_t)t->lo.size();
    sizes[7] = (int64_t)t->hi.size();
    return GCABEM_OK;
}

int gcabem_tree_fetch(gcabem_tree_t t, int64_t *a, int64_t *b, int64_t *c, int64_t *d,
                      int64_t *e, int64_t *f, double *lo, double *hi) {
    if (!t) return GCABEM_ERR_ARG;
    auto cp = [](auto *dst, const auto &v) {
        if (dst) std::copy(v.begin(), v.end(), dst);
    };
    cp(a, t->a);
    cp(b, t->b);
    cp(c, t->c);
    cp(d, t->d);
    cp(e, t->e);
    cp(f, t->f);
    cp(lo, t->lo);
    cp(hi, t->hi);
    return GCABEM_OK;
}

int gcabem_tree_free(gcabem_tree_t t) {
    delete t;
    return GCABEM_OK;
}

}  // extern "C"
