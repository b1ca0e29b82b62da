// Host-side work packaging (the CPU half of scheduler.run_assembly), native.
//
// Bit-exact restatement of what the reference scheduler does on the host
// (pkg/src/gcabem/scheduler.py): leaf enumeration in block-tree preorder
// (_leaf_blocks :425-439, make_payloads :411-422), split_block (:153-175),
// ListBuilder greedy byte budget (:178-208), the corrective shared-vertex
// scan of flagged blocks in argwhere order (distribute_disjoint :334-359)
// and classify_pair permutations (quadrature.py:197-220). The scan runs on
// std::thread workers with a count / prefix-sum / fill pass so item order is
// independent of the thread count.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <functional>
#include <thread>
#include <vector>

#include "gcabem_b200.h"

int gcabem_internal_error(int code, const char *msg);  // api.cu

namespace {

struct Packages {
    int64_t L = 0, payload_len = 0, nlists = 0;
    // panel base array [row perm | row pivots | col perm | col pivots]: owned,
    // or the caller's (gcabem_packages_build_on: shared by the leaf ranges of
    // one assembly, kept alive by the caller until free)
    std::vector<int64_t> panels_own;
    const int64_t *panels = nullptr;
    int64_t npanels = 0;
    std::vector<int64_t> leaf_shape;    // L x 2
    std::vector<int64_t> leaf_base;     // L + 1
    std::vector<int64_t> rows_at, cols_at;
    std::vector<uint8_t> flagged;       // L
    std::vector<int64_t> blk;           // B x 5 {leaf, r0, nr, c0, nc}
    std::vector<int64_t> blk_list;      // B
    // corrective items are counted at build time and written straight into
    // the caller's arrays at fetch time (no intermediate copy)
    std::vector<int64_t> fb;            // flagged blocks
    std::vector<int64_t> cnt;           // item prefix sums over fb (F + 1)
    std::vector<int64_t> tri_own;       // nt x 3 copy for the fill pass (or borrowed:)
    const int64_t *tri = nullptr;
    int nthreads = 1;
    int64_t S = 0;
};

constexpr int64_t BYTES_PER_PAIR = 32;

void split(int64_t leaf, int64_t r0, int64_t nr, int64_t c0, int64_t nc, int64_t maxsize,
           std::vector<int64_t> &out) {
    if (nr * nc * BYTES_PER_PAIR <= maxsize) {
        out.insert(out.end(), {leaf, r0, nr, c0, nc});
        return;
    }
    if (nr >= nc) {
        const int64_t h = nr / 2;
        split(leaf, r0, h, c0, nc, maxsize, out);
        split(leaf, r0 + h, nr - h, c0, nc, maxsize, out);
    } else {
        const int64_t h = nc / 2;
        split(leaf, r0, nr, c0, h, maxsize, out);
        split(leaf, r0, nr, c0 + h, nc - h, maxsize, out);
    }
}

// classify_pair permutation of one side: shared slots first by global vertex
// id, then unshared slots in original order.
inline void perm_for(const int64_t *v, const bool *shared, uint8_t *perm) {
    int k = 0;
    uint8_t lead[3];
    int nl = 0;
    for (int s = 0; s < 3; ++s)
        if (shared[s]) lead[nl++] = (uint8_t)s;
    std::sort(lead, lead + nl, [&](uint8_t a, uint8_t b) { return v[a] < v[b]; });
    for (int s = 0; s < nl; ++s) perm[k++] = lead[s];
    for (int s = 0; s < 3; ++s)
        if (!shared[s]) perm[k++] = (uint8_t)s;
}

inline int count3(const int64_t *a, const int64_t *b) {
    return (a[0] == b[0]) + (a[0] == b[1]) + (a[0] == b[2]) + (a[1] == b[0]) + (a[1] == b[1]) +
           (a[1] == b[2]) + (a[2] == b[0]) + (a[2] == b[1]) + (a[2] == b[2]);
}

void parallel_for(int64_t n, int nthreads, const std::function<void(int64_t, int64_t)> &fn) {
    if (nthreads <= 1 || n < 1024) {
        fn(0, n);
        return;
    }
    std::vector<std::thread> th;
    const int64_t chunk = (n + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t) {
        const int64_t a = t * chunk, b = std::min(n, a + chunk);
        if (a >= b) break;
        th.emplace_back(fn, a, b);
    }
    for (auto &x : th) x.join();
}

}  // namespace

struct gcabem_packages_s : Packages {};

extern "C" {

int gcabem_packages_build(int64_t nt, const int64_t *triangles, int64_t nleaves,
                          const int64_t *leaves, int64_t nrow, const int64_t *row_start,
                          const int64_t *row_size, const double *row_lo, const double *row_hi,
                          const int64_t *row_perm, const int64_t *row_op_at,
                          const int64_t *row_piv, int64_t ncol, const int64_t *col_start,
                          const int64_t *col_size, const double *col_lo, const double *col_hi,
                          const int64_t *col_perm, const int64_t *col_op_at,
                          const int64_t *col_piv, int64_t maxsize, int nthreads,
                          gcabem_packages_t *out) {
    return gcabem_packages_build_on(nt, triangles, nleaves, leaves, nrow, row_start, row_size,
                                    row_lo, row_hi, row_perm, row_op_at, row_piv, ncol,
                                    col_start, col_size, col_lo, col_hi, col_perm, col_op_at,
                                    col_piv, maxsize, nthreads, nullptr, 0, out);
}

int gcabem_packages_build_on(int64_t nt, const int64_t *triangles, int64_t nleaves,
                             const int64_t *leaves, int64_t nrow, const int64_t *row_start,
                             const int64_t *row_size, const double *row_lo,
                             const double *row_hi, const int64_t *row_perm,
                             const int64_t *row_op_at, const int64_t *row_piv, int64_t ncol,
                             const int64_t *col_start, const int64_t *col_size,
                             const double *col_lo, const double *col_hi,
                             const int64_t *col_perm, const int64_t *col_op_at,
                             const int64_t *col_piv, int64_t maxsize, int nthreads,
                             const int64_t *panel_base, int64_t npanel_base,
                             gcabem_packages_t *out) {
    auto fail = [](const char *m) { return gcabem_internal_error(GCABEM_ERR_ARG, m); };
    static const bool trace = std::getenv("GCABEM_TRACE") != nullptr;
    auto t_start = std::chrono::steady_clock::now();
    auto mark = [&](const char *what) {
        if (!trace) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[packages] %-10s %8.2f ms\n", what,
                     std::chrono::duration<double, std::milli>(now - t_start).count());
        t_start = now;
    };
    if (!out) return fail("null output");
    *out = nullptr;
    if (maxsize < BYTES_PER_PAIR) return fail("maxsize smaller than one pair record (32 B)");
    if (nthreads <= 0) nthreads = (int)std::max(1u, std::thread::hardware_concurrency());
    const bool shared_tree = (row_start == col_start && row_perm == col_perm);
    auto *pk = new gcabem_packages_s();
    Packages &P = *pk;
    P.L = nleaves;
    // panel base array: row perm, row pivots, (col perm, col pivots)
    const int64_t nrp = row_op_at[nrow];
    int64_t col_perm_at = 0, col_piv_at = nt, nbase = nt + nrp;
    const bool own_cols = !shared_tree || col_piv != row_piv;
    if (own_cols) {
        col_perm_at = nt + nrp;
        col_piv_at = col_perm_at + nt;
        nbase = col_piv_at + col_op_at[ncol];
    }
    if (panel_base) {
        if (npanel_base != nbase) {
            delete pk;
            return fail("panel base array does not match the trees and operators");
        }
        P.panels = panel_base;
        P.tri = triangles;
    } else {
        P.panels_own.reserve(nbase);
        P.panels_own.insert(P.panels_own.end(), row_perm, row_perm + nt);
        P.panels_own.insert(P.panels_own.end(), row_piv, row_piv + nrp);
        if (own_cols) {
            P.panels_own.insert(P.panels_own.end(), col_perm, col_perm + nt);
            P.panels_own.insert(P.panels_own.end(), col_piv, col_piv + col_op_at[ncol]);
        }
        P.panels = P.panels_own.data();
        P.tri_own.assign(triangles, triangles + 3 * nt);
        P.tri = P.tri_own.data();
    }
    P.npanels = nbase;
    P.leaf_shape.resize(2 * nleaves);
    P.leaf_base.resize(nleaves + 1);
    P.rows_at.resize(nleaves);
    P.cols_at.resize(nleaves);
    P.flagged.resize(nleaves);
    P.leaf_base[0] = 0;
    std::atomic<int> leaf_err{0};  // 1: cluster index out of range, 2: no operator
    parallel_for(nleaves, nthreads, [&](int64_t lo, int64_t hi) {
        for (int64_t k = lo; k < hi; ++k) {
            const int64_t r = leaves[3 * k], c = leaves[3 * k + 1], dense = leaves[3 * k + 2];
            if (r < 0 || r >= nrow || c < 0 || c >= ncol) {
                leaf_err = 1;
                return;
            }
            int64_t nr, nc;
            if (dense) {
                nr = row_size[r];
                nc = col_size[c];
                P.rows_at[k] = row_start[r];
                P.cols_at[k] = col_perm_at + col_start[c];
            } else {
                nr = row_op_at[r + 1] - row_op_at[r];
                nc = col_op_at[c + 1] - col_op_at[c];
                P.rows_at[k] = nt + row_op_at[r];
                P.cols_at[k] = col_piv_at + col_op_at[c];
                if (nr <= 0 || nc <= 0) {
                    leaf_err = 2;
                    return;
                }
            }
            P.leaf_shape[2 * k] = nr;
            P.leaf_shape[2 * k + 1] = nc;
            // box_distance(t, s) == 0.0  <=>  boxes touch on every axis (exact)
            bool touch = true;
            for (int a = 0; a < 3; ++a)
                touch = touch && row_lo[3 * r + a] <= col_hi[3 * c + a] &&
                        col_lo[3 * c + a] <= row_hi[3 * r + a];
            P.flagged[k] = touch ? 1 : 0;
        }
    });
    if (leaf_err) {
        delete pk;
        return fail(leaf_err == 1 ? "leaf cluster index out of range"
                                  : "admissible leaf without an interpolation operator");
    }
    for (int64_t k = 0; k < nleaves; ++k)
        P.leaf_base[k + 1] = P.leaf_base[k] + P.leaf_shape[2 * k] * P.leaf_shape[2 * k + 1];
    P.payload_len = P.leaf_base[nleaves];
    mark("leaves");
    // split (per leaf, on the pool: per-thread block lists joined in leaf
    // order) + greedy lists (sequential: the byte budget runs across leaves)
    {
        const int nparts = nleaves >= 4096 ? std::max(1, nthreads) : 1;
        std::vector<std::vector<int64_t>> parts(nparts);
        std::atomic<bool> tiny{false};
        const int64_t per = (nleaves + nparts - 1) / nparts;
        auto run = [&](int64_t t) {
            std::vector<int64_t> &out = parts[t];
            const int64_t lo = t * per, hi = std::min(nleaves, lo + per);
            out.reserve(5 * std::max<int64_t>(hi - lo, 0) + 16);
            for (int64_t k = lo; k < hi; ++k) {
                const int64_t nr = P.leaf_shape[2 * k], nc = P.leaf_shape[2 * k + 1];
                if (nr * nc > 1 || nr * nc * BYTES_PER_PAIR <= maxsize)
                    split(k, 0, nr, 0, nc, maxsize, out);
                else
                    tiny = true;
            }
        };
        if (nparts == 1) {
            run(0);
        } else {
            std::vector<std::thread> th;
            for (int t = 1; t < nparts; ++t) th.emplace_back(run, t);
            run(0);
            for (auto &x : th) x.join();
        }
        if (tiny) {
            delete pk;
            return fail("maxsize smaller than one pair record (32 B)");
        }
        size_t total = 0;
        for (auto &v : parts) total += v.size();
        P.blk.reserve(total);
        for (auto &v : parts) P.blk.insert(P.blk.end(), v.begin(), v.end());
    }
    const int64_t B = (int64_t)P.blk.size() / 5;
    P.blk_list.resize(B);
    {
        int64_t cur = 0, cnt = 0, lid = 0;
        for (int64_t b = 0; b < B; ++b) {
            const int64_t nb = P.blk[5 * b + 2] * P.blk[5 * b + 4] * BYTES_PER_PAIR;
            if (cur + nb > maxsize && cnt) {
                ++lid;
                cur = cnt = 0;
            }
            P.blk_list[b] = lid;
            cur += nb;
            ++cnt;
        }
        P.nlists = B ? lid + 1 : 0;
    }
    mark("split");
    // corrective scan of flagged blocks: count, prefix sum, fill
    std::vector<int64_t> fb;
    for (int64_t b = 0; b < B; ++b)
        if (P.flagged[P.blk[5 * b]]) fb.push_back(b);
    const int64_t F = (int64_t)fb.size();
    std::vector<int64_t> cnt(F + 1, 0);
    const int64_t *T = triangles;
    auto row_tri = [&](int64_t b, int64_t i) {
        const int64_t *q = &P.blk[5 * b];
        return P.panels[P.rows_at[q[0]] + q[1] + i];
    };
    auto col_tri = [&](int64_t b, int64_t j) {
        const int64_t *q = &P.blk[5 * b];
        return P.panels[P.cols_at[q[0]] + q[3] + j];
    };
    bool bad_index = false;
    bool three_shared = false;
    // vertex triples of one block's row/col panels, staged contiguously
    auto stage = [&](int64_t b, std::vector<int64_t> &ra, std::vector<int64_t> &ca,
                     std::vector<int64_t> &rt, std::vector<int64_t> &ct) {
        const int64_t nr = P.blk[5 * b + 2], nc = P.blk[5 * b + 4];
        ra.resize(3 * nr);
        ca.resize(3 * nc);
        rt.resize(nr);
        ct.resize(nc);
        for (int64_t i = 0; i < nr; ++i) {
            const int64_t tx = row_tri(b, i);
            if (tx < 0 || tx >= nt) return false;
            rt[i] = tx;
            std::memcpy(&ra[3 * i], T + 3 * tx, 24);
        }
        for (int64_t j = 0; j < nc; ++j) {
            const int64_t ty = col_tri(b, j);
            if (ty < 0 || ty >= nt) return false;
            ct[j] = ty;
            std::memcpy(&ca[3 * j], T + 3 * ty, 24);
        }
        return true;
    };
    parallel_for(F, nthreads, [&](int64_t lo, int64_t hi) {
        std::vector<int64_t> ra, ca, rt, ct;
        for (int64_t f = lo; f < hi; ++f) {
            const int64_t b = fb[f];
            if (!stage(b, ra, ca, rt, ct)) {
                bad_index = true;
                return;
            }
            const int64_t nr = (int64_t)rt.size(), nc = (int64_t)ct.size();
            int64_t n = 0;
            for (int64_t i = 0; i < nr; ++i)
                for (int64_t j = 0; j < nc; ++j) {
                    const int s = count3(&ra[3 * i], &ca[3 * j]);
                    n += s > 0;
                    if (s >= 3 && rt[i] != ct[j]) three_shared = true;
                }
            cnt[f + 1] = n;
        }
    });
    if (bad_index) {
        delete pk;
        return fail("panel index out of range");
    }
    if (three_shared) {
        delete pk;
        return fail("distinct triangles share 3 vertices");
    }
    mark("count");
    for (int64_t f = 0; f < F; ++f) cnt[f + 1] += cnt[f];
    P.S = cnt[F];
    P.fb = std::move(fb);
    P.cnt = std::move(cnt);
    P.nthreads = nthreads;
    *out = pk;
    return GCABEM_OK;
}

// sizes[9] = {L, payload_len, npanels, nblocks, nlists, nitems, 0, 0, 0}
int gcabem_packages_sizes(gcabem_packages_t pk, int64_t *sizes) {
    if (!pk || !sizes) return GCABEM_ERR_ARG;
    sizes[0] = pk->L;
    sizes[1] = pk->payload_len;
    sizes[2] = pk->npanels;
    sizes[3] = (int64_t)pk->blk.size() / 5;
    sizes[4] = pk->nlists;
    sizes[5] = pk->S;
    sizes[6] = sizes[7] = sizes[8] = 0;
    return GCABEM_OK;
}

// Copy every array out (caller-allocated with the sizes above).
int gcabem_packages_fetch(gcabem_packages_t pk, int64_t *panels, int64_t *leaf_shape,
                          int64_t *leaf_base, int64_t *rows_at, int64_t *cols_at,
                          uint8_t *flagged, int64_t *blocks, int64_t *blk_list, int64_t *items,
                          uint8_t *perms) {
    if (!pk) return GCABEM_ERR_ARG;
    Packages &P = *pk;
    auto cp = [](void *dst, const void *src, size_t bytes) {
        if (dst && bytes) std::memcpy(dst, src, bytes);
    };
    cp(panels, P.panels, P.npanels * 8);
    cp(leaf_shape, P.leaf_shape.data(), P.leaf_shape.size() * 8);
    cp(leaf_base, P.leaf_base.data(), P.leaf_base.size() * 8);
    cp(rows_at, P.rows_at.data(), P.rows_at.size() * 8);
    cp(cols_at, P.cols_at.data(), P.cols_at.size() * 8);
    cp(flagged, P.flagged.data(), P.flagged.size());
    // field-major: each field is one contiguous array on the Python side
    const int64_t B = (int64_t)P.blk.size() / 5, S = P.S;
    if (blocks)
        for (int f = 0; f < 5; ++f)
            for (int64_t b = 0; b < B; ++b) blocks[f * B + b] = P.blk[5 * b + f];
    cp(blk_list, P.blk_list.data(), P.blk_list.size() * 8);
    if (!items || !perms || S == 0) return GCABEM_OK;
    // corrective items of the flagged blocks in argwhere (row-major) order,
    // block after block; block f's items start at cnt[f]
    const int64_t F = (int64_t)P.fb.size();
    const int64_t *T = P.tri;
    int64_t *o_case = items, *o_tx = items + S, *o_ty = items + 2 * S, *o_leaf = items + 3 * S,
            *o_off = items + 4 * S, *o_blk = items + 5 * S;
    parallel_for(F, P.nthreads, [&](int64_t lo, int64_t hi) {
        std::vector<int64_t> ra, ca, rt, ct;
        for (int64_t f = lo; f < hi; ++f) {
            if (P.cnt[f + 1] == P.cnt[f]) continue;
            const int64_t b = P.fb[f];
            const int64_t leaf = P.blk[5 * b], r0 = P.blk[5 * b + 1], nr = P.blk[5 * b + 2];
            const int64_t c0 = P.blk[5 * b + 3], nc = P.blk[5 * b + 4];
            const int64_t ld = P.leaf_shape[2 * leaf + 1];
            ra.resize(3 * nr);
            ca.resize(3 * nc);
            rt.resize(nr);
            ct.resize(nc);
            for (int64_t i = 0; i < nr; ++i) {
                rt[i] = P.panels[P.rows_at[leaf] + r0 + i];
                std::memcpy(&ra[3 * i], T + 3 * rt[i], 24);
            }
            for (int64_t j = 0; j < nc; ++j) {
                ct[j] = P.panels[P.cols_at[leaf] + c0 + j];
                std::memcpy(&ca[3 * j], T + 3 * ct[j], 24);
            }
            int64_t w = P.cnt[f];
            for (int64_t i = 0; i < nr; ++i) {
                const int64_t *va = &ra[3 * i];
                for (int64_t j = 0; j < nc; ++j) {
                    const int64_t *vb = &ca[3 * j];
                    const int s = count3(va, vb);
                    if (!s) continue;
                    const int64_t tx = rt[i], ty = ct[j];
                    uint8_t *pm = perms + 6 * w;
                    if (tx == ty) {
                        o_case[w] = 3;
                        for (int q = 0; q < 3; ++q) pm[q] = pm[3 + q] = (uint8_t)q;
                    } else {
                        o_case[w] = std::min(s, 3);
                        bool sa[3], sb[3];
                        for (int q = 0; q < 3; ++q) {
                            sa[q] = va[q] == vb[0] || va[q] == vb[1] || va[q] == vb[2];
                            sb[q] = vb[q] == va[0] || vb[q] == va[1] || vb[q] == va[2];
                        }
                        perm_for(va, sa, pm);
                        perm_for(vb, sb, pm + 3);
                    }
                    o_tx[w] = tx;
                    o_ty[w] = ty;
                    o_leaf[w] = leaf;
                    o_off[w] = (r0 + i) * ld + c0 + j;
                    o_blk[w] = b;
                    ++w;
                }
            }
        }
    });
    return GCABEM_OK;
}

int gcabem_packages_free(gcabem_packages_t pk) {
    delete pk;
    return GCABEM_OK;
}

int gcabem_leaf_layout(int64_t nleaves, const int64_t *leaves, int64_t nrow,
                       const int64_t *row_size, const int64_t *row_op_at, int64_t ncol,
                       const int64_t *col_size, const int64_t *col_op_at, int64_t *leaf_shape,
                       int64_t *leaf_base) {
    if (nleaves < 0 || (nleaves > 0 && (!leaves || !leaf_shape || !leaf_base)))
        return gcabem_internal_error(GCABEM_ERR_ARG, "leaf_layout: bad arguments");
    leaf_base[0] = 0;
    for (int64_t k = 0; k < nleaves; ++k) {
        const int64_t r = leaves[3 * k], c = leaves[3 * k + 1];
        if (r < 0 || r >= nrow || c < 0 || c >= ncol)
            return gcabem_internal_error(GCABEM_ERR_ARG, "leaf cluster index out of range");
        const int64_t nr = leaves[3 * k + 2] ? row_size[r] : row_op_at[r + 1] - row_op_at[r];
        const int64_t nc = leaves[3 * k + 2] ? col_size[c] : col_op_at[c + 1] - col_op_at[c];
        leaf_shape[2 * k] = nr;
        leaf_shape[2 * k + 1] = nc;
        leaf_base[k + 1] = leaf_base[k] + nr * nc;
    }
    return GCABEM_OK;
}

}  // extern "C"
