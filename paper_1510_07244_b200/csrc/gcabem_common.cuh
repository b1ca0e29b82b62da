// Shared device-side definitions of the gcabem_b200 library (sm_100a).
//
// Data layout in HBM:
//   Chart[nt]      128 B per triangle = one L2 line: origin, edge1, edge2,
//                  unit normal, Gramian (mesh.chart_arrays, reference
//                  mesh.py:207-222, identity permutation; normals/gramians
//                  from make_surface_mesh mesh.py:111-116).
//   BlockDesc[]    one per WorkBlock (scheduler.py:87-103).
//   payload        double2[payload_len]: all block-tree leaves back to back
//                  in preorder, row-major (make_payloads scheduler.py:411-422).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gcabem {

struct __align__(16) Chart {
    double o[3], e1[3], e2[3], n[3], gram;
    double radius;  // bounding-sphere radius about the centroid (upper bound)
    double enorm;   // |e1| + |e2| (upper bound)
    double pad;
};
static_assert(sizeof(Chart) == 128, "Chart must be one 128 B line");

// Mirror roles of a block (symmetric evaluation): on a shared
// cluster tree with shared operators, leaf (t, s) and leaf (s, t) hold the
// integrals of the same panel pairs with the roles of x and y swapped (the
// disjoint rule is a symmetric tensor product), so one thread evaluates pair
// (i, j) and its transpose (j, i) together: the single layer is the same
// value, the double layer of (j, i) shares r, 1/r and the phase and differs
// only in d . n (the normal of panel i instead of j).
enum BlockRole { ROLE_NORMAL = 0,   // no mirror in this layout: evaluated alone
                 ROLE_PRIMARY = 1,  // writes its entries and the mirror leaf's
                 ROLE_SELF = 2,     // diagonal leaf (t, t): the upper triangle
                                    // writes both (i, j) and (j, i)
                 ROLE_SKIP = 3 };   // written by its (earlier) primary

struct BlockDesc {
    int64_t base;     // payload index of entry (0,0)
    int64_t rows_at;  // offset of the row panels in the panel array
    int64_t cols_at;  // offset of the column panels
    int32_t ld;       // payload row stride (leaf ncols)
    int32_t nr, nc;
    int32_t role;     // BlockRole
    int64_t mbase;    // PRIMARY/SELF: payload index of the transposed entry (0,0)
    int32_t mld;      //   its row stride: entry (i, j) mirrors to mbase + j mld + i
    int32_t dr;       // SELF: r0 - c0 (leaf row minus leaf column of entry (0,0))
};
static_assert(sizeof(BlockDesc) == 56, "BlockDesc layout");

// one disjoint task: its block's descriptor and the task's first pair, so a
// disjoint CTA's prologue loads one record instead of task -> block (one
// dependent global load fewer before the panel indices and charts)
struct __align__(16) TaskDesc {
    BlockDesc b;
    int32_t k0;   // first pair of the task (row-major in the block)
    int32_t pad;
};
static_assert(sizeof(TaskDesc) == 64, "TaskDesc layout");

struct SingItem {
    int64_t out;          // payload index (leaf base + WorkItem.offset)
    int32_t tri_x, tri_y;
    uint8_t px[3], py[3]; // classify_pair permutations
    uint8_t pad[2];
};
static_assert(sizeof(SingItem) == 24, "SingItem layout");

struct GreenBox {
    double center[3], half[3];  // enlarged box of one cluster (gca.py:103-107)
};

enum Kind { L_SLP = 0, L_DLP = 1, H_SLP = 2, H_DLP = 3,
            // fused SLP + DLP of one equation: one evaluation of r, 1/r and the
            // phase feeds both operators' accumulators (two payloads)
            L_PAIR = 4, H_PAIR = 5 };
__host__ __device__ constexpr bool kind_helm(int k) { return k == H_SLP || k == H_DLP || k == H_PAIR; }
__host__ __device__ constexpr bool kind_normal(int k) { return k == L_DLP || k == H_DLP || k >= L_PAIR; }
__host__ __device__ constexpr bool kind_pair(int k) { return k >= L_PAIR; }
constexpr int MAX_ORDER = 12;
// pairs per disjoint task = threads per CTA of the disjoint, P1 and key kernels:
// one warp, so a block's last task wastes at most 31 lanes (the coupling
// blocks are rank x rank, any size) and CTAs start and retire at a fine grain
// (C3 step 28.53 -> 28.11 ms, C2 9.02 -> 8.93 ms against 128-pair tasks)
constexpr int DISJOINT_TPB = 32;
#ifndef GCABEM_GENERIC_TPB
#define GCABEM_GENERIC_TPB 128
#endif
constexpr int GENERIC_TPB = GCABEM_GENERIC_TPB;
constexpr int GREEN_TPB = 128;
#ifndef GCABEM_RULE_CHUNK
#define GCABEM_RULE_CHUNK 256
#endif
constexpr int RULE_CHUNK = GCABEM_RULE_CHUNK;  // rule points staged in shared memory at once

inline int kind_of(int equation, int layer) { return equation * 2 + layer; }

// ---- launchers (kernels.cu) ------------------------------------------------
cudaError_t upload_disjoint_rule(int order, const double *gauss_pts, const double *gauss_wts);
// kind L_PAIR / H_PAIR: payload gets the single layer, payload2 the double
// layer (payload2 unused otherwise). kind + MIRRORED: the mirrored kernel over
// ROLE_PRIMARY / ROLE_SELF tasks (orders <= MAX_MIRROR_ORDER).
constexpr int MIRRORED = 8;
constexpr int MAX_MIRROR_ORDER = 8;
// symmetric download: SKIP-leaf runs of at least this many payload entries
// (256 KB) are written on the host from their PRIMARY instead of copied
#ifndef GCABEM_SYM_MIN_RUN
#define GCABEM_SYM_MIN_RUN 16384
#endif
constexpr int64_t SYM_MIN_RUN = GCABEM_SYM_MIN_RUN;
cudaError_t launch_disjoint(int kind, int order, const Chart *charts, const int32_t *T,
                            const TaskDesc *tasks, int64_t ntasks, const int32_t *panels,
                            double2 *payload, double2 *payload2, double kappa, cudaStream_t s);
// Generic-rule pair integrals: singular lists (vertex/edge/identical) and the
// index-based batch. Charts gathered with permutations from V/T.
// same_chart: every item has tri_x == tri_y and perm_x == perm_y (identical case).
// grouped form of a singular rule (kernels.cu generic_pair_grouped): groups
// {a, b, first row, row count, side} (doubles; side 0: x point (a, b) fixed,
// rows {ys, yt, w}; side 1: y point fixed, rows {xs, xt, w}), chunks
// {row0, row1, group0, group1} of at most RULE_CHUNK rows / groups each.
constexpr int GROUP_REC = 5;
struct GroupedRule {
    const double *rows = nullptr;
    const double *groups = nullptr;
    const int4 *chunks = nullptr;
    int nchunks = 0;
    // identical case (SAME): the rule passed is the base half of a rule whose
    // terms come in swapped pairs (quadrature.py:132-143): single layer x 2,
    // double layer 0 (exactly cancelling pairs; see generic_kernel)
    int sym_half = 0;
};
cudaError_t launch_generic(int kind, bool same_chart, const double *V, const int32_t *T,
                           const Chart *charts, const SingItem *items, int64_t n,
                           const double *rule, int64_t q, double2 *payload, double2 *payload2,
                           double kappa, cudaStream_t s, GroupedRule grouped = GroupedRule());
// one singular list of a fused launch (launch_singular_fused)
struct SingularSeg {
    const SingItem *items = nullptr;
    const int64_t *mout = nullptr;   // mirrored vertex items (else nullptr)
    int64_t n = 0;
    const double *rule = nullptr;    // staged rule (ungrouped / identical)
    int64_t q = 0;
    int same = 0;                    // identical items (exact-difference form)
    GroupedRule grouped;
};
struct SingularBatch {
    SingularSeg seg[4];
    int64_t cta_at[5] = {0, 0, 0, 0, 0};
};
cudaError_t launch_singular_fused(int kind, const double *V, const int32_t *T,
                                  const Chart *charts, const SingularBatch &b,
                                  double2 *payload, double2 *payload2, double kappa,
                                  cudaStream_t s);
// mirrored vertex items: item idx also writes the transposed pair at mout[idx]
cudaError_t launch_generic_mirror(int kind, const double *V, const int32_t *T,
                                  const Chart *charts, const SingItem *items,
                                  const int64_t *mout, int64_t n, double2 *payload,
                                  double2 *payload2, double kappa, cudaStream_t s,
                                  GroupedRule grouped);
// Raw charts (gcabem_pair_values): per pair 22 doubles
// {ox,e1x,e2x, oy,e1y,e2y, ny} (21) + gx, gy packed as 24 doubles.
cudaError_t launch_raw(int kind, const double *pairs, int64_t n, const double *rule, int64_t q,
                       double2 *out, double kappa, cudaStream_t s);
cudaError_t launch_green(int equation, const Chart *charts, const int2 *tasks, int64_t ntasks,
                         const int64_t *panel_at, const int32_t *panels, const int64_t *out_at,
                         int nsrc, const double *src, const double *duffy, int nq, double *out,
                         double kappa, cudaStream_t s);
// Green matrices of a batch of clusters with device-generated sources;
// out (per cluster |t| x 12 m^2, row-major) at out_at[c] elements (double or
// double2 by equation). Panels of cluster c: perm[cl_first[c] + i].
cudaError_t launch_green_box(int equation, const Chart *charts, const int2 *tasks, int64_t ntasks,
                             const int64_t *cl_first, const int32_t *cl_size, const int32_t *perm,
                             const GreenBox *boxes, int m, const double *gq, const double *duffy,
                             int nq, const int64_t *out_at, double *out, double kappa,
                             cudaStream_t s);
cudaError_t launch_potential(int kind, int order, const Chart *charts, int64_t nt,
                             const double *pts, int64_t npts, double xw, double2 *out,
                             double kappa, cudaStream_t s);
cudaError_t launch_fp64_probe(double *sink, int iters, int blocks, cudaStream_t s);

}  // namespace gcabem
