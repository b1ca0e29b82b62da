/*
 * gcabem_b200 — C ABI of the B200 (sm_100a) BEM setup hot path.
 *
 * Drop-in boundary for the reference package `gcabem` (pure Python + numba,
 * /root/reference/pkg/src/gcabem). Each entry point names the reference
 * interface it replaces. Plain pointers and sizes only; every call returns a
 * status (0 = ok) and never throws; gcabem_last_error() holds the message of
 * the calling thread's last failure. All entry points are thread-safe; work
 * on one mesh/plan handle is ordered on that handle's CUDA stream.
 *
 * Conventions
 *   equation: 0 = laplace, 1 = helmholtz          (kernels.py:23-43 KernelSpec)
 *   layer:    0 = single, 1 = double
 *   case:     0 = disjoint, 1 = vertex, 2 = edge, 3 = identical (quadrature.py:50)
 *   complex values are interleaved (re, im) float64 pairs (numpy complex128).
 *   Triangle charts follow mesh.py:3-10: Phi(s,t) = v0 + s(v1-v0) + t(v2-v1).
 */
#ifndef GCABEM_B200_H
#define GCABEM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GCABEM_OK 0
#define GCABEM_ERR_ARG 1      /* invalid argument (ValueError on the Python side) */
#define GCABEM_ERR_CUDA 2     /* CUDA runtime failure (BackendError) */
#define GCABEM_ERR_NODEV 3    /* no CUDA device visible (BackendError) */
#define GCABEM_ERR_GCA 4      /* GCA construction failure (gca.GcaError, gca.py:43) */

typedef struct gcabem_mesh_s *gcabem_mesh_t;
typedef struct gcabem_plan_s *gcabem_plan_t;
typedef struct gcabem_layout_s *gcabem_layout_t;
typedef struct gcabem_gca_s *gcabem_gca_t;
typedef struct gcabem_h2_s *gcabem_h2_t;
typedef struct gcabem_p1_s *gcabem_p1_t;

/* ---- library / device ------------------------------------------------- */
int gcabem_version(void);
const char *gcabem_last_error(void);
int gcabem_device_count(int *count);
/* name (>= 256 bytes), SM count, SM clock kHz */
int gcabem_device_info(int device, char *name, int *sm_count, int *clock_khz);

/* Return the caches the library keeps across calls to the driver: the
 * device memory pool's free blocks (payloads and layouts are pool
 * allocations that stay cached), the GCA staging ring and the pinned layout
 * arena of `device`. Live plans, layouts and matrices are unaffected. */
int gcabem_release_cached(int device);

/* Pinned host memory for payload buffers (cudaHostAlloc / cudaFreeHost). */
int gcabem_host_alloc(int64_t nbytes, void **ptr);
int gcabem_host_free(void *ptr);

/* ---- raw pair quadrature ------------------------------------------------
 * Replaces pairquad.pair_values (reference pairquad.py:95-112; numba ABI
 * pairquad.py:18-24,31). Host arrays: ox..e2y, ny are (n,3) C-order float64,
 * gx, gy (n,), ny may be NULL (zeros), xs/ys (nq,2), w (nq,). out is
 * complex128 (n,) interleaved. Coincident points give non-finite values
 * silently, as in the reference (pairquad.py:98-99). */
int gcabem_pair_values(int device, int equation, int layer, double kappa, int64_t n,
                       const double *ox, const double *e1x, const double *e2x,
                       const double *gx, const double *oy, const double *e1y,
                       const double *e2y, const double *gy, const double *ny,
                       int64_t nq, const double *xs, const double *ys, const double *w,
                       double *out);

/* ---- device mesh replica --------------------------------------------------
 * Uploads mesh.SurfaceMesh (mesh.py:39-78): vertices (nv,3) f64, triangles
 * (nt,3) i64, normals (nt,3), gramians (nt,). Builds the per-triangle chart
 * table (mesh.chart_arrays, mesh.py:207-222, identity permutation). */
int gcabem_mesh_create(int device, int64_t nv, const double *vertices, int64_t nt,
                       const int64_t *triangles, const double *normals,
                       const double *gramians, gcabem_mesh_t *out);
int gcabem_mesh_destroy(gcabem_mesh_t mesh);

/* Index-based batch. Replaces scheduler.batch_quadrature (scheduler.py:235-261):
 * charts gathered on device from (tri, perm); perm_x/perm_y (n,3) uint8 may
 * be NULL (identity). Rule (xs,ys,w) as in gcabem_pair_values. */
int gcabem_batch_quadrature(gcabem_mesh_t mesh, int equation, int layer, double kappa,
                            int64_t n, const int64_t *tri_x, const int64_t *tri_y,
                            const uint8_t *perm_x, const uint8_t *perm_y, int64_t nq,
                            const double *xs, const double *ys, const double *w,
                            double *out);

/* ---- assembly plan --------------------------------------------------------
 * The device side of scheduler.run_assembly (scheduler.py:442-505): executes
 * every disjoint work list (execute_list :368 -> batch_quadrature :235 ->
 * distribute_disjoint :334) and then every singular list (distribute_singular
 * :362, the overwrite protocol) into one device-resident payload buffer that
 * holds all block-tree leaves (make_payloads :411) back to back, complex128.
 *
 * blocks: nblocks x 7 int64 {payload_base, ld, nrows, ncols, rows_at, cols_at,
 *   leaf} — a WorkBlock (scheduler.py:87-103), in leaf (= payload) order,
 *   leaf non-decreasing: entry (i,j) goes to
 *   payload[payload_base + i*ld + j], row panel panels[rows_at+i], column
 *   panel panels[cols_at+j]. The rule is the disjoint rule of order
 *   disjoint_n given in factored form: gauss_pts/gauss_wts (disjoint_n,)
 *   = quadrature.gauss_legendre (:82). Orders 1..12.
 * items: nitems x 4 int64 {case, tri_x, tri_y, payload_index} — WorkItem
 *   (scheduler.py:106-117) with payload_index = leaf base + offset;
 *   perms: nitems x 6 uint8 (perm_x, perm_y) from classify_pair (:197).
 *   Any order (the plan groups them by case and payload index).
 * singular rules: for case c in 1..3, sq[c-1] points, rows of 5 float64
 *   (sx, sy... see below) in srule[c-1]: {x_s, x_t, y_s, y_t, w}
 *   (quadrature.build_rule, :170). */
int gcabem_plan_create(gcabem_mesh_t mesh, int equation, int layer, double kappa,
                       int disjoint_n, const double *gauss_pts, const double *gauss_wts,
                       int64_t payload_len, int64_t nblocks, const int64_t *blocks,
                       int64_t npanels, const int64_t *panels, int64_t nitems,
                       const int64_t *items, const uint8_t *perms, const int64_t *sq,
                       const double *const *srule, gcabem_plan_t *out);
/* The same in two steps: upload the packages once as a device layout, then
 * create any number of plans (operators: SLP, DLP, orders) on it; each plan
 * holds a reference, gcabem_layout_release drops the caller's. */
int gcabem_layout_create(gcabem_mesh_t mesh, int64_t payload_len, int64_t nblocks,
                         const int64_t *blocks, int64_t npanels, const int64_t *panels,
                         int64_t nitems, const int64_t *items, const uint8_t *perms,
                         gcabem_layout_t *out);
/* The same from the flat package arrays of packaging.make_packages (leaves
 * [leaf_lo, leaf_hi) only; payload indices relative to leaf_lo): the block
 * and item gathers run natively instead of in numpy.
 * leaf_mirror (nullable, nleaves entries): for each leaf the index of the leaf
 * of the transposed cluster pair (same cluster tree and operators on both
 * sides), or -1. Leaves whose mirror lies in [leaf_lo, leaf_hi) are evaluated
 * together with it (symmetric evaluation: the reference scheduler.py:425-439
 * assembles leaf (t, s) and leaf (s, t) separately; their panel pairs are the
 * same with x and y swapped under the symmetric disjoint rule,
 * quadrature.py:108). */
int gcabem_layout_from_packages(gcabem_mesh_t mesh, int64_t leaf_lo, int64_t leaf_hi,
                                int64_t nleaves, const int64_t *leaf_shape,
                                const int64_t *leaf_base, const int64_t *leaf_rows_at,
                                const int64_t *leaf_cols_at, int64_t npanels,
                                const int64_t *panels, int64_t nblocks, const int64_t *blk_leaf,
                                const int64_t *blk_r0, const int64_t *blk_nr,
                                const int64_t *blk_c0, const int64_t *blk_nc, int64_t nitems,
                                const int8_t *item_case, const int64_t *item_tri_x,
                                const int64_t *item_tri_y, const int64_t *item_leaf,
                                const int64_t *item_offset, const uint8_t *perms,
                                const int64_t *leaf_mirror, gcabem_layout_t *out);
/* {payload_len, blocks, tasks, disjoint pairs, vertex, edge, identical items,
 * uploaded bytes} */
int gcabem_layout_info(gcabem_layout_t layout, int64_t *info8);
/* {disjoint evaluations of the mirrored kernel (each gives a pair and its
 * transpose), of the plain kernel, pairs of mirrored (PRIMARY/SELF upper)
 * blocks, pairs of blocks written by their mirror, tasks of the mirrored
 * kernel, tasks of the plain kernel on a mirrored plan} */
int gcabem_layout_mirror_info(gcabem_layout_t layout, int64_t *info6);
int gcabem_layout_release(gcabem_layout_t layout);
/* Mirrored evaluation of the layout's mirrored leaves (default: on when the
 * layout has any and the disjoint order is <= 8); 0 evaluates every block on
 * its own (the reference's one-pair-at-a-time order). */
int gcabem_plan_set_mirror(gcabem_plan_t plan, int enable);
/* {vertex items evaluated with their transpose (the vertex rule is symmetric),
 * vertex items alone, edge items, identical items, rule points evaluated per
 * identical item (half the rule: its terms come in x <-> y swapped pairs)} of
 * one execute */
int gcabem_plan_singular_evals(gcabem_plan_t plan, int64_t *out5);
int gcabem_plan_mirrored(gcabem_plan_t plan, int *out);
int gcabem_plan_create_on(gcabem_layout_t layout, int equation, int layer, double kappa,
                          int disjoint_n, const double *gauss_pts, const double *gauss_wts,
                          const int64_t *sq, const double *const *srule, gcabem_plan_t *out);
/* Fused plan of BOTH layers of one equation (the pipelines that need V and K,
 * solver.py:279-282): every kernel evaluates r, 1/r and the phase once per
 * quadrature point and accumulates the single and the double layer into two
 * payloads (same layout). Download with gcabem_plan_execute_download2 /
 * gcabem_plan_download2 (host = single layer, host2 = double layer). */
int gcabem_plan_create_pair(gcabem_layout_t layout, int equation, double kappa, int disjoint_n,
                            const double *gauss_pts, const double *gauss_wts, const int64_t *sq,
                            const double *const *srule, gcabem_plan_t *out);
/* Launch all kernels on the plan stream (async). The payload is zeroed first
 * (make_payloads semantics), then disjoint, then singular overwrites. */
int gcabem_plan_execute(gcabem_plan_t plan);
/* Execute AND stream the payload to `host` (payload_len complex128, pinned
 * for full PCIe rate) in `nchunks` leaf-aligned chunks: chunk k's D2H runs
 * on a copy stream while chunk k+1 computes. Asynchronous: call
 * gcabem_plan_synchronize before reading `host`. */
int gcabem_plan_execute_download(gcabem_plan_t plan, double *host, int nchunks);
int gcabem_plan_execute_download2(gcabem_plan_t plan, double *host, double *host2, int nchunks);
/* Symmetric download (replaces nothing in the reference: its payloads are host
 * arrays from the start, make_payloads scheduler.py:411-422; this is how the
 * device payload reaches that host image). Mirrored plans whose first payload is a single layer:
 * L/H single layer and the pair kinds): execute_download copies neither the
 * SKIP leaves of runs of at least 16384 entries nor their value: a host
 * thread of the plan writes each as the transpose of its PRIMARY leaf (the
 * mirrored kernels write one value to both entries) plus its singular entries,
 * gathered on the device (the edge rule is not symmetric). The host buffer
 * ends up bitwise equal to the device payload; gcabem_plan_synchronize also
 * waits for the host thread. enable = 0 restores full copies. */
int gcabem_plan_set_symmetric_download(gcabem_plan_t plan, int enable);
/* Bytes the last execute_download moved device -> host (both payloads and
 * the singular patch of a symmetric download). */
int gcabem_plan_d2h_bytes(gcabem_plan_t plan, int64_t *out);
/* Copy the payload (payload_len complex128) to host memory and wait. */
int gcabem_plan_download(gcabem_plan_t plan, double *host);
int gcabem_plan_download2(gcabem_plan_t plan, double *host, double *host2);
int gcabem_plan_synchronize(gcabem_plan_t plan);
/* CUDA-event durations of the last execute, ms: [disjoint, singular, total]. */
int gcabem_plan_timing(gcabem_plan_t plan, float *ms3);
/* Launch this plan's kernels on the caller's stream (a cudaStream_t; NULL
 * restores the plan's own stream) so callers can order and time several
 * plans on one timeline. */
int gcabem_plan_set_stream(gcabem_plan_t plan, void *stream);
/* Device pointer of the payload (for device-resident consumers). */
int gcabem_plan_payload(gcabem_plan_t plan, void **dev_ptr);
int gcabem_plan_destroy(gcabem_plan_t plan);

/* ---- host work packaging (CPU) -------------------------------------------
 * Native restatement of the reference scheduler's host work, bit-exact:
 * _leaf_blocks (scheduler.py:425-439), make_payloads layout (:411-422),
 * split_block (:153-175), ListBuilder (:178-208), the corrective scan of
 * distribute_disjoint (:334-359) and classify_pair (quadrature.py:197-220).
 * leaves: L x 3 {row cluster, col cluster, dense?1:0} in block-tree preorder.
 * Trees: per node start/size (int64), box lo/hi (n x 3), permutation (nt).
 * Operators: op_at (n+1) offsets into piv (pivots_global, ACA order);
 * empty range = no operator. Pass identical pointers for a shared tree.
 * Panel indices of leaf k: panels[rows_at[k] + i], panels[cols_at[k] + j]. */
typedef struct gcabem_packages_s *gcabem_packages_t;
int gcabem_packages_build(int64_t nt, const int64_t *triangles, int64_t nleaves,
                          const int64_t *leaves, int64_t nrow, const int64_t *row_start,
                          const int64_t *row_size, const double *row_lo, const double *row_hi,
                          const int64_t *row_perm, const int64_t *row_op_at,
                          const int64_t *row_piv, int64_t ncol, const int64_t *col_start,
                          const int64_t *col_size, const double *col_lo, const double *col_hi,
                          const int64_t *col_perm, const int64_t *col_op_at,
                          const int64_t *col_piv, int64_t maxsize, int nthreads,
                          gcabem_packages_t *out);
/* The same, with the panel base array [row perm | row pivots | col perm |
 * col pivots] (the col part only when the trees or operators differ) and the
 * triangles BORROWED from the caller (alive until gcabem_packages_free): the
 * leaf ranges of one staged assembly share them instead of copying them per
 * range; gcabem_packages_fetch then skips the panels (pass NULL). Replaces
 * nothing in the reference (its packaging is per-list Python,
 * scheduler.py:153-232). */
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
                             gcabem_packages_t *out);
/* sizes[9]: {L, payload_len, npanels, nblocks, nlists, nitems, 0, 0, 0} */
int gcabem_packages_sizes(gcabem_packages_t pk, int64_t *sizes);
/* Planar (field-major) outputs: blocks 5 x nblocks {leaf, r0, nr, c0, nc};
 * items 6 x nitems {case 1..3, tri_x, tri_y, leaf, offset in leaf,
 * generating block}; perms nitems x 6 (perm_x, perm_y). */
int gcabem_packages_fetch(gcabem_packages_t pk, int64_t *panels, int64_t *leaf_shape,
                          int64_t *leaf_base, int64_t *rows_at, int64_t *cols_at,
                          uint8_t *flagged, int64_t *blocks, int64_t *blk_list, int64_t *items,
                          uint8_t *perms);
int gcabem_packages_free(gcabem_packages_t pk);
/* Payload layout of the leaves alone (the leaf loop of gcabem_packages_build,
 * make_payloads scheduler.py:411-422): leaf_shape L x 2 {rows, cols} (dense
 * |t| x |s|, admissible rank_t x rank_s), leaf_base L + 1 prefix offsets. */
int gcabem_leaf_layout(int64_t nleaves, const int64_t *leaves, int64_t nrow,
                       const int64_t *row_size, const int64_t *row_op_at, int64_t ncol,
                       const int64_t *col_size, const int64_t *col_op_at, int64_t *leaf_shape,
                       int64_t *leaf_base);

/* ---- GCA Green matrices ---------------------------------------------------
 * Replaces gca.build_green_matrix (gca.py:136-179), batched over clusters.
 * Cluster c owns panels[panel_at[c] .. panel_at[c+1]) and nsrc sources at
 * src + c*nsrc*8, each {px,py,pz, nx,ny,nz, weight, role} (role 0 monopole,
 * 1 dipole; GreenSourceSet gca.py:47-52). Output for cluster c starts at
 * entry out_at[c] (entries, row-major |t| x nsrc), real float64 for laplace,
 * complex128 for helmholtz: A[i,j] = w_j * gram_i * sum_q wq k_j(X_iq).
 * duffy (order^2 x 3 rows {s, t, wq}) = quadrature.duffy_panel_rule(order). */
int gcabem_green_matrices(gcabem_mesh_t mesh, int equation, double kappa, int64_t nclusters,
                          const int64_t *panel_at, const int64_t *panels, int64_t nsrc,
                          const double *src, int64_t nduffy, const double *duffy,
                          const int64_t *out_at, int64_t out_len, double *out_host);

/* ---- cluster / block trees (host) -------------------------------------------
 * Bit-exact restatements of cluster.build_cluster_tree (cluster.py:87-122)
 * and cluster.build_block_tree (:125-152), preorder node numbering. The
 * block tree takes node diameters precomputed by the host's own norm and a
 * norm_variant (0..3) for the distances that the caller verified reproduces
 * np.linalg.norm bit for bit (gcabem_norm3 probes the variants). */
typedef struct gcabem_tree_s *gcabem_tree_t;
int gcabem_cluster_tree(int64_t nt, const double *tri_lo, const double *tri_hi,
                        const double *mid, int64_t leaf_size, gcabem_tree_t *out);
/* The same from the mesh: triangles (nt x 3, int64) and vertices (nv x 3);
 * the bounds and midpoints are formed natively (mesh.py:65-73). */
int gcabem_cluster_tree_mesh(int64_t nt, const int64_t *triangles, const double *vertices,
                             int64_t leaf_size, gcabem_tree_t *out);
int gcabem_block_tree(int64_t nrow, const int64_t *row_c0, const int64_t *row_c1,
                      const double *row_lo, const double *row_hi, const double *row_diam,
                      int64_t ncol, const int64_t *col_c0, const int64_t *col_c1,
                      const double *col_lo, const double *col_hi, const double *col_diam,
                      double eta, int norm_variant, gcabem_tree_t *out);
int gcabem_norm3(int64_t n, const double *v, int variant, double *out);
int gcabem_tree_sizes(gcabem_tree_t t, int64_t *sizes);
int gcabem_tree_fetch(gcabem_tree_t t, int64_t *a, int64_t *b, int64_t *c, int64_t *d,
                      int64_t *e, int64_t *f, double *lo, double *hi);
int gcabem_tree_free(gcabem_tree_t t);

/* ---- ACA (host, threaded) ---------------------------------------------------
 * Partially pivoted ACA of many Green matrices (gca.aca, gca.py:182-245; the
 * CPU keeps the pivoting per north_star). Cluster c's matrix is rows
 * [rows_at[c], rows_at[c+1]) x ncols, row-major, starting at entry
 * rows_at[c]*ncols of A (float64, or interleaved complex128 if is_complex).
 * Pivots of cluster c are written at out_rows/out_cols + rows_at[c], its rank
 * to out_rank[c] and the last |u||v| to out_resid[c]. max_rank <= 0: none. */
int gcabem_aca_batch(int is_complex, int64_t ncl, const int64_t *rows_at, int64_t ncols,
                     const double *A, double epsilon, int64_t max_rank, int nthreads,
                     int64_t *out_rank, int64_t *out_rows, int64_t *out_cols,
                     double *out_resid);

/* ---- GCA interpolation operators of many clusters -------------------------
 * Replaces gca.build_interpolation_operators' per-cluster loop (reference
 * gca.py:285-310 -> build_interpolation_operator :259-282): for every
 * cluster c (ids cl_ids, panels perm[cl_first[c] .. + cl_size[c]], bounding
 * box box_lo/box_hi (ncl,3)) the device evaluates the Green matrix against
 * green_sources(box, delta, m) (gca.py:83-133; Gauss rule gauss_pts/wts of
 * order m on [0,1], scene_diameter for degenerate boxes) with the Duffy
 * panel rule (nduffy rows {s, t, w}); the host runs ACA (epsilon, one retry
 * at epsilon/10), the cond <= 1e14 pivot check and the refined V solve on
 * nthreads threads, overlapped with the next batch (batch_bytes of Green
 * matrix per launch, 4 launches in flight; 0 = 32 MiB).
 * Results: gcabem_gca_sizes (rank per
 * cluster, phase6 {device wait s, pipeline wall s, total s, batches, host
 * thread-seconds, threads}), then
 * gcabem_gca_fetch (row pivots concatenated; V blocks |t| x rank row-major,
 * float64 for Laplace, complex128 for Helmholtz, concatenated).
 * GCABEM_ERR_GCA: "cluster <id>: zero Green matrix" / "singular ACA pivot
 * block" as the reference's GcaError. */
int gcabem_gca_build(gcabem_mesh_t mesh, int equation, double kappa, int64_t ncl,
                     const int64_t *cl_ids, const int64_t *cl_first, const int64_t *cl_size,
                     const double *box_lo, const double *box_hi, int64_t nperm,
                     const int64_t *perm, double delta, int m, const double *gauss_pts,
                     const double *gauss_wts, double scene_diameter, int64_t nduffy,
                     const double *duffy, double epsilon, int nthreads, int64_t batch_bytes,
                     gcabem_gca_t *out);
int gcabem_gca_sizes(gcabem_gca_t g, int64_t *ranks, double *phase6);
int gcabem_gca_fetch(gcabem_gca_t g, int64_t *rows, double *V);
/* Per cluster (order of cl_ids): 1 if one of its ACA decisions (an argmax
 * over a residual row/column, the stopping test) had a margin inside the
 * roundoff of the device's Green matrix, i.e. the reference's numpy bits
 * could decide it the other way. Such clusters were redone by the pipeline
 * on entries evaluated in the reference's arithmetic (gcabem_green_exact). */
int gcabem_gca_flags(gcabem_gca_t g, int8_t *ambiguous);
/* Host only: one cluster's Green matrix with every entry evaluated in the
 * reference's numpy arithmetic (gca.py:136-179, kernels.py:46-64; the
 * sources of gca.py:83-133 from the box [box_lo, box_hi]), written to A
 * (nr x 12 m^2, float64 or interleaved complex128; may be NULL), and, when
 * rank/rows/V are given, the operator the GCA pipeline computes for a
 * cluster it redoes on these entries (ACA + check + V solve). The pipeline
 * uses the same evaluation internally for the clusters gcabem_gca_flags
 * reports. */
int gcabem_green_exact(int equation, double kappa, int64_t nv, const double *vertices,
                       int64_t nt, const int64_t *triangles, const double *gramians, int64_t nr,
                       const int64_t *panels, const double *box_lo, const double *box_hi,
                       double delta, int m, const double *gauss_pts, const double *gauss_wts,
                       double scene_diameter, int64_t nduffy, const double *duffy,
                       double epsilon, double *A, int64_t *rank, int64_t *rows, double *V);
int gcabem_gca_free(gcabem_gca_t g);
/* One cluster's operator from a host Green matrix A (nr x nc row-major,
 * float64 or interleaved complex128): ACA + cond check + refined V solve
 * (gca.py:259-282). rows and V must hold min(nr, nc) pivots / nr x min(nr, nc)
 * values; *rank receives the rank. */
int gcabem_gca_operator(int is_complex, const double *A, int64_t nr, int64_t nc, double epsilon,
                        int64_t *rank, int64_t *rows, double *V);

/* ---- device-resident compressed operator and matvec ------------------------
 * Replaces h2.matvec (reference h2.py:49-71): y = sum over leaves of dense
 * P x[s] and admissible V_t (P (V_s^T x[s])), in the permuted index space of
 * the row / column trees (row_perm, col_perm). leaf_desc (nleaves x 7):
 * {row_start, row_size, col_start, col_size, dense, row_op, col_op};
 * leaf_base: payload offset per leaf (complex128 payload, payload_len);
 * rowop_desc / colop_desc (n x 4): {cluster start, size, rank, offset in V};
 * V: all bases stacked (complex128, v_len). The product is a sequence of
 * gathers with a fixed summation order: bitwise reproducible. x, y host
 * complex128; device_ms (nullable) gets the device time of the product. */
int gcabem_h2_create(int device, int64_t nrows, int64_t ncols, const int64_t *row_perm,
                     const int64_t *col_perm, int64_t nleaves, const int64_t *leaf_desc,
                     const int64_t *leaf_base, int64_t payload_len, const double *payload,
                     int64_t nrowops, const int64_t *rowop_desc, int64_t ncolops,
                     const int64_t *colop_desc, int64_t v_len, const double *V,
                     gcabem_h2_t *out);
int gcabem_h2_matvec(gcabem_h2_t h, const double *x, double *y, float *device_ms);
int gcabem_h2_info(gcabem_h2_t h, double *bytes_per_product);
int gcabem_h2_free(gcabem_h2_t h);

/* ---- piecewise-linear (P1) near field ------------------------------------
 * Extension beyond the reference's P0 assembly (BASELINE
 * config 4). Per near-field pair of the layout (build it from the dense
 * leaves only), the 3 x 3 local matrix M[a][b] = g_x g_y sum_q w_q
 * lambda_a(x_q) k lambda_b(y_q), lambda = (1 - s, s - t, t) -- the reference's
 * integrate_pair(..., basis_x=lambda_a, basis_y=lambda_b) (quadrature.py:
 * 223-271) -- in the triangles' stored vertex order; then the vertex x vertex
 * near-field matrix (CSR, columns ascending) by a deterministic gather-sum
 * (fixed contribution order, no atomics). create builds the scatter plan
 * (device radix sort of the 9 entry keys); execute runs the local matrices
 * and the gather; info {nv, nnz, pairs, singular items} + ms {local, gather};
 * download: row_ptr (nv + 1), col (nnz), values (nnz complex128), local
 * (nullable; pairs x 9 complex128, payload order). */
int gcabem_p1_create(gcabem_layout_t layout, int equation, int layer, double kappa,
                     int disjoint_n, const double *gauss_pts, const double *gauss_wts,
                     const int64_t *sq, const double *const *srule, gcabem_p1_t *out);
int gcabem_p1_execute(gcabem_p1_t p1);
int gcabem_p1_info(gcabem_p1_t p1, int64_t *info4, float *ms2);
int gcabem_p1_download(gcabem_p1_t p1, int64_t *row_ptr, int32_t *col, double *values,
                       double *local);
int gcabem_p1_destroy(gcabem_p1_t p1);
/* P1 local matrices of caller-given pairs under any 4D rule (n x 9 complex128). */
int gcabem_p1_batch(gcabem_mesh_t mesh, int equation, int layer, double kappa, int64_t n,
                    const int64_t *tri_x, const int64_t *tri_y, const uint8_t *perm_x,
                    const uint8_t *perm_y, int64_t nq, const double *xs, const double *ys,
                    const double *w, double *out);

/* ---- potential evaluation --------------------------------------------------
 * Replaces scheduler.potential_batch (scheduler.py:508-534): out (npts x nt,
 * complex128 row-major) = plain panel integrals of the kernel field at each
 * point, the disjoint rule of `order` (1..8) with a zero-extent x chart and
 * gx = 2. Points on the surface give non-finite entries (the caller raises). */
int gcabem_potential(gcabem_mesh_t mesh, int equation, int layer, double kappa, int order,
                     const double *gauss_pts, const double *gauss_wts, int64_t npts,
                     const double *points, double *out);

/* ---- diagnostics ------------------------------------------------------------ */
/* Dependent-DFMA throughput probe: achieved FP64 TFLOP/s (FMA = 2 flops). */
int gcabem_fp64_probe(int device, double *tflops);

#ifdef __cplusplus
}
#endif
#endif
