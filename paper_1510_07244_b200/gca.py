"""Green cross approximation: per-cluster interpolation operators.

Drop-in for gcabem.gca (pkg/src/gcabem/gca.py). Per cluster t, monopole and
dipole sources sit on a tensor Gauss grid over the boundary of the
(1 + delta)-enlarged box; the Green matrix A_t (panel integrals of those
source fields) is compressed by partially pivoted ACA; row pivots become
the interpolation points and V = A_t[:, ct] A_t[tt, ct]^-1.

Split (north_star): the Green matrices of ALL clusters are evaluated in
batched sm_100a launches with the sources generated on the device
(csrc/kernels.cu green_box_kernel); the pivoting (ACA), the pivot-block
check and the small V solves stay on the CPU, natively on all cores
(csrc/aca.cpp), overlapped with the next batch of Green matrices
(csrc/gca_pipeline.cu, C ABI gcabem_gca_build).
"""
from __future__ import annotations

import ctypes
import time
from collections.abc import MutableMapping
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .cluster import BlockTree, ClusterTree
from .device import device_mesh
from .kernels import KernelSpec
from .mesh import SurfaceMesh
from .pairquad import default_device
from .quadrature import duffy_panel_rule, gauss_legendre

ROLE_MONOPOLE = 0
ROLE_DIPOLE = 1

DEFAULT_DELTA = 1.0
DEFAULT_FACE_POINTS = 6
DEFAULT_EPSILON = 1e-4

_PIVOT_COND_LIMIT = 1e14


class GcaError(RuntimeError):
    """Green cross approximation construction failure (gca.py:43)."""


@dataclass(frozen=True)
class GreenSourceSet:
    points: np.ndarray   # (P, 3)
    weights: np.ndarray  # (P,)
    normals: np.ndarray  # (P, 3)
    roles: np.ndarray    # (P,) uint8

    def packed(self) -> np.ndarray:
        """(P, 8) device rows {p, n, w, role}."""
        return np.column_stack([self.points, self.normals, self.weights,
                                self.roles.astype(np.float64)])


@dataclass(frozen=True)
class ACAResult:
    row_pivots: np.ndarray
    col_pivots: np.ndarray
    rank: int
    residual_estimate: float


@dataclass(frozen=True)
class InterpolationOperator:
    cluster: int
    pivots_local: np.ndarray
    pivots_global: np.ndarray
    V: np.ndarray

    @property
    def rank(self) -> int:
        return int(self.V.shape[1])


@dataclass(frozen=True)
class GcaParams:
    delta: float = DEFAULT_DELTA
    m: int = DEFAULT_FACE_POINTS
    epsilon: float = DEFAULT_EPSILON
    rule_order: int = 3


def green_sources(box_lo, box_hi, delta: float, m: int,
                  scene_diameter: float = 0.0) -> GreenSourceSet:
    """m x m Gauss points per face of the box grown by delta * (largest
    half-extent), each point twice (monopole, dipole); face order axis 0,1,2,
    negative side first (gca.py:83-133)."""
    if delta <= 0.0:
        raise ValueError("delta must be > 0")
    if m < 1:
        raise ValueError("m must be >= 1")
    lo = np.asarray(box_lo, dtype=np.float64)
    hi = np.asarray(box_hi, dtype=np.float64)
    center = 0.5 * (lo + hi)
    hmax = 0.5 * max(float(np.max(hi - lo)), 1e-8 * scene_diameter)
    if hmax <= 0.0:
        raise ValueError("degenerate box with no scene diameter to fall back on")
    half = 0.5 * (hi - lo) + delta * hmax
    g = gauss_legendre(m)
    wuv = (np.repeat(g.weights, m) * np.tile(g.weights, m))
    P, W, N = [], [], []
    for axis in range(3):
        a1, a2 = (axis + 1) % 3, (axis + 2) % 3
        u = -half[a1] + 2.0 * half[a1] * g.points
        v = -half[a2] + 2.0 * half[a2] * g.points
        face_w = wuv * (4.0 * half[a1] * half[a2])
        for sign in (-1.0, 1.0):
            pts = np.empty((m * m, 3))
            pts[:, axis] = center[axis] + sign * half[axis]
            pts[:, a1] = center[a1] + np.repeat(u, m)
            pts[:, a2] = center[a2] + np.tile(v, m)
            nrm = np.zeros((m * m, 3))
            nrm[:, axis] = sign
            P.append(np.repeat(pts, 2, axis=0))
            W.append(np.repeat(face_w, 2))
            N.append(np.repeat(nrm, 2, axis=0))
    roles = np.tile(np.array([ROLE_MONOPOLE, ROLE_DIPOLE], dtype=np.uint8), 6 * m * m)
    return GreenSourceSet(np.concatenate(P), np.concatenate(W), np.concatenate(N), roles)


def build_green_matrices(mesh: SurfaceMesh, panel_lists, source_sets, spec: KernelSpec,
                         order: int = 3, device: int | None = None, flat: bool = False):
    """Green matrices of many clusters in one device launch (gca.py:136-179).

    A[i, j] = w_j * integral over panel i of source field j: monopole
    columns use the single layer of spec.equation, dipole columns its
    derivative along the source normal (d = x - source). float64 for
    Laplace, complex128 for Helmholtz.
    """
    device = default_device() if device is None else device
    ncl = len(panel_lists)
    if ncl == 0:
        return []
    nsrc = len(source_sets[0].weights)
    if any(len(s.weights) != nsrc for s in source_sets):
        raise ValueError("all source sets of one batch must have the same size")
    dm = device_mesh(mesh, device)
    sizes = np.array([len(p) for p in panel_lists], dtype=np.int64)
    panel_at = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    panels = np.concatenate([np.asarray(p, dtype=np.int64) for p in panel_lists]) \
        if sizes.sum() else np.empty(0, np.int64)
    out_at = (panel_at[:-1] * nsrc).astype(np.int64)
    out_len = int(panel_at[-1] * nsrc)
    src = np.ascontiguousarray(np.stack([s.packed() for s in source_sets]))
    pts, wq = duffy_panel_rule(order)
    duffy = np.ascontiguousarray(np.column_stack([pts, wq]))
    complex_out = spec.is_complex
    buf = np.empty(out_len * (2 if complex_out else 1), dtype=np.float64)
    eq = 0 if spec.equation == "laplace" else 1
    nat.check(nat.lib().gcabem_green_matrices(
        dm.handle, eq, float(spec.kappa), ncl, nat.ptr(panel_at), nat.ptr(panels), nsrc,
        nat.ptr(src), duffy.shape[0], nat.ptr(duffy), nat.ptr(out_at), out_len,
        nat.ptr(buf)))
    vals = buf.view(np.complex128) if complex_out else buf
    if not np.all(np.isfinite(vals)):
        raise GcaError("source coincides with a panel quadrature point")
    mats = [vals[out_at[c]:out_at[c] + sizes[c] * nsrc].reshape(sizes[c], nsrc)
            for c in range(ncl)]
    return (mats, buf, panel_at) if flat else mats


_PANEL_CHUNK = 256


def green_matrix_exact(mesh: SurfaceMesh, panels, sources: GreenSourceSet, spec: KernelSpec,
                       order: int = 3) -> np.ndarray:
    """One cluster's Green matrix on the HOST, in the reference's own numpy
    arithmetic (gca.py:136-179 operation for operation: 256-panel chunks,
    chart_arrays, the broadcast point map, kernel_values per column group,
    einsum over the panel rule, then the Gramian and the source weights), so
    its bits are the reference's. The yardstick of the native exact entries
    (green_exact_native, csrc/green_exact.h) that settle ACA decisions the
    device's matrix leaves inside the tie window."""
    from .kernels import kernel_values
    from .mesh import chart_arrays
    panels = np.asarray(panels, dtype=np.int64)
    pts, wq = duffy_panel_rule(order)
    mono_spec = KernelSpec(spec.equation, "single", spec.kappa)
    dip_spec = KernelSpec(spec.equation, "double", spec.kappa)
    A = np.empty((len(panels), len(sources.weights)),
                 dtype=np.complex128 if spec.is_complex else np.float64)
    src, srcn = sources.points, sources.normals
    mono = sources.roles == ROLE_MONOPOLE
    dip = ~mono
    for base in range(0, len(panels), _PANEL_CHUNK):
        sel = panels[base:base + _PANEL_CHUNK]
        v0, e1, e2, gram = chart_arrays(mesh, sel)
        X = v0[:, None, :] + pts[None, :, 0, None] * e1[:, None, :] \
            + pts[None, :, 1, None] * e2[:, None, :]
        kv_m = kernel_values(mono_spec, X[:, :, None, 0] - src[None, None, mono, 0],
                             X[:, :, None, 1] - src[None, None, mono, 1],
                             X[:, :, None, 2] - src[None, None, mono, 2])
        nd = srcn[dip]
        kv_d = kernel_values(dip_spec, X[:, :, None, 0] - src[None, None, dip, 0],
                             X[:, :, None, 1] - src[None, None, dip, 1],
                             X[:, :, None, 2] - src[None, None, dip, 2],
                             nd[None, None, :, 0], nd[None, None, :, 1], nd[None, None, :, 2])
        if not (np.all(np.isfinite(kv_m)) and np.all(np.isfinite(kv_d))):
            raise GcaError("source coincides with a panel quadrature point")
        im = np.einsum("q,pqs->ps", wq, kv_m) * gram[:, None]
        idp = np.einsum("q,pqs->ps", wq, kv_d) * gram[:, None]
        A[base:base + len(sel), mono] = im * sources.weights[mono]
        A[base:base + len(sel), dip] = idp * sources.weights[dip]
    return A


def green_exact_native(mesh: SurfaceMesh, panels, box_lo, box_hi, spec: KernelSpec,
                       params: GcaParams, scene_diameter: float, operator: bool = True):
    """The native host-exact path of one cluster (C ABI gcabem_green_exact):
    its full Green matrix from csrc/green_exact.h and, with operator=True, the
    operator (row pivots, V) the GCA pipeline's tie redo computes."""
    panels = np.ascontiguousarray(panels, dtype=np.int64)
    nr = panels.size
    nc = 12 * params.m * params.m
    w = 2 if spec.is_complex else 1
    A = np.empty(nr * nc * w, np.float64)
    g = gauss_legendre(params.m)
    pts, wq = duffy_panel_rule(params.rule_order)
    duffy = np.ascontiguousarray(np.column_stack([pts, wq]))
    cap = min(nr, nc)
    rank = np.zeros(1, np.int64)
    rows = np.zeros(cap, np.int64)
    V = np.zeros(nr * cap * w, np.float64)
    p = nat.ptr
    T = np.ascontiguousarray(mesh.triangles, dtype=np.int64)
    nat.check(nat.lib().gcabem_green_exact(
        0 if spec.equation == "laplace" else 1, float(spec.kappa), mesh.num_vertices,
        p(nat.f64(mesh.vertices)), mesh.num_triangles, p(T), p(nat.f64(mesh.gramians)), nr,
        p(panels), p(nat.f64(box_lo)), p(nat.f64(box_hi)), float(params.delta), int(params.m),
        p(nat.f64(g.points)), p(nat.f64(g.weights)), float(scene_diameter), duffy.shape[0],
        p(duffy), float(params.epsilon), p(A), p(rank) if operator else None,
        p(rows) if operator else None, p(V) if operator else None))
    Am = (A.view(np.complex128) if spec.is_complex else A).reshape(nr, nc)
    if not operator:
        return Am
    r = int(rank[0])
    Vv = (V.view(np.complex128) if spec.is_complex else V)[:nr * r].reshape(nr, r)
    return Am, rows[:r].copy(), Vv


def build_green_matrix(mesh: SurfaceMesh, panels, sources: GreenSourceSet, spec: KernelSpec,
                       order: int = 3) -> np.ndarray:
    """One cluster's Green matrix (gca.py:136), on the device."""
    return build_green_matrices(mesh, [np.asarray(panels, dtype=np.int64)], [sources],
                                spec, order)[0]


def aca_batch(flat: np.ndarray, rows_at: np.ndarray, ncols: int, is_complex: bool,
              epsilon: float, max_rank: int | None = None, nthreads: int = 0):
    """Native threaded ACA of many matrices (C ABI gcabem_aca_batch):
    returns [(row_pivots, col_pivots, residual)] per matrix."""
    if epsilon <= 0.0:
        raise ValueError("epsilon must be > 0")
    rows_at = np.ascontiguousarray(rows_at, dtype=np.int64)
    ncl = rows_at.size - 1
    total = int(rows_at[-1])
    rank = np.zeros(ncl, np.int64)
    rows = np.zeros(max(total, 1), np.int64)
    cols = np.zeros(max(total, 1), np.int64)
    resid = np.zeros(ncl, np.float64)
    flat = np.ascontiguousarray(flat, dtype=np.float64)
    nat.check(nat.lib().gcabem_aca_batch(
        int(is_complex), ncl, nat.ptr(rows_at), int(ncols), nat.ptr(flat), float(epsilon),
        int(max_rank or 0), int(nthreads), nat.ptr(rank), nat.ptr(rows), nat.ptr(cols),
        nat.ptr(resid)))
    return [(rows[rows_at[c]:rows_at[c] + rank[c]].copy(),
             cols[rows_at[c]:rows_at[c] + rank[c]].copy(), float(resid[c])) for c in range(ncl)]


def aca(matrix: np.ndarray, epsilon: float, max_rank: int | None = None) -> ACAResult:
    """Partially pivoted ACA (gca.py:182-245): next row = largest residual
    column entry among unused rows, next column = largest residual row entry
    (ties to the lowest index); stop when |u||v| <= eps * sqrt(estimate).
    Native (csrc/aca.cpp)."""
    A = np.asarray(matrix)
    is_complex = np.iscomplexobj(A)
    flat = np.ascontiguousarray(A, dtype=np.complex128 if is_complex else np.float64)
    (r, c, res), = aca_batch(flat.view(np.float64).ravel(), np.array([0, A.shape[0]]),
                             A.shape[1], is_complex, epsilon, max_rank, nthreads=1)
    return ACAResult(r, c, int(r.size), res)


def _solve_with_refinement(A_cols: np.ndarray, pivot_block: np.ndarray) -> np.ndarray:
    """V = A_cols inv(pivot_block) plus two refinement sweeps (gca.py:248-256)."""
    V = np.linalg.solve(pivot_block.T, A_cols.T).T
    for _ in range(2):
        R = A_cols - V @ pivot_block
        if np.max(np.abs(R)) <= 1e-15 * max(np.max(np.abs(A_cols)), 1.0):
            break
        V = V + np.linalg.solve(pivot_block.T, R.T).T
    return V


def _operator_from_green(cluster_index: int, panels: np.ndarray, A: np.ndarray,
                         epsilon: float) -> InterpolationOperator:
    """ACA, pivot-block check and refined V solve with one tighter ACA retry
    (gca.py:268-282), natively (C ABI gcabem_gca_operator)."""
    A = np.asarray(A)
    is_complex = np.iscomplexobj(A)
    flat = np.ascontiguousarray(A, dtype=np.complex128 if is_complex else np.float64)
    nr, nc = flat.shape
    cap = min(nr, nc)
    rank = np.zeros(1, np.int64)
    rows = np.zeros(cap, np.int64)
    V = np.zeros(nr * cap, np.complex128 if is_complex else np.float64)
    try:
        nat.check(nat.lib().gcabem_gca_operator(int(is_complex), nat.ptr(flat), nr, nc,
                                                float(epsilon), nat.ptr(rank), nat.ptr(rows),
                                                nat.ptr(V)))
    except GcaError as exc:
        raise GcaError(f"cluster {cluster_index}: {exc}") from None
    r = int(rank[0])
    rows = rows[:r].copy()
    return InterpolationOperator(cluster_index, rows, np.asarray(panels)[rows],
                                 V[:nr * r].reshape(nr, r))


def build_interpolation_operator(mesh: SurfaceMesh, cluster_index: int, panels, box_lo, box_hi,
                                 spec: KernelSpec, params: GcaParams,
                                 scene_diameter: float = 0.0) -> InterpolationOperator:
    """One cluster: sources, device Green matrix, host ACA (gca.py:259-282)."""
    panels = np.asarray(panels, dtype=np.int64)
    src = green_sources(box_lo, box_hi, params.delta, params.m, scene_diameter)
    A = build_green_matrix(mesh, panels, src, spec, params.rule_order)
    return _operator_from_green(cluster_index, panels, A, params.epsilon)


last_build_phases: dict = {}


class OperatorMap(MutableMapping):
    """dict[cluster id -> InterpolationOperator] over the flat arrays one GCA
    build returns (sorted ids, ranks, local pivots, V), materialising an
    operator on first access (16k clusters at C3: building them all eagerly
    costs more than packaging needs). pivot_arrays() hands the packaging the
    flat pivot table directly. Assignment and deletion work as on a dict."""

    def __init__(self, ids, starts, sizes, ranks, rows, perm, V):
        self._ids = np.asarray(ids, dtype=np.int64)
        self._starts, self._sizes = np.asarray(starts), np.asarray(sizes)
        self._ranks = np.asarray(ranks, dtype=np.int64)
        self._rows, self._perm, self._V = rows, perm, V
        self._ro = np.concatenate([[0], np.cumsum(self._ranks)])
        self._vo = np.concatenate([[0], np.cumsum(self._sizes * self._ranks)])
        self._made: dict = {}
        self._over: dict = {}
        self._gone: set = set()
        self._pivots = None

    def _pos(self, key) -> int:
        k = int(key)
        i = int(np.searchsorted(self._ids, k))
        return i if i < self._ids.size and self._ids[i] == k else -1

    def __getitem__(self, key):
        k = int(key)
        if k in self._over:
            return self._over[k]
        op = self._made.get(k)
        if op is not None:
            return op
        i = self._pos(k)
        if i < 0 or k in self._gone:
            raise KeyError(key)
        r0, r1 = int(self._ro[i]), int(self._ro[i + 1])
        loc = self._rows[r0:r1]
        n, r = int(self._sizes[i]), r1 - r0
        op = InterpolationOperator(k, loc, self._perm[int(self._starts[i]) + loc],
                                   self._V[int(self._vo[i]):int(self._vo[i + 1])].reshape(n, r))
        self._made[k] = op
        return op

    def __setitem__(self, key, value):
        self._over[int(key)] = value
        self._gone.discard(int(key))
        self._pivots = None

    def __delitem__(self, key):
        k = int(key)
        if k not in self:
            raise KeyError(key)
        self._over.pop(k, None)
        self._gone.add(k)
        self._pivots = None

    def __contains__(self, key):
        try:
            k = int(key)
        except (TypeError, ValueError):
            return False
        return k in self._over or (self._pos(k) >= 0 and k not in self._gone)

    def __iter__(self):
        if not self._over and not self._gone:
            return iter(self._ids.tolist())
        keys = set(self._ids.tolist()) - self._gone | set(self._over)
        return iter(sorted(keys))

    def __len__(self):
        if not self._over and not self._gone:
            return int(self._ids.size)
        return len(set(self._ids.tolist()) - self._gone | set(self._over))

    def pivot_arrays(self, nnodes: int):
        """(at, pivots) as packaging._op_arrays builds them: at[c+1] - at[c]
        = rank of cluster c, pivots_global in cluster-id order; None once the
        map was modified (the generic path then walks the operators)."""
        if self._over or self._gone:
            return None
        if self._pivots is None or self._pivots[0] != nnodes:
            ok = (self._ids >= 0) & (self._ids < nnodes)
            at = np.zeros(nnodes + 1, dtype=np.int64)
            at[self._ids[ok] + 1] = self._ranks[ok]
            np.cumsum(at, out=at)
            glob = self._perm[np.repeat(self._starts, self._ranks) + self._rows[:self._ro[-1]]]
            keep = np.repeat(ok, self._ranks)
            piv = np.ascontiguousarray(glob[keep].astype(np.int64)) if glob.size else \
                np.zeros(1, np.int64)
            self._pivots = (nnodes, (at, piv if piv.size else np.zeros(1, np.int64)))
        return self._pivots[1]


def _host_threads() -> int:
    """Host threads for the ACA pool (packaging.host_threads: this process's
    share of the node's CPU set)."""
    from .packaging import host_threads
    return host_threads()


def _ops_for_tree(mesh, tree: ClusterTree, ids, spec, params, scene, device,
                  batch_bytes: int = 0, threads: int | None = None) -> dict:
    """All clusters in one native pipeline (C ABI gcabem_gca_build): device
    Green matrices per batch (sources generated on the device, bit-identical
    to green_sources), host ACA + pivot check + refined V solve on all cores,
    overlapped with the next batch's kernels and D2H."""
    t0 = time.perf_counter()
    ids = np.array(sorted(ids), dtype=np.int64)
    if ids.size == 0:
        return {}
    dm = device_mesh(mesh, device)
    t_mesh = time.perf_counter() - t0
    starts = np.fromiter((tree.nodes[c].start for c in ids), dtype=np.int64, count=ids.size)
    sizes = np.fromiter((tree.nodes[c].size for c in ids), dtype=np.int64, count=ids.size)
    lo = np.ascontiguousarray([tree.nodes[c].lo for c in ids], dtype=np.float64)
    hi = np.ascontiguousarray([tree.nodes[c].hi for c in ids], dtype=np.float64)
    perm = np.ascontiguousarray(tree.permutation, dtype=np.int64)
    g = gauss_legendre(params.m)
    gp, gw = nat.f64(g.points), nat.f64(g.weights)
    pts, wq = duffy_panel_rule(params.rule_order)
    duffy = np.ascontiguousarray(np.column_stack([pts, wq]))
    eq = 0 if spec.equation == "laplace" else 1
    h = ctypes.c_void_p()
    p = nat.ptr
    t1 = time.perf_counter()
    nat.check(nat.lib().gcabem_gca_build(
        dm.handle, eq, float(spec.kappa), ids.size, p(ids), p(starts), p(sizes), p(lo), p(hi),
        perm.size, p(perm), float(params.delta), int(params.m), p(gp), p(gw), float(scene),
        duffy.shape[0], p(duffy), float(params.epsilon), threads or _host_threads(),
        int(batch_bytes),
        ctypes.byref(h)))
    try:
        ranks = np.empty(ids.size, np.int64)
        phase = np.zeros(6, np.float64)
        nat.check(nat.lib().gcabem_gca_sizes(h, p(ranks), p(phase)))
        rows = np.empty(max(int(ranks.sum()), 1), np.int64)
        width = 2 if spec.is_complex else 1
        vlen = int(np.sum(sizes * ranks)) * width
        V = np.empty(max(vlen, 1), np.float64)
        nat.check(nat.lib().gcabem_gca_fetch(h, p(rows), p(V)))
        amb = np.zeros(ids.size, np.int8)
        nat.check(nat.lib().gcabem_gca_flags(h, p(amb)))
    finally:
        nat.lib().gcabem_gca_free(h)
    t2 = time.perf_counter()
    Vv = V.view(np.complex128) if spec.is_complex else V
    ops = OperatorMap(ids, starts, sizes, ranks, rows, perm, Vv)
    # clusters with an ACA decision inside the tie window (a tie on the
    # device's bits, e.g. from the mesh's symmetry) were redone natively on
    # entries in the reference's own arithmetic (csrc/green_exact.h), so the
    # pivots are the reference's (package assignment bit-exact)
    t3 = time.perf_counter()
    redo = ids[amb != 0]
    last_build_phases.update(device_wait_s=float(phase[0]), pipeline_s=float(phase[1]),
                             native_total_s=float(phase[2]), batches=int(phase[3]),
                             host_thread_s=float(phase[4]), threads=int(phase[5]),
                             clusters=int(ids.size), mesh_s=t_mesh, prep_s=t1 - t0 - t_mesh,
                             call_s=t2 - t1, wrap_s=t3 - t2, ties=int(redo.size),
                             ties_panels=int(sizes[amb != 0].sum()),
                             ties_s=time.perf_counter() - t3)
    return ops


def partition_clusters(tree: ClusterTree, ids, nparts: int) -> list:
    """Sorted cluster ids split into `nparts` contiguous ranges balanced by
    panel count (the Green matrix rows and most of the ACA work scale with
    |t|). Deterministic: every process computes the same parts."""
    ids = np.array(sorted(ids), dtype=np.int64)
    if nparts <= 1:
        return [ids]
    w = np.cumsum([tree.nodes[int(c)].size for c in ids]).astype(np.float64)
    cuts = np.searchsorted(w, w[-1] * np.arange(1, nparts) / nparts) + 1 if ids.size else \
        np.zeros(nparts - 1, np.int64)
    return np.split(ids, np.minimum(cuts, ids.size))


def exchange_pivots(local_ops: dict, is_complex: bool, group=None) -> dict:
    """All-gather of the pivots of each process's clusters (torch.distributed,
    the job's process group: NCCL over NVLink, or gloo): the one exchange
    step of a GCA split over processes, since packaging a leaf window needs
    the pivots (rows/cols) of every cluster its coupling leaves touch. A few
    MB at C3 (sum of ranks x 2 int64). Remote clusters come back as
    InterpolationOperators whose V has zero rows (V stays with the process
    that built it; assembly uses pivots only)."""
    import torch
    import torch.distributed as dist
    cids = sorted(local_ops)
    meta = np.array([[c, local_ops[c].pivots_global.size] for c in cids],
                    dtype=np.int64).reshape(-1, 2)
    flat = np.concatenate([np.array([meta.shape[0]], np.int64), meta.ravel()] +
                          [np.asarray(local_ops[c].pivots_global, np.int64) for c in cids] +
                          [np.asarray(local_ops[c].pivots_local, np.int64) for c in cids])
    world = dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend(group) == "nccl" else torch.device("cpu")
    n = torch.tensor([flat.size], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    nmax = int(max(int(x.item()) for x in sizes))
    buf = torch.zeros(nmax, dtype=torch.int64, device=dev)
    buf[:flat.size] = torch.from_numpy(flat).to(dev)
    got = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(got, buf, group=group)
    vt = np.complex128 if is_complex else np.float64
    ops = {}
    for g, sz in zip(got, sizes):
        a = g[:int(sz.item())].cpu().numpy()
        k = int(a[0])
        m = a[1:1 + 2 * k].reshape(k, 2)
        tot = int(m[:, 1].sum())
        pg = a[1 + 2 * k:1 + 2 * k + tot]
        pl = a[1 + 2 * k + tot:1 + 2 * k + 2 * tot]
        at = 0
        for c, r in m.tolist():
            ops[c] = local_ops[c] if c in local_ops else InterpolationOperator(
                c, pl[at:at + r].copy(), pg[at:at + r].copy(), np.zeros((0, r), vt))
            at += r
    return dict(sorted(ops.items()))


def _ops_multi(mesh, tree, ids, spec, params, scene, devices) -> dict:
    """Clusters split into contiguous id ranges balanced by panel count, one
    native pipeline per device running concurrently (the ctypes call releases
    the GIL; no exchange step: every cluster is independent, gca.py:295-302),
    host threads shared evenly."""
    ids = sorted(ids)
    if len(devices) == 1 or len(ids) < 2 * len(devices):
        return _ops_for_tree(mesh, tree, ids, spec, params, scene, devices[0])
    parts = partition_clusters(tree, ids, len(devices))
    share = max(1, _host_threads() // len(devices))
    out, errs = [None] * len(parts), []

    def run(k):
        try:
            out[k] = _ops_for_tree(mesh, tree, parts[k].tolist(), spec, params, scene,
                                   devices[k], threads=share)
        except BaseException as exc:  # re-raised on the caller's thread
            errs.append(exc)
    import threading
    th = [threading.Thread(target=run, args=(k,)) for k in range(len(parts)) if parts[k].size]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    ops: dict = {}
    for o in out:
        if o:
            ops.update(o)
    return dict(sorted(ops.items()))


def build_interpolation_operators(mesh: SurfaceMesh, block_tree: BlockTree, spec: KernelSpec,
                                  params: GcaParams, device=None, shard=None, group=None):
    """Operators for every cluster in an admissible block (gca.py:285-310);
    (row_ops, col_ops) — the same dict for a shared cluster tree. `device`
    may be a sequence of devices: the clusters are then partitioned across
    them (balanced by panel count) and built concurrently.

    shard = (rank, world): one job split over processes (torch.distributed
    initialised, `group` or the default group): this process builds only its
    part of the clusters (partition_clusters) and exchange_pivots gathers the
    others' pivots, so every process can package any leaf window; V is kept
    only for the own clusters."""
    if shard is not None and int(shard[1]) > 1:
        rank, world = int(shard[0]), int(shard[1])
        if not 0 <= rank < world:
            raise GcaError(f"shard {shard}: need 0 <= rank < world")
        full_r, full_c = _build_ops(mesh, block_tree, spec, params, device, (rank, world))
        t0 = time.perf_counter()
        row = exchange_pivots(full_r, spec.is_complex, group)
        col = row if full_c is full_r else exchange_pivots(full_c, spec.is_complex, group)
        last_build_phases["exchange_s"] = time.perf_counter() - t0
        return row, col
    return _build_ops(mesh, block_tree, spec, params, device, None)


def _build_ops(mesh, block_tree, spec, params, device, part):
    devices = tuple(device) if isinstance(device, (tuple, list)) else \
        (default_device() if device is None else device,)
    t0 = time.perf_counter()
    scene = mesh.diameter()
    native = getattr(block_tree, "_native_leaves", None)
    if native is not None:  # native block tree: leaf arrays, no per-leaf objects
        arr = native[0]
        adm = arr[:, 2] == 0
        row_ids = set(np.unique(arr[adm, 0]).tolist())
        col_ids = set(np.unique(arr[adm, 1]).tolist())
    else:
        row_ids = {b.row for b in block_tree.leaves if b.kind == "admissible"}
        col_ids = {b.col for b in block_tree.leaves if b.kind == "admissible"}
    last_build_phases.clear()
    last_build_phases["ids_s"] = time.perf_counter() - t0

    def mine(tree, ids):   # this process's part of a job split over processes
        if part is None:
            return ids
        return partition_clusters(tree, ids, part[1])[part[0]].tolist()
    if block_tree.row_tree is block_tree.col_tree:
        ops = _ops_multi(mesh, block_tree.row_tree, mine(block_tree.row_tree, row_ids | col_ids),
                         spec, params, scene, devices)
        return ops, ops
    return (_ops_multi(mesh, block_tree.row_tree, mine(block_tree.row_tree, row_ids), spec,
                       params, scene, devices),
            _ops_multi(mesh, block_tree.col_tree, mine(block_tree.col_tree, col_ids), spec,
                       params, scene, devices))

