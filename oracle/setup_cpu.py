"""ORACLE — CPU restatement of the reference's SETUP pipeline (mesh, cluster
and block trees, GCA interpolation operators, work packaging). TEST
INFRASTRUCTURE ONLY, like the rest of oracle/: tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference leg may use it, as the checker
or as the timed CPU baseline. It imports nothing from paper_1510_07244_b200 and
loads no library but oracle/liboracle.so, so the reference arm of the bench
runs without the product (no libgcabem_b200.so, no GPU).

Each function cites the reference code it restates (pkg/src/gcabem/...):

* sphere_mesh           mesh.py:142-189 (+ make_surface_mesh :92-121)
* build_cluster_tree    cluster.py:87-122
* build_block_tree      cluster.py:125-152 (admissible :79-84)
* green_sources         gca.py:83-133
* green_matrix          gca.py:136-179 (oracle.green_matrix, in 256-panel chunks)
* aca                   gca.py:182-245
* interpolation_operator  gca.py:248-282
* build_operators       gca.py:285-310 (clusters spread over worker processes)
* make_packages         scheduler.py:153-232, :334-359, :411-439 (numpy;
                        pinned against the reference's inline list composition
                        and checksums in tests/test_host.py)
"""
from __future__ import annotations

import os
import sys
from dataclasses import dataclass, field

import numpy as np

from . import green_matrix, gauss01

# ---------------------------------------------------------------------------
# mesh


@dataclass(frozen=True)
class Mesh:
    vertices: np.ndarray
    triangles: np.ndarray
    normals: np.ndarray
    gramians: np.ndarray

    @property
    def num_triangles(self) -> int:
        return int(self.triangles.shape[0])

    def diameter(self) -> float:
        """mesh.py:75-78."""
        return float(np.linalg.norm(self.vertices.max(axis=0) - self.vertices.min(axis=0)))


def make_mesh(vertices, triangles) -> Mesh:
    """make_surface_mesh (mesh.py:92-121) without the orientation check:
    gram = |(v1-v0) x (v2-v1)|, normal = cross / gram."""
    V = np.ascontiguousarray(vertices, dtype=np.float64)
    T = np.ascontiguousarray(triangles, dtype=np.int64)
    c = V[T]
    e1 = c[:, 1] - c[:, 0]
    e2 = c[:, 2] - c[:, 1]
    cr = np.cross(e1, e2)
    g = np.linalg.norm(cr, axis=1)
    return Mesh(V, T, cr / g[:, None], g)


def sphere_mesh(level: int) -> Mesh:
    """Octahedron refined `level` times; edge midpoints (keyed by sorted
    index pairs) normalised onto the unit sphere (mesh.py:142-189)."""
    verts = [np.array(v, dtype=np.float64) for v in
             ((1.0, 0.0, 0.0), (-1.0, 0.0, 0.0), (0.0, 1.0, 0.0), (0.0, -1.0, 0.0),
              (0.0, 0.0, 1.0), (0.0, 0.0, -1.0))]
    tris = [(0, 2, 4), (2, 1, 4), (1, 3, 4), (3, 0, 4),
            (2, 0, 5), (1, 2, 5), (3, 1, 5), (0, 3, 5)]
    for _ in range(level):
        mids: dict = {}

        def mid(i, j):
            key = (i, j) if i < j else (j, i)
            k = mids.get(key)
            if k is None:
                v = verts[i] + verts[j]
                v /= np.linalg.norm(v)
                k = len(verts)
                verts.append(v)
                mids[key] = k
            return k
        out = []
        for a, b, c in tris:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            out += [(a, ab, ca), (ab, b, bc), (ca, bc, c), (ab, bc, ca)]
        tris = out
    return make_mesh(np.array(verts), np.array(tris, dtype=np.int64))


# ---------------------------------------------------------------------------
# trees


@dataclass(frozen=True)
class ClusterNode:
    index: int
    start: int
    size: int
    lo: np.ndarray
    hi: np.ndarray
    children: tuple = ()

    @property
    def is_leaf(self) -> bool:
        return not self.children


@dataclass(frozen=True)
class ClusterTree:
    nodes: list
    permutation: np.ndarray
    leaf_size: int

    def panels(self, node: ClusterNode) -> np.ndarray:
        return self.permutation[node.start:node.start + node.size]


@dataclass(frozen=True)
class BlockNode:
    index: int
    row: int
    col: int
    kind: str
    children: tuple = ()


@dataclass(frozen=True)
class BlockTree:
    nodes: list
    row_tree: ClusterTree
    col_tree: ClusterTree
    eta: float
    leaves: list = field(default_factory=list)


def build_cluster_tree(mesh: Mesh, leaf_size: int = 16) -> ClusterTree:
    """Geometric bisection in preorder: split at the median midpoint along
    the box's longest axis, ties to the lower triangle index
    (cluster.py:87-122)."""
    c = mesh.vertices[mesh.triangles]
    tlo, thi = c.min(axis=1), c.max(axis=1)
    mid = (c[:, 0] + c[:, 1] + c[:, 2]) / 3.0
    nt = mesh.num_triangles
    nodes: list = []
    perm = np.empty(nt, dtype=np.int64)
    cursor = [0]

    def build(idx):
        me = len(nodes)
        nodes.append(None)
        lo, hi = tlo[idx].min(axis=0), thi[idx].max(axis=0)
        start = cursor[0]
        if len(idx) <= leaf_size:
            perm[start:start + len(idx)] = idx
            cursor[0] += len(idx)
            nodes[me] = ClusterNode(me, start, len(idx), lo, hi)
            return me
        axis = int(np.argmax(hi - lo))
        order = idx[np.lexsort((idx, mid[idx, axis]))]
        h = len(order) // 2
        kids = (build(order[:h]), build(order[h:]))
        nodes[me] = ClusterNode(me, start, len(idx), lo, hi, kids)
        return me
    old = sys.getrecursionlimit()
    sys.setrecursionlimit(max(old, 10000))
    try:
        build(np.arange(nt, dtype=np.int64))
    finally:
        sys.setrecursionlimit(old)
    return ClusterTree(nodes, perm, leaf_size)


def _admissible(t: ClusterNode, s: ClusterNode, eta: float) -> bool:
    """cluster.py:70-84: max(diam) <= eta * box distance."""
    gap = np.maximum(0.0, np.maximum(t.lo - s.hi, s.lo - t.hi))
    dist = float(np.linalg.norm(gap))
    diam = max(float(np.linalg.norm(t.hi - t.lo)), float(np.linalg.norm(s.hi - s.lo)))
    return diam <= eta * dist


def build_block_tree(row_tree: ClusterTree, col_tree: ClusterTree,
                     eta: float = 2.0) -> BlockTree:
    """Recursive descent (cluster.py:125-152)."""
    nodes: list = []
    leaves: list = []

    def build(ti, si):
        me = len(nodes)
        nodes.append(None)
        t, s = row_tree.nodes[ti], col_tree.nodes[si]
        if _admissible(t, s, eta):
            node = BlockNode(me, ti, si, "admissible")
            leaves.append(node)
        elif t.is_leaf and s.is_leaf:
            node = BlockNode(me, ti, si, "dense")
            leaves.append(node)
        else:
            tk = t.children or (ti,)
            sk = s.children or (si,)
            node = BlockNode(me, ti, si, "split", tuple(build(a, b) for a in tk for b in sk))
        nodes[me] = node
        return me
    old = sys.getrecursionlimit()
    sys.setrecursionlimit(max(old, 10000))
    try:
        build(0, 0)
    finally:
        sys.setrecursionlimit(old)
    return BlockTree(nodes, row_tree, col_tree, eta, leaves)


# ---------------------------------------------------------------------------
# GCA


def green_sources(box_lo, box_hi, delta: float, m: int, scene_diameter: float = 0.0):
    """gca.py:83-133: (points (12m^2,3), weights, normals, roles 0/1)."""
    lo = np.asarray(box_lo, dtype=np.float64)
    hi = np.asarray(box_hi, dtype=np.float64)
    center = 0.5 * (lo + hi)
    hmax = 0.5 * max(float(np.max(hi - lo)), 1e-8 * scene_diameter)
    half = 0.5 * (hi - lo) + delta * hmax
    x, w = np.polynomial.legendre.leggauss(m)
    gp, gw = (x + 1.0) / 2.0, w / 2.0
    gu, gv = np.meshgrid(gw, gw, indexing="ij")
    guv = (gu * gv).ravel()
    pts, wts, nrm, roles = [], [], [], []
    for axis in range(3):
        a1, a2 = (axis + 1) % 3, (axis + 2) % 3
        u = -half[a1] + 2.0 * half[a1] * gp
        v = -half[a2] + 2.0 * half[a2] * gp
        ua, va = np.meshgrid(u, v, indexing="ij")
        face_w = guv * (4.0 * half[a1] * half[a2])
        for sign in (-1.0, 1.0):
            face = np.empty((m * m, 3))
            face[:, axis] = center[axis] + sign * half[axis]
            face[:, a1] = center[a1] + ua.ravel()
            face[:, a2] = center[a2] + va.ravel()
            normal = np.zeros(3)
            normal[axis] = sign
            pts.append(np.repeat(face, 2, axis=0))
            wts.append(np.repeat(face_w, 2))
            nrm.append(np.tile(normal, (2 * m * m, 1)))
            roles.append(np.tile([0, 1], m * m))
    return (np.concatenate(pts), np.concatenate(wts), np.concatenate(nrm),
            np.concatenate(roles).astype(np.uint8))


def green_matrix_chunked(mesh: Mesh, panels, sources, equation, kappa, order, chunk=256):
    """build_green_matrix (gca.py:136-179): 256-panel chunks, each by the
    numpy restatement oracle.green_matrix."""
    panels = np.asarray(panels, dtype=np.int64)
    pts, wts, nrm, roles = sources
    parts = [green_matrix(mesh.vertices, mesh.triangles, mesh.gramians, panels[b:b + chunk],
                          pts, wts, nrm, roles, equation, kappa, order)
             for b in range(0, panels.size, chunk)]
    return parts[0] if len(parts) == 1 else np.concatenate(parts)


def aca(A, epsilon, max_rank=None):
    """Partially pivoted ACA (gca.py:182-245): (row pivots, col pivots)."""
    A = np.asarray(A)
    nr, nc = A.shape
    cap = min(nr, nc) if max_rank is None else min(max_rank, nr, nc)
    dtype = np.result_type(A.dtype, np.float64)
    U, W, rows, cols = [], [], [], []
    taken = np.zeros(nr, dtype=bool)
    est2 = 0.0
    cand = 0
    while len(rows) < cap:
        if cand >= nr or taken[cand]:
            free = np.flatnonzero(~taken)
            if free.size == 0:
                break
            cand = int(free[0])
        i = cand
        r = A[i, :].astype(dtype, copy=True)
        for u, w in zip(U, W):
            r -= u[i] * w
        j = int(np.argmax(np.abs(r)))
        taken[i] = True
        if r[j] == 0.0:
            cand = nr
            continue
        w = r / r[j]
        c = A[:, j].astype(dtype, copy=True)
        for u, ww in zip(U, W):
            c -= ww[j] * u
        U.append(c)
        W.append(w)
        rows.append(i)
        cols.append(j)
        nu, nw = float(np.linalg.norm(c)), float(np.linalg.norm(w))
        mix = 0.0
        for u, ww in zip(U[:-1], W[:-1]):
            mix += (np.vdot(u, c) * np.vdot(ww, w)).real
        est2 = max(est2 + nu * nu * nw * nw + 2.0 * mix, 0.0)
        if nu * nw <= epsilon * np.sqrt(est2):
            break
        mag = np.abs(c)
        mag[taken] = 0.0
        cand = int(np.argmax(mag))
        if mag[cand] == 0.0:
            cand = nr
    return np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64)


def solve_operator(A, epsilon):
    """gca.py:248-282 after the Green matrix: ACA, cond check (retry once at
    epsilon/10), V = A[:, c] A[r, c]^-1 with two refinement sweeps.
    Returns (row pivots (local), V)."""
    eps = epsilon
    for _ in range(2):
        rows, cols = aca(A, eps)
        if rows.size == 0:
            raise ValueError("zero Green matrix")
        block = A[np.ix_(rows, cols)]
        if np.linalg.cond(block) <= 1e14:
            A_cols = A[:, cols]
            V = np.linalg.solve(block.T, A_cols.T).T
            for _ in range(2):
                R = A_cols - V @ block
                if np.max(np.abs(R)) <= 1e-15 * max(np.max(np.abs(A_cols)), 1.0):
                    break
                V = V + np.linalg.solve(block.T, R.T).T
            return rows, V
        eps *= 0.1
    raise ValueError("singular ACA pivot block")


@dataclass(frozen=True)
class Operator:
    cluster: int
    pivots_local: np.ndarray
    pivots_global: np.ndarray
    V: np.ndarray


def interpolation_operator(mesh: Mesh, tree: ClusterTree, cid: int, equation: str,
                           kappa: float, delta=1.0, m=6, epsilon=1e-4, rule_order=3,
                           scene=None) -> Operator:
    """build_interpolation_operator (gca.py:248-282) of cluster `cid`."""
    node = tree.nodes[cid]
    panels = tree.panels(node)
    src = green_sources(node.lo, node.hi, delta, m,
                        mesh.diameter() if scene is None else scene)
    A = green_matrix_chunked(mesh, panels, src, equation, kappa, rule_order)
    rows, V = solve_operator(A, epsilon)
    return Operator(cid, rows, panels[rows], V)


def admissible_clusters(bt: BlockTree):
    """gca.py:303-306 (shared tree): clusters of the admissible leaves."""
    return sorted({l.row for l in bt.leaves if l.kind == "admissible"} |
                  {l.col for l in bt.leaves if l.kind == "admissible"})


_POOL_STATE: dict = {}


def _pool_job(cids):
    st = _POOL_STATE
    return [interpolation_operator(st["mesh"], st["tree"], c, st["eq"], st["kappa"],
                                   scene=st["scene"]) for c in cids]


def build_operators(mesh: Mesh, tree: ClusterTree, cids, equation: str, kappa: float,
                    workers: int = 1, timeout: float = 3600.0) -> dict:
    """Operators of `cids` (gca.py:285-310; the reference loops serially),
    spread over `workers` forked processes (one BLAS thread each)."""
    cids = [int(c) for c in cids]
    scene = mesh.diameter()
    if workers <= 1 or len(cids) < 2 * workers:
        return {c: interpolation_operator(mesh, tree, c, equation, kappa, scene=scene)
                for c in cids}
    import multiprocessing as mp
    _POOL_STATE.update(mesh=mesh, tree=tree, eq=equation, kappa=kappa, scene=scene)
    # interleaved chunks: cluster sizes vary along the id order
    nchunks = workers * 8
    chunks = [cids[k::nchunks] for k in range(nchunks)]
    ctx = mp.get_context("fork")
    from threadpoolctl import threadpool_limits
    # one BLAS thread in the parent across the fork: a forked child must not
    # inherit a multi-threaded BLAS pool (it deadlocks in its first solve)
    try:
        with threadpool_limits(limits=1):
            pool = ctx.Pool(workers)
            try:
                res = pool.map_async(_pool_job, chunks).get(timeout)
            finally:
                pool.terminate()
                pool.join()
    finally:
        _POOL_STATE.clear()
    return dict(sorted((op.cluster, op) for part in res for op in part))


# ---------------------------------------------------------------------------
# packaging (scheduler.py:153-232, 334-359, 411-439)

PAIR_RECORD_BYTES = 24
VALUE_BYTES = 8
BYTES_PER_PAIR = PAIR_RECORD_BYTES + VALUE_BYTES
SINGULAR_CASES = ("vertex", "edge", "identical")
_SCAN_CHUNK = 1 << 21   # flagged pairs scanned per vectorised step


class SchedulerConfigError(ValueError):
    pass


def classify_pairs(triangles, tri_a, tri_b):
    """quadrature.py:197-220 over index arrays: (case int8: 0 disjoint,
    1 vertex, 2 edge, 3 identical; perm_x, perm_y uint8 (n,3)). Shared
    vertices first in global-index order, the others in stored order."""
    tri_a = np.asarray(tri_a, dtype=np.int64)
    tri_b = np.asarray(tri_b, dtype=np.int64)
    va, vb = triangles[tri_a], triangles[tri_b]
    eq = va[:, :, None] == vb[:, None, :]
    a_sh, b_sh = eq.any(axis=2), eq.any(axis=1)
    nsh = a_sh.sum(axis=1)
    same = tri_a == tri_b
    if np.any((nsh == 3) & ~same):
        raise ValueError("distinct triangles share 3 vertices")
    slot = np.arange(3, dtype=np.int64)
    big = np.int64(1) << 62
    px = np.argsort(np.where(a_sh & ~same[:, None], va, big + slot), axis=1,
                    kind="stable").astype(np.uint8)
    py = np.argsort(np.where(b_sh & ~same[:, None], vb, big + slot), axis=1,
                    kind="stable").astype(np.uint8)
    return np.where(same, 3, nsh).astype(np.int8), px, py


@dataclass
class AssemblyPackages:
    """Flat package description of one assembly."""
    maxsize: int
    leaf_ids: np.ndarray        # (L,) BlockNode.index, preorder
    leaf_kind: np.ndarray       # (L,) 1 dense, 0 admissible
    leaf_shape: np.ndarray      # (L, 2)
    leaf_base: np.ndarray       # (L+1,) payload offsets (entries)
    panels: np.ndarray          # concatenated leaf rows then cols
    leaf_rows_at: np.ndarray    # (L,)
    leaf_cols_at: np.ndarray    # (L,)
    leaf_flagged: np.ndarray    # (L,) bool
    blk_leaf: np.ndarray        # (B,) disjoint WorkBlocks after splitting, list order
    blk_r0: np.ndarray
    blk_c0: np.ndarray
    blk_nr: np.ndarray
    blk_nc: np.ndarray
    blk_list: np.ndarray        # (B,) disjoint list number
    n_disjoint_lists: int
    item_case: np.ndarray       # (S,) 1 vertex, 2 edge, 3 identical (generation order)
    item_tri_x: np.ndarray
    item_tri_y: np.ndarray
    item_leaf: np.ndarray       # (S,) leaf position
    item_offset: np.ndarray     # (S,) flat offset inside the leaf payload
    item_src_block: np.ndarray  # (S,) disjoint block that generated the item
    perms: np.ndarray           # (S, 6) uint8 perm_x, perm_y
    extra: dict = field(default_factory=dict)

    @property
    def payload_len(self) -> int:
        return int(self.leaf_base[-1])

    @property
    def num_blocks(self) -> int:
        return int(self.blk_leaf.size)

    @property
    def num_items(self) -> int:
        return int(self.item_case.size)

    def block_pairs(self) -> int:
        return int(np.sum(self.leaf_shape[:, 0] * self.leaf_shape[:, 1]))

    def device_blocks(self, leaf_lo: int = 0, leaf_hi: int | None = None) -> np.ndarray:
        """(B', 7) int64 {payload_base, ld, nr, nc, rows_at, cols_at, leaf}."""
        leaf_hi = self.leaf_ids.size if leaf_hi is None else leaf_hi
        sel = (self.blk_leaf >= leaf_lo) & (self.blk_leaf < leaf_hi)
        lf = self.blk_leaf[sel]
        ld = self.leaf_shape[lf, 1]
        base = self.leaf_base[lf] - self.leaf_base[leaf_lo] + self.blk_r0[sel] * ld + \
            self.blk_c0[sel]
        return np.ascontiguousarray(np.stack(
            [base, ld, self.blk_nr[sel], self.blk_nc[sel],
             self.leaf_rows_at[lf] + self.blk_r0[sel], self.leaf_cols_at[lf] + self.blk_c0[sel],
             lf], axis=1).astype(np.int64))

    def device_items(self, leaf_lo: int = 0, leaf_hi: int | None = None):
        """((S', 4) int64 {case, tri_x, tri_y, payload_index}, (S', 6) uint8),
        grouped by case."""
        leaf_hi = self.leaf_ids.size if leaf_hi is None else leaf_hi
        sel = np.flatnonzero((self.item_leaf >= leaf_lo) & (self.item_leaf < leaf_hi))
        sel = sel[np.argsort(self.item_case[sel], kind="stable")]
        idx = self.leaf_base[self.item_leaf[sel]] - self.leaf_base[leaf_lo] + \
            self.item_offset[sel]
        items = np.stack([self.item_case[sel].astype(np.int64), self.item_tri_x[sel],
                          self.item_tri_y[sel], idx], axis=1).astype(np.int64)
        return np.ascontiguousarray(items), np.ascontiguousarray(self.perms[sel])

    def singular_lists(self):
        cap = max(self.maxsize // BYTES_PER_PAIR, 1)
        out = {}
        for code, name in enumerate(SINGULAR_CASES, start=1):
            n = int(np.count_nonzero(self.item_case == code))
            out[name] = [(a, min(a + cap, n)) for a in range(0, n, cap)]
        return out


def _split(nr: int, nc: int, maxsize: int, r0=0, c0=0, out=None):
    """split_block (scheduler.py:153-175) on index ranges, depth-first."""
    if out is None:
        out = []
    if nr * nc * BYTES_PER_PAIR <= maxsize:
        out.append((r0, nr, c0, nc))
        return out
    if nr * nc <= 1:
        raise SchedulerConfigError(
            f"maxsize {maxsize} smaller than one pair record ({BYTES_PER_PAIR} B)")
    if nr >= nc:
        h = nr // 2
        _split(h, nc, maxsize, r0, c0, out)
        _split(nr - h, nc, maxsize, r0 + h, c0, out)
    else:
        h = nc // 2
        _split(nr, h, maxsize, r0, c0, out)
        _split(nr, nc - h, maxsize, r0, c0 + h, out)
    return out


def _greedy_lists(nbytes: np.ndarray, maxsize: int):
    """ListBuilder._add (scheduler.py:197-201): flush when the next item would
    overflow a non-empty list."""
    lid = np.empty(nbytes.size, dtype=np.int64)
    cur, cnt, k = 0, 0, 0
    for b, nb in enumerate(nbytes.tolist()):
        if cur + nb > maxsize and cnt:
            k += 1
            cur, cnt = 0, 0
        lid[b] = k
        cur += nb
        cnt += 1
    return lid, (k + 1 if nbytes.size else 0)


def make_packages(triangles: np.ndarray, block_tree, row_ops, col_ops,
                  maxsize: int) -> AssemblyPackages:
    """Leaves in preorder (rows/cols = cluster panels or ACA pivots), the
    flagged touch test, split_block + greedy disjoint lists, the corrective
    scan of flagged blocks (row-major), classification permutations.
    `block_tree`: anything with .leaves (index,row,col,kind), .row_tree /
    .col_tree (.nodes[lo,hi], .panels(node)); ops: cid -> .pivots_global."""
    if maxsize < BYTES_PER_PAIR:
        raise SchedulerConfigError(
            f"maxsize {maxsize} smaller than one pair record ({BYTES_PER_PAIR} B)")
    rt, ct = block_tree.row_tree, block_tree.col_tree
    leaves = block_tree.leaves
    L = len(leaves)
    leaf_ids = np.fromiter((l.index for l in leaves), dtype=np.int64, count=L)
    kind = np.fromiter((l.kind == "dense" for l in leaves), dtype=bool, count=L)
    rows_list, cols_list = [], []
    shape = np.empty((L, 2), dtype=np.int64)
    for k, leaf in enumerate(leaves):
        if kind[k]:
            r = rt.panels(rt.nodes[leaf.row])
            c = ct.panels(ct.nodes[leaf.col])
        else:
            r = np.asarray(row_ops[leaf.row].pivots_global, dtype=np.int64)
            c = np.asarray(col_ops[leaf.col].pivots_global, dtype=np.int64)
        rows_list.append(r)
        cols_list.append(c)
        shape[k] = (r.size, c.size)
    seg = np.empty(2 * L, dtype=np.int64)
    seg[0::2], seg[1::2] = shape[:, 0], shape[:, 1]
    starts = np.concatenate([[0], np.cumsum(seg)])
    inter = [None] * (2 * L)
    inter[0::2], inter[1::2] = rows_list, cols_list
    panels = np.concatenate(inter).astype(np.int64) if L else np.empty(0, np.int64)
    rows_at, cols_at = starts[0:-1:2], starts[1::2]
    base = np.concatenate([[0], np.cumsum(shape[:, 0] * shape[:, 1])]).astype(np.int64)

    # touch test per leaf (box_distance == 0.0), exact without the norm
    rlo = np.array([n.lo for n in rt.nodes])
    rhi = np.array([n.hi for n in rt.nodes])
    clo = np.array([n.lo for n in ct.nodes])
    chi = np.array([n.hi for n in ct.nodes])
    lr = np.fromiter((l.row for l in leaves), dtype=np.int64, count=L)
    lc = np.fromiter((l.col for l in leaves), dtype=np.int64, count=L)
    flagged = np.all((rlo[lr] <= chi[lc]) & (clo[lc] <= rhi[lr]), axis=1) if L else \
        np.zeros(0, bool)

    npairs = shape[:, 0] * shape[:, 1]
    big = np.flatnonzero(npairs * BYTES_PER_PAIR > maxsize)
    if big.size == 0:
        b_leaf = np.arange(L, dtype=np.int64)
        b_r0, b_c0 = np.zeros(L, np.int64), np.zeros(L, np.int64)
        b_nr, b_nc = shape[:, 0].copy(), shape[:, 1].copy()
    else:
        parts = {int(k): _split(int(shape[k, 0]), int(shape[k, 1]), maxsize) for k in big}
        recs = []
        for k in range(L):
            if k in parts:
                recs += [(k,) + p for p in parts[k]]
            else:
                recs.append((k, 0, int(shape[k, 0]), 0, int(shape[k, 1])))
        arr = np.array(recs, dtype=np.int64).reshape(-1, 5)
        b_leaf, b_r0, b_nr, b_c0, b_nc = (arr[:, i].copy() for i in range(5))
    blk_list, n_lists = _greedy_lists(b_nr * b_nc * BYTES_PER_PAIR, maxsize)

    T = np.asarray(triangles, dtype=np.int64)
    fb = np.flatnonzero(flagged[b_leaf])
    it_case, it_tx, it_ty, it_leaf, it_off, it_blk = [], [], [], [], [], []
    sizes = b_nr[fb] * b_nc[fb]
    cut = 0
    while cut < fb.size:
        acc, stop = 0, cut
        while stop < fb.size and (acc == 0 or acc + sizes[stop] <= _SCAN_CHUNK):
            acc += int(sizes[stop])
            stop += 1
        blk = fb[cut:stop]
        cnt = b_nr[blk] * b_nc[blk]
        owner = np.repeat(blk, cnt)
        k = np.arange(owner.size, dtype=np.int64) - np.repeat(np.cumsum(cnt) - cnt, cnt)
        ncol = b_nc[owner]
        i, j = k // ncol, k % ncol
        lf = b_leaf[owner]
        tx = panels[rows_at[lf] + b_r0[owner] + i]
        ty = panels[cols_at[lf] + b_c0[owner] + j]
        ta, tb = T[tx], T[ty]
        shared = np.zeros(owner.size, dtype=np.int8)
        for a in range(3):
            for b in range(3):
                shared += (ta[:, a] == tb[:, b])
        hit = np.flatnonzero(shared > 0)
        it_case.append(np.minimum(shared[hit], 3).astype(np.int8))
        it_tx.append(tx[hit])
        it_ty.append(ty[hit])
        it_leaf.append(lf[hit])
        it_off.append((b_r0[owner[hit]] + i[hit]) * shape[lf[hit], 1] + b_c0[owner[hit]]
                      + j[hit])
        it_blk.append(owner[hit])
        cut = stop

    def cat(xs, dt):
        return np.concatenate(xs).astype(dt) if xs else np.empty(0, dt)
    item_case = cat(it_case, np.int8)
    item_tx, item_ty = cat(it_tx, np.int64), cat(it_ty, np.int64)
    case_chk, px, py = classify_pairs(T, item_tx, item_ty)
    if item_case.size and not np.array_equal(case_chk, item_case):
        raise AssertionError("shared-vertex count and classification disagree")
    perms = np.concatenate([px, py], axis=1).astype(np.uint8) if item_case.size else \
        np.empty((0, 6), np.uint8)
    return AssemblyPackages(
        maxsize=maxsize, leaf_ids=leaf_ids, leaf_kind=kind.astype(np.int8), leaf_shape=shape,
        leaf_base=base, panels=panels, leaf_rows_at=rows_at, leaf_cols_at=cols_at,
        leaf_flagged=flagged, blk_leaf=b_leaf, blk_r0=b_r0, blk_c0=b_c0, blk_nr=b_nr,
        blk_nc=b_nc, blk_list=blk_list, n_disjoint_lists=n_lists, item_case=item_case,
        item_tri_x=item_tx, item_tri_y=item_ty, item_leaf=cat(it_leaf, np.int64),
        item_offset=cat(it_off, np.int64), item_src_block=cat(it_blk, np.int64), perms=perms)


def shard_leaves(pk: AssemblyPackages, nshards: int, disjoint_q: int, singular_q=None):
    """Contiguous leaf ranges balanced by quadrature points."""
    L = pk.leaf_ids.size
    if nshards <= 1 or L == 0:
        return [(0, L)]
    w = (pk.leaf_shape[:, 0] * pk.leaf_shape[:, 1]).astype(np.float64) * disjoint_q
    if singular_q is not None and pk.num_items:
        q = np.asarray([0] + list(singular_q), dtype=np.float64)
        np.add.at(w, pk.item_leaf, q[pk.item_case])
    cum = np.cumsum(w)
    cuts = np.searchsorted(cum, cum[-1] * np.arange(1, nshards) / nshards, side="left") + 1
    edges = np.maximum.accumulate(np.concatenate([[0], np.minimum(cuts, L), [L]]))
    return [(int(edges[k]), int(edges[k + 1])) for k in range(nshards)]


def inline_lists(pk: AssemblyPackages) -> list:
    """Lists in the order the reference executes them inline
    (workers_per_backend=0, scheduler.py:474-497): each disjoint list, then
    any singular list its corrective items filled up, then the partial
    singular lists in SINGULAR_CASES order. Entries: ("disjoint", block
    indices) or (case, item indices into the generation order)."""
    cap = max(pk.maxsize // BYTES_PER_PAIR, 1)
    by_list = [[] for _ in range(pk.n_disjoint_lists)]
    for b, lid in enumerate(pk.blk_list.tolist()):
        by_list[lid].append(b)
    triggered = {k: [] for k in range(pk.n_disjoint_lists)}
    tail = []
    for code, name in enumerate(SINGULAR_CASES, start=1):
        idx = np.flatnonzero(pk.item_case == code)
        for a in range(0, idx.size, cap):
            members = idx[a:a + cap]
            if a + cap < idx.size:
                trig = int(idx[a + cap])
                lid = int(pk.blk_list[pk.item_src_block[trig]])
                triggered[lid].append((trig, name, members))
            else:
                tail.append((name, members))
    out = []
    for lid in range(pk.n_disjoint_lists):
        out.append(("disjoint", np.array(by_list[lid], dtype=np.int64)))
        for _, name, members in sorted(triggered[lid], key=lambda t: t[0]):
            out.append((name, members))
    return out + tail


def pivot_operators(cids, ranks, pivots) -> dict:
    """Operators carrying given pivots (e.g. the reference's own, from
    tests/golden/gca_levels.npz); V is not needed to package."""
    at = np.concatenate([[0], np.cumsum(ranks)])
    return {int(c): Operator(int(c), np.empty(0, np.int64),
                             np.asarray(pivots[at[k]:at[k + 1]], dtype=np.int64),
                             np.zeros((0, int(ranks[k]))))
            for k, c in enumerate(cids)}
