"""Work packages: the CPU half of scheduler.run_assembly.

The host builds exactly the reference scheduler's packages
(pkg/src/gcabem/scheduler.py): leaves in block-tree preorder with the
``flagged`` touch test (_leaf_blocks :425-439), the payload layout
(make_payloads :411-422), split WorkBlocks and greedy byte-budgeted
disjoint lists (split_block :153-175, ListBuilder :178-208), the corrective
shared-vertex scan of flagged blocks in argwhere order (distribute_disjoint
:334-359) and the classify_pair permutations of every singular item
(quadrature.py:197-220). The work is done natively
(csrc/packaging.cpp, C ABI gcabem_packages_*, threaded corrective scan);
this module marshals trees/operators in and the flat arrays out.

Panel indices are not copied per leaf: ``panels`` is the concatenation
[row permutation | row pivots (| col permutation | col pivots)] and each
leaf points into it (rows_at / cols_at), so the device upload is O(nt).
"""
from __future__ import annotations

import ctypes
import os
import sys
import threading
import time
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .cluster import BlockTree, ClusterTree

PAIR_RECORD_BYTES = 24
VALUE_BYTES = 8
BYTES_PER_PAIR = PAIR_RECORD_BYTES + VALUE_BYTES
SINGULAR_CASES = ("vertex", "edge", "identical")


class SchedulerConfigError(ValueError):
    pass


@dataclass
class AssemblyPackages:
    """Flat package description of one assembly."""
    maxsize: int
    leaf_ids: np.ndarray        # (L,) BlockNode.index, preorder
    leaf_shape: np.ndarray      # (L, 2)
    leaf_base: np.ndarray       # (L+1,) payload offsets (entries)
    panels: np.ndarray          # panel base array (see module docstring)
    leaf_rows_at: np.ndarray    # (L,)
    leaf_cols_at: np.ndarray    # (L,)
    leaf_flagged: np.ndarray    # (L,) bool
    blk_leaf: np.ndarray        # (B,) WorkBlocks after splitting, in list order
    blk_r0: np.ndarray
    blk_nr: np.ndarray
    blk_c0: np.ndarray
    blk_nc: np.ndarray
    blk_list: np.ndarray        # (B,) disjoint list number
    n_disjoint_lists: int
    item_case: np.ndarray       # (S,) 1 vertex, 2 edge, 3 identical — generation order
    item_tri_x: np.ndarray
    item_tri_y: np.ndarray
    item_leaf: np.ndarray       # (S,) leaf position
    item_offset: np.ndarray     # (S,) flat offset inside the leaf payload
    item_src_block: np.ndarray  # (S,) block whose scan generated the item
    perms: np.ndarray           # (S, 6) uint8 perm_x, perm_y
    extra: dict = field(default_factory=dict)
    # (L,) position of the leaf of the transposed cluster pair in these
    # packages, -1 if none (or outside a leaf range); None when the two sides
    # differ (different trees or operators): see leaf_mirrors()
    leaf_mirror: np.ndarray | None = None

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
        """(B', 7) int64 {payload_base, ld, nr, nc, rows_at, cols_at, leaf} for
        the blocks of leaves [leaf_lo, leaf_hi), bases relative to leaf_lo."""
        leaf_hi = self.leaf_ids.size if leaf_hi is None else leaf_hi
        if leaf_lo == 0 and leaf_hi == self.leaf_ids.size:
            sel = slice(None)
        else:
            sel = (self.blk_leaf >= leaf_lo) & (self.blk_leaf < leaf_hi)
        lf = self.blk_leaf[sel]
        ld = self.leaf_shape[lf, 1]
        r0, c0 = self.blk_r0[sel], self.blk_c0[sel]
        out = np.empty((lf.size, 7), dtype=np.int64)
        out[:, 0] = self.leaf_base[lf] - self.leaf_base[leaf_lo] + r0 * ld + c0
        out[:, 1] = ld
        out[:, 2] = self.blk_nr[sel]
        out[:, 3] = self.blk_nc[sel]
        out[:, 4] = self.leaf_rows_at[lf] + r0
        out[:, 5] = self.leaf_cols_at[lf] + c0
        out[:, 6] = lf
        return out

    def device_items(self, leaf_lo: int = 0, leaf_hi: int | None = None):
        """Singular items of leaves [leaf_lo, leaf_hi), grouped by case:
        ((S', 4) int64 {case, tri_x, tri_y, payload_index}, (S', 6) uint8)."""
        leaf_hi = self.leaf_ids.size if leaf_hi is None else leaf_hi
        sel = np.flatnonzero((self.item_leaf >= leaf_lo) & (self.item_leaf < leaf_hi))
        sel = sel[np.argsort(self.item_case[sel], kind="stable")]
        items = np.empty((sel.size, 4), dtype=np.int64)
        items[:, 0] = self.item_case[sel]
        items[:, 1] = self.item_tri_x[sel]
        items[:, 2] = self.item_tri_y[sel]
        items[:, 3] = (self.leaf_base[self.item_leaf[sel]] - self.leaf_base[leaf_lo]
                       + self.item_offset[sel])
        return items, np.ascontiguousarray(self.perms[sel])

    def singular_lists(self):
        """Per case: (start, stop) ranges into that case's items in generation
        order, as ListBuilder cuts them."""
        cap = max(self.maxsize // BYTES_PER_PAIR, 1)
        out = {}
        for code, name in enumerate(SINGULAR_CASES, start=1):
            n = int(np.count_nonzero(self.item_case == code))
            out[name] = [(a, min(a + cap, n)) for a in range(0, n, cap)]
        return out


# ---------------------------------------------------------------------------
# marshalling caches (trees are immutable; keyed on the live objects)

_tree_cache: dict = {}
_leaf_cache: dict = {}
_mirror_cache: dict = {}
_cache_lock = threading.Lock()


def _cached(cache, obj, build):
    key = id(obj)
    with _cache_lock:
        hit = cache.get(key)
    if hit is not None and hit[0]() is obj:
        return hit[1]
    val = build(obj)
    with _cache_lock:
        cache[key] = (weakref.ref(obj), val)
    weakref.finalize(obj, lambda k=key: cache.pop(k, None))
    return val


def _tree_arrays(tree: ClusterTree):
    def build(t):
        n = len(t.nodes)
        start = np.fromiter((x.start for x in t.nodes), dtype=np.int64, count=n)
        size = np.fromiter((x.size for x in t.nodes), dtype=np.int64, count=n)
        lo = np.ascontiguousarray(np.array([x.lo for x in t.nodes], dtype=np.float64))
        hi = np.ascontiguousarray(np.array([x.hi for x in t.nodes], dtype=np.float64))
        return start, size, lo, hi, np.ascontiguousarray(t.permutation, dtype=np.int64)
    return _cached(_tree_cache, tree, build)


def _leaf_arrays(bt: BlockTree):
    native = getattr(bt, "_native_leaves", None)
    if native is not None:
        return native

    def build(b):
        L = len(b.leaves)
        arr = np.empty((L, 3), dtype=np.int64)
        arr[:, 0] = np.fromiter((l.row for l in b.leaves), dtype=np.int64, count=L)
        arr[:, 1] = np.fromiter((l.col for l in b.leaves), dtype=np.int64, count=L)
        arr[:, 2] = np.fromiter((l.kind == "dense" for l in b.leaves), dtype=np.int64, count=L)
        ids = np.fromiter((l.index for l in b.leaves), dtype=np.int64, count=L)
        return arr, ids
    return _cached(_leaf_cache, bt, build)


_op_cache: dict = {}


def _op_arrays(ops: dict, nnodes: int):
    """Pivot arrays of an operator dict, cached while the dict holds the same
    operator objects (ops dicts cannot be weak-referenced: the entry keeps a
    fingerprint of (cluster, operator identity) pairs and is replaced when it
    no longer matches)."""
    fast = getattr(ops, "pivot_arrays", None)
    if fast is not None:   # gca.OperatorMap: the flat table, no per-operator walk
        arrs = fast(nnodes)
        if arrs is not None:
            return arrs
    fp = (nnodes, tuple(ops.keys()), tuple(map(id, ops.values())))
    with _cache_lock:
        hit = _op_cache.get(id(ops))
    if hit is not None and hit[0] == fp:
        return hit[2]
    val = _op_arrays_build(ops, nnodes)
    with _cache_lock:
        if len(_op_cache) > 16:
            _op_cache.clear()
        _op_cache[id(ops)] = (fp, ops, val)
    return val


def _op_arrays_build(ops: dict, nnodes: int):
    at = np.zeros(nnodes + 1, dtype=np.int64)
    pivs = []
    for cid in sorted(ops):
        if not 0 <= cid < nnodes:   # not a node of this tree: no leaf can use it
            continue
        p = np.asarray(ops[cid].pivots_global, dtype=np.int64)
        at[cid + 1] = p.size
        pivs.append(p)
    np.cumsum(at, out=at)
    # pivots must sit in cluster-id order to match `at`
    piv = np.concatenate(pivs) if pivs else np.zeros(1, np.int64)
    return at, np.ascontiguousarray(piv)


def host_threads() -> int:
    """Host threads for the native host work of this process: its CPU set,
    shared evenly by the processes of one node (torchrun LOCAL_WORLD_SIZE)."""
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count() or 1
    return max(1, min(32, n // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))))


@dataclass
class PackageInputs:
    """The flat arrays make_packages hands to the native builder (triangles,
    leaves, both trees, both operators' pivots), gathered once so that
    several leaf ranges can be packaged without re-deriving them."""
    T: np.ndarray
    leaves: np.ndarray
    leaf_ids: np.ndarray
    row: tuple      # start, size, lo, hi, perm
    col: tuple
    row_ops: tuple  # at, pivots
    col_ops: tuple
    _panel_base: np.ndarray | None = None

    @property
    def panel_base(self) -> np.ndarray:
        """[row perm | row pivots (| col perm | col pivots)]: the panel base
        array every leaf range's packages index (the col part only when the
        trees or the operators differ, as gcabem_packages_build lays it out);
        built once, shared by the ranges (gcabem_packages_build_on)."""
        if self._panel_base is None:
            # (an operator table without pivots holds one placeholder entry)
            parts = [self.row[4], self.row_ops[1][:int(self.row_ops[0][-1])]]
            shared = self.col[0] is self.row[0] and self.col[4] is self.row[4]
            if not shared or self.col_ops[1] is not self.row_ops[1]:
                parts += [self.col[4], self.col_ops[1][:int(self.col_ops[0][-1])]]
            self._panel_base = np.ascontiguousarray(np.concatenate(parts), dtype=np.int64)
        return self._panel_base


def package_inputs(triangles: np.ndarray, block_tree: BlockTree, row_ops, col_ops):
    leaves, leaf_ids = _leaf_arrays(block_tree)
    row = _tree_arrays(block_tree.row_tree)
    col = row if block_tree.col_tree is block_tree.row_tree else \
        _tree_arrays(block_tree.col_tree)
    rop = _op_arrays(row_ops, row[0].size)
    cop = rop if (col_ops is row_ops and col is row) else _op_arrays(col_ops, col[0].size)
    return PackageInputs(np.ascontiguousarray(triangles, dtype=np.int64), leaves, leaf_ids,
                         row, col, rop, cop)


def leaf_layout(block_tree: BlockTree, row_ops, col_ops, inputs: PackageInputs | None = None):
    """(leaf_ids, leaf_shape, leaf_base) of the whole payload without building
    packages: a dense leaf holds |t| x |s| entries, an admissible leaf the
    coupling matrix rank(t) x rank(s) (make_packages' leaf loop)."""
    x = inputs or package_inputs(np.zeros((0, 3), np.int64), block_tree, row_ops, col_ops)
    L = x.leaves.shape[0]
    shape = np.empty((L, 2), np.int64)
    base = np.empty(L + 1, np.int64)
    p = nat.ptr
    nat.check(nat.lib().gcabem_leaf_layout(L, p(x.leaves), x.row[1].size, p(x.row[1]),
                                           p(x.row_ops[0]), x.col[1].size, p(x.col[1]),
                                           p(x.col_ops[0]), p(shape), p(base)))
    return x.leaf_ids, shape, base


def leaf_mirrors(block_tree: BlockTree, row_ops, col_ops, inputs: PackageInputs | None = None,
                 leaf_range=None, leaf_index=None):
    """Position of each leaf's mirror, the leaf (s, t) of leaf (t, s), or
    None when the block tree's two sides differ. With one cluster tree and
    one operator set on both sides (the reference's pipelines:
    build_block_tree(tree, tree), gca.py:303-306 returning the same dict
    twice), leaf (s, t) holds the transposed panel pairs of leaf (t, s):
    dense leaves the same panels, admissible leaves the same pivots. The
    admissibility test and the subdivision are symmetric, so every leaf has
    its mirror (a diagonal leaf (t, t) is its own)."""
    if block_tree.row_tree is not block_tree.col_tree or row_ops is not col_ops:
        return None
    x = inputs or package_inputs(np.zeros((0, 3), np.int64), block_tree, row_ops, col_ops)

    def build(bt):   # whole-tree map, once per block tree (it does not depend on ops)
        leaves = x.leaves
        n = np.int64(len(bt.row_tree.nodes))
        key = leaves[:, 0] * n + leaves[:, 1]
        order = np.argsort(key, kind="stable")
        want = leaves[:, 1] * n + leaves[:, 0]
        pos = np.minimum(np.searchsorted(key[order], want), max(key.size - 1, 0))
        hit = key[order][pos] == want if key.size else np.zeros(0, bool)
        m = np.where(hit, order[pos], -1)
        if not np.all(hit) or not np.array_equal(leaves[m, 2], leaves[:, 2]):
            return None      # not a symmetric block tree: no mirrored evaluation
        return m.astype(np.int64)
    full = _cached(_mirror_cache, block_tree, build)
    if full is None:
        return None
    if leaf_index is not None:   # a leaf set (sorted positions): mirrors inside it
        idx = np.asarray(leaf_index, dtype=np.int64)
        pos = np.full(full.size, -1, np.int64)
        pos[idx] = np.arange(idx.size)
        return np.ascontiguousarray(pos[full[idx]], dtype=np.int64)
    lo, hi = (0, full.size) if leaf_range is None else leaf_range
    m = full[lo:hi] - lo
    m[(m < 0) | (m >= hi - lo)] = -1
    return np.ascontiguousarray(m, dtype=np.int64)


def full_leaf_mirrors(block_tree: BlockTree, row_ops, col_ops, inputs=None):
    """Whole-tree mirror positions (leaf_mirrors without a range), or None."""
    return leaf_mirrors(block_tree, row_ops, col_ops, inputs)


def shard_leaf_set(block_tree: BlockTree, row_ops, col_ops, shard, disjoint_q: int,
                   inputs: PackageInputs | None = None) -> np.ndarray:
    """Leaves of process `rank` of `world` when one assembly is split over
    processes: sorted preorder positions. Each leaf travels with its mirror
    (leaf (s, t) of leaf (t, s)), so the mirrored evaluation stays inside a
    process: the leaf pairs, keyed by their first leaf in the preorder, are
    cut into `world` contiguous runs balanced by disjoint-rule points (one
    evaluation per mirrored pair). Without mirrors (different trees or
    operators) the sets are contiguous preorder ranges. Every process
    computes the same sets from the payload layout alone."""
    rank, world = int(shard[0]), int(shard[1])
    if not 0 <= rank < world:
        raise SchedulerConfigError(f"shard {shard}: need 0 <= rank < world")
    x = inputs or package_inputs(np.zeros((0, 3), np.int64), block_tree, row_ops, col_ops)
    _, shape, _ = leaf_layout(block_tree, row_ops, col_ops, x)
    L = shape.shape[0]
    if world == 1 or L == 0:
        return np.arange(L, dtype=np.int64)
    m = leaf_mirrors(block_tree, row_ops, col_ops, x)
    work = (shape[:, 0] * shape[:, 1]).astype(np.float64) * disjoint_q
    if m is None:
        first = np.arange(L, dtype=np.int64)
    else:
        first = np.flatnonzero(m >= np.arange(L))     # primaries and diagonal leaves
    cum = np.cumsum(work[first])
    cuts = np.searchsorted(cum, cum[-1] * np.arange(1, world) / world, side="left") + 1
    edges = np.maximum.accumulate(np.concatenate([[0], np.minimum(cuts, first.size),
                                                  [first.size]]))
    mine = first[edges[rank]:edges[rank + 1]]
    if m is not None:
        mine = np.union1d(mine, m[mine])
    return np.ascontiguousarray(mine, dtype=np.int64)


class _Trace:
    """GCABEM_TRACE=1: phase times of the host packaging on stderr."""

    def __init__(self, who: str):
        self.who, self.on = who, bool(os.environ.get("GCABEM_TRACE"))
        self.t = time.perf_counter()

    def mark(self, what: str) -> None:
        if self.on:
            now = time.perf_counter()
            print(f"[{self.who}] {what:<12} {(now - self.t) * 1e3:8.2f} ms", file=sys.stderr)
            self.t = now


def make_packages(triangles: np.ndarray, block_tree: BlockTree, row_ops, col_ops,
                  maxsize: int, nthreads: int = 0, leaf_range=None,
                  inputs: PackageInputs | None = None, leaf_index=None) -> AssemblyPackages:
    """Packages of the block tree's leaves (or of the leaves [lo, hi) of
    leaf_range, payload offsets then relative to leaf lo: the same blocks and
    corrective items those leaves get in the whole-tree packages, list ids
    counted from 0; or of the leaf set `leaf_index`, sorted preorder
    positions, payload laid out leaf after leaf in that order).
    `inputs`: package_inputs() of the same arguments."""
    if maxsize < BYTES_PER_PAIR:
        raise SchedulerConfigError(
            f"maxsize {maxsize} smaller than one pair record ({BYTES_PER_PAIR} B)")
    x = inputs or package_inputs(triangles, block_tree, row_ops, col_ops)
    T, leaves, leaf_ids = x.T, x.leaves, x.leaf_ids
    if leaf_index is not None:
        leaf_index = np.asarray(leaf_index, dtype=np.int64)
        leaves = np.ascontiguousarray(leaves[leaf_index])
        leaf_ids = leaf_ids[leaf_index]
    elif leaf_range is not None:
        lo, hi = leaf_range
        leaves, leaf_ids = leaves[lo:hi], leaf_ids[lo:hi]
    rs, rz, rlo, rhi, rperm = x.row
    cs, cz, clo, chi, cperm = x.col
    rat, rpiv = x.row_ops
    cat, cpiv = x.col_ops
    nthreads = nthreads or host_threads()
    h = ctypes.c_void_p()
    p = nat.ptr
    tr = _Trace("make_packages")
    pbase = x.panel_base   # shared by every range of these inputs (borrowed natively)
    nat.check(nat.lib().gcabem_packages_build_on(
        T.shape[0], p(T), leaves.shape[0], p(leaves), rs.size, p(rs), p(rz), p(rlo), p(rhi),
        p(rperm), p(rat), p(rpiv), cs.size, p(cs), p(cz), p(clo), p(chi), p(cperm), p(cat),
        p(cpiv), int(maxsize), int(nthreads), p(pbase), pbase.size, ctypes.byref(h)))
    try:
        sz = np.zeros(9, dtype=np.int64)
        nat.check(nat.lib().gcabem_packages_sizes(h, p(sz)))
        L, plen, npan, nblk, nlists, nit = (int(v) for v in sz[:6])
        panels = pbase
        shape = np.empty((L, 2), np.int64)
        base = np.empty(L + 1, np.int64)
        rows_at = np.empty(L, np.int64)
        cols_at = np.empty(L, np.int64)
        flagged = np.empty(L, np.uint8)
        blocks = np.empty((5, nblk), np.int64)   # field-major
        blk_list = np.empty(nblk, np.int64)
        items = np.empty((6, nit), np.int64)
        perms = np.empty((nit, 6), np.uint8)
        tr.mark("build+alloc")
        nat.check(nat.lib().gcabem_packages_fetch(
            h, None, p(shape), p(base), p(rows_at), p(cols_at), p(flagged), p(blocks),
            p(blk_list), p(items), p(perms)))
        tr.mark("fetch")
    finally:
        nat.lib().gcabem_packages_free(h)
    mirrors = leaf_mirrors(block_tree, row_ops, col_ops, x, leaf_range, leaf_index)
    tr.mark("mirrors")
    return AssemblyPackages(
        maxsize=int(maxsize), leaf_ids=leaf_ids, leaf_shape=shape, leaf_base=base,
        panels=panels, leaf_rows_at=rows_at, leaf_cols_at=cols_at,
        leaf_flagged=flagged.astype(bool), blk_leaf=blocks[0], blk_r0=blocks[1],
        blk_nr=blocks[2], blk_c0=blocks[3], blk_nc=blocks[4], blk_list=blk_list,
        n_disjoint_lists=nlists, item_case=items[0].astype(np.int8), item_tri_x=items[1],
        item_tri_y=items[2], item_leaf=items[3], item_offset=items[4],
        item_src_block=items[5], perms=perms, leaf_mirror=mirrors)


def shard_leaves(pk: AssemblyPackages, nshards: int, disjoint_q: int, singular_q=None):
    """Contiguous leaf ranges [(lo, hi)], balanced by quadrature points.

    Packages shard with no exchange: each leaf payload has one writer per
    phase (scheduler.py:9-12), so a leaf range owns its payload range and the
    singular items that overwrite inside it."""
    L = pk.leaf_ids.size
    if nshards <= 1 or L == 0:
        return [(0, L)]
    w = (pk.leaf_shape[:, 0] * pk.leaf_shape[:, 1]).astype(np.float64) * disjoint_q
    if singular_q is not None and pk.num_items:
        q = np.asarray([0] + list(singular_q), dtype=np.float64)
        np.add.at(w, pk.item_leaf, q[pk.item_case])
    cum = np.cumsum(w)
    cuts = np.searchsorted(cum, cum[-1] * np.arange(1, nshards) / nshards, side="left") + 1
    edges = np.concatenate([[0], np.minimum(cuts, L), [L]])
    edges = np.maximum.accumulate(edges)
    return [(int(edges[k]), int(edges[k + 1])) for k in range(nshards)]


def inline_lists(pk: AssemblyPackages) -> list:
    """Lists in the order the reference executes them inline
    (workers_per_backend=0): each disjoint list, then any singular list its
    corrective items filled up (ListBuilder flushes when the next item does
    not fit), finally the partial singular lists in SINGULAR_CASES order
    (scheduler.py:474-497). Entries: ("disjoint", block indices) or
    (case, item indices into the generation order)."""
    cap = max(pk.maxsize // BYTES_PER_PAIR, 1)
    order = np.argsort(pk.blk_list, kind="stable")
    bounds = np.searchsorted(pk.blk_list[order], np.arange(pk.n_disjoint_lists + 1))
    triggered = {k: [] for k in range(pk.n_disjoint_lists)}
    tail = []
    for code, name in enumerate(SINGULAR_CASES, start=1):
        idx = np.flatnonzero(pk.item_case == code)
        for a in range(0, idx.size, cap):
            members = idx[a:a + cap]
            if a + cap < idx.size:   # flushed by the item that did not fit
                trig = int(idx[a + cap])
                lid = int(pk.blk_list[pk.item_src_block[trig]])
                triggered[lid].append((trig, name, members))
            else:
                tail.append((name, members))
    out = []
    for lid in range(pk.n_disjoint_lists):
        out.append(("disjoint", order[bounds[lid]:bounds[lid + 1]]))
        for _, name, members in sorted(triggered[lid], key=lambda t: t[0]):
            out.append((name, members))
    return out + tail
