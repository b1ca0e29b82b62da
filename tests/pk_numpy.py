"""TEST-SIDE numpy restatement of the host work packaging (cross-check for
the native builder in csrc/packaging.cpp at sizes without golden fixtures).
Pinned itself against the reference's inline list composition at L3.

Work packages: the CPU half of scheduler.run_assembly, vectorised.

Reproduces, bit for bit, what the reference scheduler does on the host
before and between quadrature calls (pkg/src/gcabem/scheduler.py):

* leaf enumeration in block-tree preorder with rows/cols = cluster panels
  (dense) or ACA pivots (admissible) and the ``flagged`` touch test
  (_leaf_blocks :425-439; make_payloads :411-422 for the payload layout);
* WorkBlock splitting along the longer dimension (split_block :153-175) and
  greedy byte-budgeted disjoint lists (ListBuilder :178-208);
* the corrective scan of flagged blocks: every pair sharing 1-3 vertices
  becomes a WorkItem in argwhere (row-major) order (distribute_disjoint
  :334-359), appended to per-case singular lists in inline-mode order;
* classification permutations of every singular item (classify_pair,
  quadrature.py:197-220; _merge_singular :223-232).

The result is a set of flat arrays the device consumes directly (C ABI
gcabem_plan_create) plus the list composition for stats and parity tests.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_1510_07244_b200.cluster import BlockTree
from paper_1510_07244_b200.quadrature import classify_pairs

PAIR_RECORD_BYTES = 24
VALUE_BYTES = 8
BYTES_PER_PAIR = PAIR_RECORD_BYTES + VALUE_BYTES
SINGULAR_CASES = ("vertex", "edge", "identical")
_SCAN_CHUNK = 1 << 21   # flagged pairs scanned per vectorised step


class SchedulerConfigError(ValueError):
    pass


@dataclass
class AssemblyPackages:
    """Flat package description of one assembly (see module docstring)."""
    maxsize: int
    leaf_ids: np.ndarray        # (L,) BlockNode.index, preorder
    leaf_kind: np.ndarray       # (L,) 1 dense, 0 admissible
    leaf_shape: np.ndarray      # (L, 2)
    leaf_base: np.ndarray       # (L+1,) payload offsets (entries)
    panels: np.ndarray          # concatenated leaf rows then cols
    leaf_rows_at: np.ndarray    # (L,)
    leaf_cols_at: np.ndarray    # (L,)
    leaf_flagged: np.ndarray    # (L,) bool
    # disjoint WorkBlocks after splitting, in list order
    blk_leaf: np.ndarray        # (B,) leaf position
    blk_r0: np.ndarray
    blk_c0: np.ndarray
    blk_nr: np.ndarray
    blk_nc: np.ndarray
    blk_list: np.ndarray        # (B,) disjoint list number
    n_disjoint_lists: int
    # singular WorkItems in generation order
    item_case: np.ndarray       # (S,) 1 vertex, 2 edge, 3 identical
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
        """(B', 6) int64 {payload_base, ld, nr, nc, rows_at, cols_at} for the
        blocks of leaves [leaf_lo, leaf_hi), bases relative to leaf_lo."""
        leaf_hi = self.leaf_ids.size if leaf_hi is None else leaf_hi
        sel = (self.blk_leaf >= leaf_lo) & (self.blk_leaf < leaf_hi)
        lf = self.blk_leaf[sel]
        ld = self.leaf_shape[lf, 1]
        base = self.leaf_base[lf] - self.leaf_base[leaf_lo] + self.blk_r0[sel] * ld + self.blk_c0[sel]
        return np.ascontiguousarray(np.stack(
            [base, ld, self.blk_nr[sel], self.blk_nc[sel],
             self.leaf_rows_at[lf] + self.blk_r0[sel], self.leaf_cols_at[lf] + self.blk_c0[sel],
             lf], axis=1).astype(np.int64))

    def device_items(self, leaf_lo: int = 0, leaf_hi: int | None = None):
        """Singular items of leaves [leaf_lo, leaf_hi), grouped by case:
        ((S', 4) int64 {case, tri_x, tri_y, payload_index}, (S', 6) uint8)."""
        leaf_hi = self.leaf_ids.size if leaf_hi is None else leaf_hi
        sel = np.flatnonzero((self.item_leaf >= leaf_lo) & (self.item_leaf < leaf_hi))
        sel = sel[np.argsort(self.item_case[sel], kind="stable")]
        idx = self.leaf_base[self.item_leaf[sel]] - self.leaf_base[leaf_lo] + self.item_offset[sel]
        items = np.stack([self.item_case[sel].astype(np.int64), self.item_tri_x[sel],
                          self.item_tri_y[sel], idx], axis=1).astype(np.int64)
        return np.ascontiguousarray(items), np.ascontiguousarray(self.perms[sel])

    def singular_lists(self):
        """Per case: list of (start, stop) ranges into that case's items in
        generation order, as ListBuilder cuts them."""
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


def _greedy_lists(nbytes: np.ndarray, maxsize: int) -> tuple[np.ndarray, int]:
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


def make_packages(triangles: np.ndarray, block_tree: BlockTree, row_ops, col_ops,
                  maxsize: int) -> AssemblyPackages:
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
    # panels: rows_0, cols_0, rows_1, cols_1, ...
    seg = np.empty(2 * L, dtype=np.int64)
    seg[0::2], seg[1::2] = shape[:, 0], shape[:, 1]
    starts = np.concatenate([[0], np.cumsum(seg)])
    inter = [None] * (2 * L)
    inter[0::2], inter[1::2] = rows_list, cols_list
    panels = np.concatenate(inter).astype(np.int64) if L else np.empty(0, np.int64)
    rows_at, cols_at = starts[0:-1:2], starts[1::2]
    base = np.concatenate([[0], np.cumsum(shape[:, 0] * shape[:, 1])]).astype(np.int64)

    # touch test per leaf (box_distance == 0.0), exact without the norm
    rlo = np.array([n.lo for n in rt.nodes]); rhi = np.array([n.hi for n in rt.nodes])
    clo = np.array([n.lo for n in ct.nodes]); chi = np.array([n.hi for n in ct.nodes])
    lr = np.fromiter((l.row for l in leaves), dtype=np.int64, count=L)
    lc = np.fromiter((l.col for l in leaves), dtype=np.int64, count=L)
    flagged = np.all((rlo[lr] <= chi[lc]) & (clo[lc] <= rhi[lr]), axis=1) if L else \
        np.zeros(0, bool)

    # split + greedy disjoint lists
    npairs = shape[:, 0] * shape[:, 1]
    big = np.flatnonzero(npairs * BYTES_PER_PAIR > maxsize)
    if big.size == 0:
        b_leaf = np.arange(L, dtype=np.int64)
        b_r0 = np.zeros(L, np.int64); b_c0 = np.zeros(L, np.int64)
        b_nr = shape[:, 0].copy(); b_nc = shape[:, 1].copy()
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

    # corrective scan of flagged blocks, row-major within each block
    T = np.asarray(triangles, dtype=np.int64)
    fb = np.flatnonzero(flagged[b_leaf])
    it_case, it_tx, it_ty, it_leaf, it_off, it_blk = [], [], [], [], [], []
    sizes = b_nr[fb] * b_nc[fb]
    cut = 0
    while cut < fb.size:
        acc, stop = 0, cut
        while stop < fb.size and (acc == 0 or acc + sizes[stop] <= _SCAN_CHUNK):
            acc += int(sizes[stop]); stop += 1
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
        it_tx.append(tx[hit]); it_ty.append(ty[hit]); it_leaf.append(lf[hit])
        it_off.append((b_r0[owner[hit]] + i[hit]) * shape[lf[hit], 1] + b_c0[owner[hit]] + j[hit])
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
    """Contiguous leaf ranges [(lo, hi)], balanced by quadrature points.

    Packages shard with no exchange: each leaf payload has one writer per
    phase (scheduler.py:9-12), so a leaf range owns its payload range and
    the singular items that overwrite inside it."""
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
    not fit), and finally the partial singular lists in SINGULAR_CASES order
    (scheduler.py:474-497). Entries: ("disjoint", block indices) or
    (case, item indices into the generation order)."""
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
            if a + cap < idx.size:   # flushed by the item that did not fit
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
