"""Compressed operator container (drop-in for gcabem.h2, pkg/src/gcabem/h2.py).

GCAMatrix.payloads maps block-leaf index -> complex128 C-ordered array,
dense (|t|, |s|) or coupling (rank_t, rank_s), exactly as the reference
(h2.py:28-46). On this implementation every payload is a VIEW into one
contiguous buffer (leaves in block-tree preorder, row-major), the host
image of the device payload the kernels write; ``buffer`` exposes it.
"""
from __future__ import annotations

import hashlib
from collections.abc import MutableMapping
from dataclasses import dataclass, field

import numpy as np

from .cluster import BlockTree

DENSE_EXPANSION_CAP = 4096


class LeafPayloads(MutableMapping):
    """dict[leaf index -> payload] whose values are views of one buffer,
    materialised on access (100k+ leaves: building every view eagerly would
    cost more than the device assembly). Assignment replaces an entry, as
    on the reference's plain dict."""

    def __init__(self, buffer: np.ndarray, leaf_ids: np.ndarray, leaf_base: np.ndarray,
                 leaf_shape: np.ndarray):
        self.buffer = buffer
        self._ids = np.asarray(leaf_ids, dtype=np.int64)
        self._sorted = bool(np.all(self._ids[1:] > self._ids[:-1]))
        self._pos = None if self._sorted else {int(k): i for i, k in enumerate(self._ids)}
        self._base = leaf_base
        self._shape = leaf_shape
        self._over: dict = {}
        self._gone: set = set()

    def _index(self, key) -> int:
        k = int(key)
        if self._sorted:
            i = int(np.searchsorted(self._ids, k))
            if i < self._ids.size and self._ids[i] == k:
                return i
            return -1
        return self._pos.get(k, -1)

    def __getitem__(self, key):
        if key in self._over:
            return self._over[key]
        i = self._index(key)
        if i < 0 or int(key) in self._gone:
            raise KeyError(key)
        a, b = int(self._base[i]), int(self._base[i + 1])
        return self.buffer[a:b].reshape(int(self._shape[i, 0]), int(self._shape[i, 1]))

    def __setitem__(self, key, value):
        self._over[key] = value
        self._gone.discard(int(key))

    def __delitem__(self, key):
        if key in self._over:
            del self._over[key]
        if self._index(key) >= 0:
            self._gone.add(int(key))
        elif key not in self._over:
            raise KeyError(key)

    def __iter__(self):
        for k in self._ids.tolist():
            if k not in self._gone and k not in self._over:
                yield k
        yield from self._over

    def __len__(self):
        return self._ids.size - len(self._gone) + sum(
            1 for k in self._over if self._index(k) < 0)

    def __contains__(self, key):
        try:
            self[key]
        except (KeyError, TypeError, ValueError):
            return False
        return True


@dataclass
class GCAMatrix:
    block_tree: BlockTree
    row_ops: dict
    col_ops: dict
    payloads: dict
    buffer: np.ndarray | None = field(default=None, repr=False)

    @property
    def shape(self) -> tuple[int, int]:
        return (len(self.block_tree.row_tree.permutation),
                len(self.block_tree.col_tree.permutation))

    def checksum(self) -> str:
        """sha256 over all leaf payloads in block-tree preorder (h2.py:40-46)."""
        h = hashlib.sha256()
        for leaf in self.block_tree.leaves:
            h.update(np.ascontiguousarray(self.payloads[leaf.index]).tobytes())
        return h.hexdigest()


def _coupling_block(M: GCAMatrix, leaf) -> np.ndarray:
    return M.row_ops[leaf.row].V @ M.payloads[leaf.index] @ M.col_ops[leaf.col].V.T


def matvec(M: GCAMatrix, x: np.ndarray) -> np.ndarray:
    """y = M x, leaves accumulated in preorder (h2.py:49-71). The column-side
    operator is conj(V_s), so its conjugate transpose is the plain V_s^T."""
    rows, cols = M.shape
    x = np.asarray(x)
    if x.shape != (cols,):
        raise ValueError(f"dimension mismatch: operator {M.shape}, vector {x.shape}")
    rt, ct = M.block_tree.row_tree, M.block_tree.col_tree
    xp = np.asarray(x, dtype=np.complex128)[ct.permutation]
    yp = np.zeros(rows, dtype=np.complex128)
    for leaf in M.block_tree.leaves:
        t, s = rt.nodes[leaf.row], ct.nodes[leaf.col]
        xs = xp[s.start:s.start + s.size]
        P = M.payloads[leaf.index]
        if leaf.kind == "dense":
            yp[t.start:t.start + t.size] += P @ xs
        else:
            yp[t.start:t.start + t.size] += M.row_ops[leaf.row].V @ (P @ (M.col_ops[leaf.col].V.T @ xs))
    y = np.empty(rows, dtype=np.complex128)
    y[rt.permutation] = yp
    return y


def to_dense(M: GCAMatrix, cap: int = DENSE_EXPANSION_CAP) -> np.ndarray:
    """Expand every leaf into the global matrix (verification; h2.py:74-93)."""
    rows, cols = M.shape
    if rows > cap or cols > cap:
        raise ValueError(f"matrix {rows}x{cols} exceeds the expansion cap {cap}")
    rt, ct = M.block_tree.row_tree, M.block_tree.col_tree
    G = np.zeros((rows, cols), dtype=np.complex128)
    for leaf in M.block_tree.leaves:
        t, s = rt.nodes[leaf.row], ct.nodes[leaf.col]
        blk = M.payloads[leaf.index] if leaf.kind == "dense" else _coupling_block(M, leaf)
        G[np.ix_(rt.permutation[t.start:t.start + t.size],
                 ct.permutation[s.start:s.start + s.size])] = blk
    return G


def storage_bytes(M: GCAMatrix) -> dict:
    """Byte footprint by component (h2.py:96-105)."""
    near = sum(M.payloads[l.index].nbytes for l in M.block_tree.leaves if l.kind == "dense")
    coup = sum(M.payloads[l.index].nbytes for l in M.block_tree.leaves if l.kind == "admissible")
    ops = {id(op): op for op in list(M.row_ops.values()) + list(M.col_ops.values())}
    bases = sum(op.V.nbytes + op.pivots_global.nbytes for op in ops.values())
    return {"near": near, "coupling": coup, "bases": bases, "total": near + coup + bases}


# ---------------------------------------------------------------------------
# GCAMAT01 binary format (reference h2.py:195-314), byte-compatible:
# little-endian; arrays as <BB kind,ndim> <ndim q shape> data, kinds
# f8 / c16 / i8 / u1; cluster trees, block tree, operators, payloads.

import struct  # noqa: E402

_MAGIC = b"GCAMAT01"
_FORMAT_VERSION = 1
_DTYPE_OF_KIND = {0: "<f8", 1: "<c16", 2: "<i8", 3: "<u1"}
_KIND_OF_DTYPE = {"f": 0, "c": 1, "i": 2, "u": 3}
_BLOCK_KIND = {"admissible": 0, "dense": 1, "split": 2}
_BLOCK_NAME = {v: k for k, v in _BLOCK_KIND.items()}


def _put_array(out: list, a) -> None:
    a = np.asarray(a)
    code = _KIND_OF_DTYPE[a.dtype.kind]
    out.append(struct.pack("<BB", code, a.ndim))
    out.append(struct.pack(f"<{a.ndim}q", *a.shape))
    out.append(np.ascontiguousarray(a.astype(_DTYPE_OF_KIND[code], copy=False)).tobytes())


def _put_tree(out: list, tree) -> None:
    out.append(struct.pack("<qq", len(tree.nodes), tree.leaf_size))
    _put_array(out, tree.permutation)
    for n in tree.nodes:
        out.append(struct.pack("<qqq", n.start, n.size, len(n.children)))
        if n.children:
            out.append(struct.pack(f"<{len(n.children)}q", *n.children))
        _put_array(out, n.lo)
        _put_array(out, n.hi)


def dump(M: GCAMatrix, path) -> None:
    """Write M in the reference's GCAMAT01 v1 layout (h2.py:241-274)."""
    bt = M.block_tree
    shared_tree = bt.row_tree is bt.col_tree
    shared_ops = M.row_ops is M.col_ops
    out: list = [_MAGIC, struct.pack("<I", _FORMAT_VERSION),
                 struct.pack("<BB", shared_tree, shared_ops)]
    _put_tree(out, bt.row_tree)
    if not shared_tree:
        _put_tree(out, bt.col_tree)
    out.append(struct.pack("<qd", len(bt.nodes), bt.eta))
    for n in bt.nodes:
        out.append(struct.pack("<qqBq", n.row, n.col, _BLOCK_KIND[n.kind], len(n.children)))
        if n.children:
            out.append(struct.pack(f"<{len(n.children)}q", *n.children))

    def put_ops(ops):
        out.append(struct.pack("<q", len(ops)))
        for cid in sorted(ops):
            op = ops[cid]
            out.append(struct.pack("<q", cid))
            _put_array(out, op.pivots_local)
            _put_array(out, op.pivots_global)
            _put_array(out, op.V)

    put_ops(M.row_ops)
    if not shared_ops:
        put_ops(M.col_ops)
    keys = sorted(M.payloads)
    out.append(struct.pack("<q", len(keys)))
    with open(path, "wb") as fh:
        fh.write(b"".join(out))
        for k in keys:
            part: list = [struct.pack("<q", k)]
            _put_array(part, M.payloads[k])
            fh.write(b"".join(part))


class _Reader:
    def __init__(self, data: bytes):
        self.data, self.pos = data, 0

    def take(self, fmt: str):
        vals = struct.unpack_from(fmt, self.data, self.pos)
        self.pos += struct.calcsize(fmt)
        return vals

    def array(self) -> np.ndarray:
        code, ndim = self.take("<BB")
        shape = self.take(f"<{ndim}q")
        dt = np.dtype(_DTYPE_OF_KIND[code])
        count = int(np.prod(shape)) if shape else 1
        a = np.frombuffer(self.data, dtype=dt, count=count, offset=self.pos)
        self.pos += count * dt.itemsize
        return a.reshape(shape).copy()


def _get_tree(r: _Reader):
    from .cluster import ClusterNode, ClusterTree
    n_nodes, leaf_size = r.take("<qq")
    perm = r.array()
    nodes = []
    for k in range(n_nodes):
        start, size, nch = r.take("<qqq")
        ch = r.take(f"<{nch}q") if nch else ()
        lo, hi = r.array(), r.array()
        nodes.append(ClusterNode(k, start, size, lo, hi, tuple(ch)))
    return ClusterTree(nodes, perm, int(leaf_size))


def load(path) -> GCAMatrix:
    """Read a GCAMAT01 v1 file (h2.py:277-314)."""
    from .cluster import BlockNode, BlockTree
    from .gca import InterpolationOperator
    with open(path, "rb") as fh:
        r = _Reader(fh.read())
    if r.data[:8] != _MAGIC:
        raise ValueError("not a GCA matrix file")
    r.pos = 8
    (version,) = r.take("<I")
    if version != _FORMAT_VERSION:
        raise ValueError(f"unsupported format version {version}")
    shared_tree, shared_ops = r.take("<BB")
    row_tree = _get_tree(r)
    col_tree = row_tree if shared_tree else _get_tree(r)
    n_nodes, eta = r.take("<qd")
    nodes = []
    for k in range(n_nodes):
        row, col, kind, nch = r.take("<qqBq")
        ch = r.take(f"<{nch}q") if nch else ()
        nodes.append(BlockNode(k, row, col, _BLOCK_NAME[kind], tuple(ch)))
    bt = BlockTree(nodes, row_tree, col_tree, eta, [n for n in nodes if n.kind != "split"])

    def get_ops():
        (count,) = r.take("<q")
        ops = {}
        for _ in range(count):
            (cid,) = r.take("<q")
            pl, pg, V = r.array(), r.array(), r.array()
            ops[cid] = InterpolationOperator(cid, pl, pg, V)
        return ops

    row_ops = get_ops()
    col_ops = row_ops if shared_ops else get_ops()
    (npay,) = r.take("<q")
    payloads = {}
    for _ in range(npay):
        (lid,) = r.take("<q")
        payloads[lid] = r.array()
    return GCAMatrix(bt, row_ops, col_ops, payloads)
