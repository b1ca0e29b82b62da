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
        # bumped by every entry replacement/removal (device copies key on it)
        self.version = 0

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
        self.version += 1

    def __delitem__(self, key):
        present = key in self._over or (self._index(key) >= 0 and int(key) not in self._gone)
        if not present:
            raise KeyError(key)
        self._over.pop(key, None)
        if self._index(key) >= 0:
            self._gone.add(int(key))
        self.version += 1

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
    # sorted preorder positions of the block-tree leaves this matrix holds
    # (one process's shard of a job split over processes,
    # SchedulerParams.shard); None = every leaf
    shard_leaves: np.ndarray | None = field(default=None, repr=False)

    @property
    def shape(self) -> tuple[int, int]:
        return (len(self.block_tree.row_tree.permutation),
                len(self.block_tree.col_tree.permutation))

    def checksum(self) -> str:
        """sha256 over all leaf payloads in block-tree preorder (h2.py:40-46)."""
        if self.shard_leaves is not None:
            raise ValueError(f"a shard ({self.shard_leaves.size} of {len(self.block_tree.leaves)} "
                             "leaves) has no whole-matrix checksum")
        h = hashlib.sha256()
        for leaf in self.block_tree.leaves:
            h.update(np.ascontiguousarray(self.payloads[leaf.index]).tobytes())
        return h.hexdigest()


def _coupling_block(M: GCAMatrix, leaf) -> np.ndarray:
    return M.row_ops[leaf.row].V @ M.payloads[leaf.index] @ M.col_ops[leaf.col].V.T


def _leaf_arrays(M: GCAMatrix):
    """(L, 7) {row_start, row_size, col_start, col_size, dense, row_op, col_op}
    in block-tree preorder plus the flat payload and per-leaf offsets, and
    the operator tables {start, size, rank, v_offset} with their stacked V
    (complex128). Operator indices follow sorted cluster ids."""
    bt = M.block_tree
    rt, ct = bt.row_tree, bt.col_tree
    native = getattr(bt, "_native_leaves", None)
    if native is not None:
        arr = native[0]
        lrow, lcol, ldense = arr[:, 0], arr[:, 1], arr[:, 2].astype(bool)
        lids = bt.leaves._idx if hasattr(bt.leaves, "_idx") else \
            np.array([l.index for l in bt.leaves], dtype=np.int64)
    else:
        lrow = np.array([l.row for l in bt.leaves], dtype=np.int64)
        lcol = np.array([l.col for l in bt.leaves], dtype=np.int64)
        ldense = np.array([l.kind == "dense" for l in bt.leaves], dtype=bool)
        lids = np.array([l.index for l in bt.leaves], dtype=np.int64)
    rstart = np.fromiter((n.start for n in rt.nodes), np.int64, len(rt.nodes))
    rsize = np.fromiter((n.size for n in rt.nodes), np.int64, len(rt.nodes))
    if ct is rt:
        cstart, csize = rstart, rsize
    else:
        cstart = np.fromiter((n.start for n in ct.nodes), np.int64, len(ct.nodes))
        csize = np.fromiter((n.size for n in ct.nodes), np.int64, len(ct.nodes))

    def op_table(ops, start, size, used):
        ids = sorted(c for c in ops if c in used)
        pos = {c: k for k, c in enumerate(ids)}
        desc = np.zeros((max(len(ids), 1), 4), np.int64)
        Vs, off = [], 0
        for k, c in enumerate(ids):
            V = np.asarray(ops[c].V)
            desc[k] = (start[c], size[c], V.shape[1], off)
            Vs.append(np.ascontiguousarray(V, dtype=np.complex128).ravel())
            off += V.size
        return pos, desc, Vs
    adm = ~ldense
    rpos, rdesc, rV = op_table(M.row_ops, rstart, rsize, set(lrow[adm].tolist()))
    cpos, cdesc, cV = op_table(M.col_ops, cstart, csize, set(lcol[adm].tolist()))
    nr_v = sum(v.size for v in rV)
    cdesc[:, 3] += nr_v
    V = np.concatenate(rV + cV) if rV or cV else np.zeros(1, np.complex128)
    L = lrow.size
    desc = np.empty((L, 7), np.int64)
    desc[:, 0], desc[:, 1] = rstart[lrow], rsize[lrow]
    desc[:, 2], desc[:, 3] = cstart[lcol], csize[lcol]
    desc[:, 4] = ldense
    desc[:, 5] = [rpos.get(int(r), -1) if a_ else -1 for r, a_ in zip(lrow, adm)]
    desc[:, 6] = [cpos.get(int(c), -1) if a_ else -1 for c, a_ in zip(lcol, adm)]
    P = M.payloads
    if isinstance(P, LeafPayloads) and not P._over and not P._gone and \
            np.array_equal(P._ids, lids):
        buf, base = P.buffer, P._base[:-1]
    else:
        parts = [np.ascontiguousarray(P[int(k)], dtype=np.complex128).ravel() for k in lids]
        base = np.concatenate([[0], np.cumsum([q.size for q in parts])[:-1]]).astype(np.int64)
        buf = np.concatenate(parts) if parts else np.zeros(1, np.complex128)
    return (desc, np.ascontiguousarray(base, dtype=np.int64),
            np.ascontiguousarray(buf, dtype=np.complex128), (rdesc, len(rpos)),
            (cdesc, len(cpos)), np.ascontiguousarray(V))


class DeviceH2:
    """A GCAMatrix resident on one device (payload, bases, index plans) with a
    deterministic matrix-vector product (C ABI gcabem_h2_*; csrc/h2_matvec.cu)."""

    def __init__(self, M: GCAMatrix, device: int | None = None):
        import ctypes
        from . import _native as nat
        from .pairquad import default_device
        if M.shard_leaves is not None:
            raise ValueError("DeviceH2 needs the whole matrix, not a process shard "
                             f"({M.shard_leaves.size} leaves)")
        self.device = default_device() if device is None else device
        nat.require_device(self.device)
        desc, base, buf, (rdesc, nro), (cdesc, nco), V = _leaf_arrays(M)
        rows, cols = M.shape
        rp = np.ascontiguousarray(M.block_tree.row_tree.permutation, dtype=np.int64)
        cp = np.ascontiguousarray(M.block_tree.col_tree.permutation, dtype=np.int64)
        h = ctypes.c_void_p()
        p = nat.ptr
        nat.check(nat.lib().gcabem_h2_create(
            self.device, rows, cols, p(rp), p(cp), desc.shape[0], p(desc), p(base), buf.size,
            p(buf), nro, p(rdesc), nco, p(cdesc), V.size, p(V), ctypes.byref(h)))
        self.handle = h.value
        self.shape = (rows, cols)
        bpp = ctypes.c_double()
        nat.check(nat.lib().gcabem_h2_info(self.handle, ctypes.byref(bpp)))
        self.bytes_per_product = bpp.value
        self.last_device_ms = None

    def matvec(self, x: np.ndarray) -> np.ndarray:
        import ctypes
        from . import _native as nat
        x = np.asarray(x)
        if x.shape != (self.shape[1],):
            raise ValueError(f"dimension mismatch: operator {self.shape}, vector {x.shape}")
        xc = np.ascontiguousarray(x, dtype=np.complex128)
        y = np.empty(self.shape[0], dtype=np.complex128)
        ms = ctypes.c_float()
        nat.check(nat.lib().gcabem_h2_matvec(self.handle, nat.ptr(xc), nat.ptr(y),
                                             ctypes.byref(ms)))
        self.last_device_ms = ms.value
        return y

    def close(self) -> None:
        from . import _native as nat
        h, self.handle = getattr(self, "handle", None), None
        if h and getattr(nat, "_lib", None) is not None:  # nat is None at interpreter teardown
            nat._lib.gcabem_h2_free(h)

    def __del__(self):
        self.close()


def _device_key(M: GCAMatrix) -> tuple:
    """What the device copy was built from: the payload mapping (identity and
    entry version), its buffer and the operator dicts. Replacing, deleting or
    reassigning any of them invalidates the copy; writing INTO a payload
    array in place is not seen (call invalidate(M) after doing that)."""
    P = M.payloads
    return (id(P), getattr(P, "version", None), id(getattr(P, "buffer", None)),
            id(M.row_ops), id(M.col_ops), id(M.block_tree))


def invalidate(M: GCAMatrix) -> None:
    """Drop M's cached device copy (next matvec re-uploads the payloads)."""
    dev = getattr(M, "_device_h2", None)
    if dev is not None:
        dev.close()
    object.__setattr__(M, "_device_h2", None)


def device_matrix(M: GCAMatrix, device: int | None = None) -> DeviceH2:
    """The device-resident copy of M, cached on M while the payloads and
    operators it was built from are unchanged (_device_key)."""
    dev = getattr(M, "_device_h2", None)
    key = _device_key(M)
    if isinstance(M.payloads, dict):  # plain dict: no version counter, never cached
        key = None
    if dev is None or dev.key != key or key is None or \
            (device is not None and dev.device != device):
        invalidate(M)
        dev = DeviceH2(M, device)
        dev.key = key
        if key is not None:
            object.__setattr__(M, "_device_h2", dev)
    return dev


def matvec(M: GCAMatrix, x: np.ndarray) -> np.ndarray:
    """y = M x (h2.py:49-71) on the device: dense leaves P x[s], admissible
    leaves V_t (P (V_s^T x[s])), summed in a fixed order (bitwise
    reproducible). The matrix is uploaded once and cached on M."""
    rows, cols = M.shape
    x = np.asarray(x)
    if x.shape != (cols,):
        raise ValueError(f"dimension mismatch: operator {M.shape}, vector {x.shape}")
    return device_matrix(M).matvec(x)


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
