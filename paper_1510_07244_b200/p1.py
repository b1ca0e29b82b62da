"""Piecewise-linear (P1) near-field assembly on the device (BASELINE config 4).

Beyond the reference, whose scheduler and GCAMatrix are piecewise-constant
only: the reference defines the P1 pair integral through
quadrature.integrate_pair(..., basis_x, basis_y) (quadrature.py:223-271)
with the chart barycentrics lambda = (1 - s, s - t, t); this module computes
those 3 x 3 local matrices for every near-field pair (the dense leaves of
the block tree, the same Sauter-Schwab packages as the P0 assembly) and
scatter-adds them into the vertex x vertex near-field matrix with a fixed
summation order (csrc/p1.cu: device radix-sort plan + gather-sum).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .cluster import BlockTree
from .device import device_mesh
from .kernels import KernelSpec
from .mesh import SurfaceMesh
from .packaging import SINGULAR_CASES, make_packages
from .pairquad import default_device
from .quadrature import build_rule, gauss_legendre


def barycentric(points: np.ndarray) -> np.ndarray:
    """(Q, 3) chart barycentrics (1 - s, s - t, t) of reference points (s, t)."""
    p = np.asarray(points, dtype=np.float64)
    return np.stack([1.0 - p[:, 0], p[:, 0] - p[:, 1], p[:, 1]], axis=1)


def local_matrices(mesh: SurfaceMesh, spec: KernelSpec, rule, tri_x, tri_y, perms_x=None,
                   perms_y=None, device: int | None = None) -> np.ndarray:
    """(n, 3, 3) P1 local matrices of the given pairs under a 4D rule, in the
    triangles' stored vertex order: entry [a, b] is integrate_pair with
    basis_x = lambda of chart vertex a, basis_y = lambda_b (after the
    classification permutations), scattered back to stored order."""
    dev = default_device() if device is None else device
    dm = device_mesh(mesh, dev)
    tx, ty = nat.i64(tri_x), nat.i64(tri_y)
    n = tx.shape[0]
    out = np.empty((n, 3, 3), dtype=np.complex128)
    if n == 0:
        return out
    px = None if perms_x is None else nat.u8(perms_x)
    py = None if perms_y is None else nat.u8(perms_y)
    eq, layer = spec.code
    xs, ys, w = nat.f64(rule.x_points), nat.f64(rule.y_points), nat.f64(rule.weights)
    nat.check(nat.lib().gcabem_p1_batch(dm.handle, eq, layer, float(spec.kappa), n, nat.ptr(tx),
                                        nat.ptr(ty), nat.ptr(px), nat.ptr(py), w.shape[0],
                                        nat.ptr(xs), nat.ptr(ys), nat.ptr(w), nat.ptr(out)))
    return out


def near_field_tree(block_tree: BlockTree) -> BlockTree:
    """The block tree restricted to its dense (near-field) leaves."""
    native = getattr(block_tree, "_native_leaves", None)
    if native is not None:
        arr, idx = native
        keep = arr[:, 2] == 1
        leaves = [block_tree.leaves[int(k)] for k in np.flatnonzero(keep)] \
            if len(block_tree.leaves) < 4096 else _LeafSubset(block_tree.leaves, keep)
        bt = BlockTree(block_tree.nodes, block_tree.row_tree, block_tree.col_tree,
                       block_tree.eta, leaves)
        object.__setattr__(bt, "_native_leaves", (np.ascontiguousarray(arr[keep]),
                                                  np.ascontiguousarray(idx[keep])))
        return bt
    return BlockTree(block_tree.nodes, block_tree.row_tree, block_tree.col_tree,
                     block_tree.eta, [l for l in block_tree.leaves if l.kind == "dense"])


class _LeafSubset:
    """Lazy view of the kept leaves of a (lazy) leaf list."""

    def __init__(self, leaves, keep):
        self._leaves, self._pos = leaves, np.flatnonzero(keep)

    def __len__(self):
        return int(self._pos.size)

    def __getitem__(self, k):
        return self._leaves[int(self._pos[k])]

    def __iter__(self):
        for k in self._pos:
            yield self._leaves[int(k)]


class VertexCSR:
    """The P1 near-field matrix (vertex x vertex) as raw CSR arrays in pinned
    host memory: indptr, indices (int32, ascending per row), data
    (complex128). to_scipy() wraps them without copying (scipy's format
    checks cost more than the device assembly at C4, so they are not paid on
    the assembly path)."""

    def __init__(self, indptr, indices, data, n):
        self.indptr, self.indices, self.data = indptr, indices, data
        self.shape = (n, n)

    @property
    def nnz(self) -> int:
        return int(self.indices.size)

    def to_scipy(self):
        import scipy.sparse as sp
        ip = self.indptr.astype(np.int32) if self.nnz < 2 ** 31 - 1 else self.indptr
        return sp.csr_matrix((self.data, self.indices, ip), shape=self.shape, copy=False)

    def toarray(self) -> np.ndarray:
        return self.to_scipy().toarray()


class NearFieldP1:
    """Device plan of the P1 near-field matrix of one kernel: packages of the
    dense leaves, the scatter plan (CSR pattern + contribution order), and
    the local-matrix kernels. execute() may be called repeatedly."""

    def __init__(self, mesh: SurfaceMesh, block_tree: BlockTree, spec: KernelSpec,
                 orders=(3, 5), device: int | None = None, maxsize: int = 8 * 2 ** 20):
        from .scheduler import DeviceLayout
        self.device = default_device() if device is None else device
        nat.require_device(self.device)
        self.mesh, self.spec, self.orders = mesh, spec, tuple(orders)
        nf = near_field_tree(block_tree)
        self.packages = make_packages(mesh.triangles, nf, {}, {}, maxsize)
        dm = device_mesh(mesh, self.device)
        self.layout = DeviceLayout(dm, self.packages, mirror=False)
        dn, sn = self.orders
        g = gauss_legendre(dn)
        gp, gw = nat.f64(g.points), nat.f64(g.weights)
        rules = [build_rule(c, sn).packed() for c in SINGULAR_CASES]
        self.singular_q = [r.shape[0] for r in rules]
        sq = np.array(self.singular_q, dtype=np.int64)
        rptr = (ctypes.c_void_p * 3)(*[r.ctypes.data for r in rules])
        eq, layer = spec.code
        h = ctypes.c_void_p()
        nat.check(nat.lib().gcabem_p1_create(self.layout.handle, eq, layer, float(spec.kappa),
                                             dn, nat.ptr(gp), nat.ptr(gw), nat.ptr(sq),
                                             ctypes.cast(rptr, ctypes.c_void_p),
                                             ctypes.byref(h)))
        self.handle = h.value
        self._keep = rules
        info = np.zeros(4, np.int64)
        nat.check(nat.lib().gcabem_p1_info(self.handle, nat.ptr(info), None))
        self.num_vertices, self.nnz, self.num_pairs, self.num_singular = (int(x) for x in info)

    def execute(self) -> None:
        nat.check(nat.lib().gcabem_p1_execute(self.handle))

    def timing_ms(self) -> dict:
        info = np.zeros(4, np.int64)
        ms = (ctypes.c_float * 2)()
        nat.check(nat.lib().gcabem_p1_info(self.handle, nat.ptr(info), ms))
        return {"local": ms[0], "scatter": ms[1]}

    def download(self, with_local: bool = False):
        """(indptr int64, indices int32, data complex128[, local (P, 3, 3)])"""
        indptr = np.empty(self.num_vertices + 1, np.int64)
        # pinned targets: the D2H of ~0.6 GB at C4 runs at the PCIe rate
        indices = nat.pinned_empty(max(self.nnz, 1), np.int32)
        data = nat.pinned_empty(max(self.nnz, 1), np.complex128)
        local = np.empty((self.num_pairs, 3, 3), np.complex128) if with_local else None
        nat.check(nat.lib().gcabem_p1_download(self.handle, nat.ptr(indptr), nat.ptr(indices),
                                               nat.ptr(data), nat.ptr(local)))
        res = (indptr, indices[:self.nnz], data[:self.nnz])
        return res + (local,) if with_local else res

    def assemble(self) -> VertexCSR:
        """execute() + the near-field matrix (VertexCSR; .to_scipy() for scipy)."""
        self.execute()
        indptr, indices, data = self.download()
        return VertexCSR(indptr, indices, data, self.num_vertices)

    def close(self) -> None:
        h, self.handle = getattr(self, "handle", None), None
        if h and getattr(nat, "_lib", None) is not None:  # nat is None at interpreter teardown
            nat._lib.gcabem_p1_destroy(h)
        lay = getattr(self, "layout", None)
        if lay is not None:
            lay.close()

    def __del__(self):
        self.close()


def assemble_near_field(mesh: SurfaceMesh, block_tree: BlockTree, spec: KernelSpec,
                        orders=(3, 5), device: int | None = None) -> VertexCSR:
    """P1 near-field matrix (vertex x vertex CSR) of `spec` on the device."""
    plan = NearFieldP1(mesh, block_tree, spec, orders, device)
    try:
        return plan.assemble()
    finally:
        plan.close()
