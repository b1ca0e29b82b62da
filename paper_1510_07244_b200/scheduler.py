"""Case-homogeneous work packages executed on B200s (drop-in for gcabem.scheduler).

Reference: pkg/src/gcabem/scheduler.py (paper Alg. 1-4). The host builds
exactly the reference's packages — disjoint lists of WorkBlocks under the
byte budget, corrective singular lists from the shared-vertex scan of
flagged blocks — and the device executes them: one fused launch runs every
disjoint list straight into a device-resident payload buffer (all leaves
back to back), then one launch per singular case overwrites the corrected
entries (the overwrite protocol, scheduler.py:9-12, :488-494: stream order
gives the happens-before). One D2H returns the payload into pinned host
memory; GCAMatrix.payloads are views into it.

The reference's worker threads and queues (:264-408) have no counterpart:
the device is the worker pool. With several devices, leaves are statically
partitioned (no exchange step exists). There is no CPU backend: a missing
library or device raises BackendError.
"""
from __future__ import annotations

import ctypes
import os
import sys
import threading
import time
import weakref
from dataclasses import dataclass, field, replace

import numpy as np

from . import _native as nat
from ._native import BackendError
from .cluster import BlockTree
from .device import DeviceMesh, device_mesh
from .h2 import GCAMatrix, LeafPayloads
from .kernels import KernelSpec
from .mesh import SurfaceMesh
from .packaging import (BYTES_PER_PAIR, PAIR_RECORD_BYTES, SINGULAR_CASES, VALUE_BYTES,
                        AssemblyPackages, SchedulerConfigError, leaf_layout, make_packages,
                        package_inputs, shard_leaf_set, shard_leaves)
from .quadrature import QuadRule4D, build_rule, classify_pair, gauss_legendre

DEFAULT_MAXSIZE = 8 * 2 ** 20
# payload growth between consecutive ranges of a staged assembly (measured at
# C3: 1.5 with 6 ranges beats 2 with 5 by ~5% e2e)
STAGE_GROWTH = float(os.environ.get("GCABEM_STAGE_GROWTH", "1.5"))
SYM_AUTO_BYTES = int(os.environ.get("GCABEM_SYM_AUTO_BYTES", str(2 << 30)))


def _symmetric(params, payload_len: int) -> bool:
    if params.symmetric_download is None:
        return payload_len * 16 >= SYM_AUTO_BYTES
    return bool(params.symmetric_download)


# range 0 = the first 1/STAGE_FIRST of the leaves (the device and the link
# start as soon as it is packaged)
STAGE_FIRST = int(os.environ.get("GCABEM_STAGE_FIRST", "64"))
# host threads packaging leaf ranges (and building their device layouts) ahead
# of the device
PACK_WORKERS = int(os.environ.get("GCABEM_PACK_WORKERS", "2"))
# the last STAGE_TAPER ranges halve in size one after the other (a small last
# range shortens the tail: its packaging, layout and D2H follow everything else)
STAGE_TAPER = int(os.environ.get("GCABEM_STAGE_TAPER", "0"))
_CASE_OF_SHARED = {1: "vertex", 2: "edge", 3: "identical"}

__all__ = ["Backend", "SchedulerParams", "WorkBlock", "WorkItem", "WorkList", "AssemblyStats",
           "split_block", "ListBuilder", "batch_quadrature", "execute_list", "run_assembly",
           "make_payloads", "BackendError", "SchedulerConfigError", "CUDA_BACKEND",
           "BATCH_BACKEND", "SCALAR_BACKEND", "DEFAULT_MAXSIZE", "BYTES_PER_PAIR",
           "PAIR_RECORD_BYTES", "VALUE_BYTES", "SINGULAR_CASES", "AssemblyPlan",
           "DeviceLayout", "potential_batch", "clear_package_cache", "run_assembly_pair"]


BACKEND_KINDS = ("cuda", "scalar-reference", "batch")


@dataclass(frozen=True)
class Backend:
    """Execution target: the sm_100a kernels on `devices`. The reference's
    kinds (scheduler.py:51-66: "scalar-reference", "batch") are accepted so
    reference-style configs construct unchanged; every kind runs the CUDA
    path (there is no host execution path)."""
    name: str
    kind: str = "cuda"
    affinity: str = ""
    devices: tuple = (0,)

    def __post_init__(self):
        if self.kind not in BACKEND_KINDS:
            raise SchedulerConfigError(f"unknown backend kind {self.kind!r}")
        if not self.affinity:
            object.__setattr__(self, "affinity", self.name)
        if not self.devices:
            raise SchedulerConfigError("backend needs at least one device")


CUDA_BACKEND = Backend("cuda")
# Reference names kept so reference-style configs resolve; both run on CUDA.
SCALAR_BACKEND = Backend("scalar", "scalar-reference")
BATCH_BACKEND = Backend("batch", "batch")


@dataclass(frozen=True)
class SchedulerParams:
    """scheduler.py:69-84. workers_per_backend is accepted for API
    compatibility; 0 still means inline (synchronous) execution order."""
    maxsize_bytes: int = DEFAULT_MAXSIZE
    workers_per_backend: int = 2
    backends: tuple = (CUDA_BACKEND,)
    affinity: dict = field(default_factory=lambda: {
        "disjoint": "cuda", "vertex": "cuda", "edge": "cuda", "identical": "cuda"})
    # this process's share when one job is split over processes (rank, world);
    # None = the whole job on this process's devices
    shard: tuple | None = None
    # leaf-aligned chunks per device whose D2H overlaps the next chunk's kernels
    chunks: int = 8
    # leaf-range stages of a single-device assembly whose packages are not
    # cached yet: stage k+1 is packaged on a host thread while stage k's
    # kernels and D2H run (1 = package everything first)
    stages: int = 6
    # symmetric evaluation: leaf (t, s) and its mirror (s, t) in the same plan
    # from one point evaluation per pair; False evaluates each
    # pair on its own (results then bitwise independent of how leaves are
    # split into stages / devices / shards)
    mirror: bool = True
    # symmetric download of a mirrored single layer: SKIP leaves (the
    # transposes of earlier PRIMARY leaves) are written on the host instead
    # of copied over PCIe (gcabem_plan_set_symmetric_download); the host
    # buffer is bitwise the device payload either way. None = when the link
    # bounds the call: a payload of at least SYM_AUTO_BYTES per operator (a
    # smaller call is bound by its host packaging, which the host-side
    # transposes would slow down: C2 53 -> 59 ms, C3 178 -> 163 ms)
    symmetric_download: bool | None = None

    def backend_for(self, case: str) -> Backend:
        wanted = self.affinity.get(case)
        for b in self.backends:
            if b.name == wanted:
                return b
        return self.backends[0]


@dataclass
class WorkBlock:
    """Disjoint-list item (scheduler.py:87-103)."""
    leaf_id: int
    row_panels: np.ndarray
    col_panels: np.ndarray
    row_slots: np.ndarray
    col_slots: np.ndarray
    flagged: bool

    @property
    def num_pairs(self) -> int:
        return len(self.row_panels) * len(self.col_panels)

    @property
    def nbytes(self) -> int:
        return self.num_pairs * BYTES_PER_PAIR


@dataclass(frozen=True)
class WorkItem:
    """Singular corrective item (scheduler.py:106-117)."""
    case: str
    tri_x: int
    tri_y: int
    leaf_id: int
    offset: int

    @property
    def nbytes(self) -> int:
        return BYTES_PER_PAIR


@dataclass
class WorkList:
    case: str
    items: list
    nbytes: int = 0
    state: str = "filling"
    seq: int = -1
    attempts: int = 0
    backend: str = ""
    t_enqueue: float = 0.0
    t_dequeue: float = 0.0
    t_done: float = 0.0

    @property
    def num_pairs(self) -> int:
        if self.case == "disjoint":
            return sum(b.num_pairs for b in self.items)
        return len(self.items)


@dataclass
class AssemblyStats:
    lists_executed: int = 0
    pairs_executed: int = 0
    block_pairs: int = 0
    corrective_items: int = 0
    events: list = field(default_factory=list)
    device_ms: dict = field(default_factory=dict)
    phase_s: dict = field(default_factory=dict)
    # staged assembly: per range (packaged, plan created, launched, synchronized), s from start
    stage_times: list = field(default_factory=list)
    # device -> host bytes of the call (both payloads of a pair call; a
    # symmetric download moves less than the payload)
    d2h_bytes: int = 0

    def event_rows(self):
        return list(self.events)


def split_block(block: WorkBlock, maxsize: int) -> list:
    """Halve the longer index dimension until each part fits (scheduler.py:153-175)."""
    if block.nbytes <= maxsize:
        return [block]
    if block.num_pairs <= 1:
        raise SchedulerConfigError(
            f"maxsize {maxsize} smaller than one pair record ({BYTES_PER_PAIR} B)")
    if len(block.row_panels) >= len(block.col_panels):
        h = len(block.row_panels) // 2
        halves = [replace(block, row_panels=block.row_panels[s], row_slots=block.row_slots[s])
                  for s in (slice(None, h), slice(h, None))]
    else:
        h = len(block.col_panels) // 2
        halves = [replace(block, col_panels=block.col_panels[s], col_slots=block.col_slots[s])
                  for s in (slice(None, h), slice(h, None))]
    return [p for half in halves for p in split_block(half, maxsize)]


class ListBuilder:
    """Byte-budgeted list accumulation (scheduler.py:178-208)."""

    def __init__(self, case: str, maxsize: int, sink):
        if maxsize < BYTES_PER_PAIR:
            raise SchedulerConfigError(
                f"maxsize {maxsize} smaller than one pair record ({BYTES_PER_PAIR} B)")
        self.case, self.maxsize, self.sink = case, maxsize, sink
        self.current = WorkList(case, [])

    def add_block(self, block: WorkBlock) -> None:
        for part in split_block(block, self.maxsize):
            self._add(part, part.nbytes)

    def add_item(self, item: WorkItem) -> None:
        self._add(item, item.nbytes)

    def _add(self, item, nbytes: int) -> None:
        if self.current.nbytes + nbytes > self.maxsize and self.current.items:
            self.flush()
        self.current.items.append(item)
        self.current.nbytes += nbytes

    def flush(self) -> None:
        if self.current.items:
            done, self.current = self.current, WorkList(self.case, [])
            done.state = "ready"
            self.sink(done)


def make_payloads(block_tree: BlockTree, row_ops, col_ops) -> dict:
    """Zeroed payloads per leaf (scheduler.py:411-422)."""
    out = {}
    for leaf in block_tree.leaves:
        if leaf.kind == "dense":
            shape = (block_tree.row_tree.nodes[leaf.row].size,
                     block_tree.col_tree.nodes[leaf.col].size)
        else:
            shape = (row_ops[leaf.row].rank, col_ops[leaf.col].rank)
        out[leaf.index] = np.zeros(shape, dtype=np.complex128)
    return out


def batch_quadrature(backend: Backend, case: str, mesh: SurfaceMesh, spec: KernelSpec,
                     rule: QuadRule4D, tri_x, tri_y, perms_x=None, perms_y=None) -> np.ndarray:
    """One case-homogeneous batch of pair integrals on the device
    (scheduler.py:235-261): charts gathered on device from (tri, perm)."""
    dm = device_mesh(mesh, backend.devices[0])
    tx, ty = nat.i64(tri_x), nat.i64(tri_y)
    n = tx.shape[0]
    out = np.empty(n, dtype=np.complex128)
    if n == 0:
        return out
    px = None if perms_x is None else nat.u8(perms_x)
    py = None if perms_y is None else nat.u8(perms_y)
    eq, layer = spec.code
    xs, ys, w = nat.f64(rule.x_points), nat.f64(rule.y_points), nat.f64(rule.weights)
    nat.check(nat.lib().gcabem_batch_quadrature(
        dm.handle, eq, layer, float(spec.kappa), n, nat.ptr(tx), nat.ptr(ty), nat.ptr(px),
        nat.ptr(py), w.shape[0], nat.ptr(xs), nat.ptr(ys), nat.ptr(w), nat.ptr(out)))
    return out


def execute_list(lst: WorkList, backend: Backend, mesh: SurfaceMesh, spec: KernelSpec,
                 orders, payloads: dict, on_corrective=None) -> None:
    """Run ONE list on the device and distribute (scheduler.py:368-395, :334-365).
    run_assembly does not go through here (it fuses all lists); this is the
    per-list API for callers that drive lists themselves."""
    lst.t_dequeue = time.monotonic()
    lst.attempts += 1
    if lst.items:
        if lst.case == "disjoint":
            tx = np.concatenate([np.repeat(b.row_panels, len(b.col_panels)) for b in lst.items])
            ty = np.concatenate([np.tile(b.col_panels, len(b.row_panels)) for b in lst.items])
            vals = batch_quadrature(backend, "disjoint", mesh, spec,
                                    build_rule("disjoint", orders[0]), tx, ty)
            pos = 0
            tri = mesh.triangles
            for blk in lst.items:
                nr, nc = len(blk.row_panels), len(blk.col_panels)
                P = payloads[blk.leaf_id]
                P[np.ix_(blk.row_slots, blk.col_slots)] = vals[pos:pos + nr * nc].reshape(nr, nc)
                pos += nr * nc
                if not blk.flagged:
                    continue
                ta, tb = tri[blk.row_panels], tri[blk.col_panels]
                shared = sum((ta[:, a][:, None] == tb[:, b][None, :]).astype(np.int8)
                             for a in range(3) for b in range(3))
                for a, b in np.argwhere(shared > 0):
                    item = WorkItem(_CASE_OF_SHARED[int(shared[a, b])], int(blk.row_panels[a]),
                                    int(blk.col_panels[b]), blk.leaf_id,
                                    int(blk.row_slots[a]) * P.shape[1] + int(blk.col_slots[b]))
                    if on_corrective is not None:
                        on_corrective(item)
        else:
            cls = [classify_pair(mesh, it.tri_x, it.tri_y) for it in lst.items]
            vals = batch_quadrature(
                backend, lst.case, mesh, spec, build_rule(lst.case, orders[1]),
                [it.tri_x for it in lst.items], [it.tri_y for it in lst.items],
                np.array([c.perm_x for c in cls]), np.array([c.perm_y for c in cls]))
            for it, v in zip(lst.items, vals):
                payloads[it.leaf_id].flat[it.offset] = v
    lst.state = "done"
    lst.t_done = time.monotonic()


# ---------------------------------------------------------------------------
# fused device execution

class DeviceLayout:
    """Packages of a leaf range uploaded to one device (C ABI gcabem_layout_*):
    block descriptors, tasks, panel indices, singular items. Shared by every
    operator assembled from the same packages; cached on the packages."""

    def __init__(self, dm: DeviceMesh, pk: AssemblyPackages, leaf_range=None,
                 mirror: bool = True):
        t0 = time.monotonic()
        lo, hi = leaf_range if leaf_range is not None else (0, pk.leaf_ids.size)
        self.leaf_range = (lo, hi)
        self.payload_offset = int(pk.leaf_base[lo])
        self.payload_len = int(pk.leaf_base[hi] - pk.leaf_base[lo])
        self.device = dm.device
        self._dm = dm
        h = ctypes.c_void_p()
        for arr in (pk.leaf_shape, pk.leaf_base, pk.leaf_rows_at, pk.leaf_cols_at, pk.panels,
                    pk.blk_leaf, pk.blk_r0, pk.blk_nr, pk.blk_c0, pk.blk_nc, pk.item_case,
                    pk.item_tri_x, pk.item_tri_y, pk.item_leaf, pk.item_offset, pk.perms):
            if not arr.flags.c_contiguous:
                raise ValueError("package arrays must be C-contiguous")
        p = nat.ptr
        nat.check(nat.lib().gcabem_layout_from_packages(
            dm.handle, lo, hi, pk.leaf_ids.size, p(pk.leaf_shape), p(pk.leaf_base),
            p(pk.leaf_rows_at), p(pk.leaf_cols_at), pk.panels.size, p(pk.panels),
            pk.blk_leaf.size, p(pk.blk_leaf), p(pk.blk_r0), p(pk.blk_nr), p(pk.blk_c0),
            p(pk.blk_nc), pk.item_case.size, p(pk.item_case), p(pk.item_tri_x),
            p(pk.item_tri_y), p(pk.item_leaf), p(pk.item_offset), p(pk.perms),
            p(pk.leaf_mirror) if (mirror and pk.leaf_mirror is not None) else None,
            ctypes.byref(h)))
        info = np.zeros(8, np.int64)
        nat.check(nat.lib().gcabem_layout_info(h, p(info)))
        mi = np.zeros(6, np.int64)
        nat.check(nat.lib().gcabem_layout_mirror_info(h, p(mi)))
        # disjoint-kernel evaluations: mirrored (a pair and its transpose) and
        # plain; 0/0 without mirrors (then every non-sharing pair is plain)
        self.mirror_info = {"evals_mirrored": int(mi[0]), "evals_plain": int(mi[1]),
                            "pairs_mirrored": int(mi[2]), "pairs_skipped": int(mi[3]),
                            "tasks_mirrored": int(mi[4]), "tasks_plain": int(mi[5])}
        self.disjoint_pairs = int(info[3])
        self.singular_counts = [int(x) for x in info[4:7]]
        self.h2d_bytes = int(info[7])
        self.prep_s = time.monotonic() - t0
        self.handle = h.value

    @staticmethod
    def cached(dm: DeviceMesh, pk: AssemblyPackages, leaf_range=None,
               mirror: bool = True) -> "DeviceLayout":
        lo, hi = leaf_range if leaf_range is not None else (0, pk.leaf_ids.size)
        key = ("layout", dm.device, id(dm), lo, hi, bool(mirror))
        lay = pk.extra.get(key)
        if lay is None:
            lay = DeviceLayout(dm, pk, (lo, hi), mirror)
            pk.extra[key] = lay
        return lay

    def close(self) -> None:
        h, self.handle = getattr(self, "handle", None), None
        if h and getattr(nat, "_lib", None) is not None:  # nat is None at interpreter teardown
            nat._lib.gcabem_layout_release(h)

    def __del__(self):
        self.close()


class AssemblyPlan:
    """Device plan of one operator on one device: a (shared, cached) device
    layout of the packages plus this operator's payload, executable
    repeatedly (C ABI gcabem_plan_*). Payload stays in HBM until download().

    pair=True: BOTH layers of spec's equation in one fused plan (every kernel
    evaluates r, 1/r and the phase once per point for the single and the
    double layer; C ABI gcabem_plan_create_pair); download2() / the pair
    execute_download() fill two host buffers."""

    def __init__(self, dm: DeviceMesh, spec: KernelSpec, pk: AssemblyPackages, orders,
                 leaf_range=None, pair: bool = False, mirror: bool = True,
                 symmetric_download: bool = True):
        t_prep = time.monotonic()
        self.layout = DeviceLayout.cached(dm, pk, leaf_range, mirror)
        lay = self.layout
        self.leaf_range = lay.leaf_range
        self.payload_offset = lay.payload_offset
        self.payload_len = lay.payload_len
        self.disjoint_pairs = lay.disjoint_pairs
        self.singular_counts = lay.singular_counts
        dn, sn = orders
        g = gauss_legendre(dn)
        gp, gw = nat.f64(g.points), nat.f64(g.weights)
        rules = [build_rule(c, sn).packed() for c in SINGULAR_CASES]
        self.singular_q = [r.shape[0] for r in rules]
        sq = np.array(self.singular_q, dtype=np.int64)
        rptr = (ctypes.c_void_p * 3)(*[r.ctypes.data for r in rules])
        eq, layer = spec.code
        self.spec, self.orders, self.device = spec, tuple(orders), dm.device
        self._dm = dm
        self.h2d_bytes = lay.h2d_bytes + int(sum(r.nbytes for r in rules))
        self.prep_s = time.monotonic() - t_prep
        self.pair = bool(pair)
        h = ctypes.c_void_p()
        if self.pair:
            nat.check(nat.lib().gcabem_plan_create_pair(
                lay.handle, eq, float(spec.kappa), dn, nat.ptr(gp), nat.ptr(gw), nat.ptr(sq),
                ctypes.cast(rptr, ctypes.c_void_p), ctypes.byref(h)))
        else:
            nat.check(nat.lib().gcabem_plan_create_on(
                lay.handle, eq, layer, float(spec.kappa), dn, nat.ptr(gp), nat.ptr(gw),
                nat.ptr(sq), ctypes.cast(rptr, ctypes.c_void_p), ctypes.byref(h)))
        self.handle = h.value
        self._keep = rules
        m = ctypes.c_int()
        nat.check(nat.lib().gcabem_plan_mirrored(self.handle, ctypes.byref(m)))
        self.mirrored = bool(m.value)
        nat.check(nat.lib().gcabem_plan_set_symmetric_download(self.handle,
                                                               int(bool(symmetric_download))))

    def d2h_bytes(self) -> int:
        """Bytes the last execute_download moved device -> host (a symmetric
        download skips the SKIP leaves of the single layer)."""
        v = ctypes.c_int64()
        nat.check(nat.lib().gcabem_plan_d2h_bytes(self.handle, ctypes.byref(v)))
        return int(v.value)

    def launches_per_execute(self) -> int:
        """Kernel launches of one execute(): the disjoint launch(es) -- plain
        and mirrored when both kinds of blocks exist -- and one fused launch
        for all singular lists (vertex mirrored / alone, edge, identical)."""
        ev = np.zeros(5, np.int64)
        nat.check(nat.lib().gcabem_plan_singular_evals(self.handle, nat.ptr(ev)))
        ev = ev[:4]
        if self.mirrored:
            mi = self.layout.mirror_info
            dis = int(mi["tasks_plain"] > 0) + int(mi["tasks_mirrored"] > 0)
        else:
            dis = int(self.disjoint_pairs > 0)
        return dis + int(np.count_nonzero(ev) > 0)

    def execute(self) -> None:
        nat.check(nat.lib().gcabem_plan_execute(self.handle))

    def synchronize(self) -> None:
        nat.check(nat.lib().gcabem_plan_synchronize(self.handle))

    def set_stream(self, stream_handle: int | None) -> None:
        """Run on an external cudaStream_t (e.g. torch.cuda.Stream.cuda_stream)."""
        nat.check(nat.lib().gcabem_plan_set_stream(self.handle, stream_handle or None))

    def execute_download(self, out: np.ndarray, nchunks: int = 8,
                         out2: np.ndarray | None = None) -> None:
        """Execute and stream the payload into `out` chunk by chunk (D2H of
        chunk k overlaps the kernels of chunk k+1); a pair plan also streams
        the double layer into `out2`. Asynchronous: call synchronize()
        before reading the targets."""
        self._check_target(out)
        if self.pair:
            self._check_target(out2)
            nat.check(nat.lib().gcabem_plan_execute_download2(self.handle, nat.ptr(out),
                                                              nat.ptr(out2), int(nchunks)))
        else:
            nat.check(nat.lib().gcabem_plan_execute_download(self.handle, nat.ptr(out),
                                                             int(nchunks)))
        self._pinned_target = (out, out2)  # keep alive until synchronize

    def _check_target(self, out) -> None:
        if out is None or out.dtype != np.complex128 or out.size != self.payload_len or \
                not out.flags.c_contiguous:
            raise ValueError("download target must be contiguous complex128 of payload_len")

    def download(self, out: np.ndarray, out2: np.ndarray | None = None) -> None:
        """Copy the payload into `out` (complex128, payload_len, ideally
        pinned); a pair plan's double layer into `out2`."""
        self._check_target(out)
        if self.pair:
            self._check_target(out2)
        nat.check(nat.lib().gcabem_plan_download2(self.handle, nat.ptr(out), nat.ptr(out2)))

    def timing_ms(self) -> dict:
        ms = (ctypes.c_float * 3)()
        nat.check(nat.lib().gcabem_plan_timing(self.handle, ms))
        return {"disjoint": ms[0], "singular": ms[1], "total": ms[2]}

    def flops(self) -> dict:
        """Algorithmic FP64 flops of one execute (SURVEY §8(d) convention). The
        disjoint launch skips the pairs that share a vertex (it writes 0 and the
        singular pass overwrites them), so they are not credited to it."""
        from .roofline import mirror_pair_flops, pair_flops
        dq = self.orders[0] ** 4
        if self.mirrored:
            mi = self.layout.mirror_info
            dis = pair_flops(self.spec, "disjoint", dq, self.pair) * mi["evals_plain"] + \
                mirror_pair_flops(self.spec, dq, self.pair) * mi["evals_mirrored"]
        else:
            computed = self.disjoint_pairs - sum(self.singular_counts)
            dis = pair_flops(self.spec, "disjoint", dq, self.pair) * computed
        ev = np.zeros(5, np.int64)
        nat.check(nat.lib().gcabem_plan_singular_evals(self.handle, nat.ptr(ev)))
        # identical items: the points actually evaluated (the base half of a
        # symmetric rule: the minimal algorithm's work)
        qs = [self.singular_q[0], self.singular_q[1], int(ev[4])]
        sing = sum(pair_flops(self.spec, "singular", q, self.pair) * int(n)
                   for q, n in zip(qs, ev[1:4]))
        # vertex items evaluated with their transpose (symmetric vertex rule)
        sing += mirror_pair_flops(self.spec, self.singular_q[0], self.pair, "singular") * \
            int(ev[0])
        return {"disjoint": dis, "singular": sing}

    def close(self) -> None:
        h, self.handle = getattr(self, "handle", None), None
        if h and getattr(nat, "_lib", None) is not None:  # nat is None at interpreter teardown
            nat._lib.gcabem_plan_destroy(h)

    def __del__(self):
        self.close()


def _events(pk: AssemblyPackages, backend: str, t0: float, t1: float) -> list:
    """One row per executed list (scheduler.py:303-315), in inline order."""
    rows = []
    npairs = pk.blk_nr * pk.blk_nc
    per_list = np.bincount(pk.blk_list, weights=npairs, minlength=pk.n_disjoint_lists)
    nblk = np.bincount(pk.blk_list, minlength=pk.n_disjoint_lists)
    for k in range(pk.n_disjoint_lists):
        p = int(per_list[k])
        rows.append({"case": "disjoint", "items": int(nblk[k]), "pairs": p,
                     "bytes": p * BYTES_PER_PAIR, "backend": backend, "enqueue": t0,
                     "dequeue": t0, "done": t1})
    for case, ranges in pk.singular_lists().items():
        for a, b in ranges:
            rows.append({"case": case, "items": b - a, "pairs": b - a,
                         "bytes": (b - a) * BYTES_PER_PAIR, "backend": backend,
                         "enqueue": t0, "dequeue": t0, "done": t1})
    return rows


_pk_cache: dict = {}
_pk_lock = threading.Lock()
# entries kept per (kind, block tree): a new operator set on the same trees
# (e.g. a kappa sweep through assemble_operator(trees=bt)) replaces the old
# entry instead of accumulating packages and device layouts
_PK_PER_TREE = 1


def clear_package_cache() -> None:
    with _pk_lock:
        _pk_cache.clear()


def _cache_get(key, block_tree):
    with _pk_lock:
        hit = _pk_cache.get(key)
    return hit[3] if hit is not None and hit[0]() is block_tree else None


def _cache_put(key, block_tree, row_ops, col_ops, value) -> None:
    """Insert, evicting older entries of the same kind on the same block tree
    (their packages and device layouts are released with the last reference)."""
    kind = key[0]
    with _pk_lock:
        same = [k for k in _pk_cache if k[0] == kind and k[1] == key[1] and k != key]
        for k in same[:max(0, len(same) - _PK_PER_TREE + 1)]:
            _pk_cache.pop(k, None)
        _pk_cache[key] = (weakref.ref(block_tree), row_ops, col_ops, value)
    weakref.finalize(block_tree, lambda k=key: _pk_cache.pop(k, None))


def _cache_drop(key, value) -> None:
    with _pk_lock:
        hit = _pk_cache.get(key)
        if hit is not None and hit[3] is value:
            del _pk_cache[key]


def _pk_key(mesh, block_tree, row_ops, col_ops, maxsize):
    return ("packages", id(block_tree), id(row_ops), id(col_ops), int(maxsize),
            id(mesh.triangles))


def packages_for(mesh: SurfaceMesh, block_tree: BlockTree, row_ops, col_ops,
                 maxsize: int) -> AssemblyPackages:
    """Work packages of (block tree, operators, budget), cached: packages do
    not depend on the kernel or the orders, so the DLP assembly reuses the
    SLP's (as the reference pipeline reuses trees and operators,
    solver.py:280-282). The cache holds the operator dicts, so their ids
    stay valid while an entry lives; one entry per block tree (a new operator
    set replaces it), entries die with the block tree."""
    key = _pk_key(mesh, block_tree, row_ops, col_ops, maxsize)
    hit = _cache_get(key, block_tree)
    if hit is not None:
        return hit
    pk = make_packages(mesh.triangles, block_tree, row_ops, col_ops, maxsize)
    _cache_put(key, block_tree, row_ops, col_ops, pk)
    return pk


class StagedPackages:
    """Packages of contiguous leaf ranges, built one range after the other on
    a host thread (make_packages(leaf_range=...)) so that the device can work
    on range k while range k+1 is packaged. Each range's packages are exactly
    the whole-tree packages restricted to its leaves (payload offsets relative
    to the range's first leaf).

    leaf_set: only those leaves (sorted preorder positions: this process's
    shard of a job split over processes, SchedulerParams.shard); the ranges
    cut the set, and leaf_ids / leaf_shape / leaf_base / payload_len /
    offset() describe the set's payload, its leaves back to back."""

    def __init__(self, mesh: SurfaceMesh, block_tree: BlockTree, row_ops, col_ops,
                 maxsize: int, nstages: int, leaf_set=None, inputs=None, prepare=None):
        inputs = inputs or package_inputs(mesh.triangles, block_tree, row_ops, col_ops)
        L_all = inputs.leaves.shape[0]
        sel = np.arange(L_all, dtype=np.int64) if leaf_set is None else \
            np.asarray(leaf_set, dtype=np.int64)
        if sel.size and (sel[0] < 0 or sel[-1] >= L_all or np.any(np.diff(sel) <= 0)):
            raise SchedulerConfigError("leaf set must be sorted positions of the block tree")
        contiguous = sel.size == 0 or sel[-1] - sel[0] + 1 == sel.size
        self.leaf_set = sel
        L = sel.size
        n = max(1, min(int(nstages), max(L, 1)))
        # range 0 = the first L/64 leaves, packaged at once (before the layout
        # is known: the device and the PCIe link start within milliseconds);
        # the rest is cut leaf-aligned into ranges growing geometrically
        # (payload weights 1, g, g^2, ... with g = STAGE_GROWTH), each packaged
        # while the (longer) D2H of all earlier ranges runs. Ranges index the set.
        first = L if n == 1 else max(1, L // STAGE_FIRST)
        self.ranges = [(0, first)]
        # allocated once at the maximum stage count and never replaced: the
        # worker thread stores into them while the ranges are still being cut
        self._pk = [None] * n
        self._ready = [threading.Event() for _ in range(n)]
        self._layout = threading.Event()
        self._err = None
        self.key = None
        args = (mesh.triangles, block_tree, row_ops, col_ops, int(maxsize))

        def package(a, b):
            if contiguous:
                return make_packages(*args, leaf_range=(int(sel[0]) + a, int(sel[0]) + b),
                                     inputs=inputs)
            return make_packages(*args, leaf_index=sel[a:b], inputs=inputs)

        def one(k):
            pk = package(*self.ranges[k])
            if prepare is not None:   # e.g. the device layout of the range
                prepare(k, pk)
            self._pk[k] = pk
            self._ready[k].set()

        nw = max(1, PACK_WORKERS)

        claim = iter(range(1, 1 << 62))   # next range to package (under the lock)
        claim_lock = threading.Lock()

        def work(w):
            # worker 0 packages range 0 at once; ranges 1, 2, ... go in order
            # to whichever worker is free, once the cuts are known
            try:
                if w == 0:
                    one(0)
                self._layout.wait()
                while True:
                    with claim_lock:
                        k = next(claim)
                    if k >= len(self.ranges):
                        return
                    one(k)
            except BaseException as exc:  # re-raised by stage()
                self._err = exc
                for ev in self._ready:
                    ev.set()
        self._threads = [threading.Thread(target=work, args=(w,), name=f"gcabem-packaging-{w}",
                                          daemon=True) for w in range(nw)]
        for t in self._threads:
            t.start()
        try:
            ids, shape, full_base = leaf_layout(block_tree, row_ops, col_ops, inputs)
            if leaf_set is None:   # the whole tree: the layout as it is
                self.leaf_ids, self.leaf_shape, base = ids, shape, full_base
            else:
                self.leaf_ids = ids[sel]
                self.leaf_shape = shape[sel]
                base = np.zeros(L + 1, np.int64)
                np.cumsum(self.leaf_shape[:, 0] * self.leaf_shape[:, 1], out=base[1:])
            self.leaf_base = base
            self.payload_len = int(base[-1])
            ranges = list(self.ranges)
            if first < L:
                b0 = base[first]
                k = np.arange(n - 1)
                peak = max(0, n - 2 - STAGE_TAPER)
                w = STAGE_GROWTH ** np.minimum(k, peak) * 0.5 ** np.maximum(0, k - peak)
                frac = np.cumsum(w)[:-1] / w.sum()
                cuts = np.searchsorted(base, b0 + (base[L] - b0) * frac, side="left")
                edges = np.unique(np.concatenate([[first], np.clip(cuts, first + 1, L), [L]]))
                ranges += [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:])]
            self.ranges = ranges
        finally:
            self._layout.set()

    def chunks(self, k: int, total: int) -> int:
        """D2H chunks of range k: about `total` over all ranges, by size."""
        lo, hi = self.ranges[k]
        share = (self.leaf_base[hi] - self.leaf_base[lo]) / max(self.payload_len, 1)
        return max(2, int(round(total * share)))

    def stage(self, k: int) -> AssemblyPackages:
        self._ready[k].wait()
        pk = self._pk[k]
        if pk is None:
            if self.key is not None:  # a failed packaging is not served again
                _cache_drop(self.key, self)
            if self._err is not None:
                raise self._err
            raise RuntimeError(f"packaging thread produced no packages for stage {k}")
        return pk

    def offset(self, k: int) -> int:
        """Payload offset of range k in the set's payload."""
        return int(self.leaf_base[self.ranges[k][0]])


def shard_leaves_of(mesh: SurfaceMesh, block_tree: BlockTree, row_ops, col_ops, shard,
                    disjoint_q: int, inputs=None) -> np.ndarray:
    """This process's leaves (sorted preorder positions) of a job split over
    processes: packaging.shard_leaf_set (each leaf with its mirror, the
    leaf pairs cut into contiguous runs balanced by disjoint-rule points)."""
    inputs = inputs or package_inputs(mesh.triangles, block_tree, row_ops, col_ops)
    return shard_leaf_set(block_tree, row_ops, col_ops, shard, disjoint_q, inputs)


def staged_packages_for(mesh: SurfaceMesh, block_tree: BlockTree, row_ops, col_ops,
                        maxsize: int, nstages: int, leaf_set=None,
                        inputs=None, prepare=None) -> StagedPackages:
    """StagedPackages of (block tree, operators, budget, stages[, leaf set]),
    cached like packages_for (a second operator from the same packages
    packages nothing). `prepare(k, packages)` runs on the packaging thread
    after range k is packaged (a new StagedPackages only)."""
    key = ("staged", id(block_tree), id(row_ops), id(col_ops), int(maxsize),
           id(mesh.triangles), int(nstages),
           None if leaf_set is None else (int(leaf_set.size), hash(leaf_set.tobytes())))
    hit = _cache_get(key, block_tree)
    if hit is not None:
        return hit
    sp = StagedPackages(mesh, block_tree, row_ops, col_ops, maxsize, nstages, leaf_set, inputs,
                        prepare)
    sp.key = key
    _cache_put(key, block_tree, row_ops, col_ops, sp)
    return sp


def _cached_packages(mesh, block_tree, row_ops, col_ops, maxsize):
    return _cache_get(_pk_key(mesh, block_tree, row_ops, col_ops, maxsize), block_tree)


def _matrices(block_tree, row_ops, col_ops, bufs, leaf_ids, leaf_base, leaf_shape, leaf_set,
              nleaves):
    part = None if leaf_set is None or leaf_set.size == nleaves else leaf_set
    return tuple(GCAMatrix(block_tree, row_ops, col_ops,
                           LeafPayloads(buf, leaf_ids, leaf_base, leaf_shape), buffer=buf,
                           shard_leaves=part) for buf in bufs)


def _assemble_staged(mesh, block_tree, spec, pair, row_ops, col_ops, params, orders, stats,
                     device, leaf_set=None, inputs=None):
    """Single-device assembly over StagedPackages: plan k is created and
    launched (kernels + chunked D2H on its own streams) as soon as range k is
    packaged, so packaging and layout upload of later ranges overlap the
    device work and the D2H of earlier ones. The payloads are bitwise those
    of the unstaged path; AssemblyStats list counts/events are per range (each
    range's lists are cut from its own first leaf), so lists_executed depends
    on the stage count (pairs_executed does not). `leaf_set`: only those
    leaves (a process shard)."""
    t0 = time.monotonic()
    phase = {}
    dm = device_mesh(mesh, device)
    mirror = params.mirror
    # the packaging threads also build each range's device layout
    sp = staged_packages_for(mesh, block_tree, row_ops, col_ops, params.maxsize_bytes,
                             params.stages, leaf_set, inputs,
                             lambda k, pk: DeviceLayout.cached(dm, pk, None, mirror))
    ta = time.monotonic()
    outs = [nat.pinned_empty(sp.payload_len, np.complex128) for _ in range(2 if pair else 1)]
    phase["pinned_alloc"] = time.monotonic() - ta
    plans, wait = [], 0.0
    try:
        ta = time.monotonic()
        times = []
        for k in range(len(sp.ranges)):
            tw = time.monotonic()
            pk = sp.stage(k)
            tr = time.monotonic()
            wait += tr - tw
            p = AssemblyPlan(dm, spec, pk, orders, pair=pair, mirror=params.mirror,
                             symmetric_download=_symmetric(params, sp.payload_len))
            plans.append(p)
            tp = time.monotonic()
            if os.environ.get("GCABEM_TRACE"):
                print(f"[stage {k}] layout {p.layout.prep_s * 1e3:.2f} ms, plan "
                      f"{(tp - tr) * 1e3:.2f} ms", file=sys.stderr)
            if p.payload_len:
                sl = slice(sp.offset(k), sp.offset(k) + p.payload_len)
                p.execute_download(outs[0][sl], sp.chunks(k, 2 * params.chunks),
                                   outs[1][sl] if pair else None)
            times.append([tr - t0, tp - t0, time.monotonic() - t0])
        phase["packaging_wait"] = wait
        phase["plans_launched"] = time.monotonic() - ta
        for p, tk in zip(plans, times):
            p.synchronize()
            tk.append(time.monotonic() - t0)
            stats.d2h_bytes += p.d2h_bytes() if p.payload_len else 0
        stats.stage_times = [tuple(round(x, 4) for x in tk) for tk in times]
        phase["execute_download"] = time.monotonic() - ta
        ms = [p.timing_ms() for p in plans if p.payload_len]
        stats.device_ms = {f"device{device}": {key: sum(m[key] for m in ms)
                                               for key in ("disjoint", "singular", "total")}}
    finally:
        ta = time.monotonic()
        for p in plans:
            p.close()
        phase["plan_destroy"] = time.monotonic() - ta
    t1 = time.monotonic()
    mult = 2 if pair else 1
    ev = []
    for k in range(len(sp.ranges)):
        pk = sp.stage(k)
        stats.block_pairs += mult * pk.block_pairs()
        stats.corrective_items += mult * pk.num_items
        ev += _events(pk, params.backend_for("disjoint").name, t0, t1)
    stats.events.extend(ev * mult)
    stats.lists_executed += mult * len(ev)
    stats.pairs_executed += mult * sum(r["pairs"] for r in ev)
    phase["total"] = time.monotonic() - t0
    stats.phase_s = phase
    nleaves = len(block_tree.leaves)
    return _matrices(block_tree, row_ops, col_ops, outs, sp.leaf_ids, sp.leaf_base,
                     sp.leaf_shape, sp.leaf_set, nleaves)


def _use_staged(mesh, block_tree, row_ops, col_ops, params) -> bool:
    devices = params.backend_for("disjoint").devices
    return (params.stages > 1 and len(devices) == 1 and
            _cached_packages(mesh, block_tree, row_ops, col_ops, params.maxsize_bytes) is None)


def _assemble(mesh, block_tree, spec, pair, row_ops, col_ops, params, orders, stats):
    """run_assembly / run_assembly_pair. Leaves are split into contiguous
    ranges, one per device of the backend; with params.shard = (rank, world)
    this process assembles only its leaf set (packaging.shard_leaf_set: each
    leaf with its mirror) and the returned matrices hold only those leaves
    (GCAMatrix.shard_leaves)."""
    params = params or SchedulerParams()
    stats = stats if stats is not None else AssemblyStats()
    if not params.backends:
        raise SchedulerConfigError("at least one backend required")
    backend = params.backend_for("disjoint")
    leaf_set = None
    inputs = None
    if params.shard is not None:
        inputs = package_inputs(mesh.triangles, block_tree, row_ops, col_ops)
        leaf_set = shard_leaves_of(mesh, block_tree, row_ops, col_ops, params.shard,
                                   orders[0] ** 4, inputs)
    if _use_staged(mesh, block_tree, row_ops, col_ops, params):
        return _assemble_staged(mesh, block_tree, spec, pair, row_ops, col_ops, params, orders,
                                stats, backend.devices[0], leaf_set, inputs)
    t0 = time.monotonic()
    phase = {}
    if leaf_set is None:
        pk = packages_for(mesh, block_tree, row_ops, col_ops, params.maxsize_bytes)
    else:   # this process's leaves only
        pk = make_packages(mesh.triangles, block_tree, row_ops, col_ops, params.maxsize_bytes,
                           leaf_index=leaf_set, inputs=inputs)
    phase["packaging"] = time.monotonic() - t0
    devices = list(backend.devices)
    sq = [build_rule(c, orders[1]).num_points for c in SINGULAR_CASES]
    ranges = shard_leaves(pk, len(devices), orders[0] ** 4, sq)
    ta = time.monotonic()
    outs = [nat.pinned_empty(pk.payload_len, np.complex128) for _ in range(2 if pair else 1)]
    phase["pinned_alloc"] = time.monotonic() - ta
    plans = []
    try:
        ta = time.monotonic()
        for dev, rng in zip(devices, ranges):
            plans.append(AssemblyPlan(device_mesh(mesh, dev), spec, pk, orders, rng, pair=pair,
                                      mirror=params.mirror,
                                      symmetric_download=_symmetric(params, pk.payload_len)))
        phase["plan_create"] = time.monotonic() - ta
        phase["plan_host_prep"] = sum(p.prep_s for p in plans)
        ta = time.monotonic()
        for p in plans:
            if p.payload_len:
                sl = slice(p.payload_offset, p.payload_offset + p.payload_len)
                p.execute_download(outs[0][sl], params.chunks, outs[1][sl] if pair else None)
        for p in plans:
            p.synchronize()
            stats.d2h_bytes += p.d2h_bytes() if p.payload_len else 0
        phase["execute_download"] = time.monotonic() - ta
        stats.device_ms = {f"device{p.device}": p.timing_ms() for p in plans if p.payload_len}
    finally:
        ta = time.monotonic()
        for p in plans:
            p.close()
        phase["plan_destroy"] = time.monotonic() - ta
    t1 = time.monotonic()
    stats.phase_s = phase
    mult = 2 if pair else 1
    stats.block_pairs += mult * pk.block_pairs()
    stats.corrective_items += mult * pk.num_items
    ev = _events(pk, backend.name, t0, t1)
    stats.events.extend(ev * mult)
    stats.lists_executed += mult * len(ev)
    stats.pairs_executed += mult * sum(r["pairs"] for r in ev)
    phase["total"] = time.monotonic() - t0
    return _matrices(block_tree, row_ops, col_ops, outs, pk.leaf_ids, pk.leaf_base,
                     pk.leaf_shape, leaf_set, len(block_tree.leaves))


def run_assembly(mesh: SurfaceMesh, block_tree: BlockTree, spec: KernelSpec,
                 row_ops: dict, col_ops: dict, params: SchedulerParams | None = None,
                 orders: tuple = (3, 5), stats: AssemblyStats | None = None) -> GCAMatrix:
    """Assemble the compressed operator (scheduler.py:442-505) on the device(s).

    Leaves are split into contiguous ranges, one per device of the backend;
    each device streams its payload range into one pinned host buffer while
    it computes. With params.shard = (rank, world) (one job split over
    processes) only this process's leaf set is assembled and returned."""
    return _assemble(mesh, block_tree, spec, False, row_ops, col_ops, params, orders, stats)[0]


def run_assembly_pair(mesh: SurfaceMesh, block_tree: BlockTree, equation: str, kappa: float,
                      row_ops: dict, col_ops: dict, params: SchedulerParams | None = None,
                      orders: tuple = (3, 5), stats: AssemblyStats | None = None):
    """The single- and the double-layer operator of one equation, assembled
    together: (GCAMatrix SLP, GCAMatrix DLP), each identical in layout and
    within roundoff in value to run_assembly() of that layer. One fused device
    pass evaluates the distance, its inverse and the Helmholtz phase once per
    quadrature point for both operators (the pipelines that need V and K,
    reference solver.py:279-282, reuse trees and operators the same way)."""
    return _assemble(mesh, block_tree, KernelSpec(equation, "single", kappa), True, row_ops,
                     col_ops, params, orders, stats)


def _split_range(pk, rng, n, dq, sq):
    """Relative sub-ranges of a leaf range for n devices, balanced by pairs."""
    lo, hi = rng
    if n <= 1:
        return [(0, hi - lo)]
    w = (pk.leaf_shape[lo:hi, 0] * pk.leaf_shape[lo:hi, 1]).astype(np.float64)
    cum = np.cumsum(w)
    cuts = np.searchsorted(cum, cum[-1] * np.arange(1, n) / n, side="left") + 1
    edges = np.maximum.accumulate(np.concatenate([[0], np.minimum(cuts, hi - lo), [hi - lo]]))
    return [(int(edges[k]), int(edges[k + 1])) for k in range(n)]


def potential_batch(mesh: SurfaceMesh, spec: KernelSpec, points: np.ndarray,
                    order: int = 3, device: int | None = None) -> np.ndarray:
    """Per-panel potentials at off-surface points (scheduler.py:508-534), on
    the device: each point is a zero-extent target panel whose Gramian 2
    cancels the reference-triangle area of the x half; returns the
    (npoints, npanels) matrix of plain panel integrals of the kernel field."""
    from .pairquad import default_device
    points = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    dev = default_device() if device is None else device
    dm = device_mesh(mesh, dev)
    g = gauss_legendre(order)
    gp, gw = nat.f64(g.points), nat.f64(g.weights)
    out = np.empty((points.shape[0], mesh.num_triangles), dtype=np.complex128)
    eq, layer = spec.code
    nat.check(nat.lib().gcabem_potential(dm.handle, eq, layer, float(spec.kappa), int(order),
                                         nat.ptr(gp), nat.ptr(gw), points.shape[0],
                                         nat.ptr(points), nat.ptr(out)))
    bad = ~np.all(np.isfinite(out), axis=1)
    if np.any(bad):
        raise ValueError(f"evaluation point {int(np.flatnonzero(bad)[0])} lies on the surface")
    return out
