"""ctypes binding of the in-tree C-ABI library libgcabem_b200.so.

The library is the only compute path: there is no CPU fallback. If it is
missing or no CUDA device is visible, every GPU-backed call raises
BackendError (reference scheduler.py:47 BackendError).
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# GCABEM_LIB_PATH: load a variant build (occupancy / flag experiments)
LIB_PATH = os.environ.get("GCABEM_LIB_PATH") or os.path.join(HERE, "libgcabem_b200.so")

ERR_ARG, ERR_CUDA, ERR_NODEV, ERR_GCA = 1, 2, 3, 4


class BackendError(RuntimeError):
    """Device/back-end failure (reference scheduler.py:47)."""


_lib = None
_lock = threading.Lock()

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_int = ctypes.c_int
_dbl = ctypes.c_double

_SIGS = {
    "gcabem_version": ([], _int),
    "gcabem_last_error": ([], ctypes.c_char_p),
    "gcabem_device_count": ([ctypes.POINTER(_int)], _int),
    "gcabem_device_info": ([_int, ctypes.c_char_p, ctypes.POINTER(_int), ctypes.POINTER(_int)],
                           _int),
    "gcabem_host_alloc": ([_i64, ctypes.POINTER(_vp)], _int),
    "gcabem_host_free": ([_vp], _int),
    "gcabem_release_cached": ([_int], _int),
    "gcabem_pair_values": ([_int, _int, _int, _dbl, _i64] + [_vp] * 9 + [_i64] + [_vp] * 4, _int),
    "gcabem_mesh_create": ([_int, _i64, _vp, _i64, _vp, _vp, _vp, ctypes.POINTER(_vp)], _int),
    "gcabem_mesh_destroy": ([_vp], _int),
    "gcabem_batch_quadrature": ([_vp, _int, _int, _dbl, _i64, _vp, _vp, _vp, _vp, _i64,
                                 _vp, _vp, _vp, _vp], _int),
    "gcabem_plan_create": ([_vp, _int, _int, _dbl, _int, _vp, _vp, _i64, _i64, _vp, _i64, _vp,
                            _i64, _vp, _vp, _vp, _vp, ctypes.POINTER(_vp)], _int),
    "gcabem_plan_execute": ([_vp], _int),
    "gcabem_layout_create": ([_vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _vp,
                              ctypes.POINTER(_vp)], _int),
    "gcabem_layout_release": ([_vp], _int),
    "gcabem_layout_info": ([_vp, _vp], _int),
    "gcabem_layout_from_packages": ([_vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _i64]
                                    + [_vp] * 5 + [_i64] + [_vp] * 7 + [ctypes.POINTER(_vp)],
                                    _int),
    "gcabem_layout_mirror_info": ([_vp, _vp], _int),
    "gcabem_plan_set_mirror": ([_vp, _int], _int),
    "gcabem_plan_singular_evals": ([_vp, _vp], _int),
    "gcabem_plan_mirrored": ([_vp, ctypes.POINTER(_int)], _int),
    "gcabem_plan_create_on": ([_vp, _int, _int, _dbl, _int, _vp, _vp, _vp, _vp,
                               ctypes.POINTER(_vp)], _int),
    "gcabem_plan_download": ([_vp, _vp], _int),
    "gcabem_plan_download2": ([_vp, _vp, _vp], _int),
    "gcabem_plan_create_pair": ([_vp, _int, _dbl, _int, _vp, _vp, _vp, _vp, ctypes.POINTER(_vp)],
                                _int),
    "gcabem_plan_execute_download2": ([_vp, _vp, _vp, _int], _int),
    "gcabem_plan_execute_download": ([_vp, _vp, _int], _int),
    "gcabem_plan_synchronize": ([_vp], _int),
    "gcabem_plan_set_symmetric_download": ([_vp, _int], _int),
    "gcabem_plan_d2h_bytes": ([_vp, ctypes.POINTER(_i64)], _int),
    "gcabem_plan_timing": ([_vp, _vp], _int),
    "gcabem_plan_payload": ([_vp, ctypes.POINTER(_vp)], _int),
    "gcabem_plan_set_stream": ([_vp, _vp], _int),
    "gcabem_plan_destroy": ([_vp], _int),
    "gcabem_green_matrices": ([_vp, _int, _dbl, _i64, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _i64,
                               _vp], _int),
    "gcabem_fp64_probe": ([_int, ctypes.POINTER(_dbl)], _int),
    "gcabem_potential": ([_vp, _int, _int, _dbl, _int, _vp, _vp, _i64, _vp, _vp], _int),
    "gcabem_packages_build": ([_i64, _vp, _i64, _vp, _i64] + [_vp] * 7 + [_i64] + [_vp] * 7
                              + [_i64, _int, ctypes.POINTER(_vp)], _int),
    "gcabem_packages_build_on": ([_i64, _vp, _i64, _vp, _i64] + [_vp] * 7 + [_i64] + [_vp] * 7
                                 + [_i64, _int, _vp, _i64, ctypes.POINTER(_vp)], _int),
    "gcabem_packages_sizes": ([_vp, _vp], _int),
    "gcabem_packages_fetch": ([_vp] * 11, _int),
    "gcabem_packages_free": ([_vp], _int),
    "gcabem_leaf_layout": ([_i64, _vp, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _vp], _int),
    "gcabem_cluster_tree_mesh": ([_i64, _vp, _vp, _i64, ctypes.POINTER(_vp)], _int),
    "gcabem_cluster_tree": ([_i64, _vp, _vp, _vp, _i64, ctypes.POINTER(_vp)], _int),
    "gcabem_block_tree": ([_i64] + [_vp] * 5 + [_i64] + [_vp] * 5 + [_dbl, _int,
                                                                     ctypes.POINTER(_vp)], _int),
    "gcabem_norm3": ([_i64, _vp, _int, _vp], _int),
    "gcabem_tree_sizes": ([_vp, _vp], _int),
    "gcabem_tree_fetch": ([_vp] * 9, _int),
    "gcabem_tree_free": ([_vp], _int),
    "gcabem_gca_build": ([_vp, _int, _dbl, _i64] + [_vp] * 5 + [_i64, _vp, _dbl, _int, _vp, _vp,
                                                     _dbl, _i64, _vp, _dbl, _int, _i64,
                                                     ctypes.POINTER(_vp)], _int),
    "gcabem_gca_sizes": ([_vp, _vp, _vp], _int),
    "gcabem_gca_fetch": ([_vp, _vp, _vp], _int),
    "gcabem_gca_flags": ([_vp, _vp], _int),
    "gcabem_green_exact": ([_int, _dbl, _i64, _vp, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _dbl,
                            _int, _vp, _vp, _dbl, _i64, _vp, _dbl, _vp, _vp, _vp, _vp], _int),
    "gcabem_gca_free": ([_vp], _int),
    "gcabem_gca_operator": ([_int, _vp, _i64, _i64, _dbl, _vp, _vp, _vp], _int),
    "gcabem_h2_create": ([_int, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _i64, _vp, _i64, _vp,
                          _i64, _vp, _i64, _vp, ctypes.POINTER(_vp)], _int),
    "gcabem_h2_matvec": ([_vp, _vp, _vp, _vp], _int),
    "gcabem_h2_info": ([_vp, _vp], _int),
    "gcabem_h2_free": ([_vp], _int),
    "gcabem_p1_create": ([_vp, _int, _int, _dbl, _int, _vp, _vp, _vp, _vp, ctypes.POINTER(_vp)],
                         _int),
    "gcabem_p1_execute": ([_vp], _int),
    "gcabem_p1_info": ([_vp, _vp, _vp], _int),
    "gcabem_p1_download": ([_vp, _vp, _vp, _vp, _vp], _int),
    "gcabem_p1_destroy": ([_vp], _int),
    "gcabem_p1_batch": ([_vp, _int, _int, _dbl, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp,
                         _vp], _int),
    "gcabem_aca_batch": ([_int, _i64, _vp, _i64, _vp, _dbl, _i64, _int, _vp, _vp, _vp, _vp],
                         _int),
}
EXPORTED = tuple(_SIGS)


def lib():
    """Load (once) and return the library; raises BackendError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise BackendError(
                    f"{LIB_PATH} not built; run __graft_entry__.build() (no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            for name, (args, res) in _SIGS.items():
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = res
            _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().gcabem_last_error().decode(errors="replace")
    if rc == ERR_ARG:
        raise ValueError(msg)
    if rc == ERR_GCA:
        from .gca import GcaError
        raise GcaError(msg)
    raise BackendError(msg)


def device_count() -> int:
    n = _int(0)
    rc = lib().gcabem_device_count(ctypes.byref(n))
    return int(n.value) if rc == 0 else 0


def require_device(device: int = 0) -> None:
    n = device_count()
    if n == 0:
        raise BackendError("no CUDA device visible; the B200 path has no CPU fallback")
    if not 0 <= device < n:
        raise BackendError(f"device {device} not available ({n} visible)")


def ptr(a):
    """Data pointer of a numpy array (None for None)."""
    return None if a is None else a.ctypes.data


def f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def i64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.int64)


def u8(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.uint8)


# ---------------------------------------------------------------------------
# pinned host buffers (payload destinations; full PCIe rate for the D2H)

class _PinnedPool:
    """Caching allocator for pinned host blocks (cudaHostAlloc costs ~0.3 s/GB,
    far more than the transfer it enables). Freed blocks are kept and
    re-issued to requests of at least half their size."""

    CAP_BYTES = 32 << 30

    def __init__(self):
        self.free: list[tuple[int, int]] = []  # (nbytes, ptr)
        self.cached = 0
        self.lock = threading.Lock()

    def acquire(self, nbytes: int) -> tuple[int, int]:
        with self.lock:
            best = None
            for k, (size, p) in enumerate(self.free):
                if nbytes <= size <= 2 * nbytes and (best is None or size < self.free[best][0]):
                    best = k
            if best is not None:
                size, p = self.free.pop(best)
                self.cached -= size
                return size, p
        p = _vp()
        check(lib().gcabem_host_alloc(int(nbytes), ctypes.byref(p)))
        return nbytes, p.value

    def release(self, size: int, p: int) -> None:
        with self.lock:
            if self.cached + size <= self.CAP_BYTES:
                self.free.append((size, p))
                self.cached += size
                return
        if _lib is not None:
            _lib.gcabem_host_free(p)

    def clear(self) -> None:
        with self.lock:
            blocks, self.free, self.cached = self.free, [], 0
        for _, p in blocks:
            _lib.gcabem_host_free(p)


_POOL = _PinnedPool()


def pinned_pool_clear() -> None:
    """Free the cached (unused) pinned blocks."""
    _POOL.clear()


class _PinnedBlock:
    """Owner of one pinned block; returns it to the pool when the last view dies."""

    def __init__(self, nbytes: int):
        self.size, self.ptr = _POOL.acquire(nbytes)

    def __del__(self):
        # at interpreter teardown the module globals may already be gone:
        # the process exit returns the memory
        if self.ptr and _POOL is not None:
            _POOL.release(self.size, self.ptr)
        self.ptr = None


def pinned_empty(shape, dtype) -> np.ndarray:
    """Uninitialised numpy array in pinned host memory.

    The ctypes view that numpy wraps holds the owner, so the block goes back
    to the pool exactly when no numpy view of it remains (payload dict views
    included).
    """
    dtype = np.dtype(dtype)
    count = int(np.prod(shape))
    nbytes = max(count * dtype.itemsize, 1)
    owner = _PinnedBlock(nbytes)
    raw = (ctypes.c_char * nbytes).from_address(owner.ptr)
    raw._owner = owner
    return np.frombuffer(raw, dtype=np.uint8)[:count * dtype.itemsize].view(dtype).reshape(shape)
