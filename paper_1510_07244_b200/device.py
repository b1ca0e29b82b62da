"""Device-resident mesh replicas (one per (mesh, device)), cached.

A replica holds the vertex table, the int32 triangle table and the 128-byte
chart table (origin, edge1, edge2, normal, Gramian) the kernels gather
from; at 131,072 triangles it is 17 MB, so every kernel's geometry reads
stay L2-resident.
"""
from __future__ import annotations

import ctypes
import threading
import weakref

import numpy as np

from . import _native as nat
from .mesh import SurfaceMesh

_cache: dict = {}
_cache_lock = threading.Lock()


class DeviceMesh:
    def __init__(self, mesh: SurfaceMesh, device: int = 0):
        nat.require_device(device)
        self.device = device
        self.num_triangles = mesh.num_triangles
        h = ctypes.c_void_p()
        V = nat.f64(mesh.vertices)
        T = nat.i64(mesh.triangles)
        N = nat.f64(mesh.normals)
        G = nat.f64(mesh.gramians)
        nat.check(nat.lib().gcabem_mesh_create(device, V.shape[0], nat.ptr(V), T.shape[0],
                                               nat.ptr(T), nat.ptr(N), nat.ptr(G),
                                               ctypes.byref(h)))
        self.handle = h.value

    def close(self) -> None:
        h, self.handle = getattr(self, "handle", None), None
        if h and getattr(nat, "_lib", None) is not None:  # nat is None at interpreter teardown
            nat._lib.gcabem_mesh_destroy(h)

    def __del__(self):
        self.close()


def _drop(key):
    """Forget the replica of a dead mesh. The replica itself is released by
    DeviceMesh.__del__ once no plan references it any more (plans must be
    destroyed before the mesh they gather from)."""
    with _cache_lock:
        _cache.pop(key, None)


def device_mesh(mesh: SurfaceMesh, device: int = 0) -> DeviceMesh:
    """Cached replica of `mesh` on `device`; released with the mesh object."""
    key = (id(mesh), device)
    with _cache_lock:
        dm = _cache.get(key)
    if dm is None:
        dm = DeviceMesh(mesh, device)
        with _cache_lock:
            _cache[key] = dm
        weakref.finalize(mesh, _drop, key)
    return dm


def fp64_peak_tflops(device: int = 0) -> float:
    """Measured dependent-DFMA throughput of `device` (TFLOP/s, FMA = 2)."""
    nat.require_device(device)
    out = ctypes.c_double()
    nat.check(nat.lib().gcabem_fp64_probe(device, ctypes.byref(out)))
    return float(out.value)


def device_info(device: int = 0) -> dict:
    name = ctypes.create_string_buffer(256)
    sms, clk = ctypes.c_int(), ctypes.c_int()
    nat.check(nat.lib().gcabem_device_info(device, name, ctypes.byref(sms), ctypes.byref(clk)))
    return {"name": name.value.decode(), "sm_count": sms.value, "clock_khz": clk.value}


def as_i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def release_cached(device: int = 0) -> None:
    """Give the library's cross-call caches on `device` back to the driver
    (device memory pool free blocks, GCA staging ring, pinned layout arena)."""
    nat.require_device(device)
    nat.check(nat.lib().gcabem_release_cached(device))
    nat.pinned_pool_clear()
