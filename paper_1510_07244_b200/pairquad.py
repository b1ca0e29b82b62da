"""Fused panel-pair quadrature on the B200 (drop-in for gcabem.pairquad).

The reference's numba loop (pairquad.py:27-92) becomes the sm_100a kernels
in csrc/kernels.cu; this module is the per-chart entry point
``pair_values`` (pairquad.py:95-112), routed through the C ABI
``gcabem_pair_values``. No CPU fallback: without the library or a device,
calls raise BackendError.
"""
from __future__ import annotations

import os

import numpy as np

from . import _native as nat

_DEVICE = int(os.environ.get("GCABEM_DEVICE", "0"))


def default_device() -> int:
    return _DEVICE


def set_default_device(device: int) -> None:
    global _DEVICE
    _DEVICE = int(device)


def pair_values(spec, ox, e1x, e2x, gx, oy, e1y, e2y, gy, ny, xs, ys, w) -> np.ndarray:
    """Weighted pair integrals for a batch of charts; complex128 (npairs,).

    out[i] = gy_i * (gx_i * sum_q w_q k(Phi_x,i(xs_q) - Phi_y,i(ys_q), ny_i)).
    Coincident points produce non-finite entries silently, as in the
    reference (the disjoint pass over singular pairs is overwritten later).
    """
    eq, layer = spec.code
    arrs = [nat.f64(a) for a in (ox, e1x, e2x, gx, oy, e1y, e2y, gy)]
    n = arrs[0].shape[0]
    for a in arrs:
        if a.shape[0] != n:
            raise ValueError("pair arrays disagree in length")
    nyv = None if ny is None else nat.f64(ny)
    xs, ys, w = nat.f64(xs), nat.f64(ys), nat.f64(w)
    if xs.shape != (w.shape[0], 2) or ys.shape != xs.shape:
        raise ValueError("rule arrays must be (Q,2), (Q,2), (Q,)")
    out = np.empty(n, dtype=np.complex128)
    if n == 0:
        return out
    nat.require_device(_DEVICE)
    nat.check(nat.lib().gcabem_pair_values(
        _DEVICE, eq, layer, float(spec.kappa), n, *[nat.ptr(a) for a in arrs],
        nat.ptr(nyv), w.shape[0], nat.ptr(xs), nat.ptr(ys), nat.ptr(w), nat.ptr(out)))
    return out
