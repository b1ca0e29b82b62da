"""ORACLE — CPU restatement of the reference path. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg may import this package, and only as the checker or
the timed CPU baseline. The product (paper_1510_07244_b200) never imports
it and has no CPU fallback.

Contents
--------
* ``pair_values`` / ``batch_quadrature``: ctypes front-end of
  pairquad_oracle.c, a bit-exact C restatement of the reference's numba
  loop (reference pkg/src/gcabem/pairquad.py:27-112) and of the batch
  backend gather (scheduler.py:257-261, mesh.py:207-222). Pinned
  bit-for-bit against tests/golden/pair_values_L3.npz.
* ``batch_quadrature(..., high_precision=True)``: pairquad_hp.c, the same
  discrete rule on the reference's double-precision chart inputs evaluated
  in binary128 — the yardstick for entries that are roundoff-dominated in
  the reference (tests/test_reference_levels.py).
* numpy restatements of the rule construction (quadrature.py:82-194),
  the pair classification (quadrature.py:197-220) and the Green matrix
  (gca.py:136-179), pinned against golden hashes / fixtures.
* setup_cpu.py: the reference's setup pipeline restated (sphere mesh,
  cluster and block trees, GCA operators, work packaging) -- the bench's
  reference arm, runnable without the product library; p1_cpu.py: the P1
  pair integrals (C4's cpu_baseline).

Parity is pinned (see tests/test_oracle.py); it is not "unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

EQ = {"laplace": 0, "helmholtz": 1}
LAYER = {"single": 0, "double": 1}


def build() -> str:
    """Compile liboracle.so (gcc, OpenMP) in place; returns its path."""
    path = os.path.join(HERE, "liboracle.so")
    srcs = [os.path.join(HERE, f) for f in ("pairquad_oracle.c", "pairquad_hp.c", "Makefile")]
    if not os.path.exists(path) or \
            os.path.getmtime(path) < max(os.path.getmtime(s) for s in srcs):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return path


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        dp = ctypes.c_void_p
        L.oracle_pair_values.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                         ctypes.c_int64] + [dp] * 9 + [ctypes.c_int64] \
            + [dp] * 4 + [ctypes.c_int]
        L.oracle_batch_quadrature.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double] \
            + [dp] * 4 + [ctypes.c_int64] + [dp] * 4 + [ctypes.c_int64] + [dp] * 4 \
            + [ctypes.c_int]
        L.oracle_batch_quadrature_hp.argtypes = L.oracle_batch_quadrature.argtypes
        L.oracle_max_threads.restype = ctypes.c_int
        _LIB = L
    return _LIB


def _p(a):
    return None if a is None else a.ctypes.data


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def pair_values(equation, layer, kappa, ox, e1x, e2x, gx, oy, e1y, e2y, gy, ny,
                xs, ys, w, nthreads=1) -> np.ndarray:
    """Bit-exact restatement of pairquad.pair_values (pairquad.py:95)."""
    arrs = [_f64(a) for a in (ox, e1x, e2x, gx, oy, e1y, e2y, gy, ny, xs, ys, w)]
    n = arrs[0].shape[0]
    out = np.empty(n, dtype=np.complex128)
    lib().oracle_pair_values(EQ[equation], LAYER[layer], float(kappa), n,
                             *[_p(a) for a in arrs[:9]], arrs[11].shape[0],
                             *[_p(a) for a in arrs[9:]], _p(out), int(nthreads))
    return out


def batch_quadrature(equation, layer, kappa, vertices, triangles, normals, gramians,
                     tri_x, tri_y, perm_x, perm_y, xs, ys, w, nthreads=1,
                     high_precision=False) -> np.ndarray:
    """Bit-exact restatement of scheduler.batch_quadrature's batch backend.
    high_precision=True: the same discrete rule on the same double-precision
    chart inputs evaluated in binary128 (pairquad_hp.c) - the exact value the
    reference's double arithmetic approximates."""
    V = _f64(vertices)
    T = np.ascontiguousarray(triangles, dtype=np.int64)
    N = _f64(normals)
    G = _f64(gramians)
    tx = np.ascontiguousarray(tri_x, dtype=np.int64)
    ty = np.ascontiguousarray(tri_y, dtype=np.int64)
    px = None if perm_x is None else np.ascontiguousarray(perm_x, dtype=np.int64)
    py = None if perm_y is None else np.ascontiguousarray(perm_y, dtype=np.int64)
    xs, ys, w = _f64(xs), _f64(ys), _f64(w)
    out = np.empty(len(tx), dtype=np.complex128)
    fn = lib().oracle_batch_quadrature_hp if high_precision else lib().oracle_batch_quadrature
    fn(EQ[equation], LAYER[layer], float(kappa),
                                  _p(V), _p(T), _p(N), _p(G), len(tx), _p(tx), _p(ty),
                                  _p(px), _p(py), w.shape[0], _p(xs), _p(ys), _p(w),
                                  _p(out), int(nthreads))
    return out


# ---------------------------------------------------------------------------
# numpy restatements (rules, classification, Green matrix)

def gauss01(n):
    """quadrature.py:82-87: leggauss mapped to [0,1]."""
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


def rule(case, n):
    """quadrature.py:99-194 restated: (xs (Q,2), ys (Q,2), w (Q,))."""
    p, gw = gauss01(n)
    A = np.meshgrid(p, p, p, p, indexing="ij")
    W = np.meshgrid(gw, gw, gw, gw, indexing="ij")
    a, b, c, d = (v.ravel() for v in A)
    w = (W[0] * W[1] * W[2] * W[3]).ravel()
    if case == "disjoint":
        terms = [((a, a * b), (c, c * d), w * (a * c))]
    elif case == "vertex":
        x, e1, e2, e3 = a, b, c, d
        wj = w * (x ** 3 * e2)
        terms = [((x, x * e1), (x * e2, x * e2 * e3), wj),
                 ((x * e2, x * e2 * e3), (x, x * e1), wj)]
    elif case == "edge":
        x, e1, e2, e3 = a, b, c, d
        w1 = w * (x ** 3 * e1 ** 2)
        w2 = w * (x ** 3 * e1 ** 2 * e2)
        terms = [((x, x * e1 * e3), (x * (1 - e1 * e2), x * (e1 * (1 - e2))), w1),
                 ((x, x * e1), (x * (1 - e1 * e2 * e3), x * (e1 * e2 * (1 - e3))), w2),
                 ((x * (1 - e1 * e2), x * (e1 * (1 - e2))), (x, x * (e1 * e2 * e3)), w2),
                 ((x * (1 - e1 * e2 * e3), x * (e1 * e2 * (1 - e3))), (x, x * e1), w2),
                 ((x * (1 - e1 * e2 * e3), x * (e1 * (1 - e2 * e3))), (x, x * (e1 * e2)), w2)]
    elif case == "identical":
        x, e1, e2, e3 = a, b, c, d
        wj = w * (x ** 3 * e1 ** 2 * e2)
        base = [((x, x * (1 - e1 + e1 * e2)), (x * (1 - e1 * e2 * e3), x * (1 - e1))),
                ((x, x * (e1 * (1 - e2 + e2 * e3))), (x * (1 - e1 * e2), x * (e1 * (1 - e2)))),
                ((x * (1 - e1 * e2 * e3), x * (e1 * (1 - e2 * e3))), (x, x * (e1 * (1 - e2))))]
        terms = []
        for X, Y in base:
            terms += [(X, Y, wj), (Y, X, wj)]
    else:
        raise ValueError(case)
    xs = np.concatenate([np.stack(t[0], axis=1) for t in terms])
    ys = np.concatenate([np.stack(t[1], axis=1) for t in terms])
    ws = np.concatenate([t[2] for t in terms])
    return np.ascontiguousarray(xs), np.ascontiguousarray(ys), np.ascontiguousarray(ws)


def classify(triangles, a, b):
    """quadrature.py:197-220 restated with plain Python ints."""
    if a == b:
        return "identical", (0, 1, 2), (0, 1, 2)
    va = [int(v) for v in triangles[a]]
    vb = [int(v) for v in triangles[b]]
    shared = sorted(set(va) & set(vb))
    if len(shared) == 3:
        raise ValueError("distinct triangles share 3 vertices")
    if not shared:
        return "disjoint", (0, 1, 2), (0, 1, 2)

    def perm(vs):
        lead = [vs.index(g) for g in shared]
        return tuple(lead + [k for k in range(3) if k not in lead])
    return ("edge" if len(shared) == 2 else "vertex"), perm(va), perm(vb)


INV_4PI = 1.0 / (4.0 * np.pi)


def _kernel(equation, layer, kappa, d0, d1, d2, n0=None, n1=None, n2=None):
    r2 = d0 * d0 + d1 * d1 + d2 * d2
    r = np.sqrt(r2)
    if equation == "laplace":
        if layer == "single":
            return INV_4PI / r
        return INV_4PI * (d0 * n0 + d1 * n1 + d2 * n2) / (r2 * r)
    ph = np.exp(1j * (kappa * r))
    if layer == "single":
        return ph / r
    return ph * (1.0 - 1j * (kappa * r)) * (d0 * n0 + d1 * n1 + d2 * n2) / (r2 * r)


def green_matrix(vertices, triangles, gramians, panels, src_points, src_weights,
                 src_normals, src_roles, equation, kappa, order):
    """gca.py:136-179 restated: A[i,j] = w_j * gram_i * sum_q wq k_j(X_iq)."""
    p, gw = gauss01(order)
    a, b = np.meshgrid(p, p, indexing="ij")
    wa, wb = np.meshgrid(gw, gw, indexing="ij")
    pts = np.stack([a.ravel(), (a * b).ravel()], axis=1)
    wq = (wa * wb).ravel() * a.ravel()
    idx = triangles[np.asarray(panels)]
    v0 = vertices[idx[:, 0]]
    e1 = vertices[idx[:, 1]] - v0
    e2 = vertices[idx[:, 2]] - vertices[idx[:, 1]]
    X = v0[:, None, :] + pts[None, :, 0, None] * e1[:, None, :] \
        + pts[None, :, 1, None] * e2[:, None, :]
    d = X[:, :, None, :] - src_points[None, None, :, :]
    mono = src_roles == 0
    out = np.empty((len(panels), len(src_weights)),
                   dtype=np.complex128 if equation == "helmholtz" else np.float64)
    km = _kernel(equation, "single", kappa, d[..., mono, 0], d[..., mono, 1], d[..., mono, 2])
    nd = src_normals[~mono]
    kd = _kernel(equation, "double", kappa, d[..., ~mono, 0], d[..., ~mono, 1],
                 d[..., ~mono, 2], nd[:, 0], nd[:, 1], nd[:, 2])
    g = gramians[np.asarray(panels)][:, None]
    out[:, mono] = np.einsum("q,pqs->ps", wq, km) * g * src_weights[mono]
    out[:, ~mono] = np.einsum("q,pqs->ps", wq, kd) * g * src_weights[~mono]
    return out
