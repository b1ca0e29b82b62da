"""ORACLE — CPU restatement of the piecewise-linear (P1) pair integrals: the
reference's integrate_pair with P1 bases (pkg/src/gcabem/quadrature.py:223-271:
basis_x / basis_y weighting the kernel values of the rule's points) over
batches of pairs. TEST INFRASTRUCTURE ONLY (tests/ and bench.py's C4
cpu_baseline); imports nothing from paper_1510_07244_b200. The reference has
no P1 matrix assembly: this restates its per-pair P1 integral, pinned against
the reference's own integrate_pair outputs (tests/golden/p1_crank.npz)."""
from __future__ import annotations

import numpy as np

from . import _kernel, rule


def lam(points):
    """Barycentric coordinates of the P1 basis on the reference triangle
    (1 - s, s - t, t) for (s, t) in the Duffy chart."""
    p = np.asarray(points)
    return np.stack([1.0 - p[:, 0], p[:, 0] - p[:, 1], p[:, 1]], axis=1)


def local_matrices(vertices, triangles, normals, gramians, equation, layer, kappa, case,
                   order, tx, ty, px=None, py=None, chunk=512):
    """(n, 3, 3) complex local matrices, stored vertex order of each panel:
    M[a, b] = gram_x gram_y sum_q w_q k(X_q - Y_q) lam_a(x_q) lam_b(y_q), the
    chart vertices permuted by px / py (classify_pair)."""
    xs, ys, w = rule(case, order)
    tx, ty = np.asarray(tx, np.int64), np.asarray(ty, np.int64)
    n = tx.size
    px = np.tile(np.arange(3), (n, 1)) if px is None else np.asarray(px, np.int64)
    py = np.tile(np.arange(3), (n, 1)) if py is None else np.asarray(py, np.int64)
    T, V = np.asarray(triangles), np.asarray(vertices)
    lx, ly = lam(xs), lam(ys)
    out = np.zeros((n, 3, 3), dtype=np.complex128)
    for a0 in range(0, n, chunk):
        sl = slice(a0, min(n, a0 + chunk))
        ix = np.take_along_axis(T[tx[sl]], px[sl], axis=1)
        iy = np.take_along_axis(T[ty[sl]], py[sl], axis=1)
        x0, x1, x2 = V[ix[:, 0]], V[ix[:, 1]], V[ix[:, 2]]
        y0, y1, y2 = V[iy[:, 0]], V[iy[:, 1]], V[iy[:, 2]]
        X = x0[:, None] + xs[None, :, 0:1] * (x1 - x0)[:, None] + \
            xs[None, :, 1:2] * (x2 - x1)[:, None]
        Y = y0[:, None] + ys[None, :, 0:1] * (y1 - y0)[:, None] + \
            ys[None, :, 1:2] * (y2 - y1)[:, None]
        d = X - Y
        nrm = np.asarray(normals)[ty[sl]][:, None, :]
        k = _kernel(equation, layer, kappa, d[..., 0], d[..., 1], d[..., 2], nrm[..., 0],
                    nrm[..., 1], nrm[..., 2])
        M = np.einsum("pq,qa,qb->pab", k * w, lx, ly)
        M = M * (np.asarray(gramians)[tx[sl]] * np.asarray(gramians)[ty[sl]])[:, None, None]
        r = np.arange(sl.stop - sl.start)
        for a in range(3):
            for b in range(3):
                out[a0 + r, px[sl][:, a], py[sl][:, b]] = M[:, a, b]
    return out
