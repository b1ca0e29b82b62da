"""TEST-SIDE numpy restatement of the P1 local matrices (reference
quadrature.integrate_pair with basis_x / basis_y, quadrature.py:223-271) and
of the near-field vertex scatter (np.add.at), the checker for csrc/p1.cu."""
import numpy as np

from paper_1510_07244_b200 import kernels, mesh as meshmod, quadrature


def lam(points):
    p = np.asarray(points)
    return np.stack([1.0 - p[:, 0], p[:, 0] - p[:, 1], p[:, 1]], axis=1)


def local_matrix(m, spec, rule, tx, ty, perm_x=(0, 1, 2), perm_y=(0, 1, 2)):
    """3 x 3 in stored vertex order."""
    cx = meshmod.chart(m, int(tx), tuple(perm_x))
    cy = meshmod.chart(m, int(ty), tuple(perm_y))
    X = cx.map_points(rule.x_points)
    Y = cy.map_points(rule.y_points)
    d = X - Y
    n = m.normals[int(ty)]
    if spec.needs_normal:
        k = kernels.kernel_values(spec, d[:, 0], d[:, 1], d[:, 2], n[0], n[1], n[2])
    else:
        k = kernels.kernel_values(spec, d[:, 0], d[:, 1], d[:, 2])
    v = k * rule.weights
    M = np.einsum("q,qa,qb->ab", v, lam(rule.x_points), lam(rule.y_points))
    M = M * cx.gramian * cy.gramian
    out = np.zeros((3, 3), dtype=np.complex128)
    for a in range(3):
        for b in range(3):
            out[perm_x[a], perm_y[b]] = M[a, b]
    return out


def local_matrices_batch(m, spec, rule, tx, ty, px=None, py=None, chunk=512):
    """Vectorised local_matrix over pairs: (n, 3, 3), stored vertex order."""
    tx, ty = np.asarray(tx, np.int64), np.asarray(ty, np.int64)
    n = tx.size
    px = np.tile(np.arange(3), (n, 1)) if px is None else np.asarray(px, np.int64)
    py = np.tile(np.arange(3), (n, 1)) if py is None else np.asarray(py, np.int64)
    T, V = m.triangles, m.vertices
    lx, ly = lam(rule.x_points), lam(rule.y_points)
    out = np.zeros((n, 3, 3), dtype=np.complex128)
    for a0 in range(0, n, chunk):
        sl = slice(a0, min(n, a0 + chunk))
        ix = np.take_along_axis(T[tx[sl]], px[sl], axis=1)
        iy = np.take_along_axis(T[ty[sl]], py[sl], axis=1)
        x0, x1, x2 = V[ix[:, 0]], V[ix[:, 1]], V[ix[:, 2]]
        y0, y1, y2 = V[iy[:, 0]], V[iy[:, 1]], V[iy[:, 2]]
        X = x0[:, None] + rule.x_points[None, :, 0:1] * (x1 - x0)[:, None] + \
            rule.x_points[None, :, 1:2] * (x2 - x1)[:, None]
        Y = y0[:, None] + rule.y_points[None, :, 0:1] * (y1 - y0)[:, None] + \
            rule.y_points[None, :, 1:2] * (y2 - y1)[:, None]
        d = X - Y
        nrm = m.normals[ty[sl]][:, None, :]
        if spec.needs_normal:
            k = kernels.kernel_values(spec, d[..., 0], d[..., 1], d[..., 2], nrm[..., 0],
                                      nrm[..., 1], nrm[..., 2])
        else:
            k = kernels.kernel_values(spec, d[..., 0], d[..., 1], d[..., 2])
        M = np.einsum("pq,qa,qb->pab", k * rule.weights, lx, ly)
        M *= (m.gramians[tx[sl]] * m.gramians[ty[sl]])[:, None, None]
        r = np.arange(sl.stop - sl.start)
        for a in range(3):
            for b in range(3):
                out[a0 + r, px[sl][:, a], py[sl][:, b]] = M[:, a, b]
    return out


def near_field(m, pk, spec, orders):
    """Dense vertex x vertex near-field matrix: every pair of the packages'
    blocks with the rule of its case (singular items overwrite)."""
    nv = m.num_vertices
    A = np.zeros((nv, nv), dtype=np.complex128)
    blocks = pk.device_blocks()
    items, perms = pk.device_items()
    drule = quadrature.build_rule("disjoint", orders[0])
    srules = {c: quadrature.build_rule(n, orders[1])
              for c, n in ((1, "vertex"), (2, "edge"), (3, "identical"))}
    T = m.triangles
    P = pk.payload_len
    txs = np.empty(P, np.int64)
    tys = np.empty(P, np.int64)
    for base, ld, nr, nc, ra, ca, _ in blocks:
        i, j = np.divmod(np.arange(nr * nc), nc)
        p = base + i * ld + j
        txs[p], tys[p] = pk.panels[ra + i], pk.panels[ca + j]
    loc = np.empty((P, 3, 3), np.complex128)
    is_s = np.zeros(P, bool)
    for code, rule in srules.items():
        sel = items[:, 0] == code
        if np.any(sel):
            out = items[sel, 3]
            loc[out] = local_matrices_batch(m, spec, rule, items[sel, 1], items[sel, 2],
                                            perms[sel, :3], perms[sel, 3:])
            is_s[out] = True
    dis = np.flatnonzero(~is_s)
    loc[dis] = local_matrices_batch(m, spec, drule, txs[dis], tys[dis])
    rows = T[txs][:, :, None].repeat(3, axis=2)
    cols = T[tys][:, None, :].repeat(3, axis=1)
    np.add.at(A, (rows.ravel(), cols.ravel()), loc.ravel())
    return A
