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


def near_field(m, pk, spec, orders):
    """Dense vertex x vertex near-field matrix: every pair of the packages'
    blocks with the rule of its case (singular items overwrite)."""
    nv = m.num_vertices
    A = np.zeros((nv, nv), dtype=np.complex128)
    blocks = pk.device_blocks()
    items, perms = pk.device_items()
    sing = {}
    for (case, tx, ty, out), pm in zip(items, perms):
        sing[int(out)] = (int(case), pm)
    drule = quadrature.build_rule("disjoint", orders[0])
    srules = {c: quadrature.build_rule(n, orders[1])
              for c, n in ((1, "vertex"), (2, "edge"), (3, "identical"))}
    T = m.triangles
    for base, ld, nr, nc, ra, ca, _ in blocks:
        for i in range(nr):
            tx = pk.panels[ra + i]
            for j in range(nc):
                ty = pk.panels[ca + j]
                p = base + i * ld + j
                if p in sing:
                    case, pm = sing[p]
                    M = local_matrix(m, spec, srules[case], tx, ty, pm[:3], pm[3:])
                else:
                    M = local_matrix(m, spec, drule, tx, ty)
                for a in range(3):
                    for b in range(3):
                        A[T[tx, a], T[ty, b]] += M[a, b]
    return A
