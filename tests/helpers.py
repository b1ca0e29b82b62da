"""Test-side helpers: oracle-driven assembly and parity rules (tests only)."""
import hashlib

import numpy as np

import oracle
from paper_1510_07244_b200 import cluster, mesh
from paper_1510_07244_b200.gca import InterpolationOperator
from paper_1510_07244_b200.packaging import make_packages

SPECS = {
    "L-SLP": ("laplace", "single", 0.0),
    "L-DLP": ("laplace", "double", 0.0),
    "H-SLP": ("helmholtz", "single", 4.0),
    "H-DLP": ("helmholtz", "double", 4.0),
}


def golden_ops(gca_npz, equation):
    """InterpolationOperators carrying the reference's pivots (V unused here)."""
    cids = gca_npz[f"ops_{equation}_cids"]
    ranks = gca_npz[f"ops_{equation}_ranks"]
    piv = gca_npz[f"ops_{equation}_pivots"]
    ops, at = {}, 0
    for c, r in zip(cids, ranks):
        ops[int(c)] = InterpolationOperator(int(c), np.arange(r), piv[at:at + r],
                                            np.zeros((1, r)))
        at += r
    return ops


def sphere_setup(level, leaf=16, eta=2.0):
    m = mesh.build_sphere_mesh(level)
    t = cluster.build_cluster_tree(m, leaf)
    return m, t, cluster.build_block_tree(t, t, eta)


def oracle_assemble(m, pk, equation, layer, kappa, orders, nthreads=0):
    """Payload buffer computed by the bit-exact oracle over the SAME packages
    (disjoint rule over every block pair, then singular overwrites)."""
    payload = np.zeros(pk.payload_len, dtype=np.complex128)
    blocks = pk.device_blocks()
    xs, ys, w = oracle.rule("disjoint", orders[0])
    if blocks.size:
        nr, nc = blocks[:, 2], blocks[:, 3]
        cnt = nr * nc
        owner = np.repeat(np.arange(len(blocks)), cnt)
        k = np.arange(owner.size) - np.repeat(np.cumsum(cnt) - cnt, cnt)
        i, j = k // nc[owner], k % nc[owner]
        tx = pk.panels[blocks[owner, 4] + i]
        ty = pk.panels[blocks[owner, 5] + j]
        vals = oracle.batch_quadrature(equation, layer, kappa, m.vertices, m.triangles,
                                       m.normals, m.gramians, tx, ty, None, None, xs, ys, w,
                                       nthreads=nthreads)
        payload[blocks[owner, 0] + i * blocks[owner, 1] + j] = vals
    items, perms = pk.device_items()
    for code, case in ((1, "vertex"), (2, "edge"), (3, "identical")):
        sel = items[:, 0] == code
        if not np.any(sel):
            continue
        xs, ys, w = oracle.rule(case, orders[1])
        vals = oracle.batch_quadrature(equation, layer, kappa, m.vertices, m.triangles,
                                       m.normals, m.gramians, items[sel, 1], items[sel, 2],
                                       perms[sel, :3].astype(np.int64),
                                       perms[sel, 3:].astype(np.int64), xs, ys, w,
                                       nthreads=nthreads)
        payload[items[sel, 3]] = vals
    return payload


def checksum(pk, payload):
    h = hashlib.sha256()
    for k in range(pk.leaf_ids.size):
        h.update(payload[pk.leaf_base[k]:pk.leaf_base[k + 1]].tobytes())
    return h.hexdigest()


def p2_check(pk, got, ref, tol=1e-12, double_layer=False):
    """|new-ref| <= tol*|ref| per entry, except entries that
    are roundoff/cancellation-dominated in the reference, compared on the
    scale of their leaf block (tol * max|ref| over the leaf): entries with
    |ref| < 1e-9 * leaf max (DLP identical pairs), and - for double-layer
    operators - every singular corrective entry (near-coplanar pairs whose
    reference rounding grows like eps/h^2).
    Returns (ok, worst relative error, number of leaf-scaled entries)."""
    err = np.abs(got - ref)
    mag = np.abs(ref)
    leaf_of = np.repeat(np.arange(pk.leaf_ids.size), np.diff(pk.leaf_base))
    leaf_max = np.zeros(pk.leaf_ids.size)
    np.maximum.at(leaf_max, leaf_of, mag)
    fallback = mag < 1e-9 * leaf_max[leaf_of]
    if double_layer and pk.num_items:
        fallback[pk.device_items()[0][:, 3]] = True
    scale = np.where(fallback, leaf_max[leaf_of], mag)
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(scale > 0, err / scale, err)
    ok = bool(np.all(np.isfinite(got)) and np.all(rel <= tol))
    return ok, float(np.max(rel)) if rel.size else 0.0, int(np.count_nonzero(fallback))


def packages_for(level, equation, gca_npz=None, maxsize=8 * 2 ** 20, near_only=False):
    m, t, bt = sphere_setup(level)
    if near_only:
        bt = cluster.BlockTree(bt.nodes, t, t, bt.eta, [l for l in bt.leaves if l.kind == "dense"])
        ops = {}
    else:
        ops = golden_ops(gca_npz, equation)
    return m, bt, ops, make_packages(m.triangles, bt, ops, ops, maxsize)
