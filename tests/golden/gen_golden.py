"""Generate golden fixtures by running the UNMODIFIED reference package.

This script is the only place that imports the reference (`gcabem`, pure
Python + numba, /root/reference/pkg/src). It runs in the dev container
only; the fixtures it writes (tests/golden/*.npz, *.json) are committed and
travel to the GPU box, where /root/reference does not exist.

    NUMBA_CACHE_DIR=/tmp/numba PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/gen_golden.py

(NUMBA_CACHE_DIR keeps numba's cache=True from writing into the reference
tree.)  Every fixture records which reference function produced it.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

import gcabem  # noqa: E402  (reference package)
from gcabem import cluster, gca, h2, kernels, mesh, quadrature, scheduler  # noqa: E402
from gcabem.pairquad import pair_values  # noqa: E402


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


SPECS = {
    "L-SLP": kernels.KernelSpec("laplace", "single"),
    "L-DLP": kernels.KernelSpec("laplace", "double"),
    "H-SLP": kernels.KernelSpec("helmholtz", "single", 4.0),
    "H-DLP": kernels.KernelSpec("helmholtz", "double", 4.0),
}
CASE_CODE = {"disjoint": 0, "vertex": 1, "edge": 2, "identical": 3}


def gen_hashes(meta):
    # mesh.py:142 build_sphere_mesh, bitwise
    meta["sphere"] = {}
    for L in range(0, 6):
        m = mesh.build_sphere_mesh(L)
        meta["sphere"][str(L)] = {
            "nv": m.num_vertices, "nt": m.num_triangles,
            "vertices": sha(m.vertices), "triangles": sha(m.triangles),
            "normals": sha(m.normals), "gramians": sha(m.gramians)}
    # quadrature.py:82 gauss_legendre, :170 build_rule, :90 duffy_panel_rule
    meta["gauss"] = {str(n): sha(quadrature.gauss_legendre(n).points,
                                 quadrature.gauss_legendre(n).weights)
                     for n in range(1, 33)}
    meta["rules"] = {}
    for case in quadrature.CASES:
        for n in range(1, 13):
            r = quadrature.build_rule(case, n)
            meta["rules"][f"{case}/{n}"] = sha(r.x_points, r.y_points, r.weights)
    meta["duffy"] = {str(n): sha(*quadrature.duffy_panel_rule(n)) for n in range(1, 9)}


def gen_rules_npz():
    out = {}
    for case in quadrature.CASES:
        for n in (2, 3):
            r = quadrature.build_rule(case, n)
            out[f"{case}_{n}_x"] = r.x_points
            out[f"{case}_{n}_y"] = r.y_points
            out[f"{case}_{n}_w"] = r.weights
    np.savez_compressed(os.path.join(HERE, "rules.npz"), **out)


def gen_classification():
    # quadrature.py:197 classify_pair over all pairs of the level-2 sphere
    m = mesh.build_sphere_mesh(2)
    nt = m.num_triangles
    cls = np.zeros((nt, nt, 7), dtype=np.int8)
    for a in range(nt):
        for b in range(nt):
            c = quadrature.classify_pair(m, a, b)
            cls[a, b, 0] = CASE_CODE[c.case]
            cls[a, b, 1:4] = c.perm_x
            cls[a, b, 4:7] = c.perm_y
    np.savez_compressed(os.path.join(HERE, "classify_L2.npz"), cls=cls)


def _pick_pairs(m, rng):
    """Pairs of the level-3 sphere per case, with reference classification."""
    nt = m.num_triangles
    tri = m.triangles
    shared = np.zeros((nt, nt), dtype=np.int8)
    for a in range(3):
        for b in range(3):
            shared += (tri[:, a][:, None] == tri[:, b][None, :]).astype(np.int8)
    picks = {}
    # disjoint: 48 random far pairs + 48 nearest disjoint pairs (2-ring)
    mid = m.midpoints()
    dist = np.linalg.norm(mid[:, None, :] - mid[None, :, :], axis=2)
    disj = np.argwhere(shared == 0)
    far = disj[rng.choice(len(disj), 48, replace=False)]
    near_order = np.argsort(dist[disj[:, 0], disj[:, 1]], kind="stable")
    near = disj[near_order[rng.choice(2000, 48, replace=False)]]
    picks["disjoint"] = np.concatenate([far, near])
    for case, cnt in (("vertex", 1), ("edge", 2)):
        cand = np.argwhere(shared == cnt)
        picks[case] = cand[rng.choice(len(cand), 64, replace=False)]
    ids = rng.choice(nt, 64, replace=False)
    picks["identical"] = np.stack([ids, ids], axis=1)
    return picks


def gen_pair_values():
    """pairquad.py:95 pair_values through scheduler.batch_quadrature's gather
    (mesh.chart_arrays with classify_pair permutations)."""
    m = mesh.build_sphere_mesh(3)
    rng = np.random.default_rng(20151024)
    picks = _pick_pairs(m, rng)
    out = {}
    for case, pairs in picks.items():
        tx = pairs[:, 0].astype(np.int64)
        ty = pairs[:, 1].astype(np.int64)
        px = np.empty((len(tx), 3), dtype=np.int64)
        py = np.empty((len(tx), 3), dtype=np.int64)
        for k in range(len(tx)):
            c = quadrature.classify_pair(m, int(tx[k]), int(ty[k]))
            assert c.case == case
            px[k] = c.perm_x
            py[k] = c.perm_y
        out[f"{case}_tri_x"] = tx
        out[f"{case}_tri_y"] = ty
        out[f"{case}_perm_x"] = px
        out[f"{case}_perm_y"] = py
        orders = (1, 2, 3, 4, 5, 7) if case == "disjoint" else (2, 3, 5, 7)
        for n in orders:
            rule = quadrature.build_rule(case, n)
            for name, spec in SPECS.items():
                if case == "disjoint":
                    vals = scheduler.batch_quadrature(scheduler.BATCH_BACKEND, case, m, spec,
                                                      rule, tx, ty, None, None)
                else:
                    vals = scheduler.batch_quadrature(scheduler.BATCH_BACKEND, case, m, spec,
                                                      rule, tx, ty, px, py)
                out[f"{case}_{n}_{name}"] = vals
    # raw A/B charts: random non-mesh geometry, ny=None for SLP
    n = 40
    ox = rng.standard_normal((n, 3)); e1x = rng.standard_normal((n, 3)) * 0.3
    e2x = rng.standard_normal((n, 3)) * 0.3
    oy = rng.standard_normal((n, 3)) + 3.0; e1y = rng.standard_normal((n, 3)) * 0.3
    e2y = rng.standard_normal((n, 3)) * 0.3
    gx = rng.uniform(0.1, 1.0, n); gy = rng.uniform(0.1, 1.0, n)
    ny = rng.standard_normal((n, 3)); ny /= np.linalg.norm(ny, axis=1, keepdims=True)
    for k, v in dict(ox=ox, e1x=e1x, e2x=e2x, oy=oy, e1y=e1y, e2y=e2y, gx=gx, gy=gy,
                     ny=ny).items():
        out[f"raw_{k}"] = v
    for rn in (3, 5):
        rule = quadrature.build_rule("disjoint", rn)
        for name, spec in SPECS.items():
            out[f"raw_{rn}_{name}"] = pair_values(
                spec, ox, e1x, e2x, gx, oy, e1y, e2y, gy,
                ny if spec.needs_normal else None,
                rule.x_points, rule.y_points, rule.weights)
    np.savez_compressed(os.path.join(HERE, "pair_values_L3.npz"), **out)


def gen_kernel_values():
    # kernels.py:46 kernel_values / :85 eval_batch
    rng = np.random.default_rng(7)
    xs = rng.standard_normal((500, 3)) + np.array([2.0, 0, 0])
    ys = rng.standard_normal((500, 3))
    ns = rng.standard_normal((500, 3)); ns /= np.linalg.norm(ns, axis=1, keepdims=True)
    out = {"xs": xs, "ys": ys, "ns": ns}
    for name, spec in SPECS.items():
        out[name] = kernels.eval_batch(spec, xs, ys, ns if spec.needs_normal else None)
    np.savez_compressed(os.path.join(HERE, "kernel_values.npz"), **out)


def _tree_arrays(prefix, tree, out):
    out[f"{prefix}_perm"] = tree.permutation
    out[f"{prefix}_start"] = np.array([n.start for n in tree.nodes], dtype=np.int64)
    out[f"{prefix}_size"] = np.array([n.size for n in tree.nodes], dtype=np.int64)
    ch = np.full((len(tree.nodes), 2), -1, dtype=np.int64)
    for i, n in enumerate(tree.nodes):
        ch[i, :len(n.children)] = n.children
    out[f"{prefix}_children"] = ch
    out[f"{prefix}_lo"] = np.array([n.lo for n in tree.nodes])
    out[f"{prefix}_hi"] = np.array([n.hi for n in tree.nodes])


def gen_trees():
    # cluster.py:87 build_cluster_tree, :125 build_block_tree
    out = {}
    for L in (3, 4):
        m = mesh.build_sphere_mesh(L)
        t = cluster.build_cluster_tree(m, 16)
        _tree_arrays(f"L{L}", t, out)
        bt = cluster.build_block_tree(t, t, 2.0)
        kind = {"admissible": 0, "dense": 1, "split": 2}
        out[f"L{L}_blocks"] = np.array([(b.row, b.col, kind[b.kind], len(b.children))
                                        for b in bt.nodes], dtype=np.int64)
        out[f"L{L}_leaves"] = np.array([b.index for b in bt.leaves], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "trees.npz"), **out)


def gen_gca(meta):
    """gca.py:83 green_sources, :136 build_green_matrix, :182 aca, :285 operators."""
    out = {}
    m = mesh.build_sphere_mesh(3)
    t = cluster.build_cluster_tree(m, 16)
    bt = cluster.build_block_tree(t, t, 2.0)
    params = gca.GcaParams()
    node = t.nodes[3]
    src = gca.green_sources(node.lo, node.hi, params.delta, params.m, m.diameter())
    out["src_points"] = src.points; out["src_weights"] = src.weights
    out["src_normals"] = src.normals; out["src_roles"] = src.roles
    out["green_cluster"] = np.array([3])
    panels = t.panels(node)
    for eq, kappa in (("laplace", 0.0), ("helmholtz", 4.0)):
        spec = kernels.KernelSpec(eq, "single", kappa)
        for order in (3, 4):
            A = gca.build_green_matrix(m, panels, src, spec, order)
            out[f"green_{eq}_{order}"] = A
        A = gca.build_green_matrix(m, panels, src, spec, 3)
        res = gca.aca(A, params.epsilon)
        out[f"aca_{eq}_rows"] = res.row_pivots
        out[f"aca_{eq}_cols"] = res.col_pivots
        ops, _ = gca.build_interpolation_operators(m, bt, spec, params)
        cids = np.array(sorted(ops), dtype=np.int64)
        out[f"ops_{eq}_cids"] = cids
        piv = [ops[c].pivots_global for c in cids]
        out[f"ops_{eq}_ranks"] = np.array([len(p) for p in piv], dtype=np.int64)
        out[f"ops_{eq}_pivots"] = np.concatenate(piv)
        out[f"ops_{eq}_V3"] = ops[int(cids[0])].V
        meta[f"ops_L3_{eq}"] = sha(*[ops[c].V for c in cids])
    np.savez_compressed(os.path.join(HERE, "gca_L3.npz"), **out)


def _inline_params(maxsize=scheduler.DEFAULT_MAXSIZE):
    return scheduler.SchedulerParams(maxsize_bytes=maxsize, workers_per_backend=0,
                                     backends=(scheduler.BATCH_BACKEND,))


def _instrumented_lists(m, bt, spec, ops, params, orders):
    """Run the reference inline and record the executed list composition."""
    seen = []
    real = scheduler.execute_list

    def spy(lst, backend, ctx):
        if lst.case == "disjoint":
            blocks = [(b.leaf_id, len(b.row_panels), len(b.col_panels),
                       int(b.row_slots[0]), int(b.col_slots[0]), int(b.flagged))
                      for b in lst.items]
            seen.append(("disjoint", blocks))
        else:
            seen.append((lst.case, [(it.tri_x, it.tri_y, it.leaf_id, it.offset)
                                    for it in lst.items]))
        return real(lst, backend, ctx)

    scheduler.execute_list = spy
    try:
        M = scheduler.run_assembly(m, bt, spec, ops, ops, params, orders)
    finally:
        scheduler.execute_list = real
    return M, seen


def gen_assembly(meta):
    """scheduler.py:442 run_assembly in inline mode: checksums, payloads, lists."""
    meta["checksums"] = {}
    out = {}
    for L in (2, 3):
        m = mesh.build_sphere_mesh(L)
        t = cluster.build_cluster_tree(m, 16)
        bt = cluster.build_block_tree(t, t, 2.0)
        for eq, kappa in (("laplace", 0.0), ("helmholtz", 4.0)):
            ops, _ = gca.build_interpolation_operators(
                m, bt, kernels.KernelSpec(eq, "single", kappa), gca.GcaParams())
            for layer in ("single", "double"):
                spec = kernels.KernelSpec(eq, layer, kappa)
                for orders in ((3, 5), (2, 3)):
                    M = scheduler.run_assembly(m, bt, spec, ops, ops, _inline_params(), orders)
                    key = f"L{L}/{eq}/{layer}/{orders[0]}-{orders[1]}"
                    meta["checksums"][key] = M.checksum()
                    if L == 2 and orders == (3, 5):
                        out[f"L2_{eq}_{layer}"] = np.concatenate(
                            [M.payloads[l.index].ravel() for l in bt.leaves])
        if L == 3:
            ops, _ = gca.build_interpolation_operators(
                m, bt, kernels.KernelSpec("laplace", "single"), gca.GcaParams())
            for maxsize, tag in ((scheduler.DEFAULT_MAXSIZE, "8M"), (4096, "4K")):
                M, seen = _instrumented_lists(m, bt, kernels.KernelSpec("laplace", "single"),
                                              ops, _inline_params(maxsize), (3, 5))
                cases, lens, rec = [], [], []
                for case, items in seen:
                    cases.append(CASE_CODE[case])
                    lens.append(len(items))
                    for it in items:
                        r = list(it) + [0] * (6 - len(it))
                        rec.append(r)
                out[f"lists_{tag}_case"] = np.array(cases, dtype=np.int64)
                out[f"lists_{tag}_len"] = np.array(lens, dtype=np.int64)
                out[f"lists_{tag}_items"] = np.array(rec, dtype=np.int64)
                meta["checksums"][f"L3/laplace/single/3-5/maxsize{tag}"] = M.checksum()
    # C1: level-4 near-field only (BASELINE config 1), SURVEY §8(d)
    m = mesh.build_sphere_mesh(4)
    t = cluster.build_cluster_tree(m, 16)
    bt = cluster.build_block_tree(t, t, 2.0)
    near = cluster.BlockTree(bt.nodes, t, t, bt.eta, [l for l in bt.leaves if l.kind == "dense"])
    M = scheduler.run_assembly(m, near, kernels.KernelSpec("laplace", "single"), {}, {},
                               _inline_params(), (3, 5))
    meta["checksums"]["L4-near/laplace/single/3-5"] = M.checksum()
    np.savez_compressed(os.path.join(HERE, "assembly.npz"), **out)


def gen_potential_and_dump():
    """scheduler.py:508 potential_batch; h2.py:195 dump (GCAMAT01 wire bytes)."""
    out = {}
    m = mesh.build_sphere_mesh(2)
    pts = np.array([[0.0, 0.0, 1.7], [1.2, -0.8, 0.9], [0.1, 0.2, 0.3], [-0.4, 0.0, -0.2],
                    [3.0, 2.0, -1.0]])
    out["points"] = pts
    for name, spec in SPECS.items():
        for order in (2, 3):
            out[f"{name}_{order}"] = scheduler.potential_batch(m, spec, pts, order)
    np.savez_compressed(os.path.join(HERE, "potential_L2.npz"), **out)
    t = cluster.build_cluster_tree(m, 16)
    bt = cluster.build_block_tree(t, t, 2.0)
    M = scheduler.run_assembly(m, bt, SPECS["L-SLP"], {}, {}, _inline_params(), (3, 5))
    h2.dump(M, os.path.join(HERE, "L2_laplace_single.gcamat"))
    m3 = mesh.build_sphere_mesh(3)
    t3 = cluster.build_cluster_tree(m3, 16)
    bt3 = cluster.build_block_tree(t3, t3, 2.0)
    ops, _ = gca.build_interpolation_operators(m3, bt3, SPECS["L-SLP"], gca.GcaParams())
    M3 = scheduler.run_assembly(m3, bt3, SPECS["L-SLP"], ops, ops, _inline_params(), (2, 3))
    import gzip
    tmp = os.path.join(HERE, "L3_laplace_single_23.gcamat")
    h2.dump(M3, tmp)
    with open(tmp, "rb") as fh, open(tmp + ".gz", "wb") as gz:
        gz.write(gzip.compress(fh.read(), 9))
    os.remove(tmp)


def gen_p1():
    """P1 local matrices M[a][b] = integrate_pair(chart_x, chart_y, spec, rule,
    normal_y, basis_x=lambda_a, basis_y=lambda_b) (quadrature.py:223-271) on a
    small crankshaft surface (geometry from our generator, everything else
    from the reference), stored in the triangles' stored vertex order."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_1510_07244_b200.mesh import build_crankshaft_mesh
    g = build_crankshaft_mesh(2048, seed=1)
    m = mesh.make_surface_mesh(g.vertices, g.triangles)
    rng = np.random.default_rng(11)
    tri = m.triangles
    nt = m.num_triangles
    shared = np.zeros((nt, nt), dtype=np.int8)
    for a_ in range(3):
        for b_ in range(3):
            shared += (tri[:, a_][:, None] == tri[:, b_][None, :]).astype(np.int8)
    mid = m.midpoints()
    picks = {}
    disj = np.argwhere(shared == 0)
    d = np.linalg.norm(mid[disj[:, 0]] - mid[disj[:, 1]], axis=1)
    near = disj[np.argsort(d, kind="stable")[rng.choice(3000, 24, replace=False)]]
    far = disj[rng.choice(len(disj), 16, replace=False)]
    picks["disjoint"] = np.concatenate([near, far])
    for case, cnt in (("vertex", 1), ("edge", 2)):
        cand = np.argwhere(shared == cnt)
        picks[case] = cand[rng.choice(len(cand), 32, replace=False)]
    ids = rng.choice(nt, 24, replace=False)
    picks["identical"] = np.stack([ids, ids], axis=1)
    lam = [lambda p: 1.0 - p[:, 0], lambda p: p[:, 0] - p[:, 1], lambda p: p[:, 1]]
    out = {"vertices": m.vertices, "triangles": m.triangles}
    for case, pairs in picks.items():
        out[f"pairs_{case}"] = pairs
        n = 3 if case == "disjoint" else 5
        rule = quadrature.build_rule(case, n)
        perms = []
        for name in ("L-SLP", "L-DLP", "H-SLP", "H-DLP"):
            spec = SPECS[name]
            vals = np.zeros((len(pairs), 3, 3), dtype=np.complex128)
            for k, (tx, ty) in enumerate(pairs):
                cls = quadrature.classify_pair(m, int(tx), int(ty))
                assert cls.case == case
                if name == "L-SLP":
                    perms.append(list(cls.perm_x) + list(cls.perm_y))
                cx = mesh.chart(m, int(tx), cls.perm_x)
                cy = mesh.chart(m, int(ty), cls.perm_y)
                for a_ in range(3):
                    for b_ in range(3):
                        v = quadrature.integrate_pair(cx, cy, spec, rule, m.normals[int(ty)],
                                                      basis_x=lam[a_], basis_y=lam[b_])
                        vals[k, cls.perm_x[a_], cls.perm_y[b_]] = v
            out[f"p1_{case}_{name}"] = vals
        out[f"perms_{case}"] = np.array(perms, dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "p1_crank.npz"), **out)


def main():
    meta = {"reference": "gcabem " + getattr(gcabem, "__version__", "0.1.0"),
            "numpy": np.__version__}
    import numba
    meta["numba"] = numba.__version__
    for step in (gen_hashes,):
        step(meta)
    gen_rules_npz()
    gen_classification()
    gen_pair_values()
    gen_kernel_values()
    gen_trees()
    gen_gca(meta)
    gen_assembly(meta)
    gen_potential_and_dump()
    gen_p1()
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("ok")


if __name__ == "__main__":
    if sys.argv[1:] == ["p1"]:
        gen_p1()
        sys.exit(0)
    sys.exit(main())
