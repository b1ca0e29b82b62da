"""Host-side (CPU) parts of the drop-in, bit-exact against the reference."""
import hashlib
import os
from pathlib import Path

import numpy as np
import pytest

import oracle.setup_cpu as pk_numpy
from helpers import golden_ops, sphere_setup
from paper_1510_07244_b200 import cluster, gca, kernels, mesh, packaging, quadrature, scheduler


def sha(*a):
    h = hashlib.sha256()
    for x in a:
        h.update(np.ascontiguousarray(x).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("level", range(6))
def test_sphere_bitwise(golden, level):
    m = mesh.build_sphere_mesh(level)
    r = golden["sphere"][str(level)]
    assert (m.num_vertices, m.num_triangles) == (r["nv"], r["nt"])
    for name in ("vertices", "triangles", "normals", "gramians"):
        assert sha(getattr(m, name)) == r[name], name


def test_gauss_and_rules_bitwise(golden):
    for n, h in golden["gauss"].items():
        g = quadrature.gauss_legendre(int(n))
        assert sha(g.points, g.weights) == h
    for key, h in golden["rules"].items():
        case, n = key.split("/")
        r = quadrature.build_rule(case, int(n))
        assert sha(r.x_points, r.y_points, r.weights) == h, key
    for n, h in golden["duffy"].items():
        assert sha(*quadrature.duffy_panel_rule(int(n))) == h


def test_rule_cache_and_bounds():
    quadrature.clear_rule_cache()
    a = quadrature.build_rule("edge", 4)
    assert quadrature.build_rule("edge", 4) is a
    assert quadrature.rule_cache_stats() == {"builds": 1, "lookups": 2}
    with pytest.raises(ValueError):
        quadrature.build_rule("disjoint", 13)
    with pytest.raises(ValueError):
        quadrature.build_rule("nearby", 3)
    for case in quadrature.CASES:
        assert abs(quadrature.build_rule(case, 5).weights.sum() - 0.25) <= 1e-13


def test_classification_all_pairs_L2(gload):
    cls = gload("classify_L2.npz")["cls"]
    m = mesh.build_sphere_mesh(2)
    nt = m.num_triangles
    a, b = np.meshgrid(np.arange(nt), np.arange(nt), indexing="ij")
    case, px, py = quadrature.classify_pairs(m.triangles, a.ravel(), b.ravel())
    got = np.concatenate([case[:, None], px, py], axis=1).reshape(nt, nt, 7)
    assert np.array_equal(got.astype(np.int8), cls)
    c = quadrature.classify_pair(m, 3, 3)
    assert c.case == "identical" and c.perm_x == (0, 1, 2)


def test_classify_rejects_three_shared():
    V = np.array([[0, 0, 0.0], [1, 0, 0], [0, 1, 0], [0, 0, 1]])
    T = np.array([[0, 1, 2], [0, 2, 1], [0, 1, 3], [1, 2, 3]])
    m = mesh.make_surface_mesh(V, T, validate=False)
    with pytest.raises(mesh.MeshError):
        quadrature.classify_pair(m, 0, 1)


@pytest.mark.parametrize("level", [3, 4])
def test_trees_bitwise(gload, level):
    g = gload("trees.npz")
    m, t, bt = sphere_setup(level)
    assert np.array_equal(t.permutation, g[f"L{level}_perm"])
    assert np.array_equal([n.start for n in t.nodes], g[f"L{level}_start"])
    assert np.array_equal([n.size for n in t.nodes], g[f"L{level}_size"])
    assert np.array_equal(np.array([n.lo for n in t.nodes]), g[f"L{level}_lo"])
    kind = {"admissible": 0, "dense": 1, "split": 2}
    got = np.array([(b.row, b.col, kind[b.kind], len(b.children)) for b in bt.nodes])
    assert np.array_equal(got, g[f"L{level}_blocks"])
    assert np.array_equal([b.index for b in bt.leaves], g[f"L{level}_leaves"])


CODE = {"disjoint": 0, "vertex": 1, "edge": 2, "identical": 3}


@pytest.mark.parametrize("tag,maxsize", [("8M", 8 * 2 ** 20), ("4K", 4096)])
def test_package_assignment_bitwise(gload, tag, maxsize):
    """Disjoint list boundaries, split blocks, singular items and singular list
    boundaries equal the reference's inline run (scheduler.py:442-505)."""
    g = gload("assembly.npz")
    m, t, bt = sphere_setup(3)
    ops = golden_ops(gload("gca_L3.npz"), "laplace")
    pk = packaging.make_packages(m.triangles, bt, ops, ops, maxsize)
    seq = packaging.inline_lists(pk)
    assert np.array_equal([CODE[c] for c, _ in seq], g[f"lists_{tag}_case"])
    assert np.array_equal([len(x) for _, x in seq], g[f"lists_{tag}_len"])
    rec = []
    for c, x in seq:
        for k in x:
            if c == "disjoint":
                lf = pk.blk_leaf[k]
                rec.append([pk.leaf_ids[lf], pk.blk_nr[k], pk.blk_nc[k], pk.blk_r0[k],
                            pk.blk_c0[k], int(pk.leaf_flagged[lf])])
            else:
                rec.append([pk.item_tri_x[k], pk.item_tri_y[k], pk.leaf_ids[pk.item_leaf[k]],
                            pk.item_offset[k], 0, 0])
    assert np.array_equal(np.array(rec), g[f"lists_{tag}_items"])


def test_split_and_listbuilder_api():
    blk = scheduler.WorkBlock(0, np.arange(10), np.arange(7), np.arange(10), np.arange(7), False)
    parts = scheduler.split_block(blk, 32 * 16)
    assert sum(p.num_pairs for p in parts) == 70
    assert all(p.nbytes <= 32 * 16 for p in parts)
    assert [(len(p.row_panels), len(p.col_panels)) for p in parts] == \
        [(r[1], r[3]) for r in pk_numpy._split(10, 7, 32 * 16)]
    out = []
    lb = scheduler.ListBuilder("disjoint", 32 * 40, out.append)
    for p in parts:
        lb._add(p, p.nbytes)
    lb.flush()
    lid, n = pk_numpy._greedy_lists(np.array([p.nbytes for p in parts]), 32 * 40)
    assert n == len(out)
    with pytest.raises(scheduler.SchedulerConfigError):
        scheduler.ListBuilder("disjoint", 16, out.append)
    with pytest.raises(scheduler.SchedulerConfigError):
        scheduler.Backend("x", "gpu-magic")


def test_reference_backend_kinds_construct():
    """Reference-style backends (scheduler.py:51-66 kinds) construct and
    resolve through SchedulerParams exactly as in the reference; they run on
    the CUDA path."""
    b = scheduler.Backend("batch", "batch")
    s = scheduler.Backend("scalar", "scalar-reference")
    assert b.affinity == "batch" and s.kind == "scalar-reference" and b.devices == (0,)
    params = scheduler.SchedulerParams(
        backends=(s, b), affinity={"disjoint": "batch", "vertex": "scalar",
                                   "edge": "scalar", "identical": "scalar"})
    assert params.backend_for("disjoint") is b and params.backend_for("edge") is s
    assert params.backend_for("unknown") is s
    assert scheduler.BATCH_BACKEND.kind == "batch"
    assert scheduler.SCALAR_BACKEND.kind == "scalar-reference"


def test_package_cache_one_entry_per_tree():
    """A new operator set on the same block tree replaces the cached packages
    (the cache grew by one entry per operator set)."""
    from paper_1510_07244_b200 import mesh as mesh_mod
    m = mesh_mod.build_sphere_mesh(2)
    t = cluster.build_cluster_tree(m, 16)
    bt = cluster.build_block_tree(t, t, 2.0)
    near = cluster.BlockTree(bt.nodes, t, t, bt.eta, [l for l in bt.leaves if l.kind == "dense"])
    scheduler.clear_package_cache()
    for _ in range(5):
        ops = {}
        scheduler.packages_for(m, near, ops, ops, scheduler.DEFAULT_MAXSIZE)
    assert sum(1 for k in scheduler._pk_cache if k[1] == id(near)) == 1
    scheduler.clear_package_cache()


def test_green_sources_bitwise(gload):
    g = gload("gca_L3.npz")
    m, t, _ = sphere_setup(3)
    node = t.nodes[int(g["green_cluster"][0])]
    s = gca.green_sources(node.lo, node.hi, 1.0, 6, m.diameter())
    for name in ("points", "weights", "normals", "roles"):
        assert np.array_equal(getattr(s, name), g[f"src_{name}"]), name


@pytest.mark.parametrize("eq", ["laplace", "helmholtz"])
def test_aca_pivots_on_reference_green(gload, eq):
    g = gload("gca_L3.npz")
    res = gca.aca(g[f"green_{eq}_3"], 1e-4)
    assert np.array_equal(res.row_pivots, g[f"aca_{eq}_rows"])
    assert np.array_equal(res.col_pivots, g[f"aca_{eq}_cols"])


def test_kernel_values_bitwise(gload):
    g = gload("kernel_values.npz")
    specs = {"L-SLP": kernels.KernelSpec("laplace", "single"),
             "L-DLP": kernels.KernelSpec("laplace", "double"),
             "H-SLP": kernels.KernelSpec("helmholtz", "single", 4.0),
             "H-DLP": kernels.KernelSpec("helmholtz", "double", 4.0)}
    for name, spec in specs.items():
        got = kernels.eval_batch(spec, g["xs"], g["ys"], g["ns"] if spec.needs_normal else None)
        assert np.array_equal(got, g[name]), name
    with pytest.raises(ValueError):
        kernels.KernelSpec("helmholtz", "single", -1.0)
    with pytest.raises(ValueError):
        kernels.eval(specs["L-SLP"], np.ones(3), np.ones(3))


def test_shard_leaves_partition():
    m, t, bt = sphere_setup(4)
    near = cluster.BlockTree(bt.nodes, t, t, bt.eta, [l for l in bt.leaves if l.kind == "dense"])
    pk = packaging.make_packages(m.triangles, near, {}, {}, 8 << 20)
    for n in (1, 2, 3, 8):
        sh = packaging.shard_leaves(pk, n, 81, [1250, 3125, 3750])
        assert sh[0][0] == 0 and sh[-1][1] == pk.leaf_ids.size
        assert all(a[1] == b[0] for a, b in zip(sh, sh[1:]))
        assert sum(len(pk.device_items(lo, hi)[0]) for lo, hi in sh) == pk.num_items
        assert sum(len(pk.device_blocks(lo, hi)) for lo, hi in sh) == pk.num_blocks


@pytest.mark.parametrize("level,maxsize", [(3, 8 << 20), (4, 8 << 20), (4, 20000), (5, 8 << 20)])
def test_native_packaging_matches_numpy(gload, level, maxsize):
    """csrc/packaging.cpp vs the numpy restatement (itself pinned at L3)."""
    m, t, bt = sphere_setup(level)
    if level == 3:
        ops = golden_ops(gload("gca_L3.npz"), "laplace")
    else:  # synthetic operators: the first min(20, |t|) panels of each cluster
        ids = {l.row for l in bt.leaves if l.kind == "admissible"} | \
              {l.col for l in bt.leaves if l.kind == "admissible"}
        ops = {c: gca.InterpolationOperator(c, None, t.panels(t.nodes[c])[::-1][:20], None)
               for c in ids}
    a = packaging.make_packages(m.triangles, bt, ops, ops, maxsize)
    b = pk_numpy.make_packages(m.triangles, bt, ops, ops, maxsize)
    assert np.array_equal(a.leaf_shape, b.leaf_shape)
    assert np.array_equal(a.leaf_base, b.leaf_base)
    assert np.array_equal(a.leaf_flagged, b.leaf_flagged)
    for f in ("blk_leaf", "blk_r0", "blk_nr", "blk_c0", "blk_nc", "blk_list", "item_case",
              "item_tri_x", "item_tri_y", "item_leaf", "item_offset", "item_src_block", "perms"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert a.n_disjoint_lists == b.n_disjoint_lists
    # same panel sequences through the two layouts
    for k in np.linspace(0, a.leaf_ids.size - 1, 200).astype(int):
        nr, nc = a.leaf_shape[k]
        assert np.array_equal(a.panels[a.leaf_rows_at[k]:a.leaf_rows_at[k] + nr],
                              b.panels[b.leaf_rows_at[k]:b.leaf_rows_at[k] + nr])
        assert np.array_equal(a.panels[a.leaf_cols_at[k]:a.leaf_cols_at[k] + nc],
                              b.panels[b.leaf_cols_at[k]:b.leaf_cols_at[k] + nc])


@pytest.mark.parametrize("nstages", [2, 3, 7])
def test_staged_packages_equal_whole_tree(nstages):
    """Leaf-range packages (the staged assembly's) are the whole-tree packages
    restricted to their leaves: same blocks, same corrective items, payload
    offsets shifted by the range's base; leaf_layout gives the same shapes."""
    m, t, bt = sphere_setup(4)
    ids = {l.row for l in bt.leaves if l.kind == "admissible"} | \
          {l.col for l in bt.leaves if l.kind == "admissible"}
    ops = {c: gca.InterpolationOperator(c, None, t.panels(t.nodes[c])[::-1][:20], None)
           for c in ids}
    full = packaging.make_packages(m.triangles, bt, ops, ops, 20000)
    lids, shape, base = packaging.leaf_layout(bt, ops, ops)
    assert np.array_equal(lids, full.leaf_ids)
    assert np.array_equal(shape, full.leaf_shape)
    assert np.array_equal(base, full.leaf_base)
    L = full.leaf_ids.size
    edges = np.linspace(0, L, nstages + 1).astype(int)
    blk, items = [], []
    for lo, hi in zip(edges[:-1], edges[1:]):
        pk = packaging.make_packages(m.triangles, bt, ops, ops, 20000, leaf_range=(lo, hi))
        assert np.array_equal(pk.leaf_shape, full.leaf_shape[lo:hi])
        assert np.array_equal(pk.leaf_base, full.leaf_base[lo:hi + 1] - full.leaf_base[lo])
        blk.append(np.stack([pk.blk_leaf + lo, pk.blk_r0, pk.blk_nr, pk.blk_c0, pk.blk_nc]))
        items.append(np.stack([pk.item_case.astype(np.int64), pk.item_tri_x, pk.item_tri_y,
                               pk.item_leaf + lo, pk.item_offset]))
    want_blk = np.stack([full.blk_leaf, full.blk_r0, full.blk_nr, full.blk_c0, full.blk_nc])
    assert np.array_equal(np.concatenate(blk, axis=1), want_blk)
    got = np.concatenate(items, axis=1)
    want = np.stack([full.item_case.astype(np.int64), full.item_tri_x, full.item_tri_y,
                     full.item_leaf, full.item_offset])
    assert got.shape == want.shape
    assert np.array_equal(got[:, np.lexsort(got[::-1])], want[:, np.lexsort(want[::-1])])


@pytest.mark.parametrize("nstages", [1, 3, 5, 9])
def test_staged_packages_ranges(nstages):
    """scheduler.StagedPackages: leaf ranges tile [0, L) in order, range 0 is
    the first L/64 leaves, later ranges grow with the payload; each stage's
    packages are make_packages(leaf_range) of its range; the layout equals the
    whole-tree packages' (native gcabem_leaf_layout)."""
    from paper_1510_07244_b200 import scheduler
    m, t, bt = sphere_setup(4)
    ids = {l.row for l in bt.leaves if l.kind == "admissible"} | \
          {l.col for l in bt.leaves if l.kind == "admissible"}
    ops = {c: gca.InterpolationOperator(c, None, t.panels(t.nodes[c])[::-1][:20], None)
           for c in ids}
    full = packaging.make_packages(m.triangles, bt, ops, ops, 20000)
    sp = scheduler.StagedPackages(m, bt, ops, ops, 20000, nstages)
    L = full.leaf_ids.size
    assert np.array_equal(sp.leaf_base, full.leaf_base)
    assert np.array_equal(sp.leaf_shape, full.leaf_shape)
    assert sp.ranges[0][0] == 0 and sp.ranges[-1][1] == L
    assert all(a[1] == b[0] and a[0] < a[1] for a, b in zip(sp.ranges, sp.ranges[1:]))
    assert len(sp.ranges) <= nstages
    if nstages > 1:
        assert sp.ranges[0] == (0, max(1, L // 64))
    for k, rng in enumerate(sp.ranges):
        pk = sp.stage(k)
        ref = packaging.make_packages(m.triangles, bt, ops, ops, 20000, leaf_range=rng)
        for f in ("blk_leaf", "blk_r0", "blk_nr", "blk_c0", "blk_nc", "item_case", "item_tri_x",
                  "item_tri_y", "item_leaf", "item_offset", "perms", "leaf_base"):
            assert np.array_equal(getattr(pk, f), getattr(ref, f)), (k, f)
        assert sp.offset(k) == full.leaf_base[rng[0]]


_ACA_BUILDS_SNIPPET = """
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1510_07244_b200 import gca
rng = np.random.default_rng(7)
mats = []
for nr in (5, 17, 40, 96):
    for cplx in (False, True):
        u = rng.standard_normal((nr, 12)) + (1j * rng.standard_normal((nr, 12)) if cplx else 0)
        v = rng.standard_normal((12, 67)) + (1j * rng.standard_normal((12, 67)) if cplx else 0)
        a = u @ v + 1e-9 * rng.standard_normal((nr, 67))
        mats.append(np.ascontiguousarray(a))
out = {}
for i, a in enumerate(mats):
    cplx = np.iscomplexobj(a)
    flat = a.view(np.float64).ravel() if cplx else a.ravel()
    r = gca.aca_batch(flat, np.array([0, a.shape[0]]), 67, cplx, 1e-6, nthreads=1)[0]
    out[f"rows{i}"], out[f"cols{i}"], out[f"res{i}"] = r[0], r[1], np.float64(r[2])
    op = gca._operator_from_green(i, np.arange(a.shape[0]), a, 1e-6)
    out[f"V{i}"] = op.V
np.savez(sys.argv[2], **out)
"""


def test_aca_builds_agree_bitwise(tmp_path):
    """The AVX2 and the baseline x86-64 builds of aca.cpp (GCABEM_ACA_BASELINE
    forces the latter) give bitwise identical pivots, residuals and V: same
    IEEE operations in the same order, vector or scalar."""
    import subprocess
    import sys
    script = tmp_path / "aca_builds.py"
    script.write_text(_ACA_BUILDS_SNIPPET)
    root = str(Path(__file__).resolve().parents[1])
    env = dict(os.environ)
    subprocess.run([sys.executable, str(script), root, str(tmp_path / "avx2.npz")], check=True,
                   env=env)
    env["GCABEM_ACA_BASELINE"] = "1"
    subprocess.run([sys.executable, str(script), root, str(tmp_path / "base.npz")], check=True,
                   env=env)
    a, b = np.load(tmp_path / "avx2.npz"), np.load(tmp_path / "base.npz")
    assert set(a.files) == set(b.files)
    for k in a.files:
        assert a[k].shape == b[k].shape and a[k].tobytes() == b[k].tobytes(), k


@pytest.mark.parametrize("eq,kappa", [("laplace", 0.0), ("helmholtz", 4.0)])
def test_native_aca_matches_numpy_restatement(eq, kappa):
    """csrc/aca.cpp (threaded batch) vs the numpy ACA on every admissible
    cluster of the L4 sphere, Green matrices from the oracle (CPU)."""
    import oracle.setup_cpu as aca_numpy
    import oracle
    m, t, bt = sphere_setup(4)
    ids = sorted({l.row for l in bt.leaves if l.kind == "admissible"})
    mats = []
    for cid in ids[:120]:
        node = t.nodes[cid]
        src = gca.green_sources(node.lo, node.hi, 1.0, 6, m.diameter())
        mats.append(oracle.green_matrix(m.vertices, m.triangles, m.gramians, t.panels(node),
                                        src.points, src.weights, src.normals, src.roles, eq,
                                        kappa, 3))
    rows_at = np.concatenate([[0], np.cumsum([a.shape[0] for a in mats])])
    flat = np.concatenate([np.ascontiguousarray(a).view(np.float64).ravel() for a in mats])
    got = gca.aca_batch(flat, rows_at, 432, eq == "helmholtz", 1e-4, nthreads=4)
    for A, (r, c, _) in zip(mats, got):
        rr, cc = aca_numpy.aca(A, 1e-4)
        assert np.array_equal(r, rr) and np.array_equal(c, cc)


@pytest.mark.parametrize("eq,kappa", [("laplace", 0.0), ("helmholtz", 4.0)])
def test_native_gca_operator_matches_numpy_restatement(eq, kappa):
    """csrc/aca.cpp gca_operator (ACA + Jacobi-SVD cond check + LU solve with
    two refinement sweeps) vs numpy/LAPACK on L4 clusters: identical pivots,
    V within roundoff x cond of the pivot block; and V reproduces the pivot
    rows (V[rows] = I), the defining property of the interpolation."""
    import oracle.setup_cpu as aca_numpy
    import oracle
    m, t, bt = sphere_setup(4)
    ids = sorted({l.row for l in bt.leaves if l.kind == "admissible"})
    for cid in ids[:40]:
        node = t.nodes[cid]
        src = gca.green_sources(node.lo, node.hi, 1.0, 6, m.diameter())
        A = oracle.green_matrix(m.vertices, m.triangles, m.gramians, t.panels(node), src.points,
                                src.weights, src.normals, src.roles, eq, kappa, 3)
        op = gca._operator_from_green(cid, t.panels(node), A, 1e-4)
        rows, V = aca_numpy.solve_operator(A, 1e-4)
        assert np.array_equal(op.pivots_local, rows)
        assert np.array_equal(op.pivots_global, t.panels(node)[rows])
        assert op.V.dtype == V.dtype and op.V.shape == V.shape
        assert np.max(np.abs(op.V - V)) <= 1e-9 * np.max(np.abs(V)), cid
        assert np.max(np.abs(op.V[rows] - np.eye(rows.size))) <= 1e-10


def test_native_gca_operator_errors():
    with pytest.raises(gca.GcaError, match="cluster 7: zero Green matrix"):
        gca._operator_from_green(7, np.arange(3), np.zeros((3, 4)), 1e-4)


@pytest.mark.parametrize("level", [5, 6])
def test_native_trees_match_python(level):
    """csrc/trees.cpp vs the Python restatements (pinned at L3/L4 by golden)."""
    m = mesh.build_sphere_mesh(level)
    a = cluster.build_cluster_tree(m, 16)
    b = cluster._build_cluster_tree_py(m, 16)
    assert np.array_equal(a.permutation, b.permutation)
    assert [(n.start, n.size, n.children) for n in a.nodes] == \
        [(n.start, n.size, n.children) for n in b.nodes]
    assert np.array_equal(np.array([n.lo for n in a.nodes]), np.array([n.lo for n in b.nodes]))
    if level == 5:
        ba = cluster.build_block_tree(a, a, 2.0)
        bb = cluster._build_block_tree_py(b, b, 2.0)
        assert len(ba.nodes) == len(bb.nodes)
        assert list(ba.nodes) == list(bb.nodes)
        assert list(ba.leaves) == list(bb.leaves)


def test_gcamat01_roundtrip_reference_files(tmp_path):
    """h2.load reads the reference's GCAMAT01 files and h2.dump writes them
    back byte for byte (h2.py:195-314)."""
    import gzip
    import os
    from paper_1510_07244_b200 import h2
    g = os.path.join(os.path.dirname(__file__), "golden")
    l3 = tmp_path / "l3.gcamat"
    l3.write_bytes(gzip.decompress(open(os.path.join(g, "L3_laplace_single_23.gcamat.gz"),
                                        "rb").read()))
    for src in (os.path.join(g, "L2_laplace_single.gcamat"), str(l3)):
        M = h2.load(src)
        out = tmp_path / "out.gcamat"
        h2.dump(M, out)
        assert out.read_bytes() == open(src, "rb").read()
    import json
    ref = json.load(open(os.path.join(g, "golden.json")))["checksums"]
    assert h2.load(str(l3)).checksum() == ref["L3/laplace/single/2-3"]


def test_device_matvec_tables_restate_reference_matvec():
    """h2._leaf_arrays (the tables the device product runs on) drive the staged
    algorithm of csrc/h2_matvec.cu to the reference leaf-loop product, on a
    GCAMATO1 reference file (L3 Laplace SLP): no device needed."""
    import gzip
    import os
    import h2_numpy
    from paper_1510_07244_b200 import h2
    g = os.path.join(os.path.dirname(__file__), "golden")
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "l3.gcamat")
        with open(path, "wb") as fh:
            fh.write(gzip.decompress(open(os.path.join(g, "L3_laplace_single_23.gcamat.gz"),
                                          "rb").read()))
        M = h2.load(path)
    rng = np.random.default_rng(3)
    x = rng.standard_normal(M.shape[1]) + 1j * rng.standard_normal(M.shape[1])
    ref = h2_numpy.matvec_reference(M, x)
    got = h2_numpy.matvec_staged(M, x)
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_crankshaft_mesh_closed_oriented_deterministic():
    m = mesh.build_crankshaft_mesh(65536, seed=0)
    assert m.num_triangles == 65536
    e = np.concatenate([m.triangles[:, [0, 1]], m.triangles[:, [1, 2]], m.triangles[:, [2, 0]]])
    key = e[:, 0] * m.num_vertices + e[:, 1]
    rev = e[:, 1] * m.num_vertices + e[:, 0]
    assert np.unique(key).size == key.size              # each directed edge once
    assert np.array_equal(np.sort(key), np.sort(rev))   # closed, consistently oriented
    assert m.num_vertices - key.size // 2 + m.num_triangles == 2
    V = m.vertices[m.triangles]
    assert np.einsum("ij,ij->i", V[:, 0], np.cross(V[:, 1], V[:, 2])).sum() > 0  # outward
    m2 = mesh.build_crankshaft_mesh(65536, seed=0)
    assert np.array_equal(m.vertices, m2.vertices)
    assert not np.array_equal(m.vertices, mesh.build_crankshaft_mesh(65536, seed=1).vertices)


def test_p1_numpy_restatement_matches_reference_golden(gload):
    """The test-side P1 oracle reproduces the reference's integrate_pair with
    P1 bases (golden p1_crank.npz, generated from the reference)."""
    import p1_numpy
    from paper_1510_07244_b200 import kernels as K, quadrature as Q
    g = gload("p1_crank.npz")
    m = mesh.make_surface_mesh(g["vertices"], g["triangles"])
    specs = {"L-SLP": K.KernelSpec("laplace", "single"), "L-DLP": K.KernelSpec("laplace", "double"),
             "H-SLP": K.KernelSpec("helmholtz", "single", 4.0),
             "H-DLP": K.KernelSpec("helmholtz", "double", 4.0)}
    for case in ("disjoint", "vertex", "edge", "identical"):
        pairs, perms = g[f"pairs_{case}"], g[f"perms_{case}"]
        rule = Q.build_rule(case, 3 if case == "disjoint" else 5)
        for name, spec in specs.items():
            ref = g[f"p1_{case}_{name}"]
            for k, (tx, ty) in enumerate(pairs):
                got = p1_numpy.local_matrix(m, spec, rule, tx, ty, perms[k, :3], perms[k, 3:])
                scale = np.max(np.abs(ref[k]))
                assert np.max(np.abs(got - ref[k])) <= 1e-12 * scale, (case, name, k)


def test_oracle_p1_batch_matches_reference_golden(gload):
    """oracle/p1_cpu.py (the C4 cpu_baseline of bench.py) reproduces the
    reference's integrate_pair with P1 bases on the golden pairs."""
    from oracle import p1_cpu
    g = gload("p1_crank.npz")
    m = mesh.make_surface_mesh(g["vertices"], g["triangles"])
    kinds = {"L-SLP": ("laplace", "single", 0.0), "L-DLP": ("laplace", "double", 0.0),
             "H-SLP": ("helmholtz", "single", 4.0), "H-DLP": ("helmholtz", "double", 4.0)}
    for case in ("disjoint", "vertex", "edge", "identical"):
        pairs, perms = g[f"pairs_{case}"], g[f"perms_{case}"]
        for name, (eq, layer, kappa) in kinds.items():
            ref = g[f"p1_{case}_{name}"]
            got = p1_cpu.local_matrices(m.vertices, m.triangles, m.normals, m.gramians, eq,
                                        layer, kappa, case, 3 if case == "disjoint" else 5,
                                        pairs[:, 0], pairs[:, 1], perms[:, :3], perms[:, 3:])
            scale = np.max(np.abs(ref), axis=(1, 2))
            assert np.all(np.max(np.abs(got - ref), axis=(1, 2)) <= 1e-12 * scale), (case, name)


def test_staged_packages_prepare_hook_and_errors(monkeypatch):
    """The packaging threads run prepare(k, packages) before range k is served
    (the staged assembly builds the device layout there); an exception in it
    reaches the caller through stage(), whichever worker raised it."""
    m, t, bt = sphere_setup(4)
    ids = {l.row for l in bt.leaves if l.kind == "admissible"} | \
          {l.col for l in bt.leaves if l.kind == "admissible"}
    ops = {c: gca.InterpolationOperator(c, None, t.panels(t.nodes[c])[::-1][:20], None)
           for c in ids}
    for workers in (1, 2, 3):
        monkeypatch.setattr(scheduler, "PACK_WORKERS", workers)
        seen = []
        sp = scheduler.StagedPackages(m, bt, ops, ops, 20000, 6,
                                      prepare=lambda k, pk: seen.append((k, pk.leaf_ids.size)))
        for k in range(len(sp.ranges)):
            pk = sp.stage(k)
            assert (k, pk.leaf_ids.size) in seen
        assert sorted(k for k, _ in seen) == list(range(len(sp.ranges)))

        def boom(k, pk):
            if k == 3:
                raise RuntimeError("layout failed")
        sp = scheduler.StagedPackages(m, bt, ops, ops, 20000, 6, prepare=boom)
        with pytest.raises(RuntimeError, match="layout failed"):
            for k in range(len(sp.ranges)):
                sp.stage(k)


def test_operator_map_behaves_like_the_dict():
    """gca.OperatorMap (the GCA build's result: operators materialised on
    access from the flat arrays) against the plain dict of the same
    operators: lookups, order, length, membership, mutation, and the flat
    pivot table packaging reads (the same as the generic walk)."""
    rng = np.random.default_rng(3)
    ids = np.array([2, 5, 6, 11, 40], np.int64)
    sizes = np.array([4, 7, 3, 9, 5], np.int64)
    ranks = np.array([2, 3, 1, 4, 2], np.int64)
    starts = np.array([0, 4, 11, 14, 23], np.int64)
    perm = rng.permutation(28).astype(np.int64)
    rows = np.concatenate([rng.choice(n, r, replace=False) for n, r in zip(sizes, ranks)])
    V = rng.standard_normal(int(np.sum(sizes * ranks))) + 1j * rng.standard_normal(
        int(np.sum(sizes * ranks)))
    om = gca.OperatorMap(ids, starts, sizes, ranks, rows, perm, V)
    ref, ro, vo = {}, 0, 0
    for c, s0, n, r in zip(ids, starts, sizes, ranks):
        loc = rows[ro:ro + r]
        ref[int(c)] = (loc, perm[s0 + loc], V[vo:vo + n * r].reshape(n, r))
        ro += r
        vo += n * r
    assert list(om) == sorted(ref) and len(om) == len(ref)
    assert 5 in om and 7 not in om and "x" not in om
    for c, (loc, glob, v) in ref.items():
        op = om[c]
        assert op is om[c]   # materialised once
        assert np.array_equal(op.pivots_local, loc) and np.array_equal(op.pivots_global, glob)
        assert np.array_equal(op.V, v)
    with pytest.raises(KeyError):
        om[3]
    at, piv = om.pivot_arrays(30)
    assert packaging._op_arrays(dict(om.items()), 30)[0].tolist() == at.tolist()
    assert np.array_equal(packaging._op_arrays(dict(om.items()), 30)[1], piv)
    # clusters outside the tree are left out, as by the generic walk
    at8, piv8 = om.pivot_arrays(8)
    g8 = packaging._op_arrays({k: v for k, v in om.items()}, 8)
    assert np.array_equal(at8, g8[0]) and np.array_equal(piv8, g8[1])
    # mutation: replace, delete, add; the flat table is withdrawn
    new = gca.InterpolationOperator(99, np.array([0]), np.array([7]), np.zeros((1, 1)))
    om[6] = new
    del om[11]
    om[50] = new
    assert om[6] is new and 11 not in om and 50 in om
    assert list(om) == [2, 5, 6, 40, 50] and len(om) == 5
    assert om.pivot_arrays(60) is None
    with pytest.raises(KeyError):
        del om[11]
