"""GPU parity: the sm_100a path through the C ABI against the oracle/golden.

Tolerance (north_star): entries within 1e-12 relative in FP64; reference
roundoff entries (|ref| < 1e-9 * leaf max, e.g. DLP identical pairs) within
1e-12 of the leaf-block max. Integer packaging is
bit-exact (tests/test_host.py).
"""
import numpy as np
import pytest

import oracle
from helpers import (SPECS, golden_ops, leaf_max_of, oracle_assemble, oracle_entries,
                     p2_check, p2_entries, packages_for, sphere_setup)
from paper_1510_07244_b200 import (cluster, gca, kernels, mesh, packaging, pairquad,
                                   quadrature, scheduler, solver)

pytestmark = pytest.mark.gpu
TOL = 1e-12


def rel_err(got, ref, floor=None):
    """Max relative error; roundoff entries (|ref| < 1e-9 max) use the max,
    and `floor` (an entry-magnitude scale) bounds the denominator from below
    for sets that are entirely reference roundoff (DLP identical pairs)."""
    mag = np.abs(ref)
    scale = np.where(mag < 1e-9 * mag.max(), mag.max(), mag)
    if floor is not None:
        scale = np.maximum(scale, floor)
    return float(np.max(np.abs(got - ref) / scale))


def spec_of(name):
    eq, layer, kappa = SPECS[name]
    return kernels.KernelSpec(eq, layer, kappa)


@pytest.fixture(scope="module")
def pv(gload):
    return gload("pair_values_L3.npz")


@pytest.mark.parametrize("name", list(SPECS))
def test_pair_values_raw_charts(pv, name):
    """pairquad.pair_values (pairquad.py:95) on caller charts vs the reference."""
    spec = spec_of(name)
    for rn in (3, 5):
        r = quadrature.build_rule("disjoint", rn)
        a = [pv[f"raw_{k}"] for k in ("ox", "e1x", "e2x", "gx", "oy", "e1y", "e2y", "gy")]
        got = pairquad.pair_values(spec, *a, pv["raw_ny"] if spec.needs_normal else None,
                                   r.x_points, r.y_points, r.weights)
        assert rel_err(got, pv[f"raw_{rn}_{name}"]) <= TOL


@pytest.mark.parametrize("case", ["disjoint", "vertex", "edge", "identical"])
@pytest.mark.parametrize("name", list(SPECS))
def test_batch_quadrature_golden(pv, case, name):
    """scheduler.batch_quadrature (scheduler.py:235) on device vs reference outputs."""
    m = mesh.build_sphere_mesh(3)
    spec = spec_of(name)
    orders = (1, 2, 3, 4, 5, 7) if case == "disjoint" else (2, 3, 5, 7)
    px = pv[f"{case}_perm_x"] if case != "disjoint" else None
    py = pv[f"{case}_perm_y"] if case != "disjoint" else None
    for n in orders:
        got = scheduler.batch_quadrature(scheduler.CUDA_BACKEND, case, m, spec,
                                         quadrature.build_rule(case, n), pv[f"{case}_tri_x"],
                                         pv[f"{case}_tri_y"], px, py)
        # coplanar identical DLP pairs are pure roundoff in the reference
        # (~1e-33); bound them by 1e-12 of the pair's SLP magnitude
        floor = np.abs(pv[f"{case}_{n}_{name[0]}-SLP"]) if spec.needs_normal else None
        assert rel_err(got, pv[f"{case}_{n}_{name}"], floor) <= TOL, (case, n)


@pytest.mark.parametrize("name", list(SPECS))
@pytest.mark.parametrize("orders", [(3, 5), (2, 3), (4, 5), (7, 7)])
def test_run_assembly_L3(gload, name, orders):
    """Full fused device assembly vs oracle over the same (bit-exact) packages."""
    eq, layer, kappa = SPECS[name]
    m, bt, ops, pk = packages_for(3, eq, gload("gca_L3.npz"))
    M = scheduler.run_assembly(m, bt, kernels.KernelSpec(eq, layer, kappa), ops, ops,
                               scheduler.SchedulerParams(), orders)
    ref = oracle_assemble(m, pk, eq, layer, kappa, orders)
    ok, worst, nfb = p2_check(pk, M.buffer, ref, TOL, m, (eq, layer, kappa), orders)
    assert ok, (worst, nfb)
    for leaf in bt.leaves:  # payload views, shapes as make_payloads
        assert M.payloads[leaf.index].base is not None
    assert set(M.payloads) == {l.index for l in bt.leaves}


def test_c1_near_field_L4():
    """BASELINE config 1: L4 sphere, Laplace SLP, near field only, orders 3/5."""
    m, bt, ops, pk = packages_for(4, "laplace", near_only=True)
    stats = scheduler.AssemblyStats()
    M = scheduler.run_assembly(m, bt, kernels.KernelSpec("laplace", "single"), {}, {},
                               scheduler.SchedulerParams(), (3, 5), stats)
    ref = oracle_assemble(m, pk, "laplace", "single", 0.0, (3, 5))
    ok, worst, _ = p2_check(pk, M.buffer, ref, TOL)
    assert ok, worst
    assert stats.corrective_items == 26576
    assert stats.block_pairs == 653312


def test_small_maxsize_split_blocks(gload):
    """4 KiB lists force split_block on every leaf; results must not change."""
    m, t, bt = sphere_setup(3)
    ops = golden_ops(gload("gca_L3.npz"), "helmholtz")
    spec = kernels.KernelSpec("helmholtz", "double", 4.0)
    a = scheduler.run_assembly(m, bt, spec, ops, ops, scheduler.SchedulerParams(), (3, 5))
    b = scheduler.run_assembly(m, bt, spec, ops, ops,
                               scheduler.SchedulerParams(maxsize_bytes=4096), (3, 5))
    assert np.array_equal(a.buffer, b.buffer)  # device arithmetic is order-free per entry


def test_multi_device_shards_equal_single(gload):
    """Leaf-range sharding (one plan per shard) gives the same payload."""
    m, t, bt = sphere_setup(3)
    ops = golden_ops(gload("gca_L3.npz"), "laplace")
    spec = kernels.KernelSpec("laplace", "double")
    # bitwise with per-pair evaluation (mirror=False): the split of the leaves
    # does not change any entry's arithmetic
    one = scheduler.run_assembly(m, bt, spec, ops, ops,
                                 scheduler.SchedulerParams(mirror=False), (3, 5))
    be = scheduler.Backend("cuda", devices=(0, 0, 0))
    three = scheduler.run_assembly(m, bt, spec, ops, ops,
                                   scheduler.SchedulerParams(backends=(be,), mirror=False), (3, 5))
    assert np.array_equal(one.buffer, three.buffer)
    # mirrored (default): mirrors inside one device's range are evaluated
    # together, the rest alone -- equal to the plain values within roundoff
    three_m = scheduler.run_assembly(m, bt, spec, ops, ops,
                                     scheduler.SchedulerParams(backends=(be,)), (3, 5))
    pk = packaging.make_packages(m.triangles, bt, ops, ops, scheduler.DEFAULT_MAXSIZE)
    ok, worst, _ = p2_check(pk, three_m.buffer, one.buffer, 1e-13, m, ("laplace", "double", 0.0),
                            (3, 5), ref_is_device=True)
    assert ok, worst


@pytest.mark.parametrize("eq,kappa", [("laplace", 0.0), ("helmholtz", 4.0)])
def test_green_matrix_vs_reference(gload, eq, kappa):
    g = gload("gca_L3.npz")
    m, t, _ = sphere_setup(3)
    node = t.nodes[int(g["green_cluster"][0])]
    src = gca.green_sources(node.lo, node.hi, 1.0, 6, m.diameter())
    for order in (3, 4):
        A = gca.build_green_matrix(m, t.panels(node), src, kernels.KernelSpec(eq, "single", kappa),
                                   order)
        ref = g[f"green_{eq}_{order}"]
        assert A.dtype == ref.dtype
        assert float(np.max(np.abs(A - ref) / np.abs(ref))) <= TOL


@pytest.mark.parametrize("eq,kappa", [("laplace", 0.0), ("helmholtz", 4.0)])
def test_gca_operators_pivots(gload, eq, kappa):
    """Device Green matrices + host ACA reproduce the reference pivots."""
    g = gload("gca_L3.npz")
    m, t, bt = sphere_setup(3)
    ops, col = gca.build_interpolation_operators(m, bt, kernels.KernelSpec(eq, "single", kappa),
                                                 gca.GcaParams())
    assert ops is col
    cids = g[f"ops_{eq}_cids"]
    assert np.array_equal(sorted(ops), cids)
    piv = np.concatenate([ops[int(c)].pivots_global for c in cids])
    assert np.array_equal(piv, g[f"ops_{eq}_pivots"])
    V3 = ops[int(cids[0])].V
    assert np.max(np.abs(V3 - g[f"ops_{eq}_V3"])) <= 1e-8 * np.max(np.abs(g[f"ops_{eq}_V3"]))


@pytest.mark.parametrize("eq,kappa", [("laplace", 0.0), ("helmholtz", 4.0)])
def test_gca_pipeline_matches_per_cluster_path(eq, kappa):
    """The native batched pipeline (device-generated sources, green_box_kernel,
    threaded host ACA/solve) reproduces the per-cluster path (host
    green_sources -> green_kernel -> native operator) on every L5 cluster:
    identical pivots, V within roundoff; several batches forced."""
    m, t, bt = sphere_setup(5)
    spec = kernels.KernelSpec(eq, "single", kappa)
    params = gca.GcaParams()
    ids = sorted({l.row for l in bt.leaves if l.kind == "admissible"})
    ops = gca._ops_for_tree(m, t, ids, spec, params, m.diameter(), 0, batch_bytes=8 << 20)
    assert gca.last_build_phases["batches"] > 1
    for cid in ids[::7]:
        node = t.nodes[cid]
        ref = gca.build_interpolation_operator(m, cid, t.panels(node), node.lo, node.hi, spec,
                                               params, m.diameter())
        assert np.array_equal(ops[cid].pivots_local, ref.pivots_local), cid
        assert np.array_equal(ops[cid].pivots_global, ref.pivots_global), cid
        assert np.max(np.abs(ops[cid].V - ref.V)) <= 1e-9 * np.max(np.abs(ref.V)), cid


def test_assemble_operator_pipeline():
    """solver.assemble_operator end to end (trees, device GCA, device assembly)."""
    m = mesh.build_sphere_mesh(3)
    cfg = solver.PipelineConfig()
    op = solver.assemble_operator(m, kernels.KernelSpec("laplace", "single"), cfg)
    bt = op.matrix.block_tree
    pk = packaging.make_packages(m.triangles, bt, op.matrix.row_ops, op.matrix.col_ops,
                                 cfg.scheduler.maxsize_bytes)
    ref = oracle_assemble(m, pk, "laplace", "single", 0.0, cfg.orders)
    ok, worst, _ = p2_check(pk, op.matrix.buffer, ref, TOL)
    assert ok, worst
    dlp = solver.assemble_operator(m, kernels.KernelSpec("laplace", "double"), cfg,
                                   trees=bt, ops=(op.matrix.row_ops, op.matrix.col_ops))
    assert dlp.matrix.buffer.shape == op.matrix.buffer.shape


@pytest.mark.parametrize("case,frozen", [("identical", 1.003065884979),
                                         ("edge", 0.483538914315),
                                         ("vertex", 0.225006419777)])
def test_singular_rules_converge_to_analytic(case, frozen):
    """Reference KAT (tests/oracles.py:71-78, test_quadrature.py:145-161)
    through integrate_pair on the device."""
    def planar(v0, v1, v2):
        v0, v1, v2 = (np.array([p[0], p[1], 0.0]) for p in (v0, v1, v2))
        return mesh.AffineChart(v0, v1 - v0, v2 - v1,
                                float(np.linalg.norm(np.cross(v1 - v0, v2 - v1))))
    charts = {"identical": (planar((0, 0), (1, 0), (0, 1)), planar((0, 0), (1, 0), (0, 1))),
              "edge": (planar((1, 0), (0, 1), (0, 0)), planar((1, 0), (0, 1), (1, 1))),
              "vertex": (planar((1, 0), (0, 1), (0, 0)), planar((1, 0), (2, 0), (1.5, 1)))}
    cx, cy = charts[case]
    spec = kernels.KernelSpec("laplace", "single")
    target = frozen * kernels.INV_4PI
    val = quadrature.integrate_pair(cx, cy, spec, quadrature.build_rule(case, 8)).real
    assert abs(val - target) / target <= 1e-4
    ref12 = quadrature.integrate_pair(cx, cy, spec, quadrature.build_rule(case, 12)).real
    diffs = [abs(quadrature.integrate_pair(cx, cy, spec, quadrature.build_rule(case, n)).real
                 - ref12) for n in range(3, 12)]
    assert all(a > b for a, b in zip(diffs, diffs[1:]))


def test_coincident_points_non_finite():
    """Disjoint rule over an identical pair: non-finite, silently (pairquad.py:98)."""
    m = mesh.build_sphere_mesh(1)
    spec = kernels.KernelSpec("laplace", "single")
    got = scheduler.batch_quadrature(scheduler.CUDA_BACKEND, "disjoint", m, spec,
                                     quadrature.build_rule("disjoint", 3), [2], [2])
    assert not np.isfinite(got[0])


def test_empty_and_single_inputs():
    m = mesh.build_sphere_mesh(1)
    spec = kernels.KernelSpec("helmholtz", "double", 2.0)
    r = quadrature.build_rule("disjoint", 3)
    assert scheduler.batch_quadrature(scheduler.CUDA_BACKEND, "disjoint", m, spec, r,
                                      [], []).shape == (0,)
    e = np.empty((0, 3))
    assert pairquad.pair_values(spec, e, e, e, np.empty(0), e, e, e, np.empty(0), e,
                                r.x_points, r.y_points, r.weights).shape == (0,)
    one = scheduler.batch_quadrature(scheduler.CUDA_BACKEND, "disjoint", m, spec, r, [0], [20])
    ref = oracle.batch_quadrature("helmholtz", "double", 2.0, m.vertices, m.triangles,
                                  m.normals, m.gramians, [0], [20], None, None, *oracle.rule(
                                      "disjoint", 3))
    assert rel_err(one, ref) <= TOL


def test_bad_arguments_raise():
    m = mesh.build_sphere_mesh(1)
    spec = kernels.KernelSpec("laplace", "single")
    with pytest.raises(ValueError):
        scheduler.batch_quadrature(scheduler.CUDA_BACKEND, "disjoint", m, spec,
                                   quadrature.build_rule("disjoint", 3), [0], [m.num_triangles])


def test_slp_block_symmetry_L5():
    """Size-independent property at L5: the disjoint-rule SLP is symmetric, so
    dense leaves (t,s) and (s,t) are transposes on uncorrected entries."""
    m, t, bt = sphere_setup(5)
    near = cluster.BlockTree(bt.nodes, t, t, bt.eta, [l for l in bt.leaves if l.kind == "dense"])
    # per-pair evaluation: with the mirrored default the transposes are equal
    # by construction
    M = scheduler.run_assembly(m, near, kernels.KernelSpec("laplace", "single"), {}, {},
                               scheduler.SchedulerParams(mirror=False), (4, 5))
    leaf = {(l.row, l.col): l.index for l in near.leaves}
    worst = 0.0
    for (r, c), idx in leaf.items():
        if r < c and (c, r) in leaf:
            A, B = M.payloads[idx], M.payloads[leaf[(c, r)]].T
            ta, tb = m.triangles[t.panels(t.nodes[r])], m.triangles[t.panels(t.nodes[c])]
            touch = (ta[:, None, :, None] == tb[None, :, None, :]).any(axis=(2, 3))
            worst = max(worst, float(np.max(np.abs(A - B)[~touch] / np.abs(A)[~touch])))
    assert worst <= 1e-13


def _near_sampled(level, eq, layer, kappa, orders, seed, n_blocks, n_items):
    """Near-field device payload vs the oracle on a deterministic sample
    (every entry of n_blocks random dense leaves + n_items random singular
    items), helpers.p2_entries rule (no blanket exemption)."""
    m, t, bt = sphere_setup(level)
    near = cluster.BlockTree(bt.nodes, t, t, bt.eta, [l for l in bt.leaves if l.kind == "dense"])
    pk = packaging.make_packages(m.triangles, near, {}, {}, 8 << 20)
    M = scheduler.run_assembly(m, near, kernels.KernelSpec(eq, layer, kappa), {}, {},
                               scheduler.SchedulerParams(), orders)
    rng = np.random.default_rng(seed)
    leaves = rng.choice(pk.leaf_ids.size, n_blocks, replace=False)
    items, _ = pk.device_items()
    idx = np.unique(np.concatenate(
        [np.arange(pk.leaf_base[l], pk.leaf_base[l + 1]) for l in leaves] +
        [items[rng.choice(len(items), n_items, replace=False), 3]]))
    ref = oracle_entries(m, pk, idx, eq, layer, kappa, orders)
    res = p2_entries(m, pk, idx, M.buffer[idx], ref, eq, layer, kappa, orders,
                     leaf_max_of(pk, M.buffer, idx), TOL)
    assert res["ok"], res
    return res


def test_sampled_parity_C2_level6():
    """BASELINE config 2 scale (L6, 32768 triangles, orders 4/5, Laplace DLP,
    near field) on a deterministic sample of entries. Double-layer edge
    entries where the reference's own rounding exceeds 1e-12
    (tests/test_reference_levels.py measures it) are checked against the
    binary128 value of the same rule."""
    _near_sampled(6, "laplace", "double", 0.0, (4, 5), 6, 300, 6000)


@pytest.mark.parametrize("layer", ["single", "double"])
def test_sampled_parity_helmholtz_small_phase(layer):
    """Fine Helmholtz mesh (L6, kappa = 2: kappa (R_x + R_y) < 1/8 for every
    pair) exercises the factored-phase path e^{i phi0} e^{i delta} in the
    disjoint and singular kernels; sampled entries vs the oracle."""
    res = _near_sampled(6, "helmholtz", layer, 2.0, (3, 5), 7, 200, 6000)
    if layer == "single":
        assert res["n_hp"] == 0


@pytest.mark.parametrize("name", list(SPECS))
def test_potential_batch_vs_reference(gload, name):
    """scheduler.potential_batch (scheduler.py:508-534) on the device."""
    g = gload("potential_L2.npz")
    m = mesh.build_sphere_mesh(2)
    for order in (2, 3):
        got = scheduler.potential_batch(m, spec_of(name), g["points"], order)
        assert rel_err(got.ravel(), g[f"{name}_{order}"].ravel()) <= TOL


def test_gcamat01_dump_of_device_matrix(tmp_path, gload):
    from paper_1510_07244_b200 import h2
    m, t, bt = sphere_setup(3)
    ops = golden_ops(gload("gca_L3.npz"), "laplace")
    M = scheduler.run_assembly(m, bt, kernels.KernelSpec("laplace", "single"), ops, ops,
                               scheduler.SchedulerParams(), (3, 5))
    h2.dump(M, tmp_path / "m.gcamat")
    L = h2.load(tmp_path / "m.gcamat")
    assert L.checksum() == M.checksum()


@pytest.mark.parametrize("eq,layer,kappa", [("laplace", "single", 0.0),
                                            ("helmholtz", "double", 4.0)])
def test_device_matvec_vs_reference(eq, layer, kappa):
    """h2.matvec on the device (csrc/h2_matvec.cu) against the reference leaf
    loop (h2.py:49-71) on an assembled L4 operator; bitwise reproducible."""
    import h2_numpy
    from paper_1510_07244_b200 import h2, solver
    m = mesh.build_sphere_mesh(4)
    op = solver.assemble_operator(m, kernels.KernelSpec(eq, layer, kappa), solver.PipelineConfig())
    M = op.matrix
    rng = np.random.default_rng(7)
    x = rng.standard_normal(M.shape[1]) + 1j * rng.standard_normal(M.shape[1])
    y = h2.matvec(M, x)
    ref = h2_numpy.matvec_reference(M, x)
    assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref))
    assert np.array_equal(y, h2.matvec(M, x))


@pytest.mark.parametrize("case", ["disjoint", "vertex", "edge", "identical"])
def test_p1_local_matrices_vs_reference_golden(gload, case):
    """csrc/p1.cu local 3x3 matrices vs the reference's integrate_pair with
    P1 bases (golden p1_crank.npz) on a crankshaft surface, 1e-12 of the
    local matrix scale."""
    from paper_1510_07244_b200 import p1, quadrature as Q
    g = gload("p1_crank.npz")
    m = mesh.make_surface_mesh(g["vertices"], g["triangles"])
    pairs, perms = g[f"pairs_{case}"], g[f"perms_{case}"]
    rule = Q.build_rule(case, 3 if case == "disjoint" else 5)
    for name, (eq, layer, kappa) in SPECS.items():
        spec = kernels.KernelSpec(eq, layer, kappa)
        got = p1.local_matrices(m, spec, rule, pairs[:, 0], pairs[:, 1], perms[:, :3],
                                perms[:, 3:])
        ref = g[f"p1_{case}_{name}"]
        scale = np.max(np.abs(ref), axis=(1, 2))
        if layer == "double":
            # P2 rule: coplanar pairs (flat parts of the crankshaft) have DLP
            # entries that are pure roundoff in the reference (~1e-21); they
            # are compared on the pair's single-layer scale
            slp = g[f"p1_{case}_{name[0]}-SLP"]
            scale = np.maximum(scale, np.max(np.abs(slp), axis=(1, 2)))
        err = np.max(np.abs(got - ref), axis=(1, 2))
        assert np.all(err <= 1e-12 * scale), (name, float(np.max(err / scale)))


@pytest.mark.parametrize("eq,layer,kappa", [("laplace", "single", 0.0),
                                            ("helmholtz", "double", 4.0)])
def test_p1_near_field_scatter_vs_oracle(eq, layer, kappa):
    """P1 near-field matrix (device local matrices + deterministic gather
    scatter) vs the numpy oracle's np.add.at scatter on a 1024-triangle
    crankshaft; row-scaled 1e-12; two executions bitwise identical."""
    import p1_numpy
    from paper_1510_07244_b200 import p1
    m = mesh.build_crankshaft_mesh(1024, seed=1, n_theta=16)
    t = cluster.build_cluster_tree(m, 16)
    bt = cluster.build_block_tree(t, t, 2.0)
    spec = kernels.KernelSpec(eq, layer, kappa)
    plan = p1.NearFieldP1(m, bt, spec, (3, 5))
    A = plan.assemble().toarray()
    ref = p1_numpy.near_field(m, plan.packages, spec, (3, 5))
    assert np.array_equal(A != 0, ref != 0) or np.all(np.abs(A[(A != 0) != (ref != 0)]) == 0)
    row = np.max(np.abs(ref), axis=1, keepdims=True)
    assert np.all(np.abs(A - ref) <= 1e-12 * row)
    plan.execute()
    _, _, d1 = plan.download()
    plan.execute()
    _, _, d2 = plan.download()
    assert np.array_equal(d1, d2)
    plan.close()


def test_gca_multi_device_partition_equals_single():
    """Clusters partitioned over several devices (here the same device
    twice: the partition and merge logic) give the single-device operators."""
    m, t, bt = sphere_setup(4)
    spec = kernels.KernelSpec("helmholtz", "single", 4.0)
    one, _ = gca.build_interpolation_operators(m, bt, spec, gca.GcaParams(), device=0)
    two, _ = gca.build_interpolation_operators(m, bt, spec, gca.GcaParams(), device=(0, 0, 0))
    assert list(one) == list(two)
    for c in one:
        assert np.array_equal(one[c].pivots_global, two[c].pivots_global)
        assert np.array_equal(one[c].V, two[c].V)


def test_release_cached_then_reassemble(gload):
    """Dropping the library's caches (pool, staging, arena) between two
    assemblies changes nothing in the result."""
    from paper_1510_07244_b200 import device as devmod
    g = gload("gca_L3.npz")
    m, t, bt = sphere_setup(3)
    ops = golden_ops(g, "laplace")
    spec = kernels.KernelSpec("laplace", "single", 0.0)
    a = scheduler.run_assembly(m, bt, spec, ops, ops, scheduler.SchedulerParams(), (3, 5))
    first = np.array(a.buffer)
    del a
    devmod.release_cached(0)
    b = scheduler.run_assembly(m, bt, spec, ops, ops, scheduler.SchedulerParams(), (3, 5))
    assert np.array_equal(first, b.buffer)


@pytest.mark.parametrize("eq,kappa", [("laplace", 0.0), ("helmholtz", 4.0)])
@pytest.mark.parametrize("orders", [(3, 5), (4, 5), (7, 5)])
def test_run_assembly_pair_vs_oracle(gload, eq, kappa, orders):
    """The fused SLP+DLP plan (one evaluation of r, 1/r and the phase per
    point for both layers) against the oracle for each layer (P2 rule), and
    against the separate single-layer plans (within roundoff)."""
    m, bt, ops, pk = packages_for(3, eq, gload("gca_L3.npz"))
    S, D = scheduler.run_assembly_pair(m, bt, eq, kappa, ops, ops,
                                       scheduler.SchedulerParams(), orders)
    for layer, M in (("single", S), ("double", D)):
        ref = oracle_assemble(m, pk, eq, layer, kappa, orders)
        ok, worst, nfb = p2_check(pk, M.buffer, ref, TOL, m, (eq, layer, kappa), orders)
        assert ok, (layer, worst, nfb)
        sep = scheduler.run_assembly(m, bt, kernels.KernelSpec(eq, layer, kappa), ops, ops,
                                     scheduler.SchedulerParams(), orders)
        ok, worst, _ = p2_check(pk, M.buffer, sep.buffer, 1e-13, m, (eq, layer, kappa), orders,
                                ref_is_device=True)
        assert ok, (layer, "vs separate", worst)
    assert set(S.payloads) == set(D.payloads) == {l.index for l in bt.leaves}


def test_run_assembly_pair_sampled_L5():
    """Fused pair plan at L5 (Helmholtz, coupling blocks included) vs the
    separate plans on every entry (1e-12, P2 rule)."""
    m, t, bt = sphere_setup(5)
    ops, _ = gca.build_interpolation_operators(m, bt, kernels.KernelSpec("helmholtz", "single",
                                                                         4.0), gca.GcaParams())
    pk = packaging.make_packages(m.triangles, bt, ops, ops, scheduler.DEFAULT_MAXSIZE)
    S, D = scheduler.run_assembly_pair(m, bt, "helmholtz", 4.0, ops, ops,
                                       scheduler.SchedulerParams(), (3, 5))
    for layer, M in (("single", S), ("double", D)):
        sep = scheduler.run_assembly(m, bt, kernels.KernelSpec("helmholtz", layer, 4.0), ops,
                                     ops, scheduler.SchedulerParams(), (3, 5))
        ok, worst, _ = p2_check(pk, M.buffer, sep.buffer, 1e-12, m, ("helmholtz", layer, 4.0),
                                (3, 5), ref_is_device=True)
        assert ok, (layer, worst)


def test_pair_plan_shards_equal_single(gload):
    """Fused pair plans: several devices of one process and process shards
    (SchedulerParams.shard) give the unsharded payloads bit for bit."""
    m, t, bt = sphere_setup(3)
    ops = golden_ops(gload("gca_L3.npz"), "helmholtz")
    S, D = scheduler.run_assembly_pair(m, bt, "helmholtz", 4.0, ops, ops,
                                       scheduler.SchedulerParams(mirror=False), (3, 5))
    be = scheduler.Backend("cuda", devices=(0, 0, 0))
    S3, D3 = scheduler.run_assembly_pair(m, bt, "helmholtz", 4.0, ops, ops,
                                         scheduler.SchedulerParams(backends=(be,), mirror=False),
                                         (3, 5))
    assert np.array_equal(S.buffer, S3.buffer) and np.array_equal(D.buffer, D3.buffer)
    L = S.payloads._ids.size
    for stages in (1, 4):   # unstaged and staged shard paths
        for world in (2, 3):
            scheduler.clear_package_cache()
            parts = [scheduler.run_assembly_pair(
                m, bt, "helmholtz", 4.0, ops, ops,
                scheduler.SchedulerParams(shard=(r, world), stages=stages, mirror=False),
                (3, 5))
                for r in range(world)]
            # each shard holds exactly its leaf set (every leaf with its
            # mirror); the sets partition the leaves, and every leaf's payload
            # is the single-process one bit for bit
            sets = [p[0].shard_leaves for p in parts]
            assert np.array_equal(np.sort(np.concatenate(sets)), np.arange(L))
            for part in parts:
                for lid in list(part[0].payloads)[::5]:
                    assert np.array_equal(part[0].payloads[lid], S.payloads[lid])
                    assert np.array_equal(part[1].payloads[lid], D.payloads[lid])
                assert part[0].buffer.size == sum(v.size for v in part[0].payloads.values())
    # mirrored (default): a shard evaluates each of its leaves with its mirror
    # (both are in the set) -- equal to the per-pair values within roundoff
    parts = [scheduler.run_assembly_pair(m, bt, "helmholtz", 4.0, ops, ops,
                                         scheduler.SchedulerParams(shard=(r, 2)), (3, 5))
             for r in range(2)]
    for part in parts:
        for M, R in ((part[0], S), (part[1], D)):
            for lid in M.payloads:
                a, b = M.payloads[lid], R.payloads[lid]
                assert np.all(np.abs(a - b) <= 1e-13 * np.maximum(np.abs(b), np.abs(b).max()))


@pytest.mark.parametrize("stages", [2, 5])
def test_staged_assembly_equals_unstaged(stages):
    """Staged assembly (leaf ranges packaged on a host thread while earlier
    ranges run on the device) gives the unstaged payloads bit for bit, for
    the single-operator and the fused pair call; a second operator reuses the
    cached stage packages."""
    m, t, bt = sphere_setup(4)
    ops, _ = gca.build_interpolation_operators(m, bt, kernels.KernelSpec("helmholtz", "single",
                                                                         4.0), gca.GcaParams())
    spec = kernels.KernelSpec("helmholtz", "double", 4.0)
    scheduler.clear_package_cache()
    ref = scheduler.run_assembly(m, bt, spec, ops, ops,
                                 scheduler.SchedulerParams(stages=1, mirror=False))
    refS, refD = scheduler.run_assembly_pair(m, bt, "helmholtz", 4.0, ops, ops,
                                             scheduler.SchedulerParams(stages=1, mirror=False))
    scheduler.clear_package_cache()
    params = scheduler.SchedulerParams(stages=stages, mirror=False)
    st = scheduler.AssemblyStats()
    got = scheduler.run_assembly(m, bt, spec, ops, ops, params, stats=st)
    assert "packaging_wait" in st.phase_s
    assert np.array_equal(got.buffer, ref.buffer)
    for lid in list(ref.payloads)[::37]:
        assert np.array_equal(got.payloads[lid], ref.payloads[lid])
    S, D = scheduler.run_assembly_pair(m, bt, "helmholtz", 4.0, ops, ops, params)
    assert np.array_equal(S.buffer, refS.buffer) and np.array_equal(D.buffer, refD.buffer)
    scheduler.clear_package_cache()


def test_bench_json_contract(tmp_path):
    """bench.py (our arm, small C1 config) prints one JSON line with the keys
    the driver reads: metric/value/unit, timing, roofline, e2e with the
    H2D/D2H byte counts, gpu_launches and the clocks sampled under load."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    out = subprocess.run([sys.executable, "bench.py", "--config", "c1", "--steps", "3",
                          "--warmup", "3", "--e2e-steps", "1", "--no-cpu", "--no-matvec"],
                         cwd=root, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    assert 0.0 < d["roofline"]["frac"] <= 1.0
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    assert d["e2e"]["d2h_bytes_per_step"] > 0 and d["gpu_launches"] > 0
    assert "workload" in d["config"]
