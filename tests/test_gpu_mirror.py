"""Mirrored (symmetric) evaluation on the device: leaf (t, s) and its mirror
(s, t) of a shared cluster tree hold the same panel pairs with x and y
swapped, and the disjoint rule is a symmetric tensor product (reference
quadrature.py:108), so one thread evaluates pair (i, j) and (j, i) together
(SchedulerParams.mirror, default on). Checked here:

* every kind (L/H x SLP/DLP, both fused pair kinds) and several orders: the
  mirrored payload against the bit-exact oracle (P2, 1e-12) and against the
  per-pair evaluation (mirror=False) within roundoff (1e-13);
* the chunked D2H path (leaf-ordered chunks: a SKIP leaf's entries are
  written by its earlier PRIMARY before that chunk's copy) equals the
  one-shot execute + download bit for bit;
* the evaluation accounting of the layout (roofline flops): every pair of a
  mirrored leaf pair is evaluated once, and so is every vertex item pair (the
  vertex rule, quadrature.py:112-117, is symmetric under x <-> y).
"""
import numpy as np
import pytest

from helpers import golden_ops, oracle_assemble, p2_check, sphere_setup
from paper_1510_07244_b200 import device as devmod
from paper_1510_07244_b200 import kernels, packaging, scheduler

pytestmark = pytest.mark.gpu

KINDS = [("laplace", "single", 0.0), ("laplace", "double", 0.0), ("helmholtz", "single", 4.0),
         ("helmholtz", "double", 4.0)]


@pytest.mark.parametrize("eq,layer,kappa", KINDS)
@pytest.mark.parametrize("orders", [(3, 5), (4, 5), (6, 5)])
def test_mirrored_single_kinds_vs_oracle_and_plain(gload, eq, layer, kappa, orders):
    m, t, bt = sphere_setup(3)
    ops = golden_ops(gload("gca_L3.npz"), eq)
    spec = kernels.KernelSpec(eq, layer, kappa)
    pk = packaging.make_packages(m.triangles, bt, ops, ops, scheduler.DEFAULT_MAXSIZE)
    assert pk.leaf_mirror is not None and np.all(pk.leaf_mirror >= 0)
    p = scheduler.SchedulerParams(stages=1)
    M = scheduler.run_assembly(m, bt, spec, ops, ops, p, orders)
    P = scheduler.run_assembly(m, bt, spec, ops, ops, scheduler.SchedulerParams(stages=1,
                                                                                mirror=False),
                               orders)
    ref = oracle_assemble(m, pk, eq, layer, kappa, orders)
    ok, worst, _ = p2_check(pk, M.buffer, ref, 1e-12, m, (eq, layer, kappa), orders)
    assert ok, ("oracle", worst)
    ok, worst, _ = p2_check(pk, M.buffer, P.buffer, 1e-13, m, (eq, layer, kappa), orders,
                            ref_is_device=True)
    assert ok, ("plain", worst)
    if layer == "single":
        # the mirror of a disjoint-rule SLP entry is the same value (entries of
        # pairs sharing a vertex come from the singular rules of (i, j) and
        # (j, i), which agree only to the rules' accuracy, as in the reference)
        for l in bt.leaves[::7]:
            if l.kind == "dense" and l.row != l.col:
                mir = next(x for x in bt.leaves if x.row == l.col and x.col == l.row)
                ta = m.triangles[t.panels(t.nodes[l.row])]
                tb = m.triangles[t.panels(t.nodes[l.col])]
                touch = (ta[:, None, :, None] == tb[None, :, None, :]).any(axis=(2, 3))
                A, B = M.payloads[l.index], M.payloads[mir.index].T
                assert np.array_equal(A[~touch], B[~touch])


@pytest.mark.parametrize("eq,kappa", [("laplace", 0.0), ("helmholtz", 4.0)])
@pytest.mark.parametrize("orders", [(3, 5), (4, 5), (7, 7), (8, 5), (9, 5)])
def test_mirrored_pair_plan_vs_oracle(gload, eq, kappa, orders):
    m, t, bt = sphere_setup(3)
    ops = golden_ops(gload("gca_L3.npz"), eq)
    pk = packaging.make_packages(m.triangles, bt, ops, ops, scheduler.DEFAULT_MAXSIZE)
    S, D = scheduler.run_assembly_pair(m, bt, eq, kappa, ops, ops,
                                       scheduler.SchedulerParams(stages=1), orders)
    for layer, M in (("single", S), ("double", D)):
        ref = oracle_assemble(m, pk, eq, layer, kappa, orders)
        ok, worst, _ = p2_check(pk, M.buffer, ref, 1e-12, m, (eq, layer, kappa), orders)
        assert ok, (layer, worst)


@pytest.mark.parametrize("eq,kappa", [("laplace", 0.0), ("helmholtz", 4.0)])
def test_mirrored_chunked_download_equals_one_shot(gload, eq, kappa):
    m, t, bt = sphere_setup(4)
    from paper_1510_07244_b200 import gca
    ops, _ = gca.build_interpolation_operators(m, bt, kernels.KernelSpec(eq, "single", kappa),
                                               gca.GcaParams())
    pk = packaging.make_packages(m.triangles, bt, ops, ops, scheduler.DEFAULT_MAXSIZE)
    dm = devmod.device_mesh(m, 0)
    plan = scheduler.AssemblyPlan(dm, kernels.KernelSpec(eq, "single", kappa), pk, (3, 5),
                                  pair=True)
    assert plan.mirrored
    from paper_1510_07244_b200 import _native as nat
    a1 = nat.pinned_empty(pk.payload_len, np.complex128)
    a2 = nat.pinned_empty(pk.payload_len, np.complex128)
    plan.execute()
    plan.download(a1, a2)
    plan.synchronize()
    one = (np.array(a1), np.array(a2))
    for nchunks in (3, 17):
        a1[:] = np.nan
        a2[:] = np.nan
        plan.execute_download(a1, nchunks, a2)
        plan.synchronize()
        assert np.array_equal(a1, one[0]) and np.array_equal(a2, one[1]), nchunks
    plan.close()


def test_mirror_evaluation_accounting(gload):
    """Layout counts: the PRIMARY leaves' pairs equal their mirrors' (written
    by them), every non-sharing pair of the matrix is covered by exactly one
    evaluation, and the flops credit the mirrored evaluations."""
    m, t, bt = sphere_setup(4)
    from paper_1510_07244_b200 import gca
    ops, _ = gca.build_interpolation_operators(m, bt, kernels.KernelSpec("helmholtz", "single",
                                                                         4.0), gca.GcaParams())
    pk = packaging.make_packages(m.triangles, bt, ops, ops, scheduler.DEFAULT_MAXSIZE)
    dm = devmod.device_mesh(m, 0)
    spec = kernels.KernelSpec("helmholtz", "single", 4.0)
    mp = scheduler.AssemblyPlan(dm, spec, pk, (3, 5), pair=True)
    pp = scheduler.AssemblyPlan(dm, spec, pk, (3, 5), pair=True, mirror=False)
    mi = mp.layout.mirror_info
    diag = [k for k, l in enumerate(pk.leaf_mirror) if l == k]
    diag_pairs = int(sum(pk.leaf_shape[k, 0] * pk.leaf_shape[k, 1] for k in diag))
    diag_upper = int(sum(pk.leaf_shape[k, 0] * (pk.leaf_shape[k, 0] - 1) // 2 for k in diag))
    assert mi["pairs_mirrored"] - diag_upper == mi["pairs_skipped"]
    total = pk.block_pairs()
    plain_pairs = total - 2 * mi["pairs_skipped"] - diag_pairs
    items = pk.num_items
    # every item is a pair sharing a vertex: the diagonal's (identical) and
    # lower-triangle items, and the SKIP leaves' items, have no evaluation
    computed = 2 * mi["evals_mirrored"] + mi["evals_plain"]
    assert computed == total - items
    assert mi["evals_plain"] <= plain_pairs
    fm, fp = mp.flops()["disjoint"], pp.flops()["disjoint"]
    assert fm < fp and fm > 0.5 * fp
    # vertex items: the symmetric vertex rule evaluates (i, j) and (j, i)
    # together; the partners are not evaluated again
    import ctypes
    from paper_1510_07244_b200 import _native as nat
    ev = np.zeros(5, np.int64)
    nat.check(nat.lib().gcabem_plan_singular_evals(mp.handle, nat.ptr(ev)))
    nv = int(np.count_nonzero(pk.item_case == 1))
    assert ev[0] > 0 and 2 * ev[0] + ev[1] == nv
    assert ev[2] == np.count_nonzero(pk.item_case == 2)
    # identical items evaluate the base half of the rule (its terms come in
    # x <-> y swapped pairs with equal weights)
    assert ev[4] * 2 == mp.singular_q[2]
    nat.check(nat.lib().gcabem_plan_singular_evals(pp.handle, nat.ptr(ev)))
    assert ev[0] == 0 and ev[1] == nv
    assert mp.flops()["singular"] < pp.flops()["singular"]
    mp.close()
    pp.close()


@pytest.mark.parametrize("min_run", ["1", "16384"])
@pytest.mark.parametrize("kind", ["pair", "single", "double"])
def test_symmetric_download_bitwise(gload, monkeypatch, min_run, kind):
    """Symmetric download (the host writes the SKIP leaves of the single layer
    from their PRIMARY plus a gathered singular patch): the host buffers are
    bitwise those of the full copy, for one and several chunks, and fewer
    bytes cross the link (the double layer is copied in full)."""
    monkeypatch.setenv("GCABEM_SYM_MIN_RUN", min_run)
    from paper_1510_07244_b200 import gca
    from paper_1510_07244_b200 import _native as nat
    m, t, bt = sphere_setup(5)
    ops, _ = gca.build_interpolation_operators(m, bt, kernels.KernelSpec("helmholtz", "single",
                                                                         4.0), gca.GcaParams())
    pk = packaging.make_packages(m.triangles, bt, ops, ops, scheduler.DEFAULT_MAXSIZE)
    dm = devmod.device_mesh(m, 0)
    layer = "single" if kind == "pair" else kind
    spec = kernels.KernelSpec("helmholtz", layer, 4.0)
    pair = kind == "pair"
    full = scheduler.AssemblyPlan(dm, spec, pk, (3, 5), pair=pair, symmetric_download=False)
    a = [nat.pinned_empty(pk.payload_len, np.complex128) for _ in range(2)]
    full.execute_download(a[0], 4, a[1] if pair else None)
    full.synchronize()
    ref = [np.array(x) for x in a]
    bytes_full = full.d2h_bytes()
    assert bytes_full == pk.payload_len * 16 * (2 if pair else 1)
    full.close()
    sym = scheduler.AssemblyPlan(dm, spec, pk, (3, 5), pair=pair)
    assert sym.mirrored
    for nchunks in (1, 7):
        for x in a:
            x[:] = np.nan
        sym.execute_download(a[0], nchunks, a[1] if pair else None)
        sym.synchronize()
        assert np.array_equal(a[0], ref[0]), nchunks
        if pair:
            assert np.array_equal(a[1], ref[1]), nchunks
        if kind == "double" or min_run != "1":
            assert sym.d2h_bytes() <= bytes_full
        else:
            # every SKIP leaf is host-filled: about a quarter (pair) / half
            # (single) of the bytes stay on the device
            saved = 1.0 - sym.d2h_bytes() / bytes_full
            assert saved > (0.2 if pair else 0.4), saved
    if kind == "double":
        assert sym.d2h_bytes() == bytes_full
    sym.close()


def test_symmetric_download_staged_public_api(gload, monkeypatch):
    """run_assembly_pair through the staged pipeline: symmetric and full
    downloads give bitwise equal matrices; the stats count the moved bytes."""
    monkeypatch.setenv("GCABEM_SYM_MIN_RUN", "64")
    from paper_1510_07244_b200 import gca
    m, t, bt = sphere_setup(5)
    ops, _ = gca.build_interpolation_operators(m, bt, kernels.KernelSpec("helmholtz", "single",
                                                                         4.0), gca.GcaParams())
    out = {}
    for sym in (False, True):
        scheduler.clear_package_cache()
        st = scheduler.AssemblyStats()
        p = scheduler.SchedulerParams(stages=4, symmetric_download=sym)
        S, D = scheduler.run_assembly_pair(m, bt, "helmholtz", 4.0, ops, ops, p, (3, 5), st)
        out[sym] = (np.array(S.buffer), np.array(D.buffer), st.d2h_bytes)
    assert np.array_equal(out[True][0], out[False][0])
    assert np.array_equal(out[True][1], out[False][1])
    assert out[False][2] == out[False][0].nbytes + out[False][1].nbytes
    assert out[True][2] < out[False][2]


def test_symmetric_download_shards_and_devices(gload, monkeypatch):
    """Process shards (leaf sets: each leaf with its mirror, payload laid out
    set-wise) and several devices of one process (leaf ranges): the
    symmetric download gives the full copy's buffers bit for bit."""
    monkeypatch.setenv("GCABEM_SYM_MIN_RUN", "32")
    from paper_1510_07244_b200 import gca
    m, t, bt = sphere_setup(5)
    ops, _ = gca.build_interpolation_operators(m, bt, kernels.KernelSpec("helmholtz", "single",
                                                                         4.0), gca.GcaParams())
    be = scheduler.Backend("cuda", devices=(0, 0))
    cases = [dict(shard=(r, 2), stages=s) for r in range(2) for s in (1, 3)]
    cases.append(dict(backends=(be,)))
    for kw in cases:
        out = {}
        for sym in (False, True):
            scheduler.clear_package_cache()
            st = scheduler.AssemblyStats()
            S, D = scheduler.run_assembly_pair(
                m, bt, "helmholtz", 4.0, ops, ops,
                scheduler.SchedulerParams(symmetric_download=sym, **kw), (3, 5), st)
            out[sym] = (np.array(S.buffer), np.array(D.buffer), st.d2h_bytes)
        assert np.array_equal(out[True][0], out[False][0]), kw
        assert np.array_equal(out[True][1], out[False][1]), kw
        assert out[True][2] < out[False][2], kw
