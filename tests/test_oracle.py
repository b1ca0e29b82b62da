"""The oracle is pinned bit-for-bit against the unmodified reference."""
import hashlib

import numpy as np
import pytest

import oracle
from helpers import SPECS, checksum, oracle_assemble, packages_for, sphere_setup
from paper_1510_07244_b200 import mesh


def sha(*a):
    h = hashlib.sha256()
    for x in a:
        h.update(np.ascontiguousarray(x).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def pv(gload):
    return gload("pair_values_L3.npz")


@pytest.mark.parametrize("case", ["disjoint", "vertex", "edge", "identical"])
def test_batch_quadrature_bitwise(pv, case):
    """pairquad.py:27-112 via scheduler.batch_quadrature: every golden set equal."""
    m = mesh.build_sphere_mesh(3)
    orders = (1, 2, 3, 4, 5, 7) if case == "disjoint" else (2, 3, 5, 7)
    px = pv[f"{case}_perm_x"] if case != "disjoint" else None
    py = pv[f"{case}_perm_y"] if case != "disjoint" else None
    for n in orders:
        xs, ys, w = oracle.rule(case, n)
        for name, (eq, layer, kappa) in SPECS.items():
            got = oracle.batch_quadrature(eq, layer, kappa, m.vertices, m.triangles, m.normals,
                                          m.gramians, pv[f"{case}_tri_x"], pv[f"{case}_tri_y"],
                                          px, py, xs, ys, w, nthreads=2)
            ref = pv[f"{case}_{n}_{name}"]
            assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)), (case, n, name)


def test_raw_pair_values_bitwise(pv):
    for rn in (3, 5):
        xs, ys, w = oracle.rule("disjoint", rn)
        for name, (eq, layer, kappa) in SPECS.items():
            a = [pv[f"raw_{k}"] for k in ("ox", "e1x", "e2x", "gx", "oy", "e1y", "e2y", "gy")]
            ny = pv["raw_ny"] if layer == "double" else None
            got = oracle.pair_values(eq, layer, kappa, *a, ny, xs, ys, w)
            assert np.array_equal(got.view(np.uint64), pv[f"raw_{rn}_{name}"].view(np.uint64))


def test_oracle_rules_match_reference_hashes(golden):
    for key, h in golden["rules"].items():
        case, n = key.split("/")
        if int(n) > 8:
            continue
        assert sha(*oracle.rule(case, int(n))) == h, key


def test_oracle_classification(gload):
    cls = gload("classify_L2.npz")["cls"]
    m = mesh.build_sphere_mesh(2)
    codes = {"disjoint": 0, "vertex": 1, "edge": 2, "identical": 3}
    rng = np.random.default_rng(0)
    for a, b in rng.integers(0, m.num_triangles, (400, 2)):
        c, px, py = oracle.classify(m.triangles, int(a), int(b))
        assert [codes[c], *px, *py] == list(cls[a, b])


def test_oracle_green_matrix(gload):
    g = gload("gca_L3.npz")
    m, t, _ = sphere_setup(3)
    panels = t.panels(t.nodes[int(g["green_cluster"][0])])
    for eq, kappa in (("laplace", 0.0), ("helmholtz", 4.0)):
        for order in (3, 4):
            A = oracle.green_matrix(m.vertices, m.triangles, m.gramians, panels, g["src_points"],
                                    g["src_weights"], g["src_normals"], g["src_roles"], eq,
                                    kappa, order)
            ref = g[f"green_{eq}_{order}"]
            assert np.max(np.abs(A - ref) / np.abs(ref)) <= 1e-14


@pytest.mark.parametrize("key", ["L2/laplace/single/3-5", "L2/helmholtz/double/3-5",
                                 "L3/laplace/single/3-5", "L3/laplace/double/3-5",
                                 "L3/helmholtz/single/3-5", "L3/helmholtz/double/3-5",
                                 "L3/laplace/single/2-3", "L3/helmholtz/double/2-3"])
def test_matrix_checksum_reproduced(golden, gload, key):
    """Host packaging + oracle values == reference GCAMatrix.checksum() bitwise."""
    level, eq, layer, orders = key.split("/")
    orders = tuple(int(x) for x in orders.split("-"))
    kappa = 4.0 if eq == "helmholtz" else 0.0
    m, bt, ops, pk = packages_for(int(level[1:]), eq, gload("gca_L3.npz"))
    pay = oracle_assemble(m, pk, eq, layer, kappa, orders)
    assert checksum(pk, pay) == golden["checksums"][key]


def test_c1_near_field_checksum(golden):
    """BASELINE config 1 (L4 sphere, Laplace SLP, near field only)."""
    m, bt, ops, pk = packages_for(4, "laplace", near_only=True)
    pay = oracle_assemble(m, pk, "laplace", "single", 0.0, (3, 5))
    assert checksum(pk, pay) == golden["checksums"]["L4-near/laplace/single/3-5"]
