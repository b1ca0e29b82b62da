"""Gauss rules, the four Sauter-Schwab pair cases, and pair classification.

Drop-in for gcabem.quadrature (pkg/src/gcabem/quadrature.py). Rules are
expanded 4D point lists on That x That (That = {0 <= t <= s <= 1}),
sub-integral-major, tensor indices (xi, e1, e2, e3) in C order; they are
built with the same elementwise numpy operations as the reference and are
bit-identical to it (pinned by tests/golden/golden.json "rules").

On the device the disjoint rule is never expanded: the kernels use its
tensor factorisation x = (a, ab), y = (c, cd), w = (wa wb a)(wc wd c)
(DESIGN.md §4). The singular rules are uploaded as expanded lists.
"""
from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

from .kernels import KernelSpec, eval_batch
from .mesh import AffineChart, MeshError, SurfaceMesh

CASES = ("disjoint", "vertex", "edge", "identical")
SUBINTEGRALS = {"disjoint": 1, "vertex": 2, "edge": 5, "identical": 6}
CASE_CODE = {c: k for k, c in enumerate(CASES)}
MAX_GAUSS_POINTS = 32
MAX_RULE_ORDER = 12


@dataclass(frozen=True)
class Rule1D:
    points: np.ndarray
    weights: np.ndarray


@dataclass(frozen=True)
class QuadRule4D:
    case: str
    order: int
    x_points: np.ndarray  # (Q, 2) test-variable reference coordinates
    y_points: np.ndarray  # (Q, 2) trial-variable reference coordinates
    weights: np.ndarray   # (Q,) with all Jacobian factors

    @property
    def num_points(self) -> int:
        return int(self.weights.shape[0])

    def packed(self) -> np.ndarray:
        """(Q, 5) rows {xs, xt, ys, yt, w}: the device layout of a generic rule."""
        return np.ascontiguousarray(np.column_stack([self.x_points, self.y_points,
                                                     self.weights]))


@dataclass(frozen=True)
class PairClassification:
    case: str
    perm_x: tuple
    perm_y: tuple


def gauss_legendre(n: int) -> Rule1D:
    """n-point Gauss-Legendre on [0, 1] (quadrature.py:82-87)."""
    if not 1 <= n <= MAX_GAUSS_POINTS:
        raise ValueError(f"point count {n} outside [1, {MAX_GAUSS_POINTS}]")
    x, w = np.polynomial.legendre.leggauss(n)
    return Rule1D(0.5 * (x + 1.0), 0.5 * w)


def duffy_panel_rule(n: int) -> tuple[np.ndarray, np.ndarray]:
    """2D Duffy rule on That: points (n*n, 2) = (a, a b), weights wa wb a."""
    g = gauss_legendre(n)
    a = np.repeat(g.points, n)
    b = np.tile(g.points, n)
    wab = np.repeat(g.weights, n) * np.tile(g.weights, n)
    return np.stack([a, a * b], axis=1), wab * a


# Sub-integral tables. Each entry maps the tensor variables (xi, e1, e2, e3)
# to ((x_s, x_t), (y_s, y_t)); the weight factor per case is separate.
# Formulas: quadrature.py:11-38 (docstring) and :108-143.
def _vertex_maps(xi, e1, e2, e3):
    u = (xi, xi * e1)
    v = (xi * e2, xi * e2 * e3)
    return [(u, v), (v, u)]


def _edge_maps(xi, e1, e2, e3):
    return [
        ((xi, xi * e1 * e3), (xi * (1 - e1 * e2), xi * (e1 * (1 - e2)))),
        ((xi, xi * e1), (xi * (1 - e1 * e2 * e3), xi * (e1 * e2 * (1 - e3)))),
        ((xi * (1 - e1 * e2), xi * (e1 * (1 - e2))), (xi, xi * (e1 * e2 * e3))),
        ((xi * (1 - e1 * e2 * e3), xi * (e1 * e2 * (1 - e3))), (xi, xi * e1)),
        ((xi * (1 - e1 * e2 * e3), xi * (e1 * (1 - e2 * e3))), (xi, xi * (e1 * e2))),
    ]


def _identical_maps(xi, e1, e2, e3):
    halves = [
        ((xi, xi * (1 - e1 + e1 * e2)), (xi * (1 - e1 * e2 * e3), xi * (1 - e1))),
        ((xi, xi * (e1 * (1 - e2 + e2 * e3))), (xi * (1 - e1 * e2), xi * (e1 * (1 - e2)))),
        ((xi * (1 - e1 * e2 * e3), xi * (e1 * (1 - e2 * e3))), (xi, xi * (e1 * (1 - e2)))),
    ]
    out = []
    for u, v in halves:
        out += [(u, v), (v, u)]
    return out


def _expand(case: str, n: int):
    g = gauss_legendre(n)
    grid = np.meshgrid(g.points, g.points, g.points, g.points, indexing="ij")
    wgrid = np.meshgrid(g.weights, g.weights, g.weights, g.weights, indexing="ij")
    xi, e1, e2, e3 = (v.ravel() for v in grid)
    w = (wgrid[0] * wgrid[1] * wgrid[2] * wgrid[3]).ravel()
    if case == "disjoint":
        maps = [((xi, xi * e1), (e2, e2 * e3))]
        weights = [w * (xi * e2)]
    elif case == "vertex":
        maps = _vertex_maps(xi, e1, e2, e3)
        weights = [w * (xi ** 3 * e2)] * 2
    elif case == "edge":
        maps = _edge_maps(xi, e1, e2, e3)
        weights = [w * (xi ** 3 * e1 ** 2)] + [w * (xi ** 3 * e1 ** 2 * e2)] * 4
    else:
        maps = _identical_maps(xi, e1, e2, e3)
        weights = [w * (xi ** 3 * e1 ** 2 * e2)] * 6
    xs = np.concatenate([np.stack(m[0], axis=1) for m in maps])
    ys = np.concatenate([np.stack(m[1], axis=1) for m in maps])
    return (np.ascontiguousarray(xs), np.ascontiguousarray(ys),
            np.ascontiguousarray(np.concatenate(weights)))


_rules: dict = {}
_rules_lock = threading.Lock()
_rule_counters = {"builds": 0, "lookups": 0}


def rule_cache_stats() -> dict:
    with _rules_lock:
        return dict(_rule_counters)


def clear_rule_cache() -> None:
    with _rules_lock:
        _rules.clear()
        _rule_counters.update(builds=0, lookups=0)


def build_rule(case: str, n: int) -> QuadRule4D:
    """Expanded 4D rule, memoised per (case, n) (quadrature.py:170-194)."""
    if case not in CASES:
        raise ValueError(f"unknown case {case!r}")
    if not 1 <= n <= MAX_RULE_ORDER:
        raise ValueError(f"order {n} outside [1, {MAX_RULE_ORDER}]")
    with _rules_lock:
        _rule_counters["lookups"] += 1
        hit = _rules.get((case, n))
        if hit is None:
            hit = QuadRule4D(case, n, *_expand(case, n))
            _rules[(case, n)] = hit
            _rule_counters["builds"] += 1
        return hit


def classify_pair(mesh: SurfaceMesh, tri_a: int, tri_b: int) -> PairClassification:
    """Case and aligning permutations of one pair (quadrature.py:197-220):
    shared vertices first, ordered by global index; others keep their order."""
    case, px, py = classify_pairs(mesh.triangles, np.array([tri_a]), np.array([tri_b]))
    return PairClassification(CASES[int(case[0])], tuple(int(v) for v in px[0]),
                              tuple(int(v) for v in py[0]))


def classify_pairs(triangles: np.ndarray, tri_a, tri_b):
    """Vectorised classify_pair over index arrays.

    Returns (case codes int8 (n,), perm_x uint8 (n,3), perm_y uint8 (n,3)).
    Raises MeshError if distinct triangles share all three vertices.
    """
    tri_a = np.asarray(tri_a, dtype=np.int64)
    tri_b = np.asarray(tri_b, dtype=np.int64)
    va = triangles[tri_a]
    vb = triangles[tri_b]
    eq = va[:, :, None] == vb[:, None, :]
    a_shared = eq.any(axis=2)
    b_shared = eq.any(axis=1)
    nshared = a_shared.sum(axis=1)
    same = tri_a == tri_b
    if np.any((nshared == 3) & ~same):
        k = int(np.flatnonzero((nshared == 3) & ~same)[0])
        raise MeshError(f"triangles {int(tri_a[k])} and {int(tri_b[k])} are distinct "
                        f"but share 3 vertices")
    slot = np.arange(3, dtype=np.int64)
    big = np.int64(1) << 62
    kx = np.where(a_shared & ~same[:, None], va, big + slot)
    ky = np.where(b_shared & ~same[:, None], vb, big + slot)
    px = np.argsort(kx, axis=1, kind="stable").astype(np.uint8)
    py = np.argsort(ky, axis=1, kind="stable").astype(np.uint8)
    case = np.where(same, 3, nshared).astype(np.int8)  # 0 disj, 1 vertex, 2 edge, 3 identical
    return case, px, py


def integrate_pair(chart_x: AffineChart, chart_y: AffineChart, kernel, rule: QuadRule4D,
                   normal_y=None, basis_x=None, basis_y=None) -> complex:
    """gram_x gram_y sum_q w_q phi(x_q) g(Phi_x(x_q), Phi_y(y_q)) psi(y_q)
    (quadrature.py:223-271). KernelSpec kernels with constant bases run on the
    device through the same fused pair kernel as the assembly; callables and
    explicit bases are host-side numpy, as in the reference."""
    if isinstance(kernel, KernelSpec):
        if kernel.needs_normal and normal_y is None:
            raise ValueError("double-layer integral requires the trial normal")
        if basis_x is None and basis_y is None:
            from .pairquad import pair_values
            ny = None if normal_y is None else np.asarray(normal_y, np.float64).reshape(1, 3)
            out = pair_values(kernel, chart_x.origin.reshape(1, 3), chart_x.edge1.reshape(1, 3),
                              chart_x.edge2.reshape(1, 3), np.array([chart_x.gramian]),
                              chart_y.origin.reshape(1, 3), chart_y.edge1.reshape(1, 3),
                              chart_y.edge2.reshape(1, 3), np.array([chart_y.gramian]),
                              ny, rule.x_points, rule.y_points, rule.weights)
            return complex(out[0])
    X = chart_x.map_points(rule.x_points)
    Y = chart_y.map_points(rule.y_points)
    if isinstance(kernel, KernelSpec):
        nrm = None
        if kernel.needs_normal:
            nrm = np.broadcast_to(np.asarray(normal_y, dtype=np.float64), X.shape)
        vals = eval_batch(kernel, X, Y, nrm)
    else:
        vals = np.asarray(kernel(X, Y))
    vals = vals * rule.weights
    if basis_x is not None:
        vals = vals * basis_x(rule.x_points)
    if basis_y is not None:
        vals = vals * basis_y(rule.y_points)
    return complex(np.sum(vals) * chart_x.gramian * chart_y.gramian)
