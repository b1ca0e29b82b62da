"""Algorithmic FP64 work per unit (SURVEY.md §8(d) convention).

+, -, x = 1 flop; FMA = 2; division, sqrt, sin, cos = 1 each. Only work the
minimal algorithm must do is counted: the disjoint rule is a tensor product
of two 2D Duffy rules, so its point mappings are hoisted out of the count;
the singular rules pay the 24-flop per-point mapping. Per pair add 4 flops
(the Gramian scaling).
"""
from __future__ import annotations

F_DISJOINT = {("laplace", "single"): 12, ("laplace", "double"): 19,
              ("helmholtz", "single"): 19, ("helmholtz", "double"): 31}
F_SINGULAR = {k: v + 24 for k, v in F_DISJOINT.items()}
# both layers of one equation from one point evaluation (fused pair plans): the
# minimal shared algorithm computes d, r^2, r (and kr, sin, cos) once, so the
# pair is credited the double layer plus what the single layer adds on top
# (its own 1/r, weight product and accumulation: 3 flops Laplace, 7 Helmholtz)
F_DISJOINT_PAIR = {"laplace": 19 + 3, "helmholtz": 31 + 7}
F_SINGULAR_PAIR = {k: v + 24 for k, v in F_DISJOINT_PAIR.items()}
# mirrored evaluation (a pair and its transpose from one point evaluation,
# DESIGN.md §4): the single layer is symmetric (one value for both entries);
# the transposed double layer adds its own d . n (5), and the product of the
# shared kernel factor with it and the weight plus the accumulation: Laplace 3,
# Helmholtz 6 (complex x real, twice) + 2 (complex add) -> +8 / +11 per point
F_MIRROR_EXTRA = {"laplace": 5 + 3, "helmholtz": 5 + 6}
PAIR_OVERHEAD = 4
# Green-matrix entry: n^2 panel points x disjoint F (monopole SLP, dipole DLP) + 2
GREEN_ENTRY_OVERHEAD = 2


def point_flops(spec, family: str, pair: bool = False) -> int:
    if pair:
        table = F_DISJOINT_PAIR if family == "disjoint" else F_SINGULAR_PAIR
        return table[spec.equation]
    table = F_DISJOINT if family == "disjoint" else F_SINGULAR
    return table[(spec.equation, spec.layer)]


def pair_flops(spec, family: str, q: int, pair: bool = False) -> int:
    """Flops of one pair integral with a Q-point rule (pair: both layers)."""
    return q * point_flops(spec, family, pair) + (2 if pair else 1) * PAIR_OVERHEAD


def mirror_pair_flops(spec, q: int, pair: bool = False, family: str = "disjoint") -> int:
    """Flops of one mirrored evaluation: pair (i, j) and its transpose (j, i)
    with a Q-point rule (pair: both layers of each); family "singular" for
    the symmetric vertex rule (mapping included)."""
    if spec.layer == "single" and not pair:
        f = point_flops(spec, family)                # symmetric: the value is shared
    else:
        f = point_flops(spec, family, pair) + F_MIRROR_EXTRA[spec.equation]
    return q * f + (4 if pair else 2) * PAIR_OVERHEAD


def p1_pair_flops(spec, family: str, q: int, order: int) -> int:
    """Flops of one P1 local (3 x 3) matrix with a Q-point rule: the P0 point
    work plus the basis weighting the minimal algorithm must do. Disjoint
    (factored) rule: per point 3 real-weighted accumulations of the kernel
    value (2 flops each, x2 for complex), per x point 9 accumulations of the
    y-side sums (36 flops complex / 18 real) shared by the N^2 y points.
    Singular rules: per point the two barycentric triples (4), the weight
    products (3), 3 scalings of the kernel value and 9 accumulations
    (complex: 6 + 36; real: 3 + 18). Per pair the 9 Gramian scalings."""
    cplx = spec.equation == "helmholtz"
    base = point_flops(spec, family)
    if family == "disjoint":
        extra = (12 if cplx else 6) + (36 if cplx else 18) / (order * order)
    else:
        extra = 7 + (42 if cplx else 21)
    return int(q * (base + extra)) + 9 * PAIR_OVERHEAD
