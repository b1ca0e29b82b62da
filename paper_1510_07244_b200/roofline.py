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
PAIR_OVERHEAD = 4
# Green-matrix entry: n^2 panel points x disjoint F (monopole SLP, dipole DLP) + 2
GREEN_ENTRY_OVERHEAD = 2


def point_flops(spec, family: str) -> int:
    table = F_DISJOINT if family == "disjoint" else F_SINGULAR
    return table[(spec.equation, spec.layer)]


def pair_flops(spec, family: str, q: int) -> int:
    """Flops of one pair integral with a Q-point rule."""
    return q * point_flops(spec, family) + PAIR_OVERHEAD
