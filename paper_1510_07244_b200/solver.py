"""Operator assembly pipeline (drop-in for gcabem.solver's setup entry).

Reference pkg/src/gcabem/solver.py:52-64 (PipelineConfig) and :203-231
(AssembledOperator, assemble_operator). Only the setup phase is in scope
(SURVEY §8(a)); the CG/GMRES solves and verification problems are the solve
phase and are not part of this package.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

from . import h2, scheduler
from .cluster import build_block_tree, build_cluster_tree
from .gca import GcaParams, build_interpolation_operators
from .kernels import KernelSpec
from .mesh import SurfaceMesh
from .scheduler import SchedulerParams


class SolverError(RuntimeError):
    pass


@dataclass(frozen=True)
class PipelineConfig:
    """eta_adm = 2.0 as in the reference pipeline (solver.py:52-64)."""
    leaf_size: int = 16
    eta_adm: float = 2.0
    orders: tuple = (3, 5)   # disjoint / singular base point counts
    gca: GcaParams = field(default_factory=GcaParams)
    scheduler: SchedulerParams = field(default_factory=SchedulerParams)
    cg_tol: float = 1e-8


@dataclass
class AssembledOperator:
    matrix: h2.GCAMatrix
    setup_ops_seconds: float
    assemble_seconds: float
    stats: scheduler.AssemblyStats


def build_trees(mesh: SurfaceMesh, config: PipelineConfig):
    tree = build_cluster_tree(mesh, config.leaf_size)
    return build_block_tree(tree, tree, config.eta_adm)


def assemble_operator(mesh: SurfaceMesh, spec: KernelSpec, config: PipelineConfig,
                      trees=None, ops=None) -> AssembledOperator:
    """Trees, GCA operators (built with the SLP of spec's equation), scheduled
    assembly (solver.py:211-231). Pass trees/ops to reuse them (the DLP
    operator reuses the SLP's, solver.py:280-282).

    config.scheduler.shard = (rank, world) splits the job over processes
    (torch.distributed initialised): each builds its part of the GCA
    clusters, the pivots are all-gathered, and each assembles its leaf
    window (the returned matrix holds only those leaves)."""
    block_tree = build_trees(mesh, config) if trees is None else trees
    t0 = time.monotonic()
    if ops is None:
        # the GCA operators use the devices of the disjoint backend: several
        # devices partition the clusters
        devices = config.scheduler.backend_for("disjoint").devices
        row_ops, col_ops = build_interpolation_operators(
            mesh, block_tree, KernelSpec(spec.equation, "single", spec.kappa), config.gca,
            device=tuple(devices), shard=config.scheduler.shard)
    else:
        row_ops, col_ops = ops
    t1 = time.monotonic()
    stats = scheduler.AssemblyStats()
    matrix = scheduler.run_assembly(mesh, block_tree, spec, row_ops, col_ops,
                                    config.scheduler, config.orders, stats)
    t2 = time.monotonic()
    return AssembledOperator(matrix, t1 - t0, t2 - t1, stats)


def assemble_operator_pair(mesh: SurfaceMesh, equation: str, kappa: float,
                           config: PipelineConfig, trees=None, ops=None):
    """Both layers of one equation (the V and K of the reference's
    Laplace DtN / Helmholtz Brakhage-Werner pipelines, solver.py:266-371,
    which reuse trees and operators between them): trees, GCA operators,
    then ONE fused device assembly (scheduler.run_assembly_pair).
    Returns (AssembledOperator single layer, AssembledOperator double layer);
    the setup seconds are reported on the first, the shared assembly time on
    both."""
    block_tree = build_trees(mesh, config) if trees is None else trees
    t0 = time.monotonic()
    if ops is None:
        devices = config.scheduler.backend_for("disjoint").devices
        row_ops, col_ops = build_interpolation_operators(
            mesh, block_tree, KernelSpec(equation, "single", kappa), config.gca,
            device=tuple(devices), shard=config.scheduler.shard)
    else:
        row_ops, col_ops = ops
    t1 = time.monotonic()
    stats = scheduler.AssemblyStats()
    slp, dlp = scheduler.run_assembly_pair(mesh, block_tree, equation, kappa, row_ops, col_ops,
                                           config.scheduler, config.orders, stats)
    t2 = time.monotonic()
    return (AssembledOperator(slp, t1 - t0, t2 - t1, stats),
            AssembledOperator(dlp, 0.0, t2 - t1, stats))
