"""Reference GCA pivots/ranks at L4-L8 (and the checksums they imply), generated
by running the UNMODIFIED reference package in this container.

    NUMBA_CACHE_DIR=/tmp/numba PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/gen_gca_levels.py [levels...]

Reference path: gca.build_interpolation_operators (gca.py:285-310) is a
serial loop over the sorted cluster ids of the admissible leaves calling
build_interpolation_operator (gca.py:258-282) per cluster; every cluster is
independent (gca.py:295-302), so this script runs that SAME per-cluster
function in a process pool (single-threaded BLAS per process) and
reassembles the dict in sorted-id order. Output: tests/golden/gca_levels.npz
with, per (level, equation):

    L{L}_{eq}_cids    int32  sorted cluster ids
    L{L}_{eq}_ranks   int32  rank per cluster
    L{L}_{eq}_pivots  int32  concatenated pivots_global (selection order)
    L{L}_{eq}_vcids   int32  clusters whose V is kept (sample: <= 32 of the clusters with id % 37 == 0, |t| <= 128)
    L{L}_{eq}_V       f64/c128 their V matrices, row-major, concatenated

Settings: the reference pipeline defaults SURVEY §8(d) uses (leaf 16,
eta 2.0, GcaParams() = delta 1, m 6, eps 1e-4, rule order 3); the spec is the
single layer of the equation, as solver.assemble_operator builds the
operators (solver.py:217-220).
"""
from __future__ import annotations

import os
import sys
import time

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

import multiprocessing as mp  # noqa: E402

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

from gcabem import cluster, gca, kernels, mesh  # noqa: E402

JOBS = {4: ("laplace", "helmholtz"), 5: ("laplace", "helmholtz"), 6: ("laplace",),
        7: ("helmholtz",), 8: ("helmholtz",)}
_CTX = {}


def _setup(level, eq):
    m = mesh.build_sphere_mesh(level)
    t = cluster.build_cluster_tree(m, 16)
    bt = cluster.build_block_tree(t, t, 2.0)
    kappa = 4.0 if eq == "helmholtz" else 0.0
    return m, t, bt, kernels.KernelSpec(eq, "single", kappa)


def _init(level, eq):
    _CTX["s"] = _setup(level, eq)


def _one(cid):
    m, t, bt, spec = _CTX["s"]
    node = t.nodes[cid]
    op = gca.build_interpolation_operator(m, cid, t.panels(node), node.lo, node.hi, spec,
                                          gca.GcaParams(), scene_diameter=m.diameter())
    keep = op.V if (op.V.shape[0] <= 128 and cid % 37 == 0) else None
    return cid, np.asarray(op.pivots_global, dtype=np.int32), keep


def run(level, eq, out, procs):
    t0 = time.time()
    m, t, bt, spec = _setup(level, eq)
    ids = sorted({l.row for l in bt.leaves if l.kind == "admissible"}
                 | {l.col for l in bt.leaves if l.kind == "admissible"})
    # largest clusters first so the pool has no long tail
    order = sorted(ids, key=lambda c: -t.nodes[c].size)
    with mp.get_context("fork").Pool(procs, initializer=_init, initargs=(level, eq)) as pool:
        res = {cid: (piv, V) for cid, piv, V in pool.imap_unordered(_one, order, chunksize=4)}
    key = f"L{level}_{eq}"
    out[f"{key}_cids"] = np.array(ids, dtype=np.int32)
    out[f"{key}_ranks"] = np.array([res[c][0].size for c in ids], dtype=np.int32)
    out[f"{key}_pivots"] = np.concatenate([res[c][0] for c in ids]).astype(np.int32)
    vc = [c for c in ids if res[c][1] is not None]
    vc = vc[::max(1, -(-len(vc) // 32))]   # at most 32 clusters' V per level
    out[f"{key}_vcids"] = np.array(vc, dtype=np.int32)
    out[f"{key}_V"] = np.concatenate([res[c][1].ravel() for c in vc])
    print(f"L{level} {eq}: {len(ids)} clusters, {out[f'{key}_pivots'].size} pivots, "
          f"{time.time() - t0:.1f} s", flush=True)


def main(levels):
    path = os.path.join(HERE, "gca_levels.npz")
    out = dict(np.load(path)) if os.path.exists(path) else {}
    procs = len(os.sched_getaffinity(0))
    for level in levels:
        for eq in JOBS[level]:
            run(level, eq, out, procs)
            np.savez_compressed(path, **out)
    print("ok")


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or sorted(JOBS))
