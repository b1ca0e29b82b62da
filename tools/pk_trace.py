"""Packaging cost at C3 (L7 sphere, Helmholtz GCA operators): whole tree vs
leaf-range stages, Python-side and native stage timings (GCABEM_TRACE=1)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np

from paper_1510_07244_b200 import cluster, gca, kernels, mesh, packaging, scheduler

lvl = int(sys.argv[1]) if len(sys.argv) > 1 else 7
m = mesh.build_sphere_mesh(lvl)
t = cluster.build_cluster_tree(m, 16)
bt = cluster.build_block_tree(t, t, 2.0)
ops, _ = gca.build_interpolation_operators(m, bt, kernels.KernelSpec("helmholtz", "single", 4.0),
                                           gca.GcaParams())
for rep in range(3):
    t0 = time.perf_counter()
    x = packaging.package_inputs(m.triangles, bt, ops, ops)
    t1 = time.perf_counter()
    lay = packaging.leaf_layout(bt, ops, ops, x)
    t2 = time.perf_counter()
    pk = packaging.make_packages(m.triangles, bt, ops, ops, scheduler.DEFAULT_MAXSIZE, inputs=x)
    t3 = time.perf_counter()
    print(f"inputs {t1-t0:.4f} layout {t2-t1:.4f} whole {t3-t2:.4f}", file=sys.stderr, flush=True)
    sp = scheduler.StagedPackages(m, bt, ops, ops, scheduler.DEFAULT_MAXSIZE, 5)
    ts = time.perf_counter()
    for k in range(len(sp.ranges)):
        sp.stage(k)
        print(f"  stage {k} {sp.ranges[k]} ready at {time.perf_counter()-ts:.4f}", file=sys.stderr,
              flush=True)
