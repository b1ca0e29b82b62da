import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
torch.cuda.set_device(0)
from paper_1510_07244_b200 import cluster, gca, kernels, mesh, device as devmod
m = mesh.build_sphere_mesh(7)
t0 = time.perf_counter(); tree = cluster.build_cluster_tree(m, 16); bt = cluster.build_block_tree(tree, tree, 2.0); print("trees", time.perf_counter()-t0, flush=True)
spec = kernels.KernelSpec("helmholtz", "single", 4.0)
for k in range(3):
    t0 = time.perf_counter()
    ops, _ = gca.build_interpolation_operators(m, bt, spec, gca.GcaParams(), device=0)
    dt = time.perf_counter() - t0
    print(f"call {k}: {dt:.3f} s", {kk: (round(v, 4) if isinstance(v, float) else v) for kk, v in gca.last_build_phases.items()}, flush=True)
