"""GCA build time on an octahedral sphere of the given level, first call
(cold: staging, pack buffers, worker buffers allocated) and second call."""
import sys, os, time
sys.path.insert(0, os.getcwd())
from paper_1510_07244_b200 import mesh, cluster, gca, kernels
lvl = int(sys.argv[1])
m = mesh.build_sphere_mesh(lvl)
t = cluster.build_cluster_tree(m, 16)
bt = cluster.build_block_tree(t, t, 2.0)
for call in ("cold", "warm"):
    t0 = time.perf_counter()
    gca.build_interpolation_operators(m, bt, kernels.KernelSpec("helmholtz", "single", 4.0),
                                      gca.GcaParams())
    print(f"gca L{lvl} {call} {time.perf_counter() - t0:.3f} s", flush=True)
