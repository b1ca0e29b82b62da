cat > /tmp/gca_only.py <<'PY'
import sys, time, os
sys.path.insert(0, os.getcwd())
from paper_1510_07244_b200 import mesh, cluster, gca, kernels
m = mesh.build_sphere_mesh(7)
t = cluster.build_cluster_tree(m, 16)
bt = cluster.build_block_tree(t, t, 2.0)
spec = kernels.KernelSpec("helmholtz", "single", 4.0)
gca.build_interpolation_operators(m, bt, spec, gca.GcaParams())
for _ in range(2):
    t0 = time.perf_counter()
    gca.build_interpolation_operators(m, bt, spec, gca.GcaParams())
    print(f"gca {time.perf_counter() - t0:.3f}", dict(gca.last_build_phases), flush=True)
PY
GCABEM_TRACE=1 python /tmp/gca_only.py
