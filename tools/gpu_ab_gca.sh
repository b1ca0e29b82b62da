# A/B of the GCA host pipeline (C3): in-tree library vs a variant build, 3 alternations
mkdir -p gpurun_out
VAR=${VAR:-build/nointrin/libgcabem_b200.so}
cat > /tmp/gca_only.py <<'PY'
import sys, time, os
sys.path.insert(0, os.getcwd())
from paper_1510_07244_b200 import mesh, cluster, gca, kernels
m = mesh.build_sphere_mesh(7)
t = cluster.build_cluster_tree(m, 16)
bt = cluster.build_block_tree(t, t, 2.0)
spec = kernels.KernelSpec("helmholtz", "single", 4.0)
gca.build_interpolation_operators(m, bt, spec, gca.GcaParams())   # warm (staging, context)
for _ in range(2):
    t0 = time.perf_counter()
    gca.build_interpolation_operators(m, bt, spec, gca.GcaParams())
    ph = gca.last_build_phases
    print(f"{sys.argv[1]} gca {time.perf_counter() - t0:.3f} s pipeline {ph['pipeline_s']:.3f} host_thread {ph['host_thread_s']:.2f}", flush=True)
PY
for k in 1 2 3; do
  unset GCABEM_LIB_PATH; python /tmp/gca_only.py base
  GCABEM_LIB_PATH=$PWD/$VAR python /tmp/gca_only.py var
done
