import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
torch.cuda.set_device(0)
from paper_1510_07244_b200 import mesh, cluster, kernels, p1, packaging, scheduler
from paper_1510_07244_b200.device import device_mesh
m = mesh.build_crankshaft_mesh(65536, seed=0)
t = cluster.build_cluster_tree(m, 16)
bt = cluster.build_block_tree(t, t, 2.0)
for rep in range(2):
    t0 = time.perf_counter()
    nf = p1.near_field_tree(bt)
    pk = packaging.make_packages(m.triangles, nf, {}, {}, 8 << 20)
    t1 = time.perf_counter()
    dm = device_mesh(m, 0)
    t2 = time.perf_counter()
    lay = scheduler.DeviceLayout(dm, pk)
    t3 = time.perf_counter()
    plan = p1.NearFieldP1(m, bt, kernels.KernelSpec("helmholtz", "double", 4.0), (3, 5), 0)
    t4 = time.perf_counter()
    print(f"rep{rep} packages {t1-t0:.3f} mesh {t2-t1:.3f} layout {t3-t2:.3f} NearFieldP1 {t4-t3:.3f}", flush=True)
