"""Where does the C4 e2e step go? (execute, download, csr)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_07244_b200 import cluster, kernels, mesh, p1  # noqa: E402

m = mesh.build_crankshaft_mesh(65536, seed=0)
t = cluster.build_cluster_tree(m, 16)
bt = cluster.build_block_tree(t, t, 2.0)
plan = p1.NearFieldP1(m, bt, kernels.KernelSpec("helmholtz", "double", 4.0), (3, 5))
A = plan.assemble()
for _ in range(3):
    A = None
    t0 = time.perf_counter()
    plan.execute()
    t1 = time.perf_counter()
    ip, ix, d = plan.download()
    t2 = time.perf_counter()
    import scipy.sparse as sp
    A = sp.csr_matrix((d, ix, ip.astype("int32")), shape=(plan.num_vertices,) * 2, copy=False)
    t3 = time.perf_counter()
    print(f"execute {t1 - t0:.4f} download {t2 - t1:.4f} csr {t3 - t2:.4f} {plan.timing_ms()}")
    ip = ix = d = None
