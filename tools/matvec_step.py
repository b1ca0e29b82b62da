"""C2 SLP operator on the device, three products (for ncu launch lists)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1510_07244_b200 import h2, kernels, scheduler  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
m, bt, ops, _ = bench.build_workload(cfg, [0], None, lambda s: None, warm_gca=False)
from paper_1510_07244_b200 import packaging as _pkg  # noqa: E402
pk = _pkg.make_packages(m.triangles, bt, ops, ops, 8 << 20)
M = scheduler.run_assembly(m, bt, kernels.KernelSpec(cfg["equation"], "single", cfg["kappa"]),
                           ops, ops, scheduler.SchedulerParams(), cfg["orders"])
D = h2.DeviceH2(M, 0)
x = np.ones(M.shape[1], np.complex128)
for _ in range(3):
    D.matvec(x)
    print(D.last_device_ms, file=sys.stderr)
