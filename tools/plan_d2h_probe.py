"""Device execute + D2H of one whole C3 pair plan (packages and layout
prepared beforehand): the link-bound floor of the e2e step, symmetric
download on and off, and a raw pinned D2H of the same bytes."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1510_07244_b200 import _native as nat  # noqa: E402
from paper_1510_07244_b200 import device as devmod, kernels, packaging, scheduler  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
m, bt, ops, _ = bench.build_workload(cfg, [0], None, lambda s: None, warm_gca=False)
pk = packaging.make_packages(m.triangles, bt, ops, ops, 8 << 20)
dm = devmod.device_mesh(m, 0)
spec = kernels.KernelSpec(cfg["equation"], "single", cfg["kappa"])
a = [nat.pinned_empty(pk.payload_len, np.complex128) for _ in range(2)]
for sym in (True, False):
    p = scheduler.AssemblyPlan(dm, spec, pk, cfg["orders"], pair=True, symmetric_download=sym)
    for nch in (8, 32):
        ts = []
        for rep in range(4):
            t0 = time.perf_counter()
            p.execute_download(a[0], nch, a[1])
            p.synchronize()
            ts.append(time.perf_counter() - t0)
        b = p.d2h_bytes()
        print(f"sym={sym} chunks={nch}: {min(ts) * 1e3:.1f} ms  {b / 1e9:.2f} GB  "
              f"{b / min(ts) / 1e9:.1f} GB/s", flush=True)
    p.close()
import torch  # noqa: E402
x = torch.empty(pk.payload_len * 2, dtype=torch.float64, device="cuda:0")
h = torch.from_numpy(a[0].view(np.float64))
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h.copy_(x, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
print(f"raw pinned D2H {h.numel() * 8 / 1e9:.2f} GB: {dt * 1e3:.1f} ms {h.numel() * 8 / dt / 1e9:.1f} GB/s")
