"""Host widening probe (the Laplace D2H question): shipping real
payloads as f64 (8 B/entry over PCIe) needs a host pass writing complex128
(16 B/entry) -- time that pass on this host against the PCIe time it saves."""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, os.getcwd())
from paper_1510_07244_b200 import _native as nat  # noqa: E402

n = 120_000_000                      # ~ C2's two operators (1.93 GB complex128)
src = nat.pinned_empty(n, np.float64)
dst = nat.pinned_empty(n, np.complex128)
src[:] = 1.0
dst[:] = 0
out = {}
for threads in (1, 4, 8, 16):
    def part(k):
        a, b = k * n // threads, (k + 1) * n // threads
        d = dst[a:b].view(np.float64)
        d[0::2] = src[a:b]
        d[1::2] = 0.0
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(part, range(threads)))          # warm
        t0 = time.perf_counter()
        list(ex.map(part, range(threads)))
        dt = time.perf_counter() - t0
    out[f"widen_{threads}t_ms"] = round(dt * 1e3, 1)
    out[f"widen_{threads}t_GBs_written"] = round(16 * n / dt / 1e9, 1)
out["pcie_saved_ms_at_52GBs"] = round(8 * n / 52e9 * 1e3, 1)
print(json.dumps(out))
