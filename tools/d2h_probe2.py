"""D2H into the library's pinned pool (nat.pinned_empty) vs torch pinned memory,
2 GiB, whole and in 256 MiB chunks; second touch of the same target."""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

from paper_1510_07244_b200 import _native as nat

dev = torch.device("cuda:0")
N = 2 << 30
src = torch.empty(N, dtype=torch.uint8, device=dev).fill_(1)
targets = {"torch_pinned": torch.empty(N, dtype=torch.uint8, pin_memory=True),
           "gcabem_pool": torch.from_numpy(nat.pinned_empty(N, np.uint8))}
res = {}
for name, dst in targets.items():
    res[name + "_is_pinned"] = bool(dst.is_pinned())
    for chunk in (N, 256 << 20):
        best = 0.0
        for rep in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for off in range(0, N, chunk):
                dst[off:off + chunk].copy_(src[off:off + chunk], non_blocking=True)
            torch.cuda.synchronize()
            best = max(best, N / (time.perf_counter() - t0) / 1e9)
        res[f"{name}_chunk{chunk >> 20}MB"] = round(best, 1)
print(json.dumps(res))
