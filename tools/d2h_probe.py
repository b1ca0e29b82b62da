"""D2H bandwidth of this box: one pinned 2 GiB target, copies of several
sizes on one and on two streams (the e2e path is D2H-bound)."""
import json
import time

import torch

dev = torch.device("cuda:0")
N = 2 << 30
src = torch.empty(N, dtype=torch.uint8, device=dev).fill_(1)
dst = torch.empty(N, dtype=torch.uint8, pin_memory=True)
res = {}
for chunk in (8 << 20, 64 << 20, 256 << 20, 1 << 30, 2 << 30):
    for nstreams in (1, 2, 4):
        ss = [torch.cuda.Stream(dev) for _ in range(nstreams)]
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for k, off in enumerate(range(0, N, chunk)):
                with torch.cuda.stream(ss[k % nstreams]):
                    dst[off:off + chunk].copy_(src[off:off + chunk], non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        res[f"chunk{chunk >> 20}MB_s{nstreams}"] = round(N / dt / 1e9, 1)
# H2D for reference
torch.cuda.synchronize()
t0 = time.perf_counter()
src.copy_(dst, non_blocking=True)
torch.cuda.synchronize()
res["h2d_2GB"] = round(N / (time.perf_counter() - t0) / 1e9, 1)
print(json.dumps(res))
