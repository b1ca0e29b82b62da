"""D2H bandwidth alone vs while FP64 compute runs on another stream."""
import json
import time

import torch

dev = torch.device("cuda:0")
N = 2 << 30
src = torch.empty(N, dtype=torch.uint8, device=dev).fill_(1)
dst = torch.empty(N, dtype=torch.uint8, pin_memory=True)
a = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
cs, ks = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
res = {}
for busy in (False, True, False, True):
    torch.cuda.synchronize()
    if busy:
        with torch.cuda.stream(ks):
            for _ in range(8):
                b = a @ a
    t0 = time.perf_counter()
    with torch.cuda.stream(cs):
        for off in range(0, N, 256 << 20):
            dst[off:off + (256 << 20)].copy_(src[off:off + (256 << 20)], non_blocking=True)
    cs.synchronize()
    dt = time.perf_counter() - t0
    res[f"busy={busy}"] = round(N / dt / 1e9, 1)
    torch.cuda.synchronize()
print(json.dumps(res))
