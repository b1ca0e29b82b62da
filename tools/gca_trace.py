"""GCA build of a config twice (first call of the process, then warm) with
the native phase trace (GCABEM_TRACE=1) on stderr."""
import os
import sys
import time

os.environ.setdefault("GCABEM_TRACE", "1")
sys.path.insert(0, os.getcwd())
import bench  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
t0 = time.perf_counter()
m, bt, ops, t = bench.build_workload(cfg, [0], None, lambda s: print(s, file=sys.stderr))
print(f"total {time.perf_counter() - t0:.3f} s {t}", file=sys.stderr)
