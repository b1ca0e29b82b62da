"""e2e (public API run_assembly_pair, host buffers) against the staging
parameters: SchedulerParams.stages x chunks, median of 3 per setting."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
from paper_1510_07244_b200 import scheduler  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = bench.CONFIGS[cfg_name]
m, bt, ops, _ = bench.build_workload(cfg, [0], None, lambda s: None, warm_gca=False)
from paper_1510_07244_b200 import packaging as _pkg  # noqa: E402
pk = _pkg.make_packages(m.triangles, bt, ops, ops, 8 << 20)
res = {}
for stages in (1, 4, 5, 6, 8):
    for chunks in (8, 16):
        p = scheduler.SchedulerParams(stages=stages, chunks=chunks)
        ts = []
        for rep in range(4):
            scheduler.clear_package_cache()
            t0 = time.perf_counter()
            out = scheduler.run_assembly_pair(m, bt, cfg["equation"], cfg["kappa"], ops, ops, p,
                                              cfg["orders"])
            ts.append(time.perf_counter() - t0)
            del out
        res[f"stages{stages}_chunks{chunks}"] = round(statistics.median(ts[1:]) * 1e3, 1)
        print(cfg_name, stages, chunks, res[f"stages{stages}_chunks{chunks}"], "ms", flush=True)
print(json.dumps(res))
