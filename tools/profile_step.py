"""One bench step (C3 by default) for ncu: builds the workload, then executes
every plan `--reps` times. Run under ncu on ONE GPU, e.g.

  ncu --set full --clock-control none --import-source on \
      -k regex:disjoint_kernel -c 2 -o gpurun_out/prof python tools/profile_step.py
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1510_07244_b200 import device as devmod  # noqa: E402
from paper_1510_07244_b200 import kernels, scheduler  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3", choices=tuple(bench.CONFIGS))
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--separate", action="store_true", help="one plan per operator")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    m, bt, ops, _ = bench.build_workload(cfg, [0], None, lambda s: print(s, file=sys.stderr),
                                         warm_gca=False)
    from paper_1510_07244_b200 import packaging
    pk = packaging.make_packages(m.triangles, bt, ops, ops, scheduler.DEFAULT_MAXSIZE)
    dm = devmod.device_mesh(m, 0)
    if len(cfg["layers"]) == 2 and not args.separate:  # the bench's fused SLP+DLP plan
        plans = [scheduler.AssemblyPlan(dm, kernels.KernelSpec(cfg["equation"], "single",
                                                               cfg["kappa"]),
                                        pk, cfg["orders"], pair=True)]
    else:
        plans = [scheduler.AssemblyPlan(dm, kernels.KernelSpec(cfg["equation"], l,
                                                               cfg["kappa"]),
                                        pk, cfg["orders"]) for l in cfg["layers"]]
    for _ in range(args.reps):
        for p in plans:
            p.execute()
            p.synchronize()
            print(p.spec.layer, p.timing_ms(), p.flops(), file=sys.stderr)


if __name__ == "__main__":
    main()
