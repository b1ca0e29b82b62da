"""Timeline of the staged e2e assembly (run_assembly_pair): per leaf range the
times (ms from the call) it was packaged, its plan created, launched and
synchronised, against the PCIe floor of its bytes."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402
from paper_1510_07244_b200 import scheduler  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = bench.CONFIGS[cfg_name]
m, bt, ops, _ = bench.build_workload(cfg, [0], None, lambda s: None, warm_gca=False)
from paper_1510_07244_b200 import packaging as _pkg  # noqa: E402
pk = _pkg.make_packages(m.triangles, bt, ops, ops, 8 << 20)
for rep in range(int(os.environ.get("REPS", "4"))):
    scheduler.clear_package_cache()
    st = scheduler.AssemblyStats()
    import resource
    r0 = resource.getrusage(resource.RUSAGE_SELF)
    t0 = time.perf_counter()
    out = scheduler.run_assembly_pair(m, bt, cfg["equation"], cfg["kappa"], ops, ops,
                                      scheduler.SchedulerParams(
                                          stages=int(os.environ.get("STAGES", "6")),
                                          symmetric_download=os.environ.get("SYM", "1") == "1"),
                                      cfg["orders"], st)
    dt = time.perf_counter() - t0
    r1 = resource.getrusage(resource.RUSAGE_SELF)
    cpu = (r1.ru_utime - r0.ru_utime) + (r1.ru_stime - r0.ru_stime)
    print(f"   host CPU {cpu:.3f} s (user {r1.ru_utime - r0.ru_utime:.3f}, sys "
          f"{r1.ru_stime - r0.ru_stime:.3f}) = {cpu / dt:.1f} cores busy on average")
    print(f"{cfg_name} total {dt * 1e3:.1f} ms  d2h {st.d2h_bytes / 1e9:.2f} GB  phases " +
          " ".join(f"{k}={v * 1e3:.1f}" for k, v in st.phase_s.items()))
    for k, t in enumerate(st.stage_times):
        print(f"   range {k}: packaged {t[0] * 1e3:6.1f}  plan {t[1] * 1e3:6.1f}  "
              f"launched {t[2] * 1e3:6.1f}  done {t[3] * 1e3:6.1f} ms")
    del out
