"""Summarise ncu output for profiles/ (run here, on the files gpurun brought back).

  python tools/ncu_summary.py launches gpurun_out/launches.csv "C2 step" > profiles/rX_launches.txt
  python tools/ncu_summary.py full gpurun_out/prof_disjoint.ncu-rep > profiles/rX_ncu.json
"""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict

FULL_METRICS = [
    "gpu__time_duration.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.per_cycle_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "launch__grid_size",
]


def _rows(text):
    lines = [l for l in text.splitlines() if l.startswith('"')]
    return list(csv.reader(io.StringIO("\n".join(lines))))


def launches(path, title):
    rows = _rows(open(path).read())
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"),
                      hdr.index("Metric Value"), hdr.index("Metric Unit"))
    gi = hdr.index("Grid Size") if "Grid Size" in hdr else None
    items = []
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0,
                 "msecond": 1.0, "s": 1e3, "second": 1e3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        items.append((v * scale, name, r[gi] if gi is not None else ""))
    tot = sum(t for t, _, _ in items) or 1.0
    print(f"# {title}: ncu --metrics gpu__time_duration.sum --clock-control none")
    print("# cold-cache, serialised per-launch times: compare SHARES with bench.py, not absolutes")
    for t, name, grid in items:
        print(f"{t:10.3f} ms  {100 * t / tot:5.1f}%  grid={grid}  {name}")
    agg = OrderedDict()
    for t, name, _ in items:
        agg[name] = agg.get(name, 0.0) + t
    print(f"# total {tot:.3f} ms over {len(items)} launches; by kernel:")
    for name, t in sorted(agg.items(), key=lambda x: -x[1]):
        print(f"#   {t:10.3f} ms  {100 * t / tot:5.1f}%  {name}")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = _rows(out)
    hdr = rows[0]
    res = []
    for r in rows[2:]:
        d = OrderedDict()
        d["Kernel Name"] = r[hdr.index("Kernel Name")]
        for m in FULL_METRICS:
            if m in hdr:
                unit = rows[1][hdr.index(m)]
                d[m] = f"{r[hdr.index(m)]} {unit}".strip()
        res.append(d)
    json.dump(res, sys.stdout, indent=1)
    print()




def metrics(path, title, last=None):
    """Per-kernel table of a multi-metric launch list (--metrics a,b,c --csv):
    one row per launch with every metric; `last` keeps only the last N
    launches (e.g. one product of a repeated step)."""
    rows = _rows(open(path).read())
    hdr = rows[0]
    ki, ii, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("ID"), hdr.index("Metric Name"),
                          hdr.index("Metric Value"), hdr.index("Metric Unit"))
    launches = OrderedDict()
    for r in rows[1:]:
        d = launches.setdefault(r[ii], {"name": r[ki].split("(")[0]})
        d[r[mi]] = (float(r[vi].replace(",", "")), r[ui])
    items = list(launches.values())
    if last:
        items = items[-int(last):]
    print(f"# {title}: ncu --metrics (cold-cache, serialised launches)")
    print("#   time_ms  dram_read_MB  dram_write_MB  fp64_pipe_%  kernel")
    for d in items:
        t, tu = d.get("gpu__time_duration.sum", (0.0, "ns"))
        t *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
              "msecond": 1.0}.get(tu, 1.0)

        def mb(key):
            v, u = d.get(key, (0.0, "byte"))
            return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1e-6)
        fp = d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", (0.0, ""))[0]
        print(f"{t:10.4f} {mb('dram__bytes_read.sum'):12.2f} {mb('dram__bytes_write.sum'):13.2f}"
              f" {fp:11.1f}  {d['name']}")
    tot = sum(1 for _ in items)
    print(f"# {tot} launches")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "launch list")
    elif sys.argv[1] == "metrics":
        metrics(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "launch list",
                sys.argv[4] if len(sys.argv) > 4 else None)
    else:
        full(sys.argv[2])
