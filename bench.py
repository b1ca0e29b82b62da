#!/usr/bin/env python
"""Benchmark: FP64 BEM setup hot path on B200 (metric of BASELINE.json).

Workload (default, BASELINE.json configs[2], "C3" -- the config north_star's
target is quoted on; it fits one GPU): Helmholtz kappa=4 SLP + DLP full H2
setup of the unit sphere with 131,072 triangles (octahedral level 7),
quadrature orders 3 (disjoint) / 5 (singular), leaf 16, eta 2.0, GCA delta 1,
m 6, eps 1e-4, Green rule order 3, 8 MiB lists. --config c2 (L6 Laplace 4/5),
c5 (L8, --order n) and c4 (P1 crankshaft) are the other configs.

* value      pair integrals/s of the device hot path with all inputs resident
             in HBM: one step = every payload entry of BOTH operators (each is
             one pair integral: the disjoint rule, or the singular rule for a
             pair sharing a vertex), near field + GCA coupling blocks. Kernel
             time from CUDA events on the launching stream; L2 flushed
             between steps.
* e2e        the same metric through the public API scheduler.run_assembly_pair
             (host packaging, H2D of the packages, kernels, D2H of all payloads
             into pinned host memory), wall clock with syncs.
* roofline   dominant kernel (disjoint pair quadrature) against the measured
             FP64 DFMA peak of the device (no FP64 figure exists in
             MEASURED_PEAKS.json; the probe runs in this process).
* h2_setup   trees + GCA operators + both assemblies, seconds.
* cpu_baseline  the bit-exact C oracle (oracle/, kind "port") with OpenMP on
             the host cores, on a deterministic sample of the same packages.

`--impl reference` runs the reference's setup path restated in oracle/ on the
host cores without the product (no libgcabem_b200.so, no GPU): trees in full,
the GCA on a sample of clusters, the packaging in full, the assembly sampled
per step; it prints the same metric plus its h2_setup seconds.

Multi-GPU (torchrun, N ranks): by default ONE job split over the ranks
(--mode strong): each rank builds its part of the GCA clusters, the pivots
are all-gathered (the only exchange), and each rank packages and assembles
its leaf window on its GPU. --mode weak: every rank its own job. Without
torchrun, --gpus N splits the job over N devices of one process.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": dict(level=4, equation="laplace", kappa=0.0, layers=("single",), orders=(3, 5),
               near_only=True,
               workload="C1: Laplace SLP near-field Sauter-Schwab only, unit sphere 2048 "
                        "triangles, orders 3/5"),
    "c2": dict(level=6, equation="laplace", kappa=0.0, layers=("single", "double"),
               orders=(4, 5), near_only=False,
               workload="C2: Laplace SLP+DLP full GCA H2-matrix setup, unit sphere 32768 "
                        "triangles, orders 4/5"),
    "c3": dict(level=7, equation="helmholtz", kappa=4.0, layers=("single", "double"),
               orders=(3, 5), near_only=False,
               workload="C3: Helmholtz kappa=4 SLP+DLP full H2 setup, sphere 131072 "
                        "triangles, orders 3/5"),
    "c5": dict(level=8, equation="helmholtz", kappa=4.0, layers=("single", "double"),
               orders=(3, 3), near_only=False,
               workload="C5: Helmholtz kappa=4 SLP+DLP scaling sweep, sphere 524288 triangles, "
                        "disjoint and singular order n swept together (--order)"),
    "c4": dict(crankshaft=65536, equation="helmholtz", kappa=4.0, layers=("double",),
               orders=(3, 5), near_only=True, p1=True,
               workload="C4: Helmholtz kappa=4 DLP, piecewise-linear basis, crankshaft-like "
                        "surface 65536 triangles (seed 0), Sauter-Schwab near field, orders 3/5"),
}
METRIC = "triangle-pair integrals/s (FP64, Sauter-Schwab near field + GCA coupling)"
UNIT = "pair-integrals/s"


# ---------------------------------------------------------------------------
# distributed plumbing (one process per GPU, torch.distributed for barrier/max)

class Dist:
    def __init__(self, cpu_only: bool = False):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.backend = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            # NCCL needs one GPU per rank; fewer GPUs than ranks (a smoke test
            # of the launch on one device) falls back to gloo for the barrier
            # and the max -- neither is on the data path
            ngpu = 0 if cpu_only else \
                (torch.cuda.device_count() if torch.cuda.is_available() else 0)
            backend = "nccl" if ngpu >= self.world else "gloo"
            if backend == "nccl":
                torch.cuda.set_device(self.local)
            dist.init_process_group(backend)
            self.torch, self.dist, self.backend = torch, dist, backend

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def _reduce(self, x: float, op) -> float:
        t = self.torch.tensor([x], dtype=self.torch.float64,
                              device="cuda" if self.backend == "nccl" else "cpu")
        self.dist.all_reduce(t, op=op)
        return float(t.item())

    def max(self, x: float) -> float:
        return x if self.world == 1 else self._reduce(x, self.dist.ReduceOp.MAX)

    def sum(self, x):
        return x if self.world == 1 else type(x)(self._reduce(x, self.dist.ReduceOp.SUM))

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


# ---------------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[3:]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def l2_flush(buf):
    if buf is not None:
        buf.zero_()


# ---------------------------------------------------------------------------

def build_workload(cfg, devices, shard, log, warm_gca=True):
    """Mesh, trees and GCA operators of the config (the setup before
    packaging). `shard` = (rank, world): this process builds its part of the
    GCA clusters and the pivots are all-gathered (gca.exchange_pivots)."""
    from paper_1510_07244_b200 import cluster, gca, kernels, mesh
    t = {}
    t0 = time.perf_counter()
    m = mesh.build_sphere_mesh(cfg["level"])
    t["mesh_s"] = time.perf_counter() - t0   # input generation, not setup
    t0 = time.perf_counter()
    tree = cluster.build_cluster_tree(m, 16)
    bt = cluster.build_block_tree(tree, tree, 2.0)
    t["trees_s"] = time.perf_counter() - t0
    if cfg["near_only"]:
        bt = cluster.BlockTree(bt.nodes, tree, tree, bt.eta,
                               [l for l in bt.leaves if l.kind == "dense"])
        ops = {}
        t["gca_s"] = 0.0
    else:
        spec = kernels.KernelSpec(cfg["equation"], "single", cfg["kappa"])
        dev = tuple(devices) if len(devices) > 1 else devices[0]
        t1 = time.perf_counter()
        ops, _ = gca.build_interpolation_operators(m, bt, spec, gca.GcaParams(), device=dev,
                                                   shard=shard)
        t["gca_s"] = time.perf_counter() - t1
        t["gca_phases"] = dict(gca.last_build_phases)
        if warm_gca:
            # the same build again: the first call of a process also pays its
            # pinned staging and worker buffers (kept for later calls)
            t1 = time.perf_counter()
            gca.build_interpolation_operators(m, bt, spec, gca.GcaParams(), device=dev,
                                              shard=shard)
            t["gca_warm_s"] = time.perf_counter() - t1
    log(f"workload: nt={m.num_triangles} leaves={len(bt.leaves)} clusters={len(ops)} "
        f"{ {k: v for k, v in t.items() if k != 'gca_phases'} }")
    return m, bt, ops, t


def cpu_sample(pk, m, cfg, target_s, nthreads, log):
    """Oracle port on a deterministic sample (every k-th block / item) of the
    packages, both layers; returns (pair integrals, seconds, description)."""
    import oracle
    blocks = pk.device_blocks()
    items, perms = pk.device_items()
    # calibrate: points/s on a small slice
    dq = cfg["orders"][0] ** 4
    xs, ys, w = oracle.rule("disjoint", cfg["orders"][0])
    b0 = blocks[:64]
    cnt = b0[:, 2] * b0[:, 3]
    own = np.repeat(np.arange(len(b0)), cnt)
    k = np.arange(own.size) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    i, j = k // b0[own, 3], k % b0[own, 3]
    tx, ty = pk.panels[b0[own, 4] + i], pk.panels[b0[own, 5] + j]
    tc = time.perf_counter()
    oracle.batch_quadrature(cfg["equation"], cfg["layers"][-1], cfg["kappa"], m.vertices,
                            m.triangles, m.normals, m.gramians, tx, ty, None, None, xs, ys, w,
                            nthreads=nthreads)
    rate = tx.size * dq / max(time.perf_counter() - tc, 1e-6)  # points/s
    sq = [oracle.rule(c, cfg["orders"][1])[2].size for c in ("vertex", "edge", "identical")]
    total_pts = (np.sum(blocks[:, 2] * blocks[:, 3]) * dq
                 + sum(np.count_nonzero(items[:, 0] == c + 1) * q for c, q in enumerate(sq)))
    total_pts *= len(cfg["layers"])
    stride = max(1, int(np.ceil(total_pts / (rate * target_s))))
    bs = blocks[::stride]
    its, pms = items[::stride], perms[::stride]
    cnt = bs[:, 2] * bs[:, 3]
    own = np.repeat(np.arange(len(bs)), cnt)
    k = np.arange(own.size) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    i, j = k // bs[own, 3], k % bs[own, 3]
    tx, ty = pk.panels[bs[own, 4] + i], pk.panels[bs[own, 5] + j]
    pairs = 0
    t0 = time.perf_counter()
    for layer in cfg["layers"]:
        oracle.batch_quadrature(cfg["equation"], layer, cfg["kappa"], m.vertices, m.triangles,
                                m.normals, m.gramians, tx, ty, None, None, xs, ys, w,
                                nthreads=nthreads)
        pairs += tx.size
        for code, case in ((1, "vertex"), (2, "edge"), (3, "identical")):
            sel = its[:, 0] == code
            if np.any(sel):
                oracle.batch_quadrature(cfg["equation"], layer, cfg["kappa"], m.vertices,
                                        m.triangles, m.normals, m.gramians, its[sel, 1],
                                        its[sel, 2], pms[sel, :3].astype(np.int64),
                                        pms[sel, 3:].astype(np.int64),
                                        *oracle.rule(case, cfg["orders"][1]), nthreads=nthreads)
                # counted above: a corrective item overwrites an entry of a sampled block
    dt = time.perf_counter() - t0
    desc = (f"every {stride}-th disjoint block ({tx.size} pairs) and singular item "
            f"({len(its)}) of the workload packages, {'+'.join(cfg['layers'])} layers")
    log(f"cpu sample: {pairs} pair integrals in {dt:.2f} s on {nthreads} threads ({desc})")
    return pairs, dt, desc, stride


def cpu_sample_p1(plan, m, cfg, target_s, log):
    """C4 CPU baseline: the oracle's numpy restatement of the reference's P1
    pair integral (integrate_pair with P1 bases, oracle/p1_cpu.py) on a
    deterministic sample of the plan's near-field pairs (every k-th disjoint
    pair and singular item), one process-wide numpy thread pool."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import p1_cpu
    pk = plan.packages
    all_blocks = pk.device_blocks()
    items, perms = pk.device_items()
    eq, layer, kappa = cfg["equation"], cfg["layers"][0], cfg["kappa"]
    nth = host_threads()

    def block_pairs(blocks):
        cnt = blocks[:, 2] * blocks[:, 3]
        own = np.repeat(np.arange(len(blocks)), cnt)
        k = np.arange(own.size) - np.repeat(np.cumsum(cnt) - cnt, cnt)
        i, j = k // blocks[own, 3], k % blocks[own, 3]
        tx, ty = pk.panels[blocks[own, 4] + i], pk.panels[blocks[own, 5] + j]
        sh = (m.triangles[tx][:, :, None] == m.triangles[ty][:, None, :]).any(axis=(1, 2))
        return tx[~sh], ty[~sh]
    # the near field is ~68 M pairs: sample blocks (every k-th) before expanding
    npairs = int(np.sum(all_blocks[:, 2] * all_blocks[:, 3]))
    bstride = max(1, len(all_blocks) // 16384)
    tx, ty = block_pairs(all_blocks[::bstride])
    scale = npairs / max(1, int(np.sum(all_blocks[::bstride, 2] * all_blocks[::bstride, 3])))

    def run(sel_tx, sel_ty, case, order, px=None, py=None):
        parts = np.array_split(np.arange(sel_tx.size), nth)
        with ThreadPoolExecutor(nth) as ex:
            list(ex.map(lambda ix: p1_cpu.local_matrices(
                m.vertices, m.triangles, m.normals, m.gramians, eq, layer, kappa, case, order,
                sel_tx[ix], sel_ty[ix], None if px is None else px[ix],
                None if py is None else py[ix]), parts))
    probe = slice(0, 4096)
    tc = time.perf_counter()
    run(tx[probe], ty[probe], "disjoint", cfg["orders"][0])
    rate = min(4096, tx.size) / max(time.perf_counter() - tc, 1e-6)
    total = tx.size + items.shape[0] * 20 / scale   # singular items ~20x the points
    stride = max(1, int(np.ceil(total / (rate * target_s))))
    t0 = time.perf_counter()
    run(tx[::stride], ty[::stride], "disjoint", cfg["orders"][0])
    n = tx[::stride].size
    for code, case in ((1, "vertex"), (2, "edge"), (3, "identical")):
        sel = np.flatnonzero(items[:, 0] == code)[::max(1, int(stride * scale))]
        if sel.size:
            run(items[sel, 1], items[sel, 2], case, cfg["orders"][1],
                perms[sel, :3].astype(np.int64), perms[sel, 3:].astype(np.int64))
            n += sel.size
    dt = time.perf_counter() - t0
    desc = (f"every {bstride}-th near-field block, every {stride}-th of its pairs "
            f"({tx[::stride].size} disjoint) and a matching share of the singular items "
            f"({n - tx[::stride].size}) of the C4 packages, oracle/p1_cpu.py (numpy), "
            f"{nth} threads")
    log(f"cpu sample (P1): {n} pairs in {dt:.2f} s ({desc})")
    return {"value": n / dt, "unit": UNIT, "cores": nth, "kind": "port", "sample": desc}


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args, cfg, dist, log):
    """--impl reference: the reference's CPU setup path restated in oracle/
    (the reference is Python + numba: nothing to compile into oracle/_ref),
    on the host cores, rank 0 only, WITHOUT the product (no
    libgcabem_b200.so, no GPU): the sphere and both trees in full
    (oracle.setup_cpu restating mesh.py / cluster.py), the GCA on a
    deterministic sample of clusters (every k-th, green matrix + ACA + pivot
    solve restating gca.py, one worker process per core; the pivots of the
    sample are checked against the reference's own), the packaging in full
    (scheduler.py restated) on the reference's pivots
    (tests/golden/gca_levels.npz, produced by running the reference), and
    each timed step a sample of the assembly (bit-exact C restatement of
    pairquad.py with OpenMP on all cores). Sampled phases are extrapolated
    by panel count / pair count and labelled."""
    if dist.rank != 0:
        return None
    if cfg.get("p1"):
        return {"impl": "reference", "unavailable": "the reference assembles P0 only (P1 exists "
                "per pair via integrate_pair bases, no matrix assembly)"}
    import oracle
    from oracle import setup_cpu as sc
    oracle.build()
    nth = host_threads()
    t0 = time.perf_counter()
    m = sc.sphere_mesh(cfg["level"])
    mesh_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    tree = sc.build_cluster_tree(m, 16)
    bt = sc.build_block_tree(tree, tree, 2.0)
    trees_s = time.perf_counter() - t0
    log(f"reference: mesh {mesh_s:.2f} s, trees {trees_s:.2f} s, {len(bt.leaves)} leaves")
    setup = {"mesh_s (input, not counted)": round(mesh_s, 3), "trees_s": round(trees_s, 3)}
    if cfg["near_only"]:
        bt = sc.BlockTree(bt.nodes, tree, tree, bt.eta,
                          [l for l in bt.leaves if l.kind == "dense"])
        ops = {}
        gca_s = 0.0
    else:
        cids = sc.admissible_clusters(bt)
        g = np.load(os.path.join(ROOT, "tests", "golden", "gca_levels.npz"))
        key = f"L{cfg['level']}_{cfg['equation']}"
        # calibrate on a few clusters, then a sample of about gca_seconds
        probe = cids[::max(1, len(cids) // 64)][:64]
        tc = time.perf_counter()
        sc.build_operators(m, tree, probe, cfg["equation"], cfg["kappa"], workers=nth)
        rate = sum(tree.nodes[c].size for c in probe) / max(time.perf_counter() - tc, 1e-6)
        total_panels = sum(tree.nodes[c].size for c in cids)
        gstride = max(1, int(np.ceil(total_panels / (rate * args.gca_seconds))))
        sample = cids[::gstride]
        tc = time.perf_counter()
        sops = sc.build_operators(m, tree, sample, cfg["equation"], cfg["kappa"], workers=nth)
        gdt = time.perf_counter() - tc
        gca_s = gdt * total_panels / sum(tree.nodes[c].size for c in sample)
        if f"{key}_cids" in g.files:
            ops = sc.pivot_operators(g[f"{key}_cids"], g[f"{key}_ranks"], g[f"{key}_pivots"])
            pivots_from = "the reference's own (tests/golden/gca_levels.npz)"
        else:   # no fixture: the restatement builds every cluster
            ops = sc.build_operators(m, tree, cids, cfg["equation"], cfg["kappa"], workers=nth)
            pivots_from = "oracle restatement, every cluster"
        match = sum(np.array_equal(sops[c].pivots_global, ops[c].pivots_global) for c in sample)
        setup.update({
            "gca_s": round(gca_s, 3),
            "gca_sample": f"every {gstride}-th of {len(cids)} clusters ({len(sample)}, "
                          f"{gdt:.2f} s on {nth} processes), extrapolated by panel count",
            "gca_sample_pivots_equal_reference": f"{match}/{len(sample)}",
            "packaging_pivots": pivots_from})
        log(f"reference GCA: {setup['gca_sample']} -> {gca_s:.1f} s; pivots {match}/{len(sample)}")
    t0 = time.perf_counter()
    pk = sc.make_packages(m.triangles, bt, ops, ops, 8 << 20)
    pack_s = time.perf_counter() - t0
    log(f"reference packaging {pack_s:.2f} s: {pk.block_pairs()} entries, {pk.num_items} items")
    vals, asm = [], []
    desc = ""
    for _ in range(args.warmup + args.steps):
        pairs, dt, desc, stride = cpu_sample(pk, m, cfg, args.cpu_seconds / max(args.steps, 1),
                                             nth, log)
        vals.append(pairs / dt)
        asm.append(dt * stride)
    v = statistics.median(vals[args.warmup:]) if len(vals) > args.warmup else vals[-1]
    asm_s = statistics.median(asm[args.warmup:]) if len(asm) > args.warmup else asm[-1]
    setup.update({"packaging_s": round(pack_s, 3),
                  "assembly_slp_dlp_s": round(asm_s, 3),
                  "assembly_sample": "each step's sampled blocks/items x the stride",
                  "total_s": round(trees_s + gca_s + pack_s + asm_s, 3)})
    return {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
        "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
        "higher_is_better": True, "scaling": args.mode, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (deterministic octahedral sphere)",
        "config": {"workload": cfg["workload"], "pairs_per_step": int(pk.block_pairs()) *
                   len(cfg["layers"]),
                   "same_config": True},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": nth, "kind": "port",
                         "sample": desc},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "h2_setup": setup,
        "native_libraries": ["oracle/liboracle.so"],
        "path": "oracle/ (C restatement of pairquad.py, numpy restatements of mesh, cluster, "
                "gca and scheduler packaging); the product package is not imported",
    }


def run_ours_p1(args, cfg, dist, log):
    """C4: P1 near field on the crankshaft surface. One step = every near-field
    pair's 3x3 local matrix (disjoint + singular rules) and the deterministic
    scatter-add into the vertex CSR matrix, on the device."""
    import torch

    from paper_1510_07244_b200 import cluster, kernels, mesh, p1
    from paper_1510_07244_b200._native import require_device
    device = dist.local % max(torch.cuda.device_count(), 1)
    require_device(device)
    torch.cuda.set_device(device)
    t0 = time.perf_counter()
    m = mesh.build_crankshaft_mesh(cfg["crankshaft"], seed=0)
    t_mesh = time.perf_counter() - t0
    t0 = time.perf_counter()
    tree = cluster.build_cluster_tree(m, 16)
    bt = cluster.build_block_tree(tree, tree, 2.0)
    t_trees = time.perf_counter() - t0
    spec = kernels.KernelSpec(cfg["equation"], cfg["layers"][0], cfg["kappa"])
    t0 = time.perf_counter()
    plan = p1.NearFieldP1(m, bt, spec, cfg["orders"], device)
    t_plan = time.perf_counter() - t0
    t0 = time.perf_counter()
    A = plan.assemble()
    t_first = time.perf_counter() - t0
    del A
    pairs = plan.num_pairs
    log(f"c4: nt={m.num_triangles} nv={m.num_vertices} near pairs={pairs} "
        f"singular={plan.num_singular} nnz={plan.nnz} plan {t_plan:.3f}s first {t_first:.3f}s")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{device}")
    for _ in range(args.warmup):
        plan.execute()
        plan.timing_ms()
    dist.barrier()
    torch.cuda.synchronize(device)
    per = []
    with ClockSampler(device) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize(device)
            plan.execute()
            tm = plan.timing_ms()
            per.append(tm)
    ms = statistics.mean(t["local"] + t["scatter"] for t in per)
    ms_max = dist.max(ms)
    value = pairs * dist.world / (ms_max * 1e-3)
    local_ms = statistics.mean(t["local"] for t in per)
    from paper_1510_07244_b200.roofline import p1_pair_flops
    nd = plan.num_pairs - plan.num_singular
    sq = plan.singular_q
    counts = [int(np.count_nonzero(plan.packages.item_case == c)) for c in (1, 2, 3)]
    n0 = cfg["orders"][0]
    fl = p1_pair_flops(spec, "disjoint", n0 ** 4, n0) * nd + \
        sum(p1_pair_flops(spec, "singular", q, cfg["orders"][1]) * c
            for q, c in zip(sq, counts))
    from paper_1510_07244_b200 import device as devmod
    peak = devmod.fp64_peak_tflops(device)
    achieved = fl / (local_ms * 1e-3) / 1e12
    e2e_t = []
    for _ in range(max(1, args.e2e_steps)):
        A = None  # release the previous matrix: its pinned buffers return to the pool
        t0 = time.perf_counter()
        A = plan.assemble()
        e2e_t.append(time.perf_counter() - t0)
    e2e_dt = dist.max(statistics.median(e2e_t))
    d2h = int((plan.num_vertices + 1) * 8 + plan.nnz * 20)
    cpu = None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu:
        cpu = cpu_sample_p1(plan, m, cfg, args.cpu_seconds, log)
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json"))).get(
            "c4/p1_disjoint")
    except (OSError, ValueError):
        traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": dist.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (deterministic crankshaft-like surface, seed 0)",
        "config": {"workload": cfg["workload"], "pairs_per_step": int(pairs),
                   "basis": "P1 (3x3 local matrix per pair, vertex CSR scatter-add)",
                   "nnz": int(plan.nnz), "l2": "flushed between steps (512 MiB device write)",
                   "parallelism": f"weak x{dist.world}, no collectives"},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "traffic_source": "ncu dram bytes of p1_disjoint_kernel<3,H_DLP> per launch "
                                       "(profiles/r2/ncu_p1_c4.txt)",
                     "kernel": "p1 local matrices (disjoint + singular launches; flops per "
                               "roofline.p1_pair_flops: P0 point work + the basis weighting)",
                     "peak_source": "measured DFMA probe (gcabem_fp64_probe), this device"},
        "e2e": {"value": pairs * dist.world / e2e_dt, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": d2h, "seconds_per_step": e2e_dt},
        "gpu_launches": int(2 + sum(1 for c in counts if c)) * args.steps,
        "clocks": clk.summary(),
        "h2_setup": {"mesh_s": round(t_mesh, 3), "trees_s": round(t_trees, 3),
                     "p1_plan_s": round(t_plan, 3), "first_assembly_s": round(t_first, 3),
                     "total_s": round(t_trees + t_plan + t_first, 3)},
        "timing_ms": {"local": local_ms,
                      "scatter": statistics.mean(t["scatter"] for t in per)},
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    plan.close()
    return line if dist.rank == 0 else None


def run_ours(args, cfg, dist, log):
    """The device path. Under torchrun (N ranks) the default is ONE job split
    over the ranks (--mode strong): each rank builds its part of the GCA
    clusters (pivots all-gathered: the only exchange), packages its leaf
    leaf set (packaging.shard_leaf_set: every leaf with its mirror, so the
    mirrored evaluation stays inside the rank) and assembles it on its GPU. Without
    torchrun, --gpus N splits the job over N devices of this process."""
    import torch

    from paper_1510_07244_b200 import device as devmod
    from paper_1510_07244_b200 import kernels, packaging, scheduler
    from paper_1510_07244_b200._native import require_device

    ndev = max(torch.cuda.device_count(), 1)
    if dist.world > 1:
        devices = [dist.local % ndev]
    else:
        if args.gpus > ndev:
            raise SystemExit(f"--gpus {args.gpus}: only {ndev} devices visible")
        devices = list(range(args.gpus))
    for d in devices:
        require_device(d)
    torch.cuda.set_device(devices[0])
    info = devmod.device_info(devices[0])
    strong = args.mode == "strong"
    shard = (dist.rank, dist.world) if (strong and dist.world > 1) else None
    m, bt, ops, setup_t = build_workload(cfg, devices, shard, log)
    specs = [kernels.KernelSpec(cfg["equation"], layer, cfg["kappa"]) for layer in cfg["layers"]]
    fused = len(specs) == 2 and {s.layer for s in specs} == {"single", "double"} and \
        not args.separate
    # this process's leaves: its window of the job (strong) or everything
    t2 = time.perf_counter()
    leaf_set = scheduler.shard_leaves_of(m, bt, ops, ops, shard, cfg["orders"][0] ** 4) \
        if shard else None
    pk = packaging.make_packages(m.triangles, bt, ops, ops, scheduler.DEFAULT_MAXSIZE,
                                 leaf_index=leaf_set)
    setup_t["packaging_s"] = time.perf_counter() - t2
    L = pk.leaf_ids.size
    sq = [scheduler.build_rule(c, cfg["orders"][1]).num_points
          for c in ("vertex", "edge", "identical")]
    dev_ranges = scheduler._split_range(pk, (0, L), len(devices), cfg["orders"][0] ** 4, sq)
    log(f"rank {dist.rank}: {'all' if leaf_set is None else 'a set of'} leaves={L} "
        f"entries={pk.payload_len} "
        f"blocks={pk.num_blocks} singular={pk.num_items} devices={devices} {dev_ranges}")

    tp = time.perf_counter()
    per_dev = []   # (device, stream, flush buffer, [plans], [separate plans])
    for d, rng in zip(devices, dev_ranges):
        dm = devmod.device_mesh(m, d)
        mir = not args.no_mirror
        sep = [scheduler.AssemblyPlan(dm, s, pk, cfg["orders"], rng, mirror=mir) for s in specs]
        main = [scheduler.AssemblyPlan(dm, specs[0], pk, cfg["orders"], rng, pair=True,
                                       mirror=mir)] if fused else sep
        st = torch.cuda.Stream(device=d)
        for p in sep + main:
            p.set_stream(st.cuda_stream)   # one timeline per device
        flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{d}")
        per_dev.append((d, st, flush, main, sep))
    plan_s = time.perf_counter() - tp
    # pair integrals per step: every payload entry of every operator is one
    # evaluated pair integral (the disjoint launch skips the entries of
    # pairs sharing a vertex, the singular pass computes exactly those)
    entries = sum(p.payload_len for dv in per_dev for p in dv[4][:1])
    pairs_local = entries * len(specs)
    pairs_job = dist.sum(pairs_local) if shard else pairs_local * (dist.world if not strong
                                                                   else 1)

    def time_plans(which, steps, warmup):
        evs = {d: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for d, *_ in per_dev}

        def step():
            for d, st, flush, main, sep in per_dev:
                with torch.cuda.device(d), torch.cuda.stream(st):
                    l2_flush(flush)
                    evs[d][0].record(st)
                    for p in (main if which == "main" else sep):
                        p.execute()
                    evs[d][1].record(st)
            for d, st, *_ in per_dev:
                st.synchronize()
            t = max(evs[d][0].elapsed_time(evs[d][1]) for d, *_ in per_dev)
            # disjoint-launch ms of each plan on the first device (the roofline's kernel)
            main, sep = per_dev[0][3], per_dev[0][4]
            return t, [p.timing_ms()["disjoint"] for p in (main if which == "main" else sep)]
        for _ in range(warmup):
            step()
        dist.barrier()
        for d, *_ in per_dev:
            torch.cuda.synchronize(d)
        per, dk = [], []
        w0 = time.perf_counter()
        for _ in range(steps):
            t, k = step()
            per.append(t)
            dk.append(k)
        for d, *_ in per_dev:
            torch.cuda.synchronize(d)
        wall_ = time.perf_counter() - w0
        dist.barrier()
        return statistics.mean(per), np.mean(np.array(dk), axis=0), wall_

    peak = devmod.fp64_peak_tflops(devices[0])
    with ClockSampler(devices[0]) as clk:
        ms, dk, wall = time_plans("main", args.steps, args.warmup)
    ms_max = dist.max(ms)
    value = pairs_job / (ms_max * 1e-3)
    single_device = dist.world == 1 and len(devices) == 1
    separate = None
    if fused and single_device and not args.no_separate:  # the same work as two single-layer plans
        ms_sep, dk_sep, _ = time_plans("sep", args.steps, 3)
        fl_sep = [p.flops() for p in per_dev[0][4]]
        kd = int(np.argmax(dk_sep))
        separate = {"value": pairs_job / (ms_sep * 1e-3), "ms_per_step": ms_sep,
                    "dominant_kernel": f"disjoint_kernel<{cfg['orders'][0]},{specs[kd].layer}>",
                    "dominant_frac": fl_sep[kd]["disjoint"] / (dk_sep[kd] * 1e-3) / 1e12 / peak}

    # roofline of the dominant kernel (the disjoint quadrature launch) on the
    # first device of this process: its algorithmic flops / its event time
    main0 = per_dev[0][3]
    fl = [p.flops() for p in main0]
    k_dom = int(np.argmax(dk))
    achieved = fl[k_dom]["disjoint"] / (dk[k_dom] * 1e-3) / 1e12
    share = float(np.sum(dk) / ms)   # of the step on the first device
    dom_name = "pair" if fused else specs[k_dom].layer
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(f"{args.config}/{dom_name}")
        except (OSError, ValueError):
            traffic = None
    h2d = sum(p.h2d_bytes for dv in per_dev for p in dv[3])
    mirrored_info = per_dev[0][3][0].layout.mirror_info if per_dev[0][3][0].mirrored else {}
    launches = args.steps * sum(p.launches_per_execute() for dv in per_dev for p in dv[3])
    for dv in per_dev:
        for p in dv[3] + dv[4]:
            p.close()
    del per_dev, pk

    # e2e through the public API, host buffers, H2D + D2H inside the step
    backend = scheduler.Backend("cuda", devices=tuple(devices))
    params = scheduler.SchedulerParams(backends=(backend,), shard=shard,
                                       mirror=not args.no_mirror,
                                       symmetric_download=False if args.no_sym_download
                                       else None)
    e2e_t, e2e_phases, d2h, payload_bytes = [], [], 0, 0

    def assemble_all(stats_list):
        if fused:
            return list(scheduler.run_assembly_pair(m, bt, cfg["equation"], cfg["kappa"], ops,
                                                    ops, params, cfg["orders"], stats_list[0]))
        return [scheduler.run_assembly(m, bt, s, ops, ops, params, cfg["orders"], st_)
                for s, st_ in zip(specs, stats_list)]
    setup_first = None
    if args.e2e_steps > 0:
        scheduler.clear_package_cache()
        st_warm = [scheduler.AssemblyStats() for _ in specs]
        warm = assemble_all(st_warm)  # path + pinned pool
        # bytes the download moved (a symmetric download skips the SKIP
        # leaves of the single layer: less than the payloads' size)
        d2h = sum(x.d2h_bytes for x in st_warm)
        payload_bytes = sum(M.buffer.nbytes for M in warm)
        del warm
    for k in range(args.e2e_steps):
        dist.barrier()
        scheduler.clear_package_cache()  # every step packages once
        t0 = time.perf_counter()
        st = [scheduler.AssemblyStats() for _ in specs]
        mats = assemble_all(st)
        dt = time.perf_counter() - t0
        e2e_phases = [dict(x.phase_s) for x in st if x.phase_s]
        e2e_t.append(dt)
        del mats
        log(f"e2e step {k}: {dt:.4f} s {e2e_phases}")
        if setup_first is None:
            setup_first = dt
    e2e_dt = dist.max(statistics.median(e2e_t)) if e2e_t else None
    e2e_value = pairs_job / e2e_dt if e2e_dt else None
    d2h_job = dist.sum(d2h) if shard else d2h * (dist.world if not strong else 1)
    payload_job = dist.sum(payload_bytes) if shard else \
        payload_bytes * (dist.world if not strong else 1)
    h2d_job = dist.sum(h2d) if shard else h2d * (dist.world if not strong else 1)

    # solve-phase product on the device-resident operator (h2.matvec, SURVEY
    # 8(f)2): HBM-bound, reported against the measured copy bandwidth
    matvec_line = None
    if not args.no_matvec and single_device:
        from paper_1510_07244_b200 import h2
        M = scheduler.run_assembly(m, bt, specs[0], ops, ops, params, cfg["orders"])
        D = h2.DeviceH2(M, devices[0])
        rng = np.random.default_rng(0)
        x = rng.standard_normal(M.shape[1]) + 1j * rng.standard_normal(M.shape[1])
        for _ in range(3):
            D.matvec(x)
        mv_ms = []
        for _ in range(10):
            D.matvec(x)
            mv_ms.append(D.last_device_ms)
        mv = statistics.median(mv_ms)
        hbm = _hbm_peak()
        gbs = D.bytes_per_product / (mv * 1e-3) / 1e9
        matvec_line = {"operator": specs[0].layer, "device_ms": mv,
                       "bytes_per_product": int(D.bytes_per_product), "GB_s": gbs,
                       "hbm_peak_GB_s": hbm, "frac": gbs / hbm if hbm else None}
        D.close()
        del M
    cpu = None
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu:
        import oracle
        oracle.build()
        nth = host_threads()
        cpk = packaging.make_packages(m.triangles, bt, ops, ops, scheduler.DEFAULT_MAXSIZE)
        pairs, dt, desc, _ = cpu_sample(cpk, m, cfg, args.cpu_seconds, nth, log)
        cpu = {"value": pairs / dt, "unit": UNIT, "cores": nth, "kind": "port", "sample": desc}
        del cpk

    gca_s = dist.max(setup_t["gca_s"])
    gca_warm = dist.max(setup_t.get("gca_warm_s", 0.0))
    trees_s = dist.max(setup_t["trees_s"])
    asm_first = dist.max(setup_first) if setup_first else None
    h2_setup = {"mesh_s (input, not counted)": round(setup_t["mesh_s"], 3),
                "trees_s": round(trees_s, 3), "gca_s": round(gca_s, 3),
                "gca_warm_s (second call)": round(gca_warm, 3),
                "gca_phases_s (rank 0)": {k: round(v, 4) if isinstance(v, float) else v
                                          for k, v in setup_t.get("gca_phases", {}).items()},
                "assembly_slp_dlp_s": round(asm_first, 4) if asm_first else None,
                "total_s": round(trees_s + gca_s + asm_first, 3) if asm_first else None,
                "total_warm_s": round(trees_s + gca_warm + e2e_dt, 3) if e2e_t else None,
                "timing": "max over ranks of each phase; GCA first call of the process "
                          "(total_s) and a second call (total_warm_s)"}
    par = (f"strong x{dist.world * len(devices)}: one job, GCA clusters and leaf sets "
           f"split over {'ranks' if dist.world > 1 else 'devices'} (pivot all-gather the only "
           f"exchange)") if strong and (dist.world > 1 or len(devices) > 1) else \
        (f"weak x{dist.world}, every rank its own job, no collectives" if dist.world > 1
         else "1 GPU")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": dist.world * len(devices),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
        "higher_is_better": True, "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (deterministic octahedral sphere level {cfg['level']})",
        "config": {"workload": cfg["workload"], "pairs_per_step": int(pairs_job),
                   "pair_count": "payload entries of both operators (each one pair integral "
                                 "evaluated once: disjoint rule, or the singular rule for "
                                 "pairs sharing a vertex)",
                   "operators": list(cfg["layers"]), "orders": list(cfg["orders"]),
                   "plan": "one fused SLP+DLP plan (scheduler.run_assembly_pair)" if fused
                   else "one plan per operator (scheduler.run_assembly)",
                   "mirrored_evaluation": bool(mirrored_info) and not args.no_mirror,
                   "mirror_counts": mirrored_info,
                   "l2": "flushed between steps (512 MiB device write)",
                   "parallelism": par},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": f"disjoint_kernel<{cfg['orders'][0]},{dom_name}>"
                               + (" (fused single+double layer: r, 1/r, phase once per point; "
                                  "flops = roofline.F_DISJOINT_PAIR)" if fused else ""),
                     "peak_source": "measured DFMA probe (gcabem_fp64_probe), this device",
                     "traffic_source": "ncu dram__bytes_read+write of this kernel and config "
                                       "(profiles/ncu_traffic.json)",
                     "kernel_share_of_step": share},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d_job),
                "d2h_bytes_per_step": int(d2h_job), "seconds_per_step": e2e_dt,
                "payload_bytes_per_step": int(payload_job),
                "symmetric_download": bool(d2h_job < payload_job),
                "phases_s": [{k: round(v, 4) for k, v in ph.items()} for ph in e2e_phases]},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "h2_setup": h2_setup,
        "device": info["name"], "wall_s_timed": wall, "plan_upload_s": plan_s,
        "flops_per_step": {("pair" if fused else s.layer): f for s, f in zip(specs, fl)},
        "separate_plans": separate,
    }
    if matvec_line is not None:
        line["matvec"] = matvec_line
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if single_device and not args.no_secondary and args.config == "c3":
        line["secondary"] = {"c5_order3": secondary_c5(devices[0], peak, log)}
    return line if dist.rank == 0 else None


def secondary_c5(device, peak, log):
    """C5 at n = 3 (BASELINE configs[4]: L8 sphere, 524,288 triangles,
    Helmholtz kappa=4 SLP+DLP, disjoint = singular order 3): the device step
    of the fused mirrored pair plan only (value and roofline, no e2e)."""
    import torch

    from paper_1510_07244_b200 import device as devmod
    from paper_1510_07244_b200 import kernels, packaging, scheduler
    cfg = dict(CONFIGS["c5"])
    t0 = time.perf_counter()
    m, bt, ops, st = build_workload(cfg, [device], None, log, warm_gca=False)
    pk = packaging.make_packages(m.triangles, bt, ops, ops, scheduler.DEFAULT_MAXSIZE)
    spec = kernels.KernelSpec(cfg["equation"], "single", cfg["kappa"])
    plan = scheduler.AssemblyPlan(devmod.device_mesh(m, device), spec, pk, cfg["orders"],
                                  pair=True)
    stream = torch.cuda.Stream(device=device)
    plan.set_stream(stream.cuda_stream)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{device}")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms, dk = [], []
    for k in range(5):
        with torch.cuda.stream(stream):
            flush.zero_()
            ev0.record(stream)
            plan.execute()
            ev1.record(stream)
        stream.synchronize()
        if k >= 2:   # 2 warm-up steps
            ms.append(ev0.elapsed_time(ev1))
            dk.append(plan.timing_ms()["disjoint"])
    fl = plan.flops()
    res = {"workload": cfg["workload"] + ", orders 3/3", "pairs_per_step": 2 * pk.payload_len,
           "ms_per_step": statistics.mean(ms),
           "value": 2 * pk.payload_len / (statistics.mean(ms) * 1e-3), "unit": UNIT,
           "roofline_frac": fl["disjoint"] / (statistics.mean(dk) * 1e-3) / 1e12 / peak,
           "gca_s": round(st["gca_s"], 3), "build_s": round(time.perf_counter() - t0, 1)}
    plan.close()
    del plan, pk
    devmod.release_cached(device)
    log(f"secondary C5 n=3: {res}")
    return res


def _hbm_peak():
    """Measured HBM copy bandwidth (GB/s) from MEASURED_PEAKS.json, else the
    profiling recipe's fallback."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6550.0


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=tuple(CONFIGS), default="c3")
    ap.add_argument("--mode", choices=("weak", "strong"), default="strong")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--gca-seconds", type=float, default=20.0,
                    help="reference arm: wall seconds of the sampled GCA clusters")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-matvec", action="store_true")
    ap.add_argument("--no-mirror", action="store_true",
                    help="evaluate every pair on its own (no symmetric evaluation of mirror "
                         "leaves)")
    ap.add_argument("--no-sym-download", action="store_true",
                    help="e2e: copy every payload entry (no symmetric download of the single "
                         "layer's mirror leaves)")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the C5 (order 3) device-step key of the default C3 line")
    ap.add_argument("--no-separate", action="store_true",
                    help="skip timing the single-layer plans next to the fused one")
    ap.add_argument("--separate", action="store_true",
                    help="time SLP and DLP as two single-layer plans (default: one fused plan)")
    ap.add_argument("--order", type=int, default=None,
                    help="override the quadrature orders (disjoint n = singular n), e.g. C5")
    args = ap.parse_args(argv)
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    cfg = dict(CONFIGS[args.config])
    if args.order is not None:
        cfg["orders"] = (args.order, args.order)
        cfg["workload"] += f", orders {args.order}/{args.order}"
    dist = Dist(cpu_only=args.impl == "reference")

    def log(msg):
        if dist.rank == 0:
            print(f"[bench] {msg}", file=sys.stderr, flush=True)

    try:
        if args.impl == "reference":
            line = run_reference(args, cfg, dist, log)
        elif cfg.get("p1"):
            line = run_ours_p1(args, cfg, dist, log)
        else:
            line = run_ours(args, cfg, dist, log)
        if line is not None and dist.rank == 0:
            print(json.dumps(line), flush=True)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
