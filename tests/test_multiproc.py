"""N>1 path on CPU (gloo, world size 2): the leaf-range sharding used by
SchedulerParams.shard / bench --mode strong partitions the work with no
data-path exchange, and the union of the shards' payloads (computed here by
the oracle on each rank's own blocks and items) equals the single-process
assembly bit for bit."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, out_path):
    import torch
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from helpers import packages_for
    from paper_1510_07244_b200.packaging import shard_leaves
    m, bt, ops, pk = packages_for(4, "laplace", near_only=True)
    lo, hi = shard_leaves(pk, world, 81, [1250, 3125, 3750])[rank]
    p0, p1 = int(pk.leaf_base[lo]), int(pk.leaf_base[hi])
    part = np.zeros(p1 - p0, dtype=np.complex128)
    blocks = pk.device_blocks(lo, hi)
    cnt = blocks[:, 2] * blocks[:, 3]
    own = np.repeat(np.arange(len(blocks)), cnt)
    k = np.arange(own.size) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    i, j = k // blocks[own, 3], k % blocks[own, 3]
    vals = oracle.batch_quadrature("laplace", "single", 0.0, m.vertices, m.triangles,
                                   m.normals, m.gramians, pk.panels[blocks[own, 4] + i],
                                   pk.panels[blocks[own, 5] + j], None, None,
                                   *oracle.rule("disjoint", 3))
    part[blocks[own, 0] + i * blocks[own, 1] + j] = vals
    items, perms = pk.device_items(lo, hi)
    for code, case in ((1, "vertex"), (2, "edge"), (3, "identical")):
        sel = items[:, 0] == code
        if np.any(sel):
            part[items[sel, 3]] = oracle.batch_quadrature(
                "laplace", "single", 0.0, m.vertices, m.triangles, m.normals, m.gramians,
                items[sel, 1], items[sel, 2], perms[sel, :3].astype(np.int64),
                perms[sel, 3:].astype(np.int64), *oracle.rule(case, 5))
    # gather (test-side only: the product has no collective on the data path)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([part.size], dtype=torch.int64))
    n_max = int(max(s.item() for s in sizes))
    buf = torch.zeros(2 * n_max, dtype=torch.float64)
    buf[:2 * part.size] = torch.from_numpy(part.view(np.float64))
    got = [torch.zeros(2 * n_max, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(got, buf)
    ranges = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(ranges, torch.tensor([lo, hi], dtype=torch.int64))
    if rank == 0:
        full = np.concatenate([g[:2 * int(s.item())].numpy() for g, s in zip(got, sizes)])
        np.save(out_path, full.view(np.complex128))
        np.save(out_path + ".ranges.npy", np.stack([r.numpy() for r in ranges]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_reassemble_bitwise(tmp_path):
    from helpers import checksum, packages_for
    out = str(tmp_path / "payload.npy")
    mp.spawn(_rank_main, args=(2, _free_port(), out), nprocs=2, join=True)
    full = np.load(out)
    ranges = np.load(out + ".ranges.npy")
    m, bt, ops, pk = packages_for(4, "laplace", near_only=True)
    assert ranges[0][0] == 0 and ranges[0][1] == ranges[1][0] and ranges[1][1] == pk.leaf_ids.size
    assert full.size == pk.payload_len
    import json
    ref = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
    assert checksum(pk, full) == ref["checksums"]["L4-near/laplace/single/3-5"]


@pytest.mark.timeout(600)
def test_bench_reference_arm_under_torchrun():
    """bench.py --impl reference launched as the driver does for N>1: rank 0
    prints one JSON line, the other rank exits 0 without work."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl",
           "reference", "--config", "c1", "--gpus", "2", "--steps", "1", "--warmup", "0",
           "--cpu-seconds", "0.5"]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    import json
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["n_gpus"] == 2
    assert d["cpu_baseline"]["kind"] == "port" and d["e2e"]["h2d_bytes_per_step"] == 0


def _pivot_rank_main(rank, world, port, out_path):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from helpers import level_ops, sphere_setup
    from paper_1510_07244_b200 import gca, scheduler
    g = np.load(os.path.join(ROOT, "tests", "golden", "gca_levels.npz"))
    m, t, bt = sphere_setup(4)
    ops_all = level_ops(lambda name: g, 4, "helmholtz")
    parts = gca.partition_clusters(t, list(ops_all), world)
    local = {int(c): ops_all[int(c)] for c in parts[rank]}
    got = gca.exchange_pivots(local, True)
    ok = sorted(got) == sorted(ops_all)
    for c, op in got.items():
        ok &= np.array_equal(op.pivots_global, ops_all[c].pivots_global)
        ok &= np.array_equal(op.pivots_local, ops_all[c].pivots_local)
        ok &= op.rank == ops_all[c].rank
        ok &= (op is local[c]) if c in local else op.V.shape == (0, ops_all[c].rank)
    from paper_1510_07244_b200 import packaging
    mine = scheduler.shard_leaves_of(m, bt, got, got, (rank, world), 81)
    # every leaf travels with its mirror
    mir = packaging.leaf_mirrors(bt, got, got)
    ok &= bool(np.all(np.isin(mir[mine], mine)))
    res = torch.tensor([int(ok), mine.size, len(local)], dtype=torch.int64)
    allres = [torch.zeros(3, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allres, res)
    L = len(bt.leaves)
    mask = torch.zeros(L, dtype=torch.int64)
    mask[torch.from_numpy(mine)] = 1
    dist.all_reduce(mask)
    if rank == 0:
        np.save(out_path, np.stack([r.numpy() for r in allres]))
        np.save(out_path + ".mask.npy", mask.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gca_shard_pivot_exchange(tmp_path, world):
    """GCA split over processes (build_interpolation_operators(shard=...)):
    the cluster parts tile the admissible clusters, exchange_pivots gives
    every rank every cluster's pivots (the reference's, here from the
    fixture) with V only for its own, and the ranks' leaf sets
    (scheduler.shard_leaves_of, computed independently per rank) partition
    the leaves, each leaf in the set of its mirror."""
    out = str(tmp_path / "res.npy")
    mp.spawn(_pivot_rank_main, args=(world, _free_port(), out), nprocs=world, join=True)
    res = np.load(out)
    assert np.all(res[:, 0] == 1)
    mask = np.load(out + ".mask.npy")
    assert np.all(mask == 1)                       # every leaf in exactly one set
    assert np.all(res[:, 1] > 0) and np.all(res[:, 2] > 0)
