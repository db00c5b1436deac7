"""The N > 1 path on CPU: world_size-2 gloo process groups shard the record stream with
parallel.shard_range and combine per-rank histograms with parallel.reduce_histogram (the
same call bench.py makes over NCCL).  Per-rank partials come from the oracle here (no
GPU); the reduced H||U must equal the single-process oracle bit for bit (integer sums are
associative, "aggregated by a second reduction")."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle
from paper_2109_06931_b200.parallel import reduce_histogram, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, records, out_path, root_less=0):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = gen.workload(name, records=records)
        a, b = shard_range(w.cfg.records, rank, world, root_less)
        rec = w.records_host(a, b - a)
        H, U, _ = oracle.attribute(w.structure, rec)
        HU = torch.from_numpy(np.concatenate([H.reshape(-1), U]).view(np.int64).copy())
        reduce_histogram(HU, dst=0)
        if rank == 0:
            np.save(out_path, HU.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,records,world,root_less", [("C2", 100_003, 2, 0), ("C4", 60_001, 2, 0), ("C1", 1, 2, 0),
                                                       ("C1", 0, 2, 0), ("C2", 100_003, 3, 20_000),
                                                       ("C4", 60_001, 2, 10 ** 9)])
def test_sharded_reduce_equals_single_process(tmp_path, name, records, world, root_less):
    """Equal shards, and bench.py's load-balanced split (rank 0 lighter by root_less records,
    down to an empty rank-0 shard), reduce to the single-process histogram."""
    out = str(tmp_path / "hu.npy")
    mp.start_processes(_worker, args=(world, _free_port(), name, records, out, root_less), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(out).view(np.uint64)
    w = gen.workload(name, records=records)
    H, U, _ = oracle.attribute(w.structure, w.records_host(0, w.cfg.records))
    assert np.array_equal(got, np.concatenate([H.reshape(-1), U]))


def test_shard_range_partitions():
    for n in [0, 1, 7, 1000, 4_000_000_000]:
        for world in [1, 2, 3, 8]:
            parts = [shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_shard_range_root_less_partitions():
    """Load-balanced split: a partition of [0, n); rank 0 holds root_less records fewer than
    the others (up to rounding), or none when root_less is too large."""
    for n in [0, 5, 1000, 4_000_000_000]:
        for world in [2, 3, 8]:
            for d in [1, 17, 143_000_000, 10 ** 12]:
                parts = [shard_range(n, r, world, d) for r in range(world)]
                assert parts[0][0] == 0 and parts[-1][1] == n
                assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
                sizes = [b - a for a, b in parts]
                assert max(sizes[1:]) - min(sizes[1:]) <= 1
                if (world - 1) * d <= n:
                    assert abs((sizes[1] - sizes[0]) - d) <= world
                else:
                    assert sizes[0] == 0


def _blame_worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from gen.trace import trace_set
        from paper_2109_06931_b200.parallel import shard_trace
        tr = trace_set("B2")
        sh = shard_trace(tr, rank, world)
        S = tr["n_scopes"]
        blame = torch.zeros((S, tr["n_routines"]), dtype=torch.float64)
        total = torch.zeros(S, dtype=torch.int64)
        if sh["n_scopes"]:
            sub = dict(sh, time=tr["time"][sh["event0"]:sh["event1"]], ctx=tr["ctx"][sh["event0"]:sh["event1"]])
            r = oracle.blame(sub)
            s0, s1 = sh["scope0"], sh["scope0"] + sh["n_scopes"]
            blame[s0:s1] = torch.from_numpy(r["blame"])
            total[s0:s1] = torch.from_numpy(r["total"].view(np.int64))
        dist.reduce(blame, dst=0)        # disjoint rows: the sum assembles them (test only)
        dist.reduce(total, dst=0)
        if rank == 0:
            np.savez(out_path, blame=blame.numpy(), total=total.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_blame_shards_by_rank(tmp_path, world):
    """f4: every trace rank lands on exactly one worker and the per-worker results, placed at
    their scope offsets, equal the single-process oracle bit for bit."""
    from gen.trace import trace_set
    out = str(tmp_path / "blame.npz")
    mp.start_processes(_blame_worker, args=(world, _free_port(), out), nprocs=world, join=True, start_method="spawn")
    got = np.load(out)
    r = oracle.blame(trace_set("B2"))
    assert np.array_equal(got["blame"].view(np.uint64), r["blame"].view(np.uint64))
    assert np.array_equal(got["total"].view(np.uint64), r["total"])


def test_shard_trace_partitions():
    from gen.trace import trace_set
    from paper_2109_06931_b200.parallel import shard_trace
    tr = trace_set("B2")
    for world in (1, 2, 3, 5, 8, 16):
        parts = [shard_trace(tr, r, world) for r in range(world)]
        assert parts[0]["scope0"] == 0 and parts[0]["event0"] == 0
        assert sum(p["n_scopes"] for p in parts) == tr["n_scopes"]
        assert parts[-1]["event1"] == len(tr["time"])
        for a, b in zip(parts, parts[1:]):
            assert a["scope0"] + a["n_scopes"] == b["scope0"] and a["event1"] == b["event0"]


# ---- distributed statistics: reduce-scatter at function-aligned bounds (R29) ---------
def _scatter_worker(rank, world, port, name, records, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2109_06931_b200 import gpa
        from paper_2109_06931_b200.parallel import reduce_scatter_histogram
        w = gen.workload(name, records=records)
        st = w.structure
        ni = len(st["inst_addr"])
        bounds = gpa.partition_structure(st, world)
        a, b = shard_range(w.cfg.records, rank, world)
        H, U, _ = oracle.attribute(st, w.records_host(a, b - a))
        HU = torch.from_numpy(np.concatenate([H.reshape(-1), U]).view(np.int64).copy())
        reduce_scatter_histogram(HU, bounds, ni)
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        mine = HU.numpy().view(np.uint64)
        # this rank's rows only: the rest of its buffer holds partial sums and must not matter
        Hr = np.zeros((ni, 16), np.uint64)
        Hr[lo:hi] = mine[:ni * 16].reshape(ni, 16)[lo:hi]
        res = {"lo": lo, "hi": hi, "H": Hr[lo:hi]}
        if rank == world - 1:
            res["U"] = mine[ni * 16:]
        for sc in ("LINE", "LOOP", "INLINE", "FUNC"):
            res[sc] = oracle.scope_hist(st, Hr, sc)[0]
        np.save(out_path.replace(".npy", f"_{rank}.npy"), np.array([res], dtype=object))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,records,world", [("C2", 100_003, 2), ("C4", 60_001, 3), ("C1", 5_000, 4)])
def test_reduce_scatter_rows_equal_single_process(tmp_path, name, records, world):
    """Every rank's reduced rows equal the single-process histogram on its function-aligned range,
    and the scope rows computed from a rank's range alone equal the full roll-up on the rows of the
    functions inside that range (so the per-rank derivation is exact); empty ranges (C1 at 4 ranks:
    3 functions) included."""
    from paper_2109_06931_b200 import gpa
    out = str(tmp_path / "rs.npy")
    mp.start_processes(_scatter_worker, args=(world, _free_port(), name, records, out), nprocs=world, join=True,
                       start_method="spawn")
    w = gen.workload(name, records=records)
    st = w.structure
    H, U, _ = oracle.attribute(st, w.records_host(0, w.cfg.records))
    bounds = gpa.partition_structure(st, world)
    for r in range(world):
        res = np.load(out.replace(".npy", f"_{r}.npy"), allow_pickle=True)[0]
        lo, hi = res["lo"], res["hi"]
        assert (lo, hi) == (int(bounds[r]), int(bounds[r + 1]))
        assert np.array_equal(res["H"], H[lo:hi])
        if r == world - 1:
            assert np.array_equal(res["U"], U)
        for sc in ("LINE", "LOOP", "INLINE", "FUNC"):
            full = oracle.scope_hist(st, H, sc)[0]
            rows = _rows_in_range(st, sc, lo, hi)
            assert np.array_equal(res[sc][rows], full[rows]), (sc, r)


def _rows_in_range(st, scope, lo, hi):
    """Rows of `scope` whose function's first instruction lies in [lo, hi) (the function layout
    of gpa_derive_metrics_range), computed from the description by walking scope parents."""
    parent = np.asarray(st["scope_parent"], np.int64)
    kind = np.asarray(st["scope_kind"])
    fscope = np.asarray(st["func_scope"], np.int64)
    func_of_root = {int(x): f for f, x in enumerate(fscope)}
    inst_scope = np.asarray(st["inst_scope"], np.int64)
    ns = len(parent)
    root = np.arange(ns)
    for _ in range(64):
        nxt = np.where(parent[root] == 0xFFFFFFFF, root, parent[root])
        if np.array_equal(nxt, root):
            break
        root = nxt
    func_first = {}
    for i, x in enumerate(inst_scope):
        f = func_of_root[int(root[x])]
        func_first.setdefault(f, i)
    if scope == "FUNC":
        return np.array([f for f in range(len(fscope)) if lo <= func_first.get(f, 1 << 40) < hi], np.int64)
    code = {"LINE": 3, "LOOP": 2, "INLINE": 1}[scope]
    ids = np.nonzero(kind == code)[0]
    return np.array([r for r, x in enumerate(ids) if lo <= func_first.get(func_of_root[int(root[x])], 1 << 40) < hi],
                    np.int64)


def test_partition_structure_bounds():
    """Host-only split: non-decreasing function starts from 0 to n_inst, near the even split."""
    from paper_2109_06931_b200 import gpa
    for name in ("C1", "C2", "C3", "C5"):
        st = gen.workload(name).structure
        ni = len(st["inst_addr"])
        for parts in (1, 2, 3, 8):
            b = gpa.partition_structure(st, parts).astype(np.int64)
            assert b[0] == 0 and b[-1] == ni and np.all(np.diff(b) >= 0)
            if name != "C1":
                assert np.abs(b[1:-1] - ni * np.arange(1, parts) / parts).max(initial=0) < ni / parts
    # a function split into two runs has no function-aligned partition
    st = dict(gen.workload("C1").structure)
    ins = np.asarray(st["inst_scope"]).copy()
    ins[[0, 150]] = ins[[150, 0]]
    st["inst_scope"] = ins
    with pytest.raises(gpa.GpaError) as ei:
        gpa.partition_structure(st, 2)
    assert ei.value.status == 2
