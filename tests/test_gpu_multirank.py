"""The N > 1 path on GPUs (a-4 cross-GPU combine; P:687 profiles distributed over
ranks, "aggregated by a second reduction" and statistics generated in parallel).

Ranks attribute record shards with the CUDA kernels, combine them with the collective bench.py
uses, and derive their function-aligned rows; the assembled result must equal the CPU oracle
(integers bit-exact, fp64 bit-identical).  With >= 2 GPUs the ranks use NCCL, one GPU each;
on a one-GPU box two ranks share cuda:0 over gloo (the same code path minus NCCL)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCOPES = ("INST", "LINE", "LOOP", "INLINE", "FUNC")


@pytest.fixture(scope="module")
def gpa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    from paper_2109_06931_b200 import gpa
    return gpa


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _world():
    n = torch.cuda.device_count()
    return (min(n, 4), "nccl") if n >= 2 else (2, "gloo")


def _worker(rank, world, backend, port, name, records, root_less, combine, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev_i = rank % torch.cuda.device_count()
    torch.cuda.set_device(dev_i)
    dev = torch.device("cuda", dev_i)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2109_06931_b200 import gpa
        from paper_2109_06931_b200.parallel import reduce_histogram, reduce_scatter_histogram, shard_range
        w = gen.workload(name, records=records)
        st = w.structure
        s = gpa.load_structure(st, dev_i)
        ni, nf, nc = s.info["n_inst"], s.info["n_func"], s.info["n_call"]
        a, b = shard_range(w.cfg.records, rank, world, root_less)
        rec = torch.empty((max(b - a, 1), 2), dtype=torch.int64, device=dev)
        if b > a:
            w.records_device(rec, a, b - a)
        HU = torch.zeros(ni * 16 + 16, dtype=torch.int64, device=dev)
        H, U = HU[:ni * 16].view(ni, 16), HU[ni * 16:]
        gpa.attribute_samples(s, rec, H, U, n=b - a)
        res = {}
        if combine == "reduce":
            reduce_histogram(HU, dst=0)
            if rank == 0:
                res["HU"] = HU.cpu().numpy().view(np.uint64).copy()
        else:
            bounds = [int(x) for x in gpa.partition_structure(st, world)]
            lo, hi = bounds[rank], bounds[rank + 1]
            reduce_scatter_histogram(HU, bounds, ni)
            res.update(lo=lo, hi=hi, H=H[lo:hi].cpu().numpy().view(np.uint64).copy())
            if rank == world - 1:
                res["U"] = U.cpu().numpy().view(np.uint64).copy()
            for sc in SCOPES:
                rows = len(s.rows(sc))
                hist = torch.full((max(rows, 1), 16), -1, dtype=torch.int64, device=dev)
                met = torch.full((max(rows, 1), 33), -7.0, dtype=torch.float64, device=dev)
                if rows:
                    gpa.derive_metrics_range(s, sc, H, lo, hi, scope_hist=hist, metrics=met)
                res[sc] = (hist.cpu().numpy().view(np.uint64), met.cpu().numpy())
            SW = torch.zeros(nf * 16 + nc, dtype=torch.int64, device=dev)
            gpa.cct_inputs(s, H, lo, hi, SW[:nf * 16].view(nf, 16), SW[nf * 16:])
            dist.reduce(SW, dst=0)
            if rank == 0:
                c = gpa.reconstruct_cct_inputs(s, SW[:nf * 16].view(nf, 16), SW[nf * 16:])
                res["cct"] = c.to_numpy()
                c.free()
        torch.cuda.synchronize()
        np.save(f"{out}_{rank}.npy", np.array([res], dtype=object))
        s.free()
    finally:
        dist.destroy_process_group()


def _run(name, records, root_less, combine, tmp_path):
    import torch.multiprocessing as mp
    world, backend = _world()
    out = str(tmp_path / "r")
    mp.start_processes(_worker, args=(world, backend, _free_port(), name, records, root_less, combine, out),
                       nprocs=world, join=True, start_method="spawn")
    return world, [np.load(f"{out}_{r}.npy", allow_pickle=True)[0] for r in range(world)]


@pytest.mark.parametrize("name,records,root_less", [("C2", 5_000_011, 0), ("C4", 4_500_000, 10 ** 10),
                                                    ("C3", 3_000_017, 400_000)])
def test_multirank_scatter_equals_oracle(gpa, tmp_path, name, records, root_less):
    """Shards (incl. an empty rank-0 shard: root_less beyond the stream) attributed on the GPU,
    reduce-scattered at function-aligned bounds, rows derived per rank and the CCT rebuilt on rank
    0 from the summed S_f || w: every piece equals the single-process oracle."""
    world, res = _run(name, records, root_less, "scatter", tmp_path)
    w = gen.workload(name, records=records)
    st = w.structure
    H, U, _ = oracle.attribute(st, w.records_host(0, w.cfg.records), threads=len(os.sched_getaffinity(0)))
    for r in range(world):
        lo, hi = res[r]["lo"], res[r]["hi"]
        assert np.array_equal(res[r]["H"], H[lo:hi]), r
    assert np.array_equal(res[world - 1]["U"], U)
    # every row of every scope is written by exactly one rank, bit-equal to the oracle's
    for sc in SCOPES:
        eh, em = oracle.scope_hist(st, H, sc)
        emet = oracle.derive_u64(eh, em)
        got_h = np.full_like(eh, 0xFFFFFFFFFFFFFFFF)
        got_m = np.full(emet.shape, -7.0)
        owners = np.zeros(len(eh), np.int64)
        for r in range(world):
            hh, mm = res[r][sc]
            wrote = ~np.all(hh[:len(eh)] == 0xFFFFFFFFFFFFFFFF, axis=1)
            owners += wrote
            got_h[wrote] = hh[:len(eh)][wrote]
            got_m[wrote] = mm[:len(eh)][wrote]
        assert np.all(owners == 1), sc
        assert np.array_equal(got_h, eh), sc
        assert np.array_equal(got_m.view(np.uint64), emet.view(np.uint64)), sc
    R = oracle.cct(st, H)
    g = res[0]["cct"]
    assert g["n"] == R["n"]
    for k in ("parent", "site", "node", "kind"):
        assert np.array_equal(g[k], R[k]), k
    for k in ("frac", "excl", "incl"):
        assert np.array_equal(g[k].view(np.uint64), R[k].view(np.uint64)), k


def test_multirank_reduce_equals_oracle(gpa, tmp_path):
    """--combine reduce: the collective sum of the GPU partials on rank 0 equals the oracle."""
    world, res = _run("C5", 3_000_001, 0, "reduce", tmp_path)
    w = gen.workload("C5", records=3_000_001)
    H, U, _ = oracle.attribute(w.structure, w.records_host(0, w.cfg.records), threads=len(os.sched_getaffinity(0)))
    assert np.array_equal(res[0]["HU"], np.concatenate([H.reshape(-1), U]))


def test_derive_metrics_range_matches_full(gpa):
    """Single process: the range entry points write exactly the range's rows, bit-equal to the
    full derive_metrics / reconstruct_cct; misaligned ranges are refused."""
    w = gen.workload("C3", records=2_000_000)
    st = w.structure
    s = gpa.load_structure(st, 0)
    rec = torch.empty((w.cfg.records, 2), dtype=torch.int64, device="cuda")
    w.records_device(rec)
    ni, nf, nc = s.info["n_inst"], s.info["n_func"], s.info["n_call"]
    H = torch.zeros((ni, 16), dtype=torch.int64, device="cuda")
    U = torch.zeros(16, dtype=torch.int64, device="cuda")
    gpa.attribute_samples(s, rec, H, U)
    b = [int(x) for x in gpa.partition_structure(st, 5)]
    for sc in SCOPES:
        rows = len(s.rows(sc))
        full = torch.empty((rows, 33), dtype=torch.float64, device="cuda")
        gpa.derive_metrics(s, sc, H, metrics=full)
        got = torch.full((rows, 33), -7.0, dtype=torch.float64, device="cuda")
        for r in range(5):
            gpa.derive_metrics_range(s, sc, H, b[r], b[r + 1], metrics=got)
        assert np.array_equal(got.cpu().numpy().view(np.uint64), full.cpu().numpy().view(np.uint64)), sc
    SF = torch.zeros((nf, 16), dtype=torch.int64, device="cuda")
    CW = torch.zeros(nc, dtype=torch.int64, device="cuda")
    for r in range(5):
        gpa.cct_inputs(s, H, b[r], b[r + 1], SF, CW)
    c1, c2 = gpa.reconstruct_cct(s, H), gpa.reconstruct_cct_inputs(s, SF, CW)
    g1, g2 = c1.to_numpy(), c2.to_numpy()
    assert g1["n"] == g2["n"] and all(np.array_equal(g1[k], g2[k]) for k in ("parent", "node", "incl"))
    c1.free(), c2.free()
    with pytest.raises(gpa.GpaError) as ei:
        gpa.derive_metrics_range(s, "LINE", H, 1, b[1], metrics=got)   # not a function start
    assert ei.value.status == 1


def test_bench_two_ranks(gpa):
    """bench.py --gpus 2 starts two ranks itself and prints one line with n_gpus = 2."""
    world, backend = _world()
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dist-backend", backend, "--config", "C2",
           "--records", "6000000", "--steps", "2", "--warmup", "3", "--no-e2e", "--no-cpu-baseline"]
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and "reduce-scatter" in d["config"]["parallelism"]


@pytest.mark.parametrize("name,records", [("C2", 3_000_000), ("C3", 2_000_000), ("C1", 50_000)])
def test_derive_scopes_matches_per_scope(gpa, name, records):
    """gpa_derive_scopes (all kinds in one launch) writes exactly what gpa_derive_metrics writes per
    scope (histograms, mixes, metrics; bit-identical), for the whole structure and for
    function-aligned ranges."""
    w = gen.workload(name, records=records)
    st = w.structure
    s = gpa.load_structure(st, 0)
    rec = torch.empty((w.cfg.records, 2), dtype=torch.int64, device="cuda")
    w.records_device(rec)
    ni = s.info["n_inst"]
    H = torch.zeros((ni, 16), dtype=torch.int64, device="cuda")
    U = torch.zeros(16, dtype=torch.int64, device="cuda")
    gpa.attribute_samples(s, rec, H, U)
    rows = {sc: len(s.rows(sc)) for sc in SCOPES}

    def outs(fill):
        return {sc: {"scope_hist": torch.full((max(rows[sc], 1), 16), fill, dtype=torch.int64, device="cuda"),
                     "scope_mix": torch.full((max(rows[sc], 1), 16), fill, dtype=torch.int64, device="cuda"),
                     "metrics": torch.full((max(rows[sc], 1), 33), float(fill), dtype=torch.float64, device="cuda")}
                for sc in SCOPES}

    ref = outs(-1)
    for sc in SCOPES:
        if rows[sc]:
            gpa.derive_metrics(s, sc, H, **ref[sc])
    got = outs(-1)
    gpa.derive_scopes(s, H, got)
    parts = outs(-1)
    b = [int(x) for x in gpa.partition_structure(st, 3)]
    for r in range(3):
        gpa.derive_scopes(s, H, parts, b[r], b[r + 1])
    torch.cuda.synchronize()
    for sc in SCOPES:
        for k in ("scope_hist", "scope_mix", "metrics"):
            a = ref[sc][k].cpu().numpy().view(np.uint64)
            assert np.array_equal(got[sc][k].cpu().numpy().view(np.uint64), a), (sc, k)
            assert np.array_equal(parts[sc][k].cpu().numpy().view(np.uint64), a), (sc, k, "ranges")
