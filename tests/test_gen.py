"""The seeded input generator: determinism, shard independence, and the workload
properties DESIGN.md §4 promises (corruption rates, full stall breakdown, the planted
> 2^32 bin, stream layout, structure validity).  CPU only (device build: test_gpu_*)."""
import numpy as np
import pytest

import gen

NONE = gen.NONE


def test_records_are_a_pure_function_of_k():
    w = gen.workload("C3", records=1_000_000)
    full = w.records_host(threads=7)
    assert np.array_equal(full, w.records_host(threads=1))
    for k0, n in [(0, 1), (4095, 3), (123_457, 10_000), (999_990, 10)]:
        assert np.array_equal(w.records_host(k0, n, threads=3), full[k0:k0 + n])


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_structure_is_well_formed(name):
    w = gen.workload(name)
    st = w.structure
    a, ln = st["inst_addr"], st["inst_len"].astype(np.uint64)
    assert (np.diff(a.astype(np.int64)) > 0).all() and (a[:-1] + ln[:-1] <= a[1:]).all()
    kind, par = st["scope_kind"], st["scope_parent"]
    assert ((par == NONE) == (kind == gen.KIND_FUNCTION)).all()
    assert (kind[st["inst_scope"]] == gen.KIND_LINE).all()
    has_p = par != NONE
    assert (kind[par[has_p]] != gen.KIND_LINE).all()
    assert sorted(st["func_scope"].tolist()) == np.nonzero(kind == gen.KIND_FUNCTION)[0].tolist()
    assert len(np.unique(st["call_inst"])) == len(st["call_inst"])
    assert (np.diff(st["call_inst"].astype(np.int64)) > 0).all()
    assert (st["inst_class"][st["call_inst"]] == gen.CLASS_CALL).all()
    assert st["call_callee"].max() < len(st["func_scope"])
    cfg = w.cfg
    assert w.meta["n_inst"] == cfg.n_inst and w.meta["n_func"] == cfg.n_func
    assert w.meta["static_contexts"] <= cfg.ctx_budget


def test_corruption_and_misalignment_rates():
    w = gen.workload("C2", records=2_000_000)
    rec = w.records_host()
    n = len(rec)
    bad_stall = (rec["stall"] >= 12).mean()
    assert 0.3e-4 < bad_stall < 3e-4
    a = w.structure["inst_addr"]
    j = np.searchsorted(a, rec["pc"], side="right") - 1
    inside = (j >= 0) & (rec["pc"] < a[np.maximum(j, 0)] + 16)
    assert 0.3e-4 < (~inside).mean() < 3e-4
    mis = inside & (rec["pc"] != a[np.maximum(j, 0)])
    assert 0.005 < mis.mean() < 0.015
    assert rec["count"].min() >= 1 and abs(rec["count"].mean() - 2.0) < 0.05
    assert n == 2_000_000


def test_c5_full_stall_breakdown_and_hot_bin():
    w = gen.workload("C5")
    cum = w.tables["stall_cum"].astype(np.int64).reshape(-1, 12)
    p = np.diff(np.concatenate([np.zeros((len(cum), 1), np.int64), cum], 1), axis=1) / 2.0 ** 31
    assert (p >= 0.0099).all()                           # every reason >= 1% everywhere
    t = w.tables
    assert t["hot_records"] == 65537 and t["hot_records"] * 65536 > 2 ** 32
    stride = t["hot_stride"]
    ks = [0, stride, stride * 65536, stride * 65536 + 1]
    recs = [w.records_host(k, 1)[0] for k in ks]
    hot_pc = w.structure["inst_addr"][t["hot_inst"]]
    assert all(r["pc"] == hot_pc and r["count"] == 65536 and r["stall"] == 5 for r in recs[:3])
    assert not (recs[3]["count"] == 65536 and recs[3]["pc"] == hot_pc)
    assert w.structure["inst_class"][t["hot_inst"]] == gen.CLASS_SYNC


def test_c4_streams():
    w = gen.workload("C4", records=50_000_000)
    sfb = w.tables["stream_first_burst"]
    assert len(sfb) == 384 and sfb[0] == 0 and (np.diff(sfb.astype(np.int64)) >= 1).all()
    for k0 in (0, 10_000_000, 49_990_000):
        s = w.records_host(k0, 10_000)["stream"]
        assert (np.diff(s.astype(np.int64)) >= 0).all() and s.max() < 384
    assert w.records_host(49_999_999, 1)["stream"][0] == 383


def test_trace_sets_are_seeded_and_well_formed():
    """f4 inputs (gen/trace.py): deterministic per seed, every line non-decreasing in time, ranks
    grouped, every rank has GPU and CPU lines, routine ids in range, mostly idle-terminated."""
    from gen.trace import TRACE_CONFIGS, trace_set
    for name in ("B1", "B2"):
        a, b = trace_set(name), trace_set(name)
        for k in ("line_off", "line_kind", "line_scope", "time", "ctx"):
            assert np.array_equal(a[k], b[k]), k
        cfg = TRACE_CONFIGS[name]
        lo = a["line_off"].astype(np.int64)
        assert lo[0] == 0 and lo[-1] == len(a["time"]) and (np.diff(lo) > 0).all()
        assert (np.diff(a["line_scope"].astype(np.int64)) >= 0).all() and a["line_scope"][-1] == cfg.scopes - 1
        for l in range(len(lo) - 1):
            t = a["time"][lo[l]:lo[l + 1]]
            assert (np.diff(t.astype(np.int64)) >= 0).all()
            c = a["ctx"][lo[l]:lo[l + 1]]
            if a["line_kind"][l] == 1:
                live = c[c != 0xFFFFFFFF]
                assert (live < cfg.n_routines).all()
        for s in range(cfg.scopes):
            kinds = a["line_kind"][a["line_scope"] == s]
            assert (kinds == 0).sum() == cfg.gpu_lines and (kinds == 1).sum() == cfg.cpu_lines
