"""Pins of oracle D1 (attribution) and D2 (roll-up) against things other than itself:
a brute-force linear scan, the worked examples in tests/golden, conservation, shard
invariance and explicit top-down scope containment.  CPU only."""
import numpy as np
import pytest

import gen
import oracle
from tests.fixtures import load_golden

NONE = oracle.NONE


def _brute_attribute(addr, ln, rec):
    """Linear scan over every instruction (no search, no sortedness assumption)."""
    n = len(addr)
    H = np.zeros((n, 16), np.uint64)
    U = np.zeros(16, np.uint64)
    ri = np.full(len(rec), NONE, np.uint32)
    for k, (pc, c, s, _) in enumerate(rec.tolist()):
        slot = s if s < 12 else 15
        hit = [i for i in range(n) if addr[i] <= pc < addr[i] + ln[i]]
        assert len(hit) <= 1
        if hit:
            H[hit[0], slot] += c
            ri[k] = hit[0]
        else:
            U[slot] += c
    return H, U, ri


def _random_table(rng, n):
    """Sorted disjoint ranges with random lengths and random gaps (incl. zero gaps)."""
    lens = rng.integers(1, 24, n).astype(np.uint64)
    gaps = rng.integers(0, 3, n).astype(np.uint64) * rng.integers(0, 9, n).astype(np.uint64)
    addr = np.cumsum(gaps + np.concatenate([[0], lens[:-1]])).astype(np.uint64) + np.uint64(rng.integers(0, 50))
    return addr, lens.astype(np.uint16)


def _random_records(rng, addr, ln, n):
    rec = np.zeros(n, gen.RECORD_DTYPE)
    hi = int(addr[-1]) + int(ln[-1]) + 20
    rec["pc"] = rng.integers(0, hi, n)
    rec["pc"][:5] = [0, int(addr[0]), hi, 2 ** 64 - 1, int(addr[-1]) + int(ln[-1])]
    rec["count"] = rng.integers(1, 70000, n)
    rec["stall"] = np.where(rng.random(n) < 0.1, rng.integers(12, 65536, n), rng.integers(0, 12, n))
    return rec


@pytest.mark.parametrize("seed", range(12))
def test_d1_matches_linear_scan(seed):
    rng = np.random.default_rng(seed)
    addr, ln = _random_table(rng, int(rng.integers(1, 40)))
    rec = _random_records(rng, addr, ln, 400)
    st = dict(inst_addr=addr, inst_len=ln)
    H, U, ri = oracle.attribute(st, rec, rec_inst=True)
    Hb, Ub, rib = _brute_attribute(addr, ln, rec)
    assert np.array_equal(H, Hb) and np.array_equal(U, Ub) and np.array_equal(ri, rib)


def test_d1_worked_example():
    g = load_golden("attribution_examples.json")
    s = g["structure"]
    st = dict(inst_addr=np.array(s["inst_addr"], np.uint64), inst_len=np.array(s["inst_len"], np.uint16))
    rec = np.zeros(len(g["records"]), gen.RECORD_DTYPE)
    for k, (pc, c, stall) in enumerate(g["records"]):
        rec[k] = (pc, c, stall, 0)
    H, U, ri = oracle.attribute(st, rec, rec_inst=True)
    He = np.zeros_like(H)
    for i, d in g["expect"]["H"].items():
        for slot, c in d.items():
            He[int(i), int(slot)] = c
    Ue = np.zeros(16, np.uint64)
    for slot, c in g["expect"]["U"].items():
        Ue[int(slot)] = c
    assert np.array_equal(H, He) and np.array_equal(U, Ue)
    assert [None if x == NONE else int(x) for x in ri] == g["expect"]["rec_inst"]


def test_d1_empty_inputs():
    st = dict(inst_addr=np.zeros(0, np.uint64), inst_len=np.zeros(0, np.uint16))
    rec = np.zeros(3, gen.RECORD_DTYPE)
    rec["pc"] = [0, 5, 2 ** 63]
    rec["count"] = [1, 2, 3]
    H, U, ri = oracle.attribute(st, rec, rec_inst=True)
    assert H.shape == (0, 16) and U[0] == 6 and (ri == NONE).all()
    H, U, _ = oracle.attribute(gen.workload("C1").structure, np.zeros(0, gen.RECORD_DTYPE))
    assert H.sum() == 0 and U.sum() == 0


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_d1_conservation_and_shards(name):
    """P2: sum(H)+U = sum(count) per slot; P3: any split into shards (some empty) sums to the
    same histogram; the multi-threaded path equals the serial one."""
    w = gen.workload(name, records=200_000)
    rec = w.records_host()
    H, U, ri = oracle.attribute(w.structure, rec, rec_inst=True)
    slot = np.where(rec["stall"] < 12, rec["stall"], 15)
    expect = np.bincount(slot, weights=rec["count"].astype(np.float64), minlength=16).astype(np.uint64)
    assert np.array_equal(H.sum(0) + U, expect)
    cuts = sorted([0, len(rec), len(rec), 7, 7, 12345, 100_000])
    Hs = np.zeros_like(H)
    Us = np.zeros_like(U)
    for a, b in zip(cuts[:-1], cuts[1:]):
        h, u, _ = oracle.attribute(w.structure, rec[a:b])
        Hs += h
        Us += u
    assert np.array_equal(Hs, H) and np.array_equal(Us, U)
    Hm, Um, _ = oracle.attribute(w.structure, rec, threads=5)
    assert np.array_equal(Hm, H) and np.array_equal(Um, U)
    # every attributed record's pc lies inside its instruction
    ok = ri != NONE
    a = w.structure["inst_addr"][ri[ok]]
    assert ((rec["pc"][ok] >= a) & (rec["pc"][ok] < a + 16)).all()


def _desc_from_golden(s):
    kinds = {"FUNCTION": 0, "INLINE": 1, "LOOP": 2, "LINE": 3}
    n = len(s["inst_addr"])
    return dict(inst_addr=np.array(s["inst_addr"], np.uint64), inst_len=np.array(s["inst_len"], np.uint16),
                inst_class=np.arange(n, dtype=np.uint8) % 16, inst_scope=np.array(s["inst_scope"], np.uint32),
                scope_parent=np.array([NONE if p is None else p for _, p in s["scopes"]], np.uint32),
                scope_kind=np.array([kinds[k] for k, _ in s["scopes"]], np.uint8),
                func_scope=np.array(s["func_scope"], np.uint32),
                call_inst=np.zeros(0, np.uint32), call_callee=np.zeros(0, np.uint32))


def test_d2_resolve_example():
    """pc 50 inside loop [40,60) of function [0,100) -> line, loop, function."""
    g = load_golden("attribution_examples.json")
    st = _desc_from_golden(g["structure"])
    rec = np.zeros(1, gen.RECORD_DTYPE)
    rec[0] = (50, 9, 3, 0)
    H, U, _ = oracle.attribute(st, rec)
    Hs, MIX = oracle.rollup(st, H)
    hit = [s for s in range(len(st["scope_parent"])) if Hs[s, 3] == 9]
    assert sorted(hit) == sorted(g["expect"]["scope_rows_for_pc50"])
    assert Hs.sum() == 9 * 3
    assert MIX[0, int(st["inst_class"][5])] == 9


def _topdown_rollup(st, H):
    """Explicit containment: collect each scope's instruction set top-down through the
    children lists, then sum H over the set (no parent walk, no accumulation order)."""
    n_scope = len(st["scope_parent"])
    children = [[] for _ in range(n_scope)]
    for s, p in enumerate(st["scope_parent"]):
        if p != NONE:
            children[p].append(s)
    direct = [[] for _ in range(n_scope)]
    for i, s in enumerate(st["inst_scope"]):
        direct[s].append(i)

    def members(s):
        out = list(direct[s])
        for c in children[s]:
            out += members(c)
        return out

    Hs = np.zeros((n_scope, 16), np.uint64)
    MIX = np.zeros((n_scope, 16), np.uint64)
    S = H[:, :12].sum(1, dtype=np.uint64)
    for s in range(n_scope):
        m = np.array(members(s), np.int64)
        if len(m):
            Hs[s] = H[m].sum(0, dtype=np.uint64)
            np.add.at(MIX[s], st["inst_class"][m].astype(np.int64), S[m])
    return Hs, MIX


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_d2_matches_topdown_containment(name):
    w = gen.workload(name, records=50_000)
    H, _, _ = oracle.attribute(w.structure, w.records_host())
    Hs, MIX = oracle.rollup(w.structure, H)
    Ht, MIXt = _topdown_rollup(w.structure, H)
    assert np.array_equal(Hs, Ht) and np.array_equal(MIX, MIXt)


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_d2_invariants(name):
    """P4: FUNC rows sum to all attributed samples; nested rows never exceed their parents;
    mix rows sum to the row's valid samples; LINE rows partition the instructions."""
    w = gen.workload(name, records=100_000)
    st = w.structure
    H, _, _ = oracle.attribute(st, w.records_host())
    Hs, MIX = oracle.rollup(st, H)
    fs = st["func_scope"].astype(np.int64)
    assert np.array_equal(Hs[fs].sum(0), H.sum(0))
    kind = st["scope_kind"]
    assert np.array_equal(Hs[kind == 3].sum(0), H.sum(0))
    par = st["scope_parent"]
    has_p = par != NONE
    assert (Hs[has_p] <= Hs[par[has_p].astype(np.int64)]).all()
    assert np.array_equal(MIX.sum(1), Hs[:, :12].sum(1))
    hist, mix = oracle.scope_hist(st, H, "FUNC")
    assert np.array_equal(hist, Hs[fs])
