"""Pins of oracle D8 (per-profile histograms + cross-profile statistics, SURVEY §8f f1;
PAPER.md P:481-487): the SPEC worked examples, a per-record brute force, conservation
against the aggregate roll-up, and a numpy two-pass statistics computation.  CPU only."""
import numpy as np
import pytest

import gen
import oracle
from tests.fixtures import load_golden


def test_stats_worked_examples():
    for case in load_golden("stats_examples.json")["cases"]:
        v = case["values"]
        Hp = np.zeros((len(v) + 1, 1, 16), np.uint64)
        Hp[:len(v), 0, 3] = v
        Hp[len(v), 0, 3] = 12345            # the overflow row never enters the statistics
        st = oracle.profile_stats(Hp, len(v))[0, :, 3]
        assert st[0] == case["sum"] and st[1] == case["min"] and st[3] == case["max"]
        assert st[2] == pytest.approx(case["mean"], rel=1e-15)
        assert st[4] == pytest.approx(case["std"], rel=1e-14, abs=1e-300)
        assert st[5] == pytest.approx(case["cv"], rel=1e-14, abs=1e-300)


def test_profiles_brute_force_small():
    w = gen.workload("C4", records=20_000)
    rec = w.records_host()
    st = w.structure
    n_prof = 300                               # some stream ids (>= 300) overflow
    Hp, Up = oracle.attribute_profiles(st, rec, n_prof)
    _, _, ri = oracle.attribute(st, rec, rec_inst=True)
    ifunc = oracle.inst_func(st)
    Hb = np.zeros_like(Hp)
    Ub = np.zeros_like(Up)
    for k, (pc, c, s, p) in enumerate(rec.tolist()):
        slot = s if s < 12 else 15
        p = p if p < n_prof else n_prof
        if ri[k] == oracle.NONE:
            Ub[p, slot] += c
        else:
            Hb[p, ifunc[ri[k]], slot] += c
    assert np.array_equal(Hp, Hb) and np.array_equal(Up, Ub)


@pytest.mark.parametrize("name,records,n_prof", [("C4", 400_000, 384), ("C2", 100_000, 1), ("C4", 50_000, 64)])
def test_profiles_conservation_and_two_pass_stats(name, records, n_prof):
    w = gen.workload(name, records=records)
    rec = w.records_host()
    st = w.structure
    Hp, Up = oracle.attribute_profiles(st, rec, n_prof)
    H, U, _ = oracle.attribute(st, rec)
    fh, _ = oracle.scope_hist(st, H, "FUNC")
    assert np.array_equal(Hp.sum(0), fh) and np.array_equal(Up.sum(0), U)
    S = oracle.profile_stats(Hp, n_prof)
    x = Hp[:n_prof].astype(np.float64)       # values < 2^53: exact in fp64
    mean = x.mean(0)
    std = np.sqrt(((x - mean) ** 2).mean(0))
    assert np.array_equal(S[:, 0], x.sum(0)) and np.array_equal(S[:, 1], x.min(0)) and np.array_equal(S[:, 3], x.max(0))
    assert np.allclose(S[:, 2], mean, rtol=1e-15, atol=0)
    assert np.allclose(S[:, 4], std, rtol=1e-10, atol=1e-9)
    cv = np.where(mean == 0, 0.0, std / np.where(mean == 0, 1, mean))
    assert np.allclose(S[:, 5], cv, rtol=1e-10, atol=1e-12)


# ---- f1 at instruction level and at CCT level (D8 inst, D11) --------------------------------
def test_profiles_inst_brute_force_and_conservation():
    w = gen.workload("C2", records=30_000)
    rec = w.records_host()
    st = w.structure
    n_prof = 3
    Hp, Up = oracle.attribute_profiles_inst(st, rec, n_prof)
    addr, ln = st["inst_addr"].astype(np.int64), st["inst_len"].astype(np.int64)
    Hb = np.zeros_like(Hp)
    Ub = np.zeros_like(Up)
    for pc, c, s, p in rec.tolist():                     # linear-scan containment (no search)
        slot = s if s < 12 else 15
        p = min(p, n_prof)
        hit = np.nonzero((addr <= pc) & (pc < addr + ln))[0]
        if len(hit):
            Hb[p, hit[0], slot] += c
        else:
            Ub[p, slot] += c
    assert np.array_equal(Hp, Hb) and np.array_equal(Up, Ub)
    H, U, _ = oracle.attribute(st, rec)
    assert np.array_equal(Hp.sum(0), H) and np.array_equal(Up.sum(0), U)
    Hf, _ = oracle.attribute_profiles(st, rec, n_prof)            # function rows = sums of their instructions
    fn = oracle.inst_func(st)
    agg = np.zeros_like(Hf)
    for i, f in enumerate(fn):
        agg[:, f] += Hp[:, i]
    assert np.array_equal(agg, Hf)


def _fig4():
    from tests.fixtures import build as build_fixture, frac
    g = load_golden("cct_fig4_narrative.json")
    st, H, _ = build_fixture(g["spec"])
    return st, H, g, frac


def test_cct_profiles_hand_worked_fractions():
    """Profile p's excl at a context = f(c) (hand-worked, golden) x p's samples of the function;
    incl = subtree sums — exact rationals vs the oracle (every f is a dyadic fraction)."""
    from fractions import Fraction
    st, H, g, frac = _fig4()
    R = oracle.cct(st, H)
    fn = oracle.inst_func(st)
    rng = np.random.default_rng(5)
    P1 = 3
    Hi = np.zeros((P1,) + H.shape, np.uint64)                   # split every bin over 3 profiles
    for i in range(H.shape[0]):
        for r in range(16):
            cuts = np.sort(rng.integers(0, int(H[i, r]) + 1, P1 - 1))
            parts = np.diff(np.concatenate([[0], cuts, [int(H[i, r])]]))
            Hi[:, i, r] = parts
    Hp = np.zeros((P1, len(st["func_scope"]), 16), np.uint64)
    for i, f in enumerate(fn):
        Hp[:, f] += Hi[:, i]
    E, I = oracle.cct_profiles(R, Hp)
    ctx = g["expect"]["contexts"]
    assert R["n"] == len(ctx)
    cf = oracle.cct_ctx_func(R)
    for p in range(P1):
        ex = [Fraction(0) if cf[c] == oracle.NONE else frac(ctx[c][4]) * int(Hp[p, cf[c], r])
              for c in range(len(ctx)) for r in range(16)]
        ex = np.array(ex, dtype=object).reshape(len(ctx), 16)
        inc = ex.copy()
        for c in range(len(ctx) - 1, -1, -1):                  # parents precede children (BFS)
            parent = int(R["parent"][c])
            if parent != oracle.NONE:
                inc[parent] = inc[parent] + inc[c]
        assert np.array_equal(E[p], ex.astype(np.float64)) and np.array_equal(I[p], inc.astype(np.float64))


def test_cct_profiles_single_profile_is_the_aggregate_tree():
    w = gen.workload("C3", records=200_000)
    st, rec = w.structure, w.records_host()
    H, _, _ = oracle.attribute(st, rec)
    R = oracle.cct(st, H)
    Hp, _ = oracle.attribute_profiles(st, rec, 1)
    Hp = Hp.sum(0, keepdims=True)                                 # one profile holding everything
    E, I = oracle.cct_profiles(R, Hp)
    assert np.array_equal(E[0].view(np.uint64), R["excl"].view(np.uint64))
    assert np.array_equal(I[0].view(np.uint64), R["incl"].view(np.uint64))


def test_cct_profiles_conservation():
    w = gen.workload("C4", records=300_000)
    st, rec = w.structure, w.records_host()
    H, _, _ = oracle.attribute(st, rec)
    R = oracle.cct(st, H)
    Hp, _ = oracle.attribute_profiles(st, rec, 16)
    E, I = oracle.cct_profiles(R, Hp)
    np.testing.assert_allclose(E.sum(0), R["excl"], rtol=1e-12, atol=1e-9)
    np.testing.assert_allclose(I.sum(0), R["incl"], rtol=1e-12, atol=1e-9)


def test_stats_f64_against_numpy_and_spec():
    rng = np.random.default_rng(9)
    X = rng.random((9, 40, 16)) * 1e6
    X[:, 3] = 7.25                                                 # equal values: std 0, cv 0
    X[:, 5] = 0.0
    n_prof = 8                                                     # row 8 = overflow, excluded
    S = oracle.profile_stats_f64(X, n_prof)
    Y = X[:n_prof]
    np.testing.assert_allclose(S[:, 0], Y.sum(0), rtol=1e-13)
    assert np.array_equal(S[:, 1], Y.min(0)) and np.array_equal(S[:, 3], Y.max(0))
    np.testing.assert_allclose(S[:, 2], Y.mean(0), rtol=1e-13)
    np.testing.assert_allclose(S[:, 4], Y.std(0), rtol=1e-10, atol=1e-9)
    assert (S[3, 4] == 0).all() and (S[5, 5] == 0).all()
    for case in load_golden("stats_examples.json")["cases"]:
        v = np.zeros((len(case["values"]), 1, 16))
        v[:, 0, 2] = case["values"]
        st = oracle.profile_stats_f64(v, len(case["values"]))[0, :, 2]
        assert st[2] == pytest.approx(case["mean"], rel=1e-15)
        assert st[4] == pytest.approx(case["std"], rel=1e-14, abs=1e-300)
        assert st[5] == pytest.approx(case["cv"], rel=1e-14, abs=1e-300)
