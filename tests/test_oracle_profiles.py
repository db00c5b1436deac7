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
