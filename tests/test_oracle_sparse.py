"""Pins of oracle D9 (PMS / CMS sparse cubes; §5.2): SPEC's worked
lookups and scans, exact round trips on random cubes, the space accounting and the
logarithmic lookup cost the paper states.  CPU only."""
import math

import numpy as np
import pytest

import oracle
from tests.fixtures import load_golden
from tests.sparse_util import decode, lookup, scan


def _cube(case):
    Hp = np.zeros((case["P"], case["C"], 16), np.uint64)
    for p, c, m, v in case["entries"]:
        Hp[p, c, m] = v
    return Hp


def test_worked_examples():
    g = load_golden("sparse_examples.json")
    pms = oracle.sparse_build(_cube(g["single"]), cms=False)
    for p, c, m, v in g["single"]["lookups"]:
        assert lookup(pms, p, c, m)[0] == v
    cms = oracle.sparse_build(_cube(g["scan"]), cms=True)
    for c, m, expect in g["scan"]["scans"]:
        assert scan(cms, c, m) == [tuple(x) for x in expect]
    for p, c, m, v in g["scan"]["lookups"]:
        assert lookup(cms, c, m, p)[0] == v                     # CMS: plane = context, leaf = profile


@pytest.mark.parametrize("density", [0.0, 0.01, 0.05, 0.2, 1.0])
def test_round_trip_space_and_lookup_cost(density):
    rng = np.random.default_rng(int(density * 1000))
    P, C = 20, 50
    Hp = np.where(rng.random((P, C, 16)) < density, rng.integers(1, 2 ** 40, (P, C, 16)), 0).astype(np.uint64)
    cms, pms = oracle.sparse_build(Hp, True), oracle.sparse_build(Hp, False)
    assert np.array_equal(decode(cms, P, C, True), Hp) and np.array_equal(decode(pms, P, C, False), Hp)
    x = int((Hp != 0).sum())
    assert cms["n_values"] == x and pms["n_values"] == x
    m_c = (Hp != 0).any(0).sum()                                # non-empty (context, metric) pairs
    k_p = (Hp != 0).any(2).sum()                                # non-empty (profile, context) pairs
    assert cms["n_index"] == m_c + C and pms["n_index"] == k_p + P   # + one sentinel per plane
    for _ in range(200):
        p, c, m = int(rng.integers(P)), int(rng.integers(C)), int(rng.integers(16))
        v = int(Hp[p, c, m]) or None
        got, comps = lookup(cms, c, m, p)
        assert got == v and comps <= math.ceil(math.log2(16 + 1)) + math.ceil(math.log2(P + 1)) + 2
        assert lookup(pms, p, c, m)[0] == v
