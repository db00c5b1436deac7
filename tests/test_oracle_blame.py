"""Pins of oracle D10 (GPU-idleness blame): SPEC's worked
examples and a hand-worked three-thread case (tests/golden/blame_examples.json), an
independent 1-ns brute force with exact rationals on random tiny traces, integer
conservation (sum_r num[r][k] = k * D_k), shares summing to 1, scope independence, and the
invalid-input errors.  CPU only."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from gen.trace import trace_set
from tests.blame_util import brute_force, from_lines, random_trace
from tests.fixtures import load_golden

G = load_golden("blame_examples.json")["cases"]


@pytest.mark.parametrize("name", sorted(G))
def test_worked_examples(name):
    case = G[name]
    R = len(case["routines"])
    r = oracle.blame(from_lines([(R, case["lines"])]))
    assert int(r["total"][0]) == case["total"] and int(r["gpu_idle"][0]) == case["gpu_idle"]
    for i, nm in enumerate(case["routines"]):
        p, q = case["blame"][nm]
        assert r["blame"][0, i] == float(Fraction(p, q))
        if case["share"][nm] is None:
            assert np.isnan(r["share"][0, i])
        else:
            assert r["share"][0, i] == pytest.approx(case["share"][nm], rel=1e-15)
        for k, v in case.get("num", {}).get(nm, {}).items():
            assert int(r["num"][0, i, int(k)]) == v


def test_scopes_are_independent():
    cases = [(len(G[n]["routines"]), G[n]["lines"]) for n in sorted(G)]
    r = oracle.blame(from_lines(cases))
    for s, (R, lines) in enumerate(cases):
        one = oracle.blame(from_lines([(R, lines)]))
        assert r["total"][s] == one["total"][0] and r["gpu_idle"][s] == one["gpu_idle"][0]
        assert np.array_equal(r["blame"][s, :R], one["blame"][0])


@pytest.mark.parametrize("seed", range(40))
def test_brute_force_exact_rationals(seed):
    rng = np.random.default_rng(seed)
    tr = random_trace(rng, int(rng.integers(1, 4)))
    r = oracle.blame(tr)
    num, total, idle, blame = brute_force(tr)
    assert list(r["total"]) == total and list(r["gpu_idle"]) == idle
    got = {(s, q, k): int(v) for (s, q, k), v in np.ndenumerate(r["num"]) if v}
    assert got == num
    for s in range(tr["n_scopes"]):
        for q in range(tr["n_routines"]):
            assert r["blame"][s, q] == pytest.approx(float(blame[s][q]), rel=1e-15, abs=0)
            exact = sum((Fraction(int(r["num"][s, q, k]), k) for k in range(1, r["kmax"] + 1)), Fraction(0))
            assert exact == blame[s][q]


def test_conservation_on_generated_traces():
    tr = trace_set("B2")
    r = oracle.blame(tr)
    num = r["num"].astype(object)
    for s in range(tr["n_scopes"]):
        per_k = num[s].sum(axis=0)                       # sum over routines, per k
        assert per_k[0] == 0
        d = [per_k[k] // k for k in range(1, r["kmax"] + 1)]
        assert all(per_k[k] % k == 0 for k in range(1, r["kmax"] + 1))   # k threads share each piece
        assert sum(d) == int(r["total"][s])
        assert r["total"][s] > 0 and r["total"][s] <= r["gpu_idle"][s]
        assert np.nansum(r["share"][s]) == pytest.approx(1.0, abs=1e-12)


def test_invalid_inputs():
    base = [("gpu", [[0, 1], [5, None]]), ("cpu", [[0, 0], [5, None]])]
    with pytest.raises(ValueError):                       # back in time
        oracle.blame(from_lines([(1, [("gpu", [[5, 1], [0, None]]), base[1]])]))
    with pytest.raises(ValueError):                       # routine id out of range
        oracle.blame(from_lines([(1, [base[0], ("cpu", [[0, 3], [5, None]])])]))
    with pytest.raises(ValueError):                       # scope without a GPU line (SPEC NoGpuLines)
        oracle.blame(from_lines([(1, [base[1]])]))
    r = oracle.blame(from_lines([(1, base)]))
    assert r["total"][0] == 0
