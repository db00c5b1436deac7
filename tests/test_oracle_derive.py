"""Pins of oracle D7 (derived metrics, §6.1) by closed forms:
W(100, 75) = 0.25, NaN at S = 0, single-reason rows, fractions summing to one, and the
mix columns against a direct class count.  CPU only."""
import math

import numpy as np
import pytest

import oracle
from tests.fixtures import load_golden

LAT = [1, 2, 3, 4, 5, 6, 7, 8, 10, 11]


def _row(d):
    v = np.zeros(16, np.uint64)
    for k, c in d.items():
        v[int(k)] = c
    return v


def test_derive_worked_examples():
    g = load_golden("derive_examples.json")
    for row in g["rows"]:
        v = _row(row["v"])
        for out in (oracle.derive_u64(v, np.zeros(16, np.uint64))[0], oracle.derive_f64(v.astype(np.float64))[0]):
            assert out[0] == row["S"]
            if row["W"] is None:
                assert math.isnan(out[1])
            else:
                assert out[1] == row["W"]
            if "latency_hiding" in row:
                assert out[2] == row["latency_hiding"] and out[3] == row["latency_stall"]
            if "invalid" in row:
                assert out[16] == row["invalid"]


def test_derive_zero_row_is_nan_everywhere_but_counts():
    out = oracle.derive_u64(np.zeros(16, np.uint64), np.zeros(16, np.uint64))[0]
    assert out[0] == 0 and out[16] == 0
    for c in list(range(1, 16)) + list(range(17, 33)):
        assert math.isnan(out[c])
        assert out[c:c + 1].view(np.uint64)[0] == 0x7FF8000000000000   # canonical quiet NaN


@pytest.mark.parametrize("r", range(12))
def test_derive_single_reason(r):
    v = np.zeros(16, np.uint64)
    v[r] = 123456789
    out = oracle.derive_u64(v, None)[0]
    for q in range(12):
        assert out[4 + q] == (1.0 if q == r else 0.0)
    assert out[1] == (1.0 if r == 0 else 0.0)
    assert out[2] == (1.0 if r in (0, 9) else 0.0)
    assert out[3] == (1.0 if r in LAT else 0.0)
    assert all(math.isnan(x) for x in out[17:])          # no mix given


def test_derive_random_rows_sum_to_one():
    rng = np.random.default_rng(7)
    V = rng.integers(0, 2 ** 40, (500, 16)).astype(np.uint64)
    V[:, 12:15] = 0
    MIX = np.zeros_like(V)
    S = V[:, :12].sum(1)
    for i in range(len(V)):                               # split S over classes
        cuts = np.sort(rng.integers(0, int(S[i]) + 1, 15))
        MIX[i] = np.diff(np.concatenate([[0], cuts, [int(S[i])]])).astype(np.uint64)
    out = oracle.derive_u64(V, MIX)
    eps = np.finfo(np.float64).eps
    assert np.all(np.abs(out[:, 4:16].sum(1) - 1) <= 12 * eps)
    assert np.all(np.abs(out[:, 2] + out[:, 3] - 1) <= 4 * eps)
    assert np.all(np.abs(out[:, 17:33].sum(1) - 1) <= 16 * eps)
    assert np.array_equal(out[:, 0], S.astype(np.float64))
    assert np.array_equal(out[:, 1], V[:, 0].astype(np.float64) / S.astype(np.float64))
    assert np.array_equal(out[:, 16], V[:, 15].astype(np.float64))
    # fp64 rows with the same integer values give the same ratios (exact sums < 2^53)
    outf = oracle.derive_f64(V.astype(np.float64))
    assert np.array_equal(outf[:, :17], out[:, :17])
    assert np.isnan(outf[:, 17:]).all()
