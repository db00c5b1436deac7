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


def _mix_fixture():
    g = load_golden("mix_example.json")
    cls = np.array(g["structure"]["inst_class"], np.uint8)
    n = len(cls)
    st = dict(inst_addr=np.arange(n, dtype=np.uint64) * 16 + 0x1000, inst_len=np.full(n, 16, np.uint16),
              inst_class=cls, inst_scope=np.ones(n, np.uint32),
              scope_parent=np.array([0xFFFFFFFF, 0], np.uint32), scope_kind=np.array([0, 3], np.uint8),
              func_scope=np.array([0], np.uint32), call_inst=np.zeros(0, np.uint32), call_callee=np.zeros(0, np.uint32))
    H = np.zeros((n, 16), np.uint64)
    for i, slots in g["structure"]["H"].items():
        for r, c in slots.items():
            H[int(i), int(r)] = c
    return g, st, H


@pytest.mark.parametrize("scope", ["FUNC", "LINE"])
def test_mix_columns_hand_worked(scope):
    """Every derived column of the one-function row, columns 17..32 included, against the values
    written out by hand: a class -> column permutation, a dropped class or counting slot 15 in
    the mix would each fail."""
    g, st, H = _mix_fixture()
    e = g["expect"]
    hist, mix = oracle.scope_hist(st, H, scope)
    assert hist.shape[0] == 1 and mix.shape[0] == 1
    for k in range(16):
        assert mix[0, k] == e["mix_counts"].get(str(k), 0), k
    out = oracle.derive_u64(hist, mix)[0]
    assert out[0] == e["S"] and out[16] == e["invalid"]
    assert out[1] == float(e["W"]) and out[2] == float(e["latency_hiding"]) and out[3] == float(e["latency_stall"])
    for r in range(12):
        assert out[4 + r] == float(e["stall_fraction"].get(str(r), "0")), r
    for c in range(17, 33):
        assert out[c] == float(e["mix_columns"][str(c)]), c


def test_inst_row_mix_hand_worked():
    """INST rows: each instruction's whole valid-sample total sits in its own class column (1.0),
    every other mix column is 0, and slot 15 counts only as 'invalid'."""
    g, st, H = _mix_fixture()
    hist, mix = oracle.scope_hist(st, H, "INST")
    out = oracle.derive_u64(hist, mix)
    for row in g["expect"]["inst_rows"]:
        i = row["inst"]
        assert out[i, 0] == row["S"] and mix[i].sum() == row["S"]
        for c in range(17, 33):
            assert out[i, c] == (1.0 if c == row["mix_col"] else 0.0), (i, c)
        assert out[i, 16] == row.get("invalid", 0)
