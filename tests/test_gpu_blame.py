"""f4 GPU parity: gpa_idleness_blame against oracle D10 on the same trace sets — the worked
examples, random tiny traces (ties, single events, many lines per rank = many merge rounds),
the generated rank traces B1-B3 (B3 = the bench size, 64 ranks, 31 M events); totals bit-exact,
blame and share bit-identical (same operation order) and within 1e-9; invalid inputs fail."""
import numpy as np
import pytest

import oracle
from gen.trace import trace_set
from tests.blame_util import NONE, from_lines, random_trace
from tests.fixtures import load_golden

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
DEV = "cuda:0"


@pytest.fixture(scope="module")
def gpa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    from paper_2109_06931_b200 import gpa
    return gpa


def _run(gpa, tr):
    S, R = tr["n_scopes"], tr["n_routines"]
    t = torch.from_numpy(tr["time"].view(np.int64)).to(DEV)
    c = torch.from_numpy(tr["ctx"].view(np.int32)).to(DEV)
    out = dict(blame=torch.empty((S, R), dtype=torch.float64, device=DEV),
               share=torch.empty((S, R), dtype=torch.float64, device=DEV),
               total=torch.empty(S, dtype=torch.int64, device=DEV),
               gpu_idle=torch.empty(S, dtype=torch.int64, device=DEV))
    gpa.idleness_blame(tr, t, c, **out)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


def _compare(gpa, tr):
    got, exp = _run(gpa, tr), oracle.blame(tr)
    assert np.array_equal(got["total"].view(np.uint64), exp["total"])
    assert np.array_equal(got["gpu_idle"].view(np.uint64), exp["gpu_idle"])
    for k in ("blame", "share"):
        assert np.array_equal(got[k].view(np.uint64), exp[k].view(np.uint64)), k
        np.testing.assert_allclose(got[k], exp[k], rtol=1e-9, atol=0)
    return got


def test_worked_examples(gpa):
    G = load_golden("blame_examples.json")["cases"]
    cases = [(len(G[n]["routines"]), G[n]["lines"]) for n in sorted(G)]
    for case in cases:
        _compare(gpa, from_lines([case]))
    got = _compare(gpa, from_lines(cases))
    three = sorted(G).index("three_threads")
    assert got["blame"][three, 0] == 95 / 6 and got["total"][three] == 30


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("GPA_FUZZ_SEEDS", "30"))))
def test_random_tiny(gpa, seed):
    rng = np.random.default_rng(1000 + seed)
    _compare(gpa, random_trace(rng, int(rng.integers(1, 6))))


@pytest.mark.parametrize("seed", range(6))
def test_random_many_lines_and_ties(gpa, seed):
    rng = np.random.default_rng(2000 + seed)
    _compare(gpa, random_trace(rng, int(rng.integers(1, 4)), max_lines=(20, 45), t_max=int(rng.choice([5, 400])),
                               max_events=200))


@pytest.mark.parametrize("name", ["B1", "B2", "B3"])
def test_generated_traces(gpa, name):
    got = _compare(gpa, trace_set(name))
    assert (got["total"] > 0).all()


def test_edge_cases(gpa):
    # empty lines everywhere (no events at all), and lines with one change point only
    tr = from_lines([(2, [("gpu", []), ("cpu", [])]), (2, [("gpu", [[5, 1]]), ("cpu", [[5, 0]])])])
    got = _compare(gpa, tr)
    assert (got["total"] == 0).all() and np.isnan(got["share"]).all()
    # a rank whose only CPU line is idle throughout
    _compare(gpa, from_lines([(1, [("gpu", [[0, 3], [10, None], [20, None]]), ("cpu", [[0, None], [30, None]])])]))


def test_invalid_inputs(gpa):
    base = [("gpu", [[0, 1], [5, None]]), ("cpu", [[0, 0], [5, None]])]
    bad = [from_lines([(1, [("gpu", [[5, 1], [0, None]]), base[1]])]),      # back in time
           from_lines([(1, [base[0], ("cpu", [[0, 3], [5, None]])])]),      # routine id >= n_routines
           from_lines([(1, [base[1]])])]                                    # no GPU line
    for tr in bad:
        with pytest.raises(gpa.GpaError):
            _run(gpa, tr)
    tr = from_lines([(1, base)])
    tr["line_scope"] = np.array([1, 0], np.uint32)
    tr["n_scopes"] = 2
    with pytest.raises(gpa.GpaError):
        _run(gpa, tr)


# ---- larger random ranks: many merge tiles per rank, equal times across and inside lines --------
@pytest.mark.parametrize("seed", range(8))
def test_random_large_ranks(gpa, seed):
    """Ranks of up to 16 lines and up to 60 k change points (several merge tiles per run and
    merge round), with equal times across lines (t_max small against the event count)."""
    rng = np.random.default_rng(3000 + seed)
    _compare(gpa, random_trace(rng, int(rng.integers(1, 4)), max_lines=(8, 9), t_max=int(rng.choice([3000, 200_000])),
                               max_events=int(rng.choice([300, 4000]))))


def test_many_equal_times(gpa):
    """3000 change points at one timestamp in a line (one merge tile is all ties)."""
    gpu = [[t, 1 if i % 2 else None] for i, t in enumerate([0] + [10] * 3000 + [20, 30])]
    cpu = [[0, 0], [5, 1], [15, 0], [25, None], [40, None]]
    _compare(gpa, from_lines([(2, [("gpu", gpu), ("cpu", cpu), ("cpu", [[1, 1], [35, None]])])]))
