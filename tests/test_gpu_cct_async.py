"""gpa_reconstruct_cct_async / gpa_cct_finish: the CCT (a-6..a-9) built without a host
synchronization, CCT metrics (a-10) derived while its size is still on the device.  Every array
of the finished tree and every metric row must be bit-identical to the synchronous
gpa_reconstruct_cct (itself pinned to the oracle by tests/test_gpu_parity.py), including a tree
the one-launch build cannot hold (rebuilt by the counted path inside gpa_cct_finish)."""
import numpy as np
import pytest

import gen
import oracle
from tests.fixtures import build as build_fixture, load_golden

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
DEV = "cuda:0"
ARRAYS = ["parent", "site", "node", "kind", "first_child", "n_children", "frac", "excl", "incl", "call_weight",
          "dag_weight", "dag_active", "func_active", "func_hist"]


@pytest.fixture(scope="module")
def gpa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    from paper_2109_06931_b200 import gpa
    return gpa


def _bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint8) if a.dtype.itemsize == 1 else a.view(f"u{a.dtype.itemsize}")


def _metrics(gpa, s, c, rows):
    out = {}
    for scope in ("CCT_EXCL", "CCT_INCL"):
        m = torch.full((max(rows, 1), 33), -7.0, dtype=torch.float64, device=DEV)
        gpa.derive_metrics(s, scope, cct=c, metrics=m)
        out[scope] = m
    return out


def _compare(gpa, s, H, mode=0, expect_rebuild=None):
    ref = gpa.reconstruct_cct(s, H, mode=mode)
    ref_np = ref.to_numpy()
    ref_m = {k: v.cpu().numpy() for k, v in _metrics(gpa, s, ref, ref.n).items()}
    c = gpa.reconstruct_cct_async(s, H, mode=mode)
    if c.pending:  # views are refused until the size is known
        with pytest.raises(gpa.GpaError):
            gpa._check(gpa._lib.gpa_get_cct_view(c.handle, gpa.ctypes.byref(gpa.CctView())), "gpa_get_cct_view")
    cap = c.capacity
    m = _metrics(gpa, s, c, cap)  # enqueued before the size is known
    rebuilt = c.finish()
    assert rebuilt == (ref.n > cap if expect_rebuild is None else expect_rebuild)
    assert c.n == ref.n and c.n <= max(cap, c.n)
    got = c.to_numpy()
    for k in ARRAYS:
        assert np.array_equal(_bits(got[k]), _bits(ref_np[k])), k
    if rebuilt:  # metrics derived on the pending build are void: derive again on the finished tree
        m = _metrics(gpa, s, c, c.n)
    else:  # rows past the size were not written
        for v in m.values():
            assert (v[c.n:] == -7.0).all()
    for k, v in m.items():
        assert np.array_equal(_bits(v.cpu().numpy()[:c.n]), _bits(ref_m[k][:c.n])), k
    c.free()
    ref.free()
    return ref_np


@pytest.mark.parametrize("name", ["cct_fig4_narrative.json", "cct_guard.json", "cct_diamond.json"])
def test_async_golden(gpa, name):
    st, H, _ = build_fixture(load_golden(name)["spec"])
    s = gpa.load_structure(st, 0)
    _compare(gpa, s, torch.from_numpy(H.view(np.int64)).to(DEV))


@pytest.mark.parametrize("exact", [0, 1])
@pytest.mark.parametrize("seed", range(12))
def test_async_random_graphs(gpa, seed, exact):
    from tests.test_oracle_cct import _random_graph
    rng = np.random.default_rng(1000 + seed)
    st, H, _ = build_fixture(_random_graph(rng))
    s = gpa.load_structure(st, 0)
    _compare(gpa, s, torch.from_numpy(H.view(np.int64)).to(DEV), mode=exact)


@pytest.mark.parametrize("name,records", [("C1", 10_000), ("C2", 1_000_000), ("C3", 2_000_000), ("C4", 2_000_000),
                                          ("C5", 2_000_000)])
def test_async_workloads(gpa, name, records):
    w = gen.workload(name, records=records)
    s = gpa.load_structure(w.structure, 0)
    rec = torch.empty((records, 2), dtype=torch.int64, device=DEV)
    w.records_device(rec)
    H = torch.zeros((s.info["n_inst"], 16), dtype=torch.int64, device=DEV)
    U = torch.zeros(16, dtype=torch.int64, device=DEV)
    gpa.attribute_samples(s, rec, H, U)
    R = _compare(gpa, s, H)
    Ro = oracle.cct(w.structure, H.cpu().numpy().view(np.uint64))
    assert R["n"] == Ro["n"]
    assert np.array_equal(R["incl"].view(np.uint64), Ro["incl"].view(np.uint64))


def test_async_overflow_rebuilds(gpa):
    """Exact counts on C3's structure with every call executed: 4.19 M contexts, far beyond the
    one-launch build's 2^16 slots -> gpa_cct_finish rebuilds with the counted path."""
    w = gen.workload("C3", records=10)
    s = gpa.load_structure(w.structure, 0)
    n_inst = s.info["n_inst"]
    rng = np.random.default_rng(9)
    cuts = np.sort(rng.choice(np.arange(1, n_inst), 20_000, replace=False))
    start = np.concatenate([[0], cuts, [n_inst]]).astype(np.uint32)
    cnt = rng.integers(1, 1000, len(start) - 1).astype(np.uint64)
    H = torch.zeros((n_inst, 16), dtype=torch.int64, device=DEV)
    gpa.block_counts(s, torch.from_numpy(start.view(np.int32)).to(DEV), torch.from_numpy(cnt.view(np.int64)).to(DEV), H)
    R = _compare(gpa, s, H, mode=1, expect_rebuild=True)
    assert R["n"] > 1 << 16
