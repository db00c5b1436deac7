"""GPU parity of the per-profile CCTs unified by call path (f1 extension, reading R30; P:872
"for each GPU kernel invocation", "unify the tree of call paths from each profile")
against oracle D12 on the same seeded inputs.  Structure and indices bit-exact; frac / excl /
incl bit-exact (every profile's tree is computed in the oracle's arithmetic order)."""
import numpy as np
import pytest

import gen
import oracle
from tests.fixtures import build as build_fixture, load_golden
from tests.test_oracle_cct_profiles import _random_structure

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
DEV = "cuda:0"
NONE = 0xFFFFFFFF


@pytest.fixture(scope="module")
def gpa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    from paper_2109_06931_b200 import gpa
    return gpa


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(DEV)


def _inputs_from_inst(gpa, s, Hp):
    """Per-profile Step-1 inputs (S_f,p, w_p) on the GPU from instruction histograms."""
    P = Hp.shape[0]
    nf, nc, ni = s.info["n_func"], s.info["n_call"], s.info["n_inst"]
    S = torch.zeros((P, max(nf, 1), 16), dtype=torch.int64, device=DEV)
    W = torch.zeros((P, max(nc, 1)), dtype=torch.int64, device=DEV)
    for p in range(P):
        gpa.cct_inputs(s, _dev(Hp[p]).reshape(-1, 16), 0, ni, S[p], W[p])
    return S, W


def _compare(g, R, P):
    n = R["n"]
    assert g["n"] == n and g["n_profiles"] == P
    for k in ("parent", "site", "node", "kind"):
        assert np.array_equal(g[k], R[k]), k
    for k in ("frac", "excl", "incl"):
        assert np.array_equal(g[k].view(np.uint64), R[k].view(np.uint64)), k
    # child ranges agree with the parent array (BFS: children contiguous)
    par = R["parent"].astype(np.int64)
    kid = np.nonzero(par != NONE)[0]
    cnt = np.bincount(par[kid], minlength=n) if n else np.zeros(0, np.int64)
    assert np.array_equal(g["n_children"].astype(np.int64), cnt)
    has = cnt > 0
    first = np.zeros(n, np.int64)
    u, idx = np.unique(par[kid], return_index=True)
    first[u] = kid[idx]
    assert np.array_equal(g["first_child"].astype(np.int64)[has], first[has])


def _run(gpa, st, Hp, exact=False):
    s = gpa.load_structure(st, 0)
    S, W = _inputs_from_inst(gpa, s, Hp)
    P = Hp.shape[0]
    mode = gpa.WEIGHTS_EXACT if exact else gpa.WEIGHTS_SAMPLES
    R = oracle.cct_per_profile(st, Hp, exact=exact)
    assert gpa.reconstruct_cct_per_profile(s, S, W, P, mode=mode, max_contexts=0) == R["n"]
    m = gpa.reconstruct_cct_per_profile(s, S, W, P, mode=mode)
    _compare(m.to_numpy(), R, P)
    m.free()
    return s, S, W, R


def test_hand_worked_golden(gpa):
    g = load_golden("cct_per_profile.json")
    spec = g["spec"]
    Hs = []
    for smp in g["profiles"]:
        sp = {"functions": [dict(f, samples=smp.get(f["name"], {})) for f in spec["functions"]], "calls": spec["calls"]}
        st, H, _ = build_fixture(sp)
        Hs.append(H)
    _run(gpa, st, np.stack(Hs))


@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("seed", range(30))
def test_random_graphs(gpa, seed, exact):
    rng = np.random.default_rng(3000 + seed)
    fns, calls = _random_structure(rng, int(rng.integers(2, 9)))
    P = int(rng.integers(1, 6))
    Hs = []
    for p in range(P):
        sp = {"functions": [dict(f, samples={str(k): int(rng.integers(0, 4)) for k in range(f["n_inst"])
                                             if rng.random() < 0.5}) for f in fns], "calls": calls}
        st, H, _ = build_fixture(sp)
        Hs.append(H)
    _run(gpa, st, np.stack(Hs), exact=exact)


def test_one_profile_is_reconstruct_cct(gpa):
    g = load_golden("cct_fig4_narrative.json")
    st, H, _ = build_fixture(g["spec"])
    s, S, W, R = _run(gpa, st, H[None])
    c = gpa.reconstruct_cct(s, _dev(H).reshape(-1, 16)).to_numpy()
    assert R["n"] == c["n"]
    for k in ("parent", "site", "node", "kind"):
        assert np.array_equal(c[k], R[k]), k
    for k in ("frac", "excl", "incl"):
        assert np.array_equal(c[k].view(np.uint64), R[k][:, 0].view(np.uint64)), k


def test_no_samples_and_capacity(gpa):
    g = load_golden("cct_fig4_narrative.json")
    st, H, _ = build_fixture(g["spec"])
    s = gpa.load_structure(st, 0)
    Hp = np.zeros((3,) + H.shape, np.uint64)
    S, W = _inputs_from_inst(gpa, s, Hp)
    assert gpa.reconstruct_cct_per_profile(s, S, W, 3, max_contexts=0) == 0
    m = gpa.reconstruct_cct_per_profile(s, S, W, 3)
    assert m.n == 0 and m.n_profiles == 3
    m.free()
    Hp = np.stack([H, H])
    S, W = _inputs_from_inst(gpa, s, Hp)
    n = gpa.reconstruct_cct_per_profile(s, S, W, 2, max_contexts=0)
    assert n > 1
    with pytest.raises(gpa.GpaError):
        gpa.reconstruct_cct_per_profile(s, S, W, 2, max_contexts=n - 1)
    with pytest.raises(gpa.GpaError):
        gpa.reconstruct_cct_per_profile(s, S, W, 0)


@pytest.mark.parametrize("name,records,n_prof", [("C2", 500_000, 4), ("C3", 3_000_000, 3), ("C4", 1_000_003, 16)])
def test_workloads_from_records(gpa, name, records, n_prof):
    """The full f1 path from records: S_f,p from gpa_attribute_profiles, w_p from
    gpa_profile_call_weights; the oracle from its own per-profile instruction histograms."""
    w = gen.workload(name, records=records)
    s = gpa.load_structure(w.structure, 0)
    rec = torch.empty((records, 2), dtype=torch.int64, device=DEV)
    w.records_device(rec, 0, records)
    nf, nc = s.info["n_func"], s.info["n_call"]
    PH = torch.zeros((n_prof + 1, nf, 16), dtype=torch.int64, device=DEV)
    PU = torch.zeros((n_prof + 1, 16), dtype=torch.int64, device=DEV)
    gpa.attribute_profiles(s, rec, n_prof, PH, PU)
    PW = torch.zeros((n_prof + 1, max(nc, 1)), dtype=torch.int64, device=DEV)
    gpa.profile_call_weights(s, rec, n_prof, PW)
    m = gpa.reconstruct_cct_per_profile(s, PH, PW, n_prof)
    g = m.to_numpy()
    torch.cuda.synchronize()
    Hp, _ = oracle.attribute_profiles_inst(w.structure, w.records_host(), n_prof)
    R = oracle.cct_per_profile(w.structure, Hp[:n_prof])
    _compare(g, R, n_prof)
    # the call weights also pin against the oracle's instruction cube directly (R10)
    ci = np.asarray(w.structure["call_inst"], np.int64)
    want = Hp[:, ci, :12].sum(axis=2) if nc else np.zeros((n_prof + 1, 0), np.uint64)
    assert np.array_equal(PW.cpu().numpy().view(np.uint64)[:, :nc], want)
    m.free()
