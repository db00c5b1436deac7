"""Pins of oracle D12 (reading R30): one approximate CCT per profile ("for each GPU kernel
invocation"), unified by call path.  A hand-worked two-profile example, the
one-profile identity with D6, and a brute force over random tiny call graphs: the unified tree's
path set is exactly the union of the profiles' path sets, numbered breadth first with children in
key order, and every profile's values sit at its own paths.  CPU only."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from tests.fixtures import build as build_fixture, load_golden

NONE = 0xFFFFFFFF


def _profiles_from_golden(g):
    spec = g["spec"]
    Hs = []
    for smp in g["profiles"]:
        sp = {"functions": [dict(f, samples=smp.get(f["name"], {})) for f in spec["functions"]], "calls": spec["calls"]}
        st, H, idx = build_fixture(sp)
        Hs.append(H)
    return st, np.stack(Hs), idx


def test_per_profile_hand_worked():
    g = load_golden("cct_per_profile.json")
    st, Hp, idx = _profiles_from_golden(g)
    R = oracle.cct_per_profile(st, Hp)
    e = g["expect"]
    assert R["n"] == len(e["contexts"])
    for u, (kind, fn, parent) in enumerate(e["contexts"]):
        assert R["kind"][u] == {"FUNC": 0, "SCC": 1, "MEMBER": 2}[kind]
        assert R["node"][u] == idx[fn]          # trivial DAG node id = function id here
        assert R["parent"][u] == (NONE if parent is None else parent)
        for p in range(2):
            assert Fraction(R["frac"][u, p]) == Fraction(e["frac"][u][p])
            assert Fraction(R["excl"][u, p, 0]) == Fraction(e["excl_slot0"][u][p])
            assert Fraction(R["incl"][u, p, 0]) == Fraction(e["incl_slot0"][u][p])


def test_one_profile_is_the_tree():
    g = load_golden("cct_fig4_narrative.json")
    st, H, _ = build_fixture(g["spec"])
    R1 = oracle.cct(st, H)
    R = oracle.cct_per_profile(st, H[None])
    assert R["n"] == R1["n"]
    for k in ("kind", "node", "parent", "site"):
        assert np.array_equal(R[k], R1[k]), k
    assert np.array_equal(R["frac"][:, 0], R1["frac"])
    assert np.array_equal(R["incl"][:, 0], R1["incl"])


def _paths(kind, node, parent, site, ci):
    """Call path of every context: root DAG node, then per step the member function (SCC parent)
    or the call instruction of the site."""
    out = []
    for c in range(len(kind)):
        if parent[c] == NONE:
            out.append((int(node[c]),))
        else:
            pk = kind[parent[c]]
            step = int(node[c]) if pk == 1 else int(ci[site[c]])
            out.append(out[parent[c]] + (step,))
    return out


def _random_structure(rng, n_func):
    fns = [{"name": f"f{i}", "n_inst": int(rng.integers(2, 5)), "samples": {}} for i in range(n_func)]
    calls, used = [], set()
    for i in range(n_func):
        for _ in range(int(rng.integers(0, 3))):
            k = int(rng.integers(0, fns[i]["n_inst"]))
            if (i, k) in used:
                continue
            used.add((i, k))
            calls.append([f"f{i}", k, f"f{int(rng.integers(0, n_func))}"])   # cycles and self calls allowed
    return fns, calls


@pytest.mark.parametrize("seed", range(30))
def test_unified_paths_are_the_union(seed):
    rng = np.random.default_rng(3000 + seed)
    fns, calls = _random_structure(rng, int(rng.integers(2, 7)))
    P = int(rng.integers(1, 5))
    Hs = []
    for p in range(P):
        sp = {"functions": [dict(f, samples={str(k): int(rng.integers(0, 4)) for k in range(f["n_inst"])
                                             if rng.random() < 0.5}) for f in fns], "calls": calls}
        st, H, _ = build_fixture(sp)
        Hs.append(H)
    Hp = np.stack(Hs)
    R = oracle.cct_per_profile(st, Hp)
    ci = np.asarray(st["call_inst"])
    upaths = _paths(R["kind"], R["node"], R["parent"], R["site"], ci)
    assert len(set(upaths)) == R["n"]                                   # a path appears once
    union = set()
    for p, T in enumerate(R["trees"]):
        tp = _paths(T["kind"], T["node"], T["parent"], T["site"], ci)
        union |= set(tp)
        at = {q: u for u, q in enumerate(upaths)}
        for c, q in enumerate(tp):                                      # p's values at its paths
            u = at[q]
            assert R["frac"][u, p] == T["frac"][c] and np.array_equal(R["incl"][u, p], T["incl"][c])
        mine = {at[q] for q in tp}
        for u in range(R["n"]):                                         # 0 where p lacks the path
            if u not in mine:
                assert R["frac"][u, p] == 0 and not R["incl"][u, p].any()
        # conservation per profile: sum of excl = samples of p's active functions
        assert np.isclose(R["excl"][:, p].sum(), T["excl"].sum(), rtol=1e-12, atol=0)
    assert set(upaths) == union
    # breadth-first numbering: parents first; siblings by key; levels non-decreasing
    depth = [len(q) for q in upaths]
    assert all(depth[u] <= depth[u + 1] for u in range(R["n"] - 1))
    for u in range(1, R["n"]):
        if R["parent"][u] != NONE:
            assert R["parent"][u] < u
        if R["parent"][u] == R["parent"][u - 1] and depth[u] == depth[u - 1]:
            assert upaths[u][-1] > upaths[u - 1][-1]
