"""Pins of oracle D3-D6 (GPU calling-context tree, §5.3):
hand-worked fixtures (tests/golden/cct_*.json), a brute-force re-derivation on random tiny
graphs with exact rationals (different algorithms: fixpoint sweeps, transitive-closure
SCCs, path enumeration), conservation and the gprof identity.  CPU only."""
from fractions import Fraction

import numpy as np
import pytest

import gen
import oracle
from tests.fixtures import build, frac, load_golden

NONE = oracle.NONE
KIND = {"FUNC": 0, "SCC": 1, "MEMBER": 2}


def _check_expected(st, H, expect, exact=False):
    R = oracle.cct(st, H, exact=exact)
    assert R["status"] == 0
    if "w_step1" in expect:
        assert R["w_step1"].tolist() == expect["w_step1"]
    assert R["w"].tolist() == expect["w"]
    if "scc_of" in expect:
        assert R["scc_of"].tolist() == expect["scc_of"]
    if "dag_weight" in expect:
        assert R["W"].tolist() == expect["dag_weight"]
    ctx = expect["contexts"]
    assert R["n"] == len(ctx)
    S_f = R["S_f"]
    for c, (kind, node, parent, site, f, ex, inc) in enumerate(ctx):
        assert R["kind"][c] == KIND[kind], c
        assert R["node"][c] == node, c
        assert R["parent"][c] == (NONE if parent is None else parent), c
        assert R["site"][c] == (NONE if site is None else site), c
        assert R["frac"][c] == pytest.approx(float(frac(f)), rel=1e-15), c
        assert R["excl"][c, :12].sum() == pytest.approx(float(frac(ex)), rel=1e-13, abs=1e-15), c
        assert R["incl"][c, :12].sum() == pytest.approx(float(frac(inc)), rel=1e-13, abs=1e-15), c
        if kind in ("FUNC", "MEMBER"):   # every slot, incl. the invalid one, scales by f
            g = node if kind == "MEMBER" else R["scc_of"].tolist().index(node)
            for r in range(16):
                assert R["excl"][c, r] == pytest.approx(float(frac(f) * int(S_f[g, r])), rel=1e-15, abs=0)
    return R


@pytest.mark.parametrize("name", ["cct_fig4_narrative.json", "cct_guard.json", "cct_diamond.json"])
def test_cct_golden(name):
    g = load_golden(name)
    st, H, _ = build(g["spec"])
    _check_expected(st, H, g["expect"])


@pytest.mark.parametrize("case", ["apportion", "single", "chain", "nonzero", "self"])
def test_cct_spec_examples(case):
    g = load_golden("cct_spec_examples.json")["cases"][case]
    st, H, _ = build(g["spec"])
    _check_expected(st, H, g["expect"])


# ---------------------------------------------------------------------------------------
# brute force with exact rationals
# ---------------------------------------------------------------------------------------
def brute_cct(st, H, exact=False):
    n_func, n_call = len(st["func_scope"]), len(st["call_inst"])
    ifunc = oracle.inst_func(st)
    callee = [int(x) for x in st["call_callee"]]
    caller = [int(ifunc[i]) for i in st["call_inst"]]
    H = np.asarray(H, np.uint64)
    S = [[0] * 16 for _ in range(n_func)]
    for i in range(len(H)):
        for r in range(16):
            S[ifunc[i]][r] += int(H[i, r])
    w = [int(H[st["call_inst"][e], :12].sum()) for e in range(n_call)]
    active = [sum(S[f][:12]) > 0 for f in range(n_func)]
    changed = not exact                     # exact counts: no Step 2, no guard (R24)
    while changed:                          # Step 2 by whole-graph sweeps to a fixpoint
        changed = False
        for f in range(n_func):
            ins = [e for e in range(n_call) if callee[e] == f]
            if active[f] and ins and all(w[e] == 0 for e in ins):
                for e in ins:
                    w[e] = 1
                    active[caller[e]] = True
                changed = True
    reach = [[False] * n_func for _ in range(n_func)]   # transitive closure (Warshall)
    for e in range(n_call):
        reach[caller[e]][callee[e]] = True
    for k in range(n_func):
        for i in range(n_func):
            if reach[i][k]:
                for j in range(n_func):
                    if reach[k][j]:
                        reach[i][j] = True
    rep = [min(j for j in range(n_func) if j == i or (reach[i][j] and reach[j][i])) for i in range(n_func)]
    reps = sorted(set(rep))
    dag = {r: d for d, r in enumerate(reps)}
    scc = [dag[rep[f]] for f in range(n_func)]
    members = {d: [f for f in range(n_func) if scc[f] == d] for d in range(len(reps))}
    nontriv = {d: len(m) > 1 or reach[m[0]][m[0]] for d, m in members.items()}
    ext_in = {d: [e for e in range(n_call) if scc[callee[e]] == d and scc[caller[e]] != d] for d in members}
    dact = {d: any(active[f] for f in m) for d, m in members.items()}
    changed = not exact
    while changed:                          # DAG guard (reading R12)
        changed = False
        for d in members:
            if dact[d] and ext_in[d] and all(w[e] == 0 for e in ext_in[d]):
                for e in ext_in[d]:
                    w[e] = 1
                    dact[scc[caller[e]]] = True
                changed = True
    W = {d: sum(w[e] for e in ext_in[d]) for d in members}
    roots = [d for d in sorted(members) if not ext_in[d] and dact[d]]
    ctxs = {}

    def visit(key, kind, node, f):
        """Enumerate every root->node path (the tree IS the set of paths)."""
        if kind == 1:
            ex = [Fraction(0)] * 16
            inc = list(ex)
            for m in members[node]:
                sub = visit(key + (("m", m),), 2, m, f)
                inc = [a + b for a, b in zip(inc, sub)]
        else:
            g = node if kind == 2 else members[node][0]
            ex = [f * S[g][r] for r in range(16)]
            inc = list(ex)
            outs = sorted((int(st["call_inst"][e]), e) for e in range(n_call) if caller[e] == g)
            for _, e in outs:
                Y = scc[callee[e]]
                if Y == scc[g] or w[e] == 0:
                    continue
                sub = visit(key + (e,), 1 if nontriv[Y] else 0, Y, f * Fraction(w[e], W[Y]))
                inc = [a + b for a, b in zip(inc, sub)]
        ctxs[key] = (kind, node, f, ex, inc)
        return inc

    for d in roots:
        visit((("root", d),), 1 if nontriv[d] else 0, d, Fraction(1))
    return ctxs, w, scc, W, S, dact


def _key_of(R, c):
    path = []
    while R["parent"][c] != NONE:
        path.append(("m", int(R["node"][c])) if R["kind"][c] == 2 else int(R["site"][c]))
        c = int(R["parent"][c])
    return (("root", int(R["node"][c])),) + tuple(reversed(path))


def _random_graph(rng):
    n_func = int(rng.integers(1, 9))
    spec = {"functions": [], "calls": []}
    sizes = [int(rng.integers(1, 5)) for _ in range(n_func)]
    n_call = int(rng.integers(0, 13))
    slots = {f: list(range(sizes[f])) for f in range(n_func)}
    for _ in range(n_call):
        c = int(rng.integers(n_func))
        if not slots[c]:
            continue
        k = slots[c].pop(int(rng.integers(len(slots[c]))))
        spec["calls"].append([f"F{c}", k, f"F{int(rng.integers(n_func))}"])
    for f in range(n_func):
        smp = {}
        cold = rng.random() < 0.3
        for k in range(sizes[f]):
            if cold or rng.random() < 0.4:
                continue
            smp[str(k)] = {str(int(r)): int(rng.integers(1, 9)) for r in rng.choice(16, 2, replace=False)}
        spec["functions"].append({"name": f"F{f}", "n_inst": sizes[f], "samples": smp})
    return spec


@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("seed", range(60))
def test_cct_brute_force_random_graphs(seed, exact):
    rng = np.random.default_rng(1000 + seed)
    st, H, _ = build(_random_graph(rng))
    R = oracle.cct(st, H, exact=exact)
    ctxs, w, scc, W, S, _ = brute_cct(st, H, exact=exact)
    assert R["w"].tolist() == w
    assert R["scc_of"].tolist() == scc
    assert R["W"].tolist() == [W[d] for d in range(len(W))]
    assert R["n"] == len(ctxs)
    for c in range(R["n"]):
        kind, node, f, ex, inc = ctxs[_key_of(R, c)]
        assert (R["kind"][c], R["node"][c]) == (kind, node)
        assert R["frac"][c] == pytest.approx(float(f), rel=1e-14)
        for r in range(16):
            assert R["excl"][c, r] == pytest.approx(float(ex[r]), rel=1e-13, abs=1e-300)
            assert R["incl"][c, r] == pytest.approx(float(inc[r]), rel=1e-13, abs=1e-300)


def _structural_checks(st, R):
    n = R["n"]
    par, fc, nc = R["parent"], R["first_child"], R["n_children"]
    depth = np.zeros(n, np.int64)
    for c in range(n):
        if par[c] != NONE:
            assert par[c] < c
            depth[c] = depth[par[c]] + 1
            assert fc[par[c]] <= c < fc[par[c]] + nc[par[c]]
    assert (np.diff(depth) >= 0).all()                     # breadth-first numbering
    ci = st["call_inst"]
    for c in range(n):
        kids = range(int(fc[c]), int(fc[c]) + int(nc[c]))
        if R["kind"][c] == 1:
            assert [int(R["node"][d]) for d in kids] == sorted(int(R["node"][d]) for d in kids)
        else:
            sites = [int(ci[R["site"][d]]) for d in kids]
            assert sites == sorted(sites)


@pytest.mark.parametrize("name,records", [("C1", 10_000), ("C2", 300_000), ("C3", 300_000), ("C4", 300_000)])
def test_cct_invariants_on_workloads(name, records):
    """P8: sum of excl over contexts = all valid samples (every sampled function is
    reachable, reading R15); gprof identity incl(c) = f(c) * T(node) via an independent
    reverse-topological DP; BFS numbering and child order (R17)."""
    w = gen.workload(name, records=records)
    st = w.structure
    H, _, _ = oracle.attribute(st, w.records_host())
    R = oracle.cct(st, H)
    assert R["status"] == 0 and R["n"] > 0
    tot = H[:, :12].sum(0).astype(np.float64)
    assert np.allclose(R["excl"][:, :12].sum(0), tot, rtol=1e-12, atol=0)
    _structural_checks(st, R)
    # gprof identity with T from a DP over the condensed DAG (reverse topological order)
    ifunc = oracle.inst_func(st)
    caller = ifunc[st["call_inst"]]
    scc = R["scc_of"]
    wv = R["w"]
    Wd = R["W"]
    n_dag = R["n_dag"]
    S_f = R["S_f"].astype(np.float64)
    memb = [[] for _ in range(n_dag)]
    for f in range(len(scc)):
        memb[scc[f]].append(f)
    out_of = [[] for _ in range(len(scc))]
    for e in range(len(caller)):
        out_of[caller[e]].append(e)
    Tf = {}
    Td = {}

    def T_func(g):
        if g not in Tf:
            t = S_f[g].copy()
            for e in out_of[g]:
                Y = scc[st["call_callee"][e]]
                if Y != scc[g] and wv[e] > 0:
                    t = t + (wv[e] / Wd[Y]) * T_dag(Y)
            Tf[g] = t
        return Tf[g]

    def T_dag(X):
        if X not in Td:
            Td[X] = sum((T_func(m) for m in memb[X]), np.zeros(16))
        return Td[X]

    import sys
    sys.setrecursionlimit(100000)
    for c in range(R["n"]):
        node = int(R["node"][c])
        T = T_func(node) if R["kind"][c] == 2 else (T_dag(node) if R["kind"][c] == 1 else T_func(memb[node][0]))
        assert np.allclose(R["incl"][c], R["frac"][c] * T, rtol=1e-10, atol=1e-9)


def test_cct_capacity_and_empty():
    g = load_golden("cct_fig4_narrative.json")
    st, H, _ = build(g["spec"])
    R = oracle.cct(st, H, max_contexts=5)
    assert R["status"] == 3 and R["n"] == 9
    R = oracle.cct(st, np.zeros_like(H))
    assert R["status"] == 0 and R["n"] == 0
    assert R["w"].tolist() == [0] * 6


def test_cct_exact_mode_fixtures():
    """R24: with consistent exact counts Step 2 is a no-op, so the exact
    tree equals the samples tree; with an executed function behind an unexecuted call,
    exact mode leaves it out."""
    g = load_golden("cct_exact.json")
    st, H, _ = build(g["consistent"])
    Rs, Re = oracle.cct(st, H), oracle.cct(st, H, exact=True)
    for k in ["parent", "site", "node", "kind", "frac", "excl", "incl", "w"]:
        assert np.array_equal(Rs[k], Re[k]), k
    st, H, _ = build(g["inconsistent"]["spec"])
    _check_expected(st, H, g["inconsistent"]["expect"], exact=True)


def test_block_counts_propagate_to_instructions():
    """a basic block's execution count is every member instruction's count."""
    rng = np.random.default_rng(3)
    for _ in range(20):
        n_inst = int(rng.integers(1, 200))
        cuts = np.sort(rng.choice(np.arange(1, n_inst), size=min(n_inst - 1, int(rng.integers(0, 20))), replace=False))
        start = np.concatenate([[0], cuts, [n_inst]]).astype(np.uint32)
        cnt = rng.integers(0, 2 ** 40, len(start) - 1).astype(np.uint64)
        H = oracle.block_counts(n_inst, start, cnt)
        expect = np.repeat(cnt, np.diff(start.astype(np.int64)))
        assert np.array_equal(H[:, 0], expect) and H[:, 1:].sum() == 0
