"""Randomised whole-path parity: random module layouts (variable instruction lengths, gaps,
random scope trees with non-contiguous lines, random call graphs with cycles and
self-calls), random records (misaligned / unmapped pcs, invalid stalls, skewed counts
including ~2^32), every entry point on the GPU vs the oracle."""
import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
NONE = 0xFFFFFFFF
DEV = "cuda:0"


@pytest.fixture(scope="module")
def gpa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    from paper_2109_06931_b200 import gpa
    return gpa


def random_structure(rng, n_func, n_inst):
    sizes = np.maximum(1, rng.multinomial(n_inst - n_func, np.ones(n_func) / n_func) + 1)
    lens = rng.choice([2, 4, 8, 16, 6], size=n_inst).astype(np.uint64)
    gaps = np.where(rng.random(n_inst) < 0.2, rng.integers(1, 40, n_inst), 0).astype(np.uint64)
    addr = (0x4000 + np.cumsum(gaps + np.concatenate([[0], lens[:-1]]))).astype(np.uint64)
    parent, kind, inst_scope, func_scope = [], [], np.empty(n_inst, np.uint32), []
    first = np.concatenate([[0], np.cumsum(sizes)])
    for f in range(n_func):
        parent.append(NONE); kind.append(0); fs = len(parent) - 1; func_scope.append(fs)
        inner = [fs]
        for _ in range(int(rng.integers(0, 4))):          # nested loops / inline scopes
            parent.append(inner[int(rng.integers(len(inner)))]); kind.append(int(rng.integers(1, 3)))
            inner.append(len(parent) - 1)
        lines = []
        for i in range(int(first[f]), int(first[f + 1])):
            if lines and rng.random() < 0.4:
                inst_scope[i] = lines[int(rng.integers(len(lines)))]   # non-contiguous line
            else:
                parent.append(inner[int(rng.integers(len(inner)))]); kind.append(3)
                lines.append(len(parent) - 1)
                inst_scope[i] = lines[-1]
    calls = {}
    for _ in range(int(rng.integers(0, 3 * n_func))):
        c = int(rng.integers(n_func))
        i = int(rng.integers(first[c], first[c + 1]))
        calls[i] = int(rng.integers(n_func))
    ci = np.array(sorted(calls), np.uint32)
    perm = rng.permutation(len(ci))                        # call sites in arbitrary order
    st = dict(inst_addr=addr, inst_len=lens.astype(np.uint16),
              inst_class=rng.integers(0, 16, n_inst).astype(np.uint8), inst_scope=inst_scope,
              scope_parent=np.array(parent, np.uint32), scope_kind=np.array(kind, np.uint8),
              func_scope=np.array(func_scope, np.uint32), call_inst=ci[perm],
              call_callee=np.array([calls[int(i)] for i in ci], np.uint32)[perm])
    return st


def random_records(rng, st, n):
    a, ln = st["inst_addr"], st["inst_len"].astype(np.uint64)
    w = rng.pareto(1.2, len(a)) + 0.01                     # heavy-tailed instruction popularity
    i = rng.choice(len(a), n, p=w / w.sum())
    rec = np.zeros(n, gen.RECORD_DTYPE)
    rec["pc"] = a[i] + (rng.integers(0, 1 << 20, n).astype(np.uint64) % ln[i])
    bad = rng.random(n) < 0.02
    rec["pc"][bad] = rng.integers(0, int(a[-1]) + 100, bad.sum())
    rec["count"] = np.where(rng.random(n) < 0.01, rng.integers(2 ** 31, 2 ** 32, n), rng.integers(0, 9, n))
    rec["stall"] = np.where(rng.random(n) < 0.01, rng.integers(12, 65536, n), rng.integers(0, 12, n))
    rec["stream"] = np.sort(rng.integers(0, 9, n))
    return rec


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("GPA_FUZZ_SEEDS", "24"))))
def test_fuzz_whole_path(gpa, seed):
    rng = np.random.default_rng(777 + seed)
    n_func = int(rng.integers(1, 60))
    n_inst = int(rng.integers(n_func, 6000))
    st = random_structure(rng, n_func, n_inst)
    n = int(rng.choice([1, 1000, 200_000, 2_300_000]))
    rec = random_records(rng, st, n)
    s = gpa.load_structure(st, 0)
    assert np.array_equal(s.scc_of(), oracle.cct(st, np.zeros((n_inst, 16), np.uint64))["scc_of"])
    dr = torch.from_numpy(rec.view(np.int64).reshape(-1, 2)).to(DEV)
    for kernel in (0, 1, 2, 3, 4, 5, 6, 7, 8, 9):
        gpa.set_attr_kernel(kernel)
        H = torch.zeros((n_inst, 16), dtype=torch.int64, device=DEV)
        U = torch.zeros(16, dtype=torch.int64, device=DEV)
        ri = torch.empty(n, dtype=torch.int32, device=DEV)
        gpa.attribute_samples(s, dr, H, U, ri)
        torch.cuda.synchronize()
        if kernel == 0:
            Ho, Uo, rio = oracle.attribute(st, rec, rec_inst=True)
        assert np.array_equal(H.cpu().numpy().view(np.uint64), Ho), kernel
        assert np.array_equal(U.cpu().numpy().view(np.uint64), Uo), kernel
        assert np.array_equal(ri.cpu().numpy().view(np.uint32), rio), kernel
    gpa.set_attr_kernel(0)
    for scope in ("INST", "LINE", "LOOP", "INLINE", "FUNC"):
        rows = len(s.rows(scope))
        if rows == 0:
            continue
        hist = torch.empty((rows, 16), dtype=torch.int64, device=DEV)
        mix = torch.empty((rows, 16), dtype=torch.int64, device=DEV)
        met = torch.empty((rows, 33), dtype=torch.float64, device=DEV)
        gpa.derive_metrics(s, scope, H, scope_hist=hist, scope_mix=mix, metrics=met)
        eh, em = oracle.scope_hist(st, Ho, scope)
        assert np.array_equal(hist.cpu().numpy().view(np.uint64), eh), scope
        assert np.array_equal(mix.cpu().numpy().view(np.uint64), em), scope
        assert np.array_equal(met.cpu().numpy().view(np.uint64), oracle.derive_u64(eh, em).view(np.uint64)), scope
    for exact in (False, True):
        R = oracle.cct(st, Ho, exact=exact)
        c = gpa.reconstruct_cct(s, H, mode=gpa.WEIGHTS_EXACT if exact else gpa.WEIGHTS_SAMPLES)
        g = c.to_numpy()
        assert g["n"] == R["n"]
        for k in ("parent", "site", "node", "kind", "first_child", "n_children"):
            assert np.array_equal(g[k], R[k]), k
        for k in ("frac", "excl", "incl"):
            assert np.array_equal(g[k].view(np.uint64), R[k].view(np.uint64)), k
        c.free()
    P = 7
    PH = torch.zeros((P + 1, n_func, 16), dtype=torch.int64, device=DEV)
    PU = torch.zeros((P + 1, 16), dtype=torch.int64, device=DEV)
    gpa.attribute_profiles(s, dr, P, PH, PU)
    Hp, Up = oracle.attribute_profiles(st, rec, P)
    assert np.array_equal(PH.cpu().numpy().view(np.uint64), Hp) and np.array_equal(PU.cpu().numpy().view(np.uint64), Up)
