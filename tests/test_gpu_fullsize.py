"""Parity at BASELINE.json's full sizes (all five configs), in the launch configuration
bench.py times (one gpa_attribute_samples call over the whole device-resident stream): the
complete histogram H || U bit-exact against the oracle run chunk by chunk on the host (all
host threads), sampled per-record attributions, the > 2^32 planted bin (C5), the CCT
(topology exact, fp64 within 1e-9) with its EXCL/INCL metrics, and every scope's roll-up and
metrics on the full histogram.  Slow (about a minute for C4 / C5)."""
import os

import numpy as np
import pytest

import gen
import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def gpa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    from paper_2109_06931_b200 import gpa
    return gpa


def _oracle_full(w, chunk=1 << 27):
    threads = len(os.sched_getaffinity(0))
    H = np.zeros((w.meta["n_inst"], 16), np.uint64)
    U = np.zeros(16, np.uint64)
    buf = np.empty(chunk, gen.RECORD_DTYPE)
    for k0 in range(0, w.cfg.records, chunk):
        n = min(chunk, w.cfg.records - k0)
        rec = w.records_host(k0, n, threads=threads, out=buf[:n])
        h, u, _ = oracle.attribute(w.structure, rec, threads=threads)
        H += h
        U += u
    return H, U


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_full_size_histogram_bit_exact(gpa, name):
    w = gen.workload(name)
    n = w.cfg.records
    s = gpa.load_structure(w.structure, 0)
    rec = torch.empty((n, 2), dtype=torch.int64, device="cuda")
    for k in range(0, n, 1 << 28):
        w.records_device(rec[k:k + (1 << 28)], k, min(1 << 28, n - k))
    H = torch.zeros((s.info["n_inst"], 16), dtype=torch.int64, device="cuda")
    U = torch.zeros(16, dtype=torch.int64, device="cuda")
    gpa.attribute_samples(s, rec, H, U)
    # per-record attributions on sampled windows (a second call over slices, rec_inst on)
    rng = np.random.default_rng(11)
    win = min(100_000, n)
    for k0 in [0, n - win] + [int(x) for x in rng.integers(0, n - win + 1, 3)]:
        ri = torch.empty(win, dtype=torch.int32, device="cuda")
        H2 = torch.zeros_like(H)
        U2 = torch.zeros_like(U)
        gpa.attribute_samples(s, rec[k0:k0 + win], H2, U2, ri)
        _, _, rio = oracle.attribute(w.structure, w.records_host(k0, win), rec_inst=True)
        assert np.array_equal(ri.cpu().numpy().view(np.uint32), rio)
    torch.cuda.synchronize()
    Hg = H.cpu().numpy().view(np.uint64)
    Ug = U.cpu().numpy().view(np.uint64)
    del rec
    torch.cuda.empty_cache()
    Ho, Uo = _oracle_full(w)
    assert np.array_equal(Ug, Uo)
    assert np.array_equal(Hg, Ho)
    if name == "C5":   # the planted barrier bin exceeds 2^32 (reading R19)
        assert Hg[w.tables["hot_inst"], 5] > 2 ** 32
    # roll-up, CCT and metrics on the full-size histogram
    R = oracle.cct(w.structure, Ho)
    c = gpa.reconstruct_cct(s, H)
    g = c.to_numpy()
    assert g["n"] == R["n"] and np.array_equal(g["parent"], R["parent"]) and np.array_equal(g["site"], R["site"])
    assert np.allclose(g["incl"], R["incl"], rtol=1e-9, atol=0)
    assert np.allclose(g["excl"], R["excl"], rtol=1e-9, atol=0) and np.allclose(g["frac"], R["frac"], rtol=1e-9, atol=0)
    for scope, V in [("CCT_EXCL", R["excl"]), ("CCT_INCL", R["incl"])]:
        met = torch.empty((max(R["n"], 1), 33), dtype=torch.float64, device="cuda")
        gpa.derive_metrics(s, scope, cct=c, metrics=met)
        assert np.allclose(met.cpu().numpy()[:R["n"]], oracle.derive_f64(V), rtol=1e-9, atol=0, equal_nan=True), scope
    c.free()
    # every scope's roll-up (u64, bit-exact) and derived metrics (closed forms on u64: bit-exact)
    for scope in ["INST", "LINE", "LOOP", "INLINE", "FUNC"]:
        rows = max(1, gpa.scope_row_count(s, scope))
        sh = torch.empty((rows, 16), dtype=torch.int64, device="cuda")
        sm = torch.empty((rows, 16), dtype=torch.int64, device="cuda")
        fm = torch.empty((rows, 33), dtype=torch.float64, device="cuda")
        gpa.derive_metrics(s, scope, H, scope_hist=sh, scope_mix=sm, metrics=fm)
        hist, mix = oracle.scope_hist(w.structure, Ho, scope)
        k = len(hist)
        assert np.array_equal(sh.cpu().numpy().view(np.uint64)[:k], hist), scope
        assert np.array_equal(sm.cpu().numpy().view(np.uint64)[:k], mix), scope
        assert np.array_equal(fm.cpu().numpy()[:k].view(np.uint64), oracle.derive_u64(hist, mix).view(np.uint64)), scope


def test_full_size_profiles_c4(gpa):
    """f1 at C4's full size in bench_next's launch configuration (1e9 records, 384 profiles, one
    call each): every profile's instruction rows summed over profiles equal the aggregate H of
    the same records (integers, exact at any size); four sampled profiles (contiguous record
    ranges of the stream field) bit-exact against the oracle at instruction and function level."""
    w = gen.workload("C4")
    n = w.cfg.records
    s = gpa.load_structure(w.structure, 0)
    rec = torch.empty((n, 2), dtype=torch.int64, device="cuda")
    for k in range(0, n, 1 << 28):
        w.records_device(rec[k:k + (1 << 28)], k, min(1 << 28, n - k))
    P, ni, nf = 384, s.info["n_inst"], s.info["n_func"]
    H = torch.zeros((ni, 16), dtype=torch.int64, device="cuda")
    U = torch.zeros(16, dtype=torch.int64, device="cuda")
    gpa.attribute_samples(s, rec, H, U)
    PH = torch.zeros((P + 1, nf, 16), dtype=torch.int64, device="cuda")
    PU = torch.zeros((P + 1, 16), dtype=torch.int64, device="cuda")
    gpa.attribute_profiles(s, rec, P, PH, PU)
    PI = torch.zeros((P + 1, ni, 16), dtype=torch.int64, device="cuda")
    PUI = torch.zeros((P + 1, 16), dtype=torch.int64, device="cuda")
    gpa.attribute_profiles_inst(s, rec, P, PI, PUI)
    torch.cuda.synchronize()
    assert torch.equal(PI.sum(0), H) and torch.equal(PUI.sum(0), U)   # int64 sums wrap like u64
    assert torch.equal(PU, PUI)
    del rec
    sfb = w.tables["stream_first_burst"].astype(np.int64)
    bounds = np.concatenate([np.minimum(sfb << int(w.tables["burst_shift"]), n), [n]])
    rng = np.random.default_rng(12)
    for p in [0, P - 1] + [int(x) for x in rng.integers(1, P - 1, 2)]:
        k0, k1 = int(bounds[p]), int(bounds[p + 1])
        Ho, Uo, _ = oracle.attribute(w.structure, w.records_host(k0, k1 - k0, threads=len(os.sched_getaffinity(0))),
                                     threads=len(os.sched_getaffinity(0)))
        assert np.array_equal(PI[p].cpu().numpy().view(np.uint64), Ho), p
        assert np.array_equal(PUI[p].cpu().numpy().view(np.uint64), Uo), p
        Fo, _ = oracle.scope_hist(w.structure, Ho, "FUNC")
        assert np.array_equal(PH[p].cpu().numpy().view(np.uint64), Fo), p
