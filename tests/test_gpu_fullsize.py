"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (one
gpa_attribute_samples call over the whole device-resident stream): the complete histogram
H || U bit-exact against the oracle run chunk by chunk on the host (16 threads), sampled
per-record attributions, the > 2^32 planted bin (C5), and CCT / metrics on the full
histogram.  Slow (about a minute each)."""
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


@pytest.mark.parametrize("name", ["C4", "C5"])
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
    for k0 in [0, n - 100_000] + [int(x) for x in rng.integers(0, n - 100_000, 3)]:
        ri = torch.empty(100_000, dtype=torch.int32, device="cuda")
        H2 = torch.zeros_like(H)
        U2 = torch.zeros_like(U)
        gpa.attribute_samples(s, rec[k0:k0 + 100_000], H2, U2, ri)
        _, _, rio = oracle.attribute(w.structure, w.records_host(k0, 100_000), rec_inst=True)
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
    fm = torch.empty((s.info["n_func"], 33), dtype=torch.float64, device="cuda")
    gpa.derive_metrics(s, "FUNC", H, metrics=fm)
    hist, mix = oracle.scope_hist(w.structure, Ho, "FUNC")
    assert np.array_equal(fm.cpu().numpy().view(np.uint64), oracle.derive_u64(hist, mix).view(np.uint64))
    c.free()
