"""GPU parity: the CUDA path through the C ABI against the CPU oracle on the same seeded
inputs.  Integers and indices bit-exact; fp64 within 1e-9 relative (north star), checked
here also for bit-equality where the arithmetic order is identical by construction."""
import numpy as np
import pytest

import gen
import oracle
from tests.fixtures import build as build_fixture, load_golden

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
RTOL = 1e-9


@pytest.fixture(scope="module")
def gpa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    from paper_2109_06931_b200 import gpa
    return gpa


DEV = "cuda:0"


def u64(t):
    return t.cpu().numpy().view(np.uint64)


def _device_records(w, k0=0, n=None):
    n = w.cfg.records - k0 if n is None else n
    rec = torch.empty((n, 2), dtype=torch.int64, device=DEV)
    w.records_device(rec, k0, n)
    return rec


def _attribute(gpa, s, rec, rec_inst=True):
    n = rec.shape[0]
    H = torch.zeros((s.info["n_inst"], 16), dtype=torch.int64, device=DEV)
    U = torch.zeros(16, dtype=torch.int64, device=DEV)
    ri = torch.empty(n, dtype=torch.int32, device=DEV) if rec_inst else None
    gpa.attribute_samples(s, rec, H, U, ri)
    torch.cuda.synchronize()
    return H, U, ri


# ---- input generator: device build == host build -------------------------------------------
@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_device_generator_matches_host(gpa, name):
    w = gen.workload(name)
    for k0, n in [(0, 10_000), (w.cfg.records - 5_000, 5_000), (w.cfg.records // 3, 7_777)]:
        if k0 < 0 or n <= 0:
            continue
        d = _device_records(w, k0, n).cpu().numpy().view(gen.RECORD_DTYPE).reshape(-1)
        assert np.array_equal(d, w.records_host(k0, n)), (name, k0)


# ---- a-1..a-3 -------------------------------------------------------------------------------
@pytest.mark.parametrize("name,records", [("C1", 10_000), ("C2", 1_000_003), ("C3", 2_000_000),
                                          ("C4", 2_000_000), ("C5", 3_000_001)])
def test_attribution_parity(gpa, name, records):
    w = gen.workload(name, records=records)
    s = gpa.load_structure(w.structure, 0)
    assert s.info["lookup_mode"] == 0
    rec = _device_records(w)
    H, U, ri = _attribute(gpa, s, rec)
    Ho, Uo, rio = oracle.attribute(w.structure, w.records_host(), rec_inst=True)
    assert np.array_equal(u64(H), Ho)
    assert np.array_equal(u64(U), Uo)
    assert np.array_equal(ri.cpu().numpy().view(np.uint32), rio)


def _random_structure(rng, n, sparse=False):
    lens = rng.integers(1, 24, n).astype(np.uint64)
    gaps = rng.integers(0, 3, n).astype(np.uint64) * rng.integers(0, 9, n).astype(np.uint64)
    if sparse:
        gaps[n // 2] = np.uint64(1 << 40)          # forces the binary-search lookup mode
    addr = (np.cumsum(gaps + np.concatenate([[0], lens[:-1]])) + 3).astype(np.uint64)
    st = dict(inst_addr=addr, inst_len=lens.astype(np.uint16), inst_class=rng.integers(0, 16, n).astype(np.uint8),
              inst_scope=np.arange(1, n + 1, dtype=np.uint32),
              scope_parent=np.concatenate([[0xFFFFFFFF], np.zeros(n)]).astype(np.uint32),
              scope_kind=np.concatenate([[0], np.full(n, 3)]).astype(np.uint8), func_scope=np.zeros(1, np.uint32),
              call_inst=np.zeros(0, np.uint32), call_callee=np.zeros(0, np.uint32))
    return st


def _random_records(rng, st, n):
    addr, ln = st["inst_addr"], st["inst_len"]
    rec = np.zeros(n, gen.RECORD_DTYPE)
    i = rng.integers(0, len(addr), n)
    rec["pc"] = addr[i] + rng.integers(0, 30, n).astype(np.uint64)
    rec["pc"][:6] = [0, int(addr[0]), int(addr[-1]) + int(ln[-1]), 2 ** 64 - 1, int(addr[0]) - 1, 1 << 39]
    rec["count"] = rng.integers(0, 70000, n)
    rec["stall"] = np.where(rng.random(n) < 0.1, rng.integers(12, 65536, n), rng.integers(0, 12, n))
    return rec


@pytest.mark.parametrize("sparse", [False, True])
@pytest.mark.parametrize("seed", range(4))
def test_attribution_random_tables_both_lookup_modes(gpa, seed, sparse):
    rng = np.random.default_rng(seed)
    st = _random_structure(rng, int(rng.integers(1, 3000)), sparse)
    s = gpa.load_structure(st, 0)
    assert s.info["lookup_mode"] == (1 if sparse else 0)
    rec = _random_records(rng, st, 100_003)
    H, U, ri = _attribute(gpa, s, torch.from_numpy(rec.view(np.int64).reshape(-1, 2)).to(DEV))
    Ho, Uo, rio = oracle.attribute(st, rec, rec_inst=True)
    assert np.array_equal(u64(H), Ho) and np.array_equal(u64(U), Uo)
    assert np.array_equal(ri.cpu().numpy().view(np.uint32), rio)


def test_attribution_worked_example(gpa):
    g = load_golden("attribution_examples.json")
    s_ = g["structure"]
    kinds = {"FUNCTION": 0, "INLINE": 1, "LOOP": 2, "LINE": 3}
    st = dict(inst_addr=np.array(s_["inst_addr"], np.uint64), inst_len=np.array(s_["inst_len"], np.uint16),
              inst_class=np.zeros(len(s_["inst_addr"]), np.uint8), inst_scope=np.array(s_["inst_scope"], np.uint32),
              scope_parent=np.array([0xFFFFFFFF if p is None else p for _, p in s_["scopes"]], np.uint32),
              scope_kind=np.array([kinds[k] for k, _ in s_["scopes"]], np.uint8),
              func_scope=np.array(s_["func_scope"], np.uint32), call_inst=np.zeros(0, np.uint32),
              call_callee=np.zeros(0, np.uint32))
    s = gpa.load_structure(st, 0)
    assert s.info["granule_shift"] == 1 and s.info["lookup_mode"] == 0
    rec = np.zeros(len(g["records"]), gen.RECORD_DTYPE)
    for k, (pc, c, stall) in enumerate(g["records"]):
        rec[k] = (pc, c, stall, 0)
    H, U, ri = _attribute(gpa, s, torch.from_numpy(rec.view(np.int64).reshape(-1, 2)).to(DEV))
    assert [None if x == 0xFFFFFFFF else int(x) for x in ri.cpu().numpy().view(np.uint32)] == g["expect"]["rec_inst"]
    Hs = torch.zeros((s.rows("LINE").size, 16), dtype=torch.int64, device=DEV)
    gpa.derive_metrics(s, "LOOP", H, scope_hist=Hs[:1])
    assert u64(Hs)[0, 3] == 4 and u64(Hs)[0, 0] == 1


def test_attribution_edge_cases(gpa):
    w = gen.workload("C2", records=300_000)
    s = gpa.load_structure(w.structure, 0)
    rec = _device_records(w)
    Ho, Uo, _ = oracle.attribute(w.structure, w.records_host())
    # chunked accumulation (ragged chunk sizes, incl. 1-record chunks) == one shot
    H = torch.zeros((s.info["n_inst"], 16), dtype=torch.int64, device=DEV)
    U = torch.zeros(16, dtype=torch.int64, device=DEV)
    cuts = [0, 1, 2, 33, 127, 128, 129, 5000, 150_001, 299_999, 300_000]
    for a, b in zip(cuts[:-1], cuts[1:]):
        gpa.attribute_samples(s, rec[a:b], H, U)
    gpa.attribute_samples(s, rec[:0], H, U)                     # n == 0 is a no-op
    torch.cuda.synchronize()
    assert np.array_equal(u64(H), Ho) and np.array_equal(u64(U), Uo)
    # host records through the C ABI (pageable and pinned)
    host = w.records_host()
    for pinned in (False, True):
        H.zero_()
        U.zero_()
        src = torch.from_numpy(host.view(np.int64).reshape(-1, 2))
        gpa.attribute_samples_host(s, src.pin_memory() if pinned else src, H, U)
        assert np.array_equal(u64(H), Ho) and np.array_equal(u64(U), Uo)
    # misaligned device buffer is rejected
    raw = torch.zeros(16 * 10 + 8, dtype=torch.uint8, device=DEV)
    with pytest.raises(gpa.GpaError):
        gpa.attribute_samples(s, raw[8:], H, U, n=10)


def test_attribution_empty_structure(gpa):
    e32 = np.zeros(0, np.uint32)
    st = dict(inst_addr=np.zeros(0, np.uint64), inst_len=np.zeros(0, np.uint16), inst_class=np.zeros(0, np.uint8),
              inst_scope=e32, scope_parent=e32, scope_kind=np.zeros(0, np.uint8), func_scope=e32,
              call_inst=e32, call_callee=e32)
    s = gpa.load_structure(st, 0)
    rng = np.random.default_rng(3)
    rec = np.zeros(1000, gen.RECORD_DTYPE)
    rec["pc"] = rng.integers(0, 2 ** 63, 1000)
    rec["count"] = 2
    rec["stall"] = rng.integers(0, 20, 1000)
    H = torch.zeros((1, 16), dtype=torch.int64, device=DEV)
    U = torch.zeros(16, dtype=torch.int64, device=DEV)
    gpa.attribute_samples(s, torch.from_numpy(rec.view(np.int64).reshape(-1, 2)).to(DEV), H, U)
    _, Uo, _ = oracle.attribute(st, rec)
    assert np.array_equal(u64(U), Uo) and u64(H).sum() == 0
    assert gpa.reconstruct_cct(s, H, max_contexts=0) == 0


# ---- a-5 + a-10 --------------------------------------------------------------------------------
@pytest.mark.parametrize("name,records", [("C1", 10_000), ("C2", 500_000), ("C3", 500_000), ("C5", 500_000)])
def test_rollup_and_derive_parity(gpa, name, records):
    w = gen.workload(name, records=records)
    st = w.structure
    s = gpa.load_structure(st, 0)
    H, _, _ = _attribute(gpa, s, _device_records(w), rec_inst=False)
    Ho = u64(H)
    for scope in ["INST", "LINE", "LOOP", "INLINE", "FUNC"]:
        rows = s.rows(scope)
        assert np.array_equal(rows, oracle.scope_rows(st, scope)), scope
        n = len(rows)
        hist = torch.full((max(n, 1), 16), -1, dtype=torch.int64, device=DEV)
        mix = torch.full((max(n, 1), 16), -1, dtype=torch.int64, device=DEV)
        met = torch.full((max(n, 1), 33), -7.0, dtype=torch.float64, device=DEV)
        gpa.derive_metrics(s, scope, H, scope_hist=hist, scope_mix=mix, metrics=met)
        torch.cuda.synchronize()
        eh, em = oracle.scope_hist(st, Ho, scope)
        assert np.array_equal(u64(hist)[:n], eh), scope
        assert np.array_equal(u64(mix)[:n], em), scope
        ed = oracle.derive_u64(eh, em)
        got = met.cpu().numpy()[:n]
        assert np.array_equal(np.isnan(got), np.isnan(ed)), scope
        assert np.allclose(got, ed, rtol=RTOL, atol=0, equal_nan=True), scope
        assert np.array_equal(got.view(np.uint64), ed.view(np.uint64)), scope      # bit-identical
        # metrics alone (no u64 outputs) give the same numbers
        met2 = torch.zeros_like(met)
        gpa.derive_metrics(s, scope, H, metrics=met2)
        assert torch.equal(met2[:n].view(torch.int64), met[:n].view(torch.int64))


# ---- a-6..a-10: CCT ----------------------------------------------------------------------------
def _cct_compare(gpa, s, st, H_np, bit_exact=True, exact=False):
    H = torch.from_numpy(H_np.view(np.int64)).to(DEV).reshape(-1, 16)
    mode = gpa.WEIGHTS_EXACT if exact else gpa.WEIGHTS_SAMPLES
    n_pred = gpa.reconstruct_cct(s, H, mode=mode, max_contexts=0)
    R = oracle.cct(st, H_np, exact=exact)
    assert n_pred == R["n"]
    c = gpa.reconstruct_cct(s, H, mode=mode)
    g = c.to_numpy()
    assert g["n"] == R["n"]
    for k in ["parent", "site", "node", "kind", "first_child", "n_children"]:
        assert np.array_equal(g[k], R[k]), k
    assert np.array_equal(g["call_weight"], R["w"])
    assert np.array_equal(g["dag_weight"], R["W"])
    assert np.array_equal(g["dag_active"], R["dag_active"])
    assert np.array_equal(g["func_active"], R["func_active"])
    assert np.array_equal(g["func_hist"], R["S_f"])
    assert np.array_equal(s.scc_of(), R["scc_of"])
    for k, o in [("frac", R["frac"]), ("excl", R["excl"]), ("incl", R["incl"])]:
        assert np.allclose(g[k], o, rtol=RTOL, atol=0), k
        if bit_exact:
            assert np.array_equal(g[k].view(np.uint64), o.view(np.uint64)), k
    for scope, V in [("CCT_EXCL", R["excl"]), ("CCT_INCL", R["incl"])]:
        met = torch.empty((max(R["n"], 1), 33), dtype=torch.float64, device=DEV)
        gpa.derive_metrics(s, scope, cct=c, metrics=met)
        got = met.cpu().numpy()[:R["n"]]
        ed = oracle.derive_f64(V)
        assert np.allclose(got, ed, rtol=RTOL, atol=0, equal_nan=True), scope
        if bit_exact:
            assert np.array_equal(got.view(np.uint64), ed.view(np.uint64)), scope
    c.free()
    return R


@pytest.mark.parametrize("name", ["cct_fig4_narrative.json", "cct_guard.json", "cct_diamond.json"])
def test_cct_golden(gpa, name):
    g = load_golden(name)
    st, H, _ = build_fixture(g["spec"])
    R = _cct_compare(gpa, gpa.load_structure(st, 0), st, H)
    assert R["n"] == len(g["expect"]["contexts"])


@pytest.mark.parametrize("case", ["apportion", "single", "chain", "nonzero", "self"])
def test_cct_spec_examples(gpa, case):
    g = load_golden("cct_spec_examples.json")["cases"][case]
    st, H, _ = build_fixture(g["spec"])
    _cct_compare(gpa, gpa.load_structure(st, 0), st, H)


@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("seed", range(40))
def test_cct_random_graphs(gpa, seed, exact):
    from tests.test_oracle_cct import _random_graph
    rng = np.random.default_rng(1000 + seed)
    st, H, _ = build_fixture(_random_graph(rng))
    _cct_compare(gpa, gpa.load_structure(st, 0), st, H, exact=exact)


def test_cct_exact_golden_and_block_counts(gpa):
    g = load_golden("cct_exact.json")
    st, H, _ = build_fixture(g["inconsistent"]["spec"])
    R = _cct_compare(gpa, gpa.load_structure(st, 0), st, H, exact=True)
    assert R["n"] == len(g["inconsistent"]["expect"]["contexts"])
    # instrumentation counts: basic blocks -> instructions, then an exact-mode CCT
    w = gen.workload("C3", records=10)
    s = gpa.load_structure(w.structure, 0)
    n_inst = s.info["n_inst"]
    rng = np.random.default_rng(9)
    cuts = np.sort(rng.choice(np.arange(1, n_inst), 20_000, replace=False))
    start = np.concatenate([[0], cuts, [n_inst]]).astype(np.uint32)
    cnt = rng.integers(0, 1000, len(start) - 1).astype(np.uint64)
    Ht = torch.zeros((n_inst, 16), dtype=torch.int64, device=DEV)
    gpa.block_counts(s, torch.from_numpy(start.view(np.int32)).to(DEV), torch.from_numpy(cnt.view(np.int64)).to(DEV), Ht)
    Ho = oracle.block_counts(n_inst, start, cnt)
    assert np.array_equal(u64(Ht), Ho)
    _cct_compare(gpa, s, w.structure, Ho, exact=True)


@pytest.mark.parametrize("name,records", [("C1", 10_000), ("C2", 1_000_000), ("C3", 2_000_000),
                                          ("C4", 2_000_000), ("C5", 2_000_000)])
def test_cct_workloads(gpa, name, records):
    w = gen.workload(name, records=records)
    s = gpa.load_structure(w.structure, 0)
    assert s.info["cct_path_bound"] == w.meta["static_contexts"]
    H, _, _ = _attribute(gpa, s, _device_records(w), rec_inst=False)
    R = _cct_compare(gpa, s, w.structure, u64(H))
    assert R["n"] > 0


def test_cct_capacity(gpa):
    g = load_golden("cct_fig4_narrative.json")
    st, H, _ = build_fixture(g["spec"])
    s = gpa.load_structure(st, 0)
    Ht = torch.from_numpy(H.view(np.int64)).to(DEV)
    with pytest.raises(gpa.GpaError) as ei:
        gpa.reconstruct_cct(s, Ht, max_contexts=5)
    assert ei.value.status == 3
    with pytest.raises(gpa.GpaError) as ei:
        gpa.reconstruct_cct(s, Ht, mode=5)
    assert ei.value.status == 1


# ---- every attribution kernel, and the u32 wrap repayment of the shared-memory rows -------------
@pytest.fixture
def attr_kernel(gpa):
    yield gpa.set_attr_kernel
    gpa.set_attr_kernel(0)


@pytest.mark.parametrize("kernel", [1, 2, 3, 4, 5, 6, 7, 8, 9])
@pytest.mark.parametrize("name,records", [("C2", 3_000_001), ("C3", 4_000_003), ("C5", 3_000_001)])
def test_attribution_each_kernel(gpa, attr_kernel, kernel, name, records):
    attr_kernel(kernel)
    w = gen.workload(name, records=records)
    s = gpa.load_structure(w.structure, 0)
    H, U, ri = _attribute(gpa, s, _device_records(w))
    Ho, Uo, rio = oracle.attribute(w.structure, w.records_host(), rec_inst=True)
    assert np.array_equal(u64(H), Ho) and np.array_equal(u64(U), Uo)
    assert np.array_equal(ri.cpu().numpy().view(np.uint32), rio)


@pytest.mark.parametrize("kernel", [1, 2, 3, 4, 5, 6, 7, 8, 9])
def test_attribution_huge_counts_exact(gpa, attr_kernel, kernel):
    """Counts near 2^32 make every shared u32 add wrap: the repaid 2^32 keeps H exact."""
    attr_kernel(kernel)
    w = gen.workload("C2" if kernel == 9 else "C3", records=2_200_000)  # 9: a structure it holds whole
    rec = w.records_host()
    rng = np.random.default_rng(5)
    rec["count"] = np.where(rng.random(len(rec)) < 0.5, 0xFFFFFFF0, rng.integers(1, 1 << 31, len(rec)))
    s = gpa.load_structure(w.structure, 0)
    H, U, _ = _attribute(gpa, s, torch.from_numpy(rec.view(np.int64).reshape(-1, 2)).to(DEV), rec_inst=False)
    Ho, Uo, _ = oracle.attribute(w.structure, rec)
    assert Ho.max() > 2 ** 40
    assert np.array_equal(u64(H), Ho) and np.array_equal(u64(U), Uo)


# ---- f1: per-profile histograms + cross-profile statistics --------------------------------------
@pytest.mark.parametrize("name,records,n_prof", [("C4", 3_000_001, 384), ("C4", 500_000, 100), ("C2", 1_000_000, 1),
                                                 ("C5", 200_000, 1)])
def test_profiles_parity(gpa, name, records, n_prof):
    w = gen.workload(name, records=records)
    s = gpa.load_structure(w.structure, 0)
    rec = _device_records(w)
    nf = s.info["n_func"]
    PH = torch.zeros((n_prof + 1, nf, 16), dtype=torch.int64, device=DEV)
    PU = torch.zeros((n_prof + 1, 16), dtype=torch.int64, device=DEV)
    gpa.attribute_profiles(s, rec, n_prof, PH, PU)
    stats = torch.empty((nf, 6, 16), dtype=torch.float64, device=DEV)
    gpa.profile_stats(s, PH, n_prof, stats)
    torch.cuda.synchronize()
    Hp, Up = oracle.attribute_profiles(w.structure, w.records_host(), n_prof)
    assert np.array_equal(u64(PH), Hp) and np.array_equal(u64(PU), Up)
    So = oracle.profile_stats(Hp, n_prof)
    got = stats.cpu().numpy()
    assert np.allclose(got, So, rtol=1e-9, atol=0)
    assert np.array_equal(got.view(np.uint64), So.view(np.uint64))       # bit-identical


def test_profile_stats_huge_values(gpa):
    """u128 sums of squares and the correctly rounded u128 -> double conversion."""
    rng = np.random.default_rng(2)
    n_prof, nf = 7, 25
    w = gen.workload("C2", records=10)
    s = gpa.load_structure(w.structure, 0)
    Hp = rng.integers(0, 2 ** 62, (n_prof + 1, nf, 16)).astype(np.uint64)
    Hp[:, 0, :] = 2 ** 62 + 12345                                          # equal values: std 0
    stats = torch.empty((nf, 6, 16), dtype=torch.float64, device=DEV)
    gpa.profile_stats(s, torch.from_numpy(Hp.view(np.int64)).to(DEV), n_prof, stats)
    So = oracle.profile_stats(Hp, n_prof)
    assert np.array_equal(stats.cpu().numpy().view(np.uint64), So.view(np.uint64))
    assert (So[0, 4] == 0).all()


@pytest.mark.parametrize("kernel", [3, 4, 5, 6, 7, 8, 9])
def test_attribution_shared_counter_overflow_patterns(gpa, attr_kernel, kernel):
    """Hot bins receive counts that drive 16- and 32-bit shared counters through many
    overflows (incl. carries between packed halves, counts of exactly 0xFFFF / 0x10000)."""
    attr_kernel(kernel)
    w = gen.workload("C2" if kernel == 9 else "C4", records=3_000_000)
    rec = w.records_host()
    rng = np.random.default_rng(8)
    choices = np.array([1, 0xFFFF, 0x10000, 0x7FFF, 0xFFFE, 2 ** 31, 0xFFFFFFFF], np.uint64)
    rec["count"] = np.where(rng.random(len(rec)) < 0.3, choices[rng.integers(0, len(choices), len(rec))],
                            rng.integers(1, 70000, len(rec)))
    s = gpa.load_structure(w.structure, 0)
    H, U, _ = _attribute(gpa, s, torch.from_numpy(rec.view(np.int64).reshape(-1, 2)).to(DEV), rec_inst=False)
    Ho, Uo, _ = oracle.attribute(w.structure, rec)
    assert np.array_equal(u64(H), Ho) and np.array_equal(u64(U), Uo)


# ---- f1 at instruction and CCT level ------------------------------------------------------------
@pytest.mark.parametrize("name,records,n_prof", [("C2", 2_000_000, 5), ("C4", 1_000_003, 64), ("C1", 1000, 0),
                                                 ("C4", 6_000_011, 48), ("C3", 4_500_001, 7), ("C5", 5_000_003, 3)])
def test_profiles_inst_parity(gpa, name, records, n_prof):
    w = gen.workload(name, records=records)
    s = gpa.load_structure(w.structure, 0)
    rec = _device_records(w)
    ni = s.info["n_inst"]
    PH = torch.zeros((n_prof + 1, ni, 16), dtype=torch.int64, device=DEV)
    PU = torch.zeros((n_prof + 1, 16), dtype=torch.int64, device=DEV)
    gpa.attribute_profiles_inst(s, rec, n_prof, PH, PU)
    stats = torch.empty((ni, 6, 16), dtype=torch.float64, device=DEV)
    gpa.profile_stats_rows(PH, n_prof, stats)
    torch.cuda.synchronize()
    Hp, Up = oracle.attribute_profiles_inst(w.structure, w.records_host(), n_prof)
    assert np.array_equal(u64(PH), Hp) and np.array_equal(u64(PU), Up)
    So = oracle.profile_stats(Hp, n_prof)
    assert np.array_equal(stats.cpu().numpy().view(np.uint64), So.view(np.uint64))


def test_profiles_inst_carries_exact(gpa):
    """Large calls count the current profile's hot bins in shared byte counters: counts of 128-255
    overflow a byte every one or two records, and the carries are repaid in the cube directly."""
    w = gen.workload("C5", records=4_400_007)
    rec = w.records_host()
    rng = np.random.default_rng(11)
    rec["count"] = np.where(rng.random(len(rec)) < 0.9, rng.integers(128, 256, len(rec)), rec["count"])
    s = gpa.load_structure(w.structure, 0)
    ni, n_prof = s.info["n_inst"], 2
    PH = torch.zeros((n_prof + 1, ni, 16), dtype=torch.int64, device=DEV)
    PU = torch.zeros((n_prof + 1, 16), dtype=torch.int64, device=DEV)
    gpa.attribute_profiles_inst(s, torch.from_numpy(rec.view(np.int64).reshape(-1, 2)).to(DEV), n_prof, PH, PU)
    torch.cuda.synchronize()
    Hp, Up = oracle.attribute_profiles_inst(w.structure, rec, n_prof)
    assert np.array_equal(u64(PH), Hp) and np.array_equal(u64(PU), Up)


@pytest.mark.parametrize("name,records,n_prof", [("C4", 2_000_000, 48), ("C3", 3_000_000, 3), ("C2", 500_000, 1)])
def test_cct_profiles_parity(gpa, name, records, n_prof):
    w = gen.workload(name, records=records)
    s = gpa.load_structure(w.structure, 0)
    rec = _device_records(w)
    H = torch.zeros((s.info["n_inst"], 16), dtype=torch.int64, device=DEV)
    U = torch.zeros(16, dtype=torch.int64, device=DEV)
    gpa.attribute_samples(s, rec, H, U)
    nf = s.info["n_func"]
    PH = torch.zeros((n_prof + 1, nf, 16), dtype=torch.int64, device=DEV)
    PU = torch.zeros((n_prof + 1, 16), dtype=torch.int64, device=DEV)
    gpa.attribute_profiles(s, rec, n_prof, PH, PU)
    c = gpa.reconstruct_cct(s, H)
    n = c.n
    E = torch.empty((n_prof + 1, n, 16), dtype=torch.float64, device=DEV)
    I = torch.empty_like(E)
    gpa.cct_profiles(s, c, PH, n_prof, E, I)
    stats = torch.empty((n, 6, 16), dtype=torch.float64, device=DEV)
    gpa.profile_stats_f64(I, n_prof, stats)
    torch.cuda.synchronize()
    R = oracle.cct(w.structure, u64(H))
    Eo, Io = oracle.cct_profiles(R, u64(PH))
    assert np.array_equal(E.cpu().numpy().view(np.uint64), Eo.view(np.uint64))
    assert np.array_equal(I.cpu().numpy().view(np.uint64), Io.view(np.uint64))
    So = oracle.profile_stats_f64(Io, n_prof)
    got = stats.cpu().numpy()
    np.testing.assert_allclose(got, So, rtol=1e-9, atol=0)
    assert np.array_equal(got.view(np.uint64), So.view(np.uint64))
    c.free()


def test_f1_invalid_args(gpa):
    w = gen.workload("C2", records=1000)
    s = gpa.load_structure(w.structure, 0)
    rec = _device_records(w)
    ni, nf = s.info["n_inst"], s.info["n_func"]
    with pytest.raises(gpa.GpaError):                  # instruction cube too small
        gpa.attribute_profiles_inst(s, rec, 4, torch.zeros((2, ni, 16), dtype=torch.int64, device=DEV),
                                    torch.zeros((5, 16), dtype=torch.int64, device=DEV))
    with pytest.raises(gpa.GpaError):                  # unaligned records
        gpa.attribute_profiles_inst(s, rec.view(-1)[1:-1], 1,
                                    torch.zeros((2, ni, 16), dtype=torch.int64, device=DEV),
                                    torch.zeros((2, 16), dtype=torch.int64, device=DEV), n=10)
    H = torch.zeros((ni, 16), dtype=torch.int64, device=DEV)
    U = torch.zeros(16, dtype=torch.int64, device=DEV)
    gpa.attribute_samples(s, rec, H, U)
    c = gpa.reconstruct_cct(s, H)
    PH = torch.zeros((3, nf, 16), dtype=torch.int64, device=DEV)
    with pytest.raises(gpa.GpaError):                  # outputs too small for the tree
        gpa.cct_profiles(s, c, PH, 2, torch.empty((1, 1, 16), dtype=torch.float64, device=DEV),
                         torch.empty((1, 1, 16), dtype=torch.float64, device=DEV))
    c.free()
    with pytest.raises(gpa.GpaError):
        gpa.profile_stats_f64(torch.zeros((2, 4, 16), dtype=torch.float64, device=DEV), 3,
                              torch.empty((4, 6, 16), dtype=torch.float64, device=DEV))


# ---- reusable attribution plans and the host-records path --------------------------------------
@pytest.mark.parametrize("name", ["C2", "C3", "C5"])
def test_attr_plan_reuse_exact(gpa, name):
    """A plan built from one batch serves other batches (and a batch from another part of the
    stream): results equal the oracle bit for bit, whatever the plan."""
    w = gen.workload(name, records=6_000_000)
    s = gpa.load_structure(w.structure, 0)
    first = _device_records(w, 0, 2_000_000)
    plan = gpa.AttrPlan(s, first)
    assert plan.variant in (7, 8, 9)
    for k0, n in [(2_000_000, 3_999_999), (0, 2_000_000), (5_999_000, 1000)]:
        rec = _device_records(w, k0, n)
        H = torch.zeros((s.info["n_inst"], 16), dtype=torch.int64, device=DEV)
        U = torch.zeros(16, dtype=torch.int64, device=DEV)
        ri = torch.empty(n, dtype=torch.int32, device=DEV)
        plan.attribute(rec, H, U, ri)
        torch.cuda.synchronize()
        Ho, Uo, rio = oracle.attribute(w.structure, w.records_host(k0, n), rec_inst=True)
        assert np.array_equal(u64(H), Ho) and np.array_equal(u64(U), Uo), (k0, n)
        assert np.array_equal(ri.cpu().numpy().view(np.uint32), rio)
    plan.free()


@pytest.mark.parametrize("name", ["C2", "C4"])
@pytest.mark.parametrize("pinned", [True, False])
def test_host_path_many_chunks(gpa, pinned, name):
    """gpa_attribute_samples_host over more than 3 x 2^22 + 17 records (several passes of the
    3-buffer staging rotation and a ragged last chunk, one plan for the whole call), pinned and
    pageable host memory."""
    n = 3 * (1 << 22) + 17 + 1_000_003
    w = gen.workload(name, records=n)
    s = gpa.load_structure(w.structure, 0)
    host = torch.empty((n, 2), dtype=torch.int64, pin_memory=pinned)
    w.records_host(0, n, out=host.numpy().view(gen.RECORD_DTYPE).reshape(-1))
    H = torch.zeros((s.info["n_inst"], 16), dtype=torch.int64, device=DEV)
    U = torch.zeros(16, dtype=torch.int64, device=DEV)
    gpa.attribute_samples_host(s, host, H, U)
    torch.cuda.synchronize()
    Ho, Uo, _ = oracle.attribute(w.structure, host.numpy().view(gen.RECORD_DTYPE).reshape(-1),
                                 threads=len(__import__("os").sched_getaffinity(0)))
    assert np.array_equal(u64(H), Ho) and np.array_equal(u64(U), Uo)


@pytest.mark.parametrize("kernel", [7, 8, 9])
@pytest.mark.parametrize("stress", [1, 8])
def test_ring_stress_exact(gpa, attr_kernel, kernel, stress):
    """Adversarial TMA-ring timing (gpa_set_ring_stress: random producer and consumer sleeps, so
    the producer runs ahead of slow consumers and consumers wait on refills): a stage refilled
    before every consumer read it would corrupt H; the result stays bit-exact."""
    attr_kernel(kernel)
    gpa.set_ring_stress(stress)
    try:
        w = gen.workload({7: "C4", 8: "C5", 9: "C2"}[kernel], records=4_200_007)
        s = gpa.load_structure(w.structure, 0)
        H, U, ri = _attribute(gpa, s, _device_records(w))
    finally:
        gpa.set_ring_stress(0)
    Ho, Uo, rio = oracle.attribute(w.structure, w.records_host(), rec_inst=True)
    assert np.array_equal(u64(H), Ho) and np.array_equal(u64(U), Uo)
    assert np.array_equal(ri.cpu().numpy().view(np.uint32), rio)


def test_scratch_reuse_across_streams(gpa):
    """Consecutive attribution calls on one structure reuse its scratch block (ScratchCache); calls
    alternating between two streams (the second waits on the first's event) and a call from a
    second host thread while one is being enqueued stay bit-exact."""
    import threading
    w = gen.workload("C2", records=3_000_000)
    s = gpa.load_structure(w.structure, 0)
    rec = _device_records(w)
    Ho, Uo, _ = oracle.attribute(w.structure, w.records_host())
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    for i in range(6):
        H = torch.zeros((s.info["n_inst"], 16), dtype=torch.int64, device=DEV)
        U = torch.zeros(16, dtype=torch.int64, device=DEV)
        st = streams[i % 2]
        st.wait_stream(torch.cuda.current_stream())
        gpa.attribute_samples(s, rec, H, U, stream=st)
        outs.append((H, U))
    errs = []

    def worker():
        try:
            H = torch.zeros((s.info["n_inst"], 16), dtype=torch.int64, device=DEV)
            U = torch.zeros(16, dtype=torch.int64, device=DEV)
            st = torch.cuda.Stream()
            st.wait_stream(torch.cuda.current_stream())
            gpa.attribute_samples(s, rec, H, U, stream=st)
            st.synchronize()
            outs.append((H, U))
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ths = [threading.Thread(target=worker) for _ in range(3)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    torch.cuda.synchronize()
    assert not errs
    for H, U in outs:
        assert np.array_equal(u64(H), Ho) and np.array_equal(u64(U), Uo)
