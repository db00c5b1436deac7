"""f3 GPU parity: gpa_sparse_build (PMS / CMS, §5.2) against oracle D9 on
the same cubes, every array bit-exact — random cubes over the density range, the degenerate
cubes (all zero, all dense, one profile row, one function row) and the per-profile cube the
f1 path produces from a full C4 record stream."""
import numpy as np
import pytest

import gen
import oracle
from tests.sparse_util import decode

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
DEV = "cuda:0"
KEYS = ("plane_off", "index_off", "vals", "ids", "index_start", "index_id")


@pytest.fixture(scope="module")
def gpa():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__
    __graft_entry__.build()
    from paper_2109_06931_b200 import gpa
    return gpa


def _check(gpa, s, Hp, cms):
    P = Hp.shape[0] - 1
    sp = gpa.sparse_build(s, torch.from_numpy(Hp.view(np.int64)).to(DEV), P, cms)
    got = sp.to_numpy()
    exp = oracle.sparse_build(Hp, cms)
    for k in ("n_planes", "n_values", "n_index"):
        assert got[k] == exp[k], k
    for k in KEYS:
        assert np.array_equal(got[k], exp[k]), k
    assert np.array_equal(decode(got, Hp.shape[0], Hp.shape[1], cms), Hp)
    sp.free()


@pytest.mark.parametrize("cms", [False, True])
@pytest.mark.parametrize("name,n_prof,density", [("C1", 0, 0.3), ("C2", 9, 0.0), ("C2", 9, 1.0), ("C2", 33, 0.02),
                                                 ("C4", 100, 0.05), ("C3", 64, 0.001), ("C5", 31, 0.01)])
def test_sparse_random_cubes(gpa, cms, name, n_prof, density):
    rng = np.random.default_rng(n_prof * 7 + int(density * 1000))
    w = gen.workload(name, records=1)
    s = gpa.load_structure(w.structure, 0)
    nf = s.info["n_func"]
    Hp = np.where(rng.random((n_prof + 1, nf, 16)) < density,
                  rng.integers(1, 2 ** 63, (n_prof + 1, nf, 16), dtype=np.uint64), 0).astype(np.uint64)
    _check(gpa, s, Hp, cms)


@pytest.mark.parametrize("cms", [False, True])
def test_sparse_from_profiles(gpa, cms):
    w = gen.workload("C4", records=2_000_003)
    s = gpa.load_structure(w.structure, 0)
    n_prof = 96
    rec = torch.empty((w.cfg.records, 2), dtype=torch.int64, device=DEV)
    w.records_device(rec, 0, w.cfg.records)
    PH = torch.zeros((n_prof + 1, s.info["n_func"], 16), dtype=torch.int64, device=DEV)
    PU = torch.zeros((n_prof + 1, 16), dtype=torch.int64, device=DEV)
    gpa.attribute_profiles(s, rec, n_prof, PH, PU)
    sp = gpa.sparse_build(s, PH, n_prof, cms)
    got = sp.to_numpy()
    Hp, _ = oracle.attribute_profiles(w.structure, w.records_host(), n_prof)
    exp = oracle.sparse_build(Hp, cms)
    for k in KEYS:
        assert np.array_equal(got[k], exp[k]), k
    assert 0 < got["n_values"] < Hp.size


def test_sparse_single_function_row(gpa):
    st = dict(inst_addr=np.array([0x100], np.uint64), inst_len=np.array([16], np.uint16),
              inst_class=np.zeros(1, np.uint8), inst_scope=np.array([1], np.uint32),
              scope_parent=np.array([0xFFFFFFFF, 0], np.uint32), scope_kind=np.array([0, 3], np.uint8),
              func_scope=np.array([0], np.uint32), call_inst=np.zeros(0, np.uint32),
              call_callee=np.zeros(0, np.uint32))
    s = gpa.load_structure(st, 0)
    Hp = np.zeros((5, 1, 16), np.uint64)
    Hp[2, 0, 15] = 7
    Hp[4, 0, 0] = 2 ** 64 - 1
    for cms in (False, True):
        _check(gpa, s, Hp, cms)


def test_sparse_invalid_args(gpa):
    w = gen.workload("C1", records=1)
    s = gpa.load_structure(w.structure, 0)
    PH = torch.zeros((3, s.info["n_func"], 16), dtype=torch.int64, device=DEV)
    with pytest.raises(gpa.GpaError):                  # buffer too small for 5 profiles
        gpa.sparse_build(s, PH, 5, True)
    import ctypes
    from paper_2109_06931_b200.gpa import _lib
    h = ctypes.c_void_p()
    assert _lib.gpa_sparse_build(s.handle, PH.data_ptr(), 2, 7, ctypes.byref(h), None) != 0   # bad major
    assert _lib.gpa_sparse_build(None, PH.data_ptr(), 2, 0, ctypes.byref(h), None) != 0       # NULL structure
