"""CPU-side checks of the C-ABI boundary: libgpa.so loads, exports every entry point
include/gpa.h declares, and its host-only structure validation rejects each malformed
description gpa.h lists (no device is touched).  The product never falls back to the CPU:
without a GPU the device entry points return GPA_ERR_CUDA / raise."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import gen
from tests.fixtures import build as build_fixture, load_golden

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gpa.h")


@pytest.fixture(scope="module")
def gpa():
    import __graft_entry__
    __graft_entry__.build_lib()
    from paper_2109_06931_b200 import gpa
    return gpa


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"GPA_API\s+[\w\s\*]*?\b(gpa_\w+)\s*\(", txt)))


def test_exports_every_declared_symbol(gpa):
    names = _declared()
    assert len(names) >= 14
    lib = ctypes.CDLL(gpa.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    nm = subprocess.run(["nm", "-D", "--defined-only", gpa.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (gpa_\w+)", nm))
    assert set(names) == exported, (set(names) ^ exported)
    assert gpa.version().startswith("libgpa")


def test_library_is_sm100a_only(gpa):
    out = subprocess.run(["cuobjdump", "--list-elf", gpa.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def _valid():
    st, _, _ = build_fixture(load_golden("cct_fig4_narrative.json")["spec"])
    return {k: np.array(v) for k, v in st.items()}


def test_validate_accepts_generated_structures(gpa):
    for name in ["C1", "C2", "C3"]:
        gpa.validate_structure(gen.workload(name).structure)
    gpa.validate_structure(_valid())


def _mutations():
    m = {}

    def mut(name, f):
        d = _valid()
        f(d)
        m[name] = d

    mut("unsorted", lambda d: d["inst_addr"].__setitem__(slice(0, 2), d["inst_addr"][1::-1].copy()))
    mut("overlap", lambda d: d["inst_len"].__setitem__(0, 17))
    mut("zero_len", lambda d: d["inst_len"].__setitem__(3, 0))
    mut("overflow", lambda d: (d["inst_addr"].__setitem__(-1, 2 ** 64 - 8)))
    mut("class", lambda d: d["inst_class"].__setitem__(0, 16))
    mut("inst_scope_not_line", lambda d: d["inst_scope"].__setitem__(0, 0))
    mut("inst_scope_range", lambda d: d["inst_scope"].__setitem__(0, 10 ** 6))
    mut("kind", lambda d: d["scope_kind"].__setitem__(1, 4))
    mut("line_parent", lambda d: d["scope_parent"].__setitem__(2, 1))
    mut("function_with_parent", lambda d: d["scope_parent"].__setitem__(0, 1))
    mut("orphan_scope", lambda d: d["scope_parent"].__setitem__(1, 0xFFFFFFFF))
    mut("parent_range", lambda d: d["scope_parent"].__setitem__(1, 10 ** 6))
    mut("func_scope_dup", lambda d: d["func_scope"].__setitem__(1, d["func_scope"][0]))
    mut("func_scope_not_function", lambda d: d["func_scope"].__setitem__(0, 1))
    mut("call_inst_range", lambda d: d["call_inst"].__setitem__(0, 10 ** 6))
    mut("call_callee_range", lambda d: d["call_callee"].__setitem__(0, 99))
    mut("call_dup", lambda d: d["call_inst"].__setitem__(1, d["call_inst"][0]))

    # cycle among non-function scopes: INLINE a -> LOOP b -> a
    def cyc(d):
        n = len(d["scope_parent"])
        d["scope_parent"] = np.concatenate([d["scope_parent"], [n + 1, n]]).astype(np.uint32)
        d["scope_kind"] = np.concatenate([d["scope_kind"], [1, 2]]).astype(np.uint8)
    mut("cycle", cyc)
    return m


@pytest.mark.parametrize("case", sorted(_mutations()))
def test_validate_rejects_malformed(gpa, case):
    d = _mutations()[case]
    with pytest.raises(gpa.GpaError) as ei:
        gpa.validate_structure(d)
    assert ei.value.status == 2, str(ei.value)


def test_validate_accepts_degenerate_empty(gpa):
    e32, e64 = np.zeros(0, np.uint32), np.zeros(0, np.uint64)
    d = dict(inst_addr=e64, inst_len=np.zeros(0, np.uint16), inst_class=np.zeros(0, np.uint8), inst_scope=e32,
             scope_parent=e32, scope_kind=np.zeros(0, np.uint8), func_scope=e32, call_inst=e32, call_callee=e32)
    gpa.validate_structure(d)


def test_no_cpu_fallback(gpa):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(gpa.GpaError) as ei:
        gpa.load_structure(_valid(), 0)
    assert ei.value.status in (1, 5)
