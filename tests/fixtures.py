"""Hand-written structures for golden tests (test helper, no method arithmetic).

A fixture spec names functions (each with a number of instructions and per-instruction
samples) and call sites (caller, instruction index inside the caller, callee).  It is
turned into gpa_structure_desc arrays plus a per-instruction histogram H:
  * function f occupies instructions laid out at 0x1000 + 0x100*f, 16 B each;
  * one FUNCTION scope per function, one LINE scope per instruction (unless the spec gives
    an explicit scope tree);
  * samples: {"<inst>": count} puts count in slot 0 (issued), or {"<inst>": {"<slot>": c}}.
"""
from __future__ import annotations

import json
import os
from fractions import Fraction

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NONE = 0xFFFFFFFF


def load_golden(name: str) -> dict:
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def build(spec: dict):
    funcs = spec["functions"]
    names = [f["name"] for f in funcs]
    idx = {n: i for i, n in enumerate(names)}
    inst_addr, inst_scope, scope_parent, scope_kind, func_scope = [], [], [], [], []
    first = []
    for fi, f in enumerate(funcs):
        scope_parent.append(NONE)
        scope_kind.append(0)
        fs = len(scope_parent) - 1
        func_scope.append(fs)
        first.append(len(inst_addr))
        for k in range(f["n_inst"]):
            inst_addr.append(0x1000 + 0x100 * fi + 16 * k)
            scope_parent.append(fs)
            scope_kind.append(3)
            inst_scope.append(len(scope_parent) - 1)
    n = len(inst_addr)
    H = np.zeros((n, 16), np.uint64)
    for fi, f in enumerate(funcs):
        for k, v in f.get("samples", {}).items():
            i = first[fi] + int(k)
            if isinstance(v, dict):
                for slot, c in v.items():
                    H[i, int(slot)] += c
            else:
                H[i, 0] += v
    calls = sorted(((first[idx[c]] + int(k), idx[v]) for c, k, v in spec.get("calls", [])))
    st = dict(inst_addr=np.array(inst_addr, np.uint64), inst_len=np.full(n, 16, np.uint16),
              inst_class=np.zeros(n, np.uint8), inst_scope=np.array(inst_scope, np.uint32),
              scope_parent=np.array(scope_parent, np.uint32), scope_kind=np.array(scope_kind, np.uint8),
              func_scope=np.array(func_scope, np.uint32),
              call_inst=np.array([c for c, _ in calls], np.uint32),
              call_callee=np.array([v for _, v in calls], np.uint32))
    for i, _ in calls:
        st["inst_class"][i] = 14
    return st, H, idx


def frac(s) -> Fraction:
    return Fraction(str(s))
