"""CPU oracle for the PC-sample attribution path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs
may import this package.  The product (paper_2109_06931_b200) never does, and the two
share no code: this is a ctypes wrapper over oracle/gpa_oracle.c, a plain C transcription
of the paper's definitions (D1-D7, see that file's header and DESIGN.md §3).

Structures are dicts of numpy arrays with the keys of gpa_structure_desc
(inst_addr, inst_len, inst_class, inst_scope, scope_parent, scope_kind, func_scope,
call_inst, call_callee); records are 16-byte (pc u64, count u32, stall u16, stream u16).
"""
from __future__ import annotations

import ctypes
import functools
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "gpa_oracle.c")
NONE = 0xFFFFFFFF
SLOTS, VALID, NCOLS = 16, 12, 33
KIND_FUNCTION, KIND_INLINE, KIND_LOOP, KIND_LINE = 0, 1, 2, 3

_u64p = ctypes.POINTER(ctypes.c_uint64)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_f64p = ctypes.POINTER(ctypes.c_double)


class _Sparse(ctypes.Structure):
    _fields_ = [("n_planes", ctypes.c_uint32), ("n_values", ctypes.c_uint64), ("n_index", ctypes.c_uint64),
                ("plane_off", _u64p), ("index_off", _u64p), ("vals", _u64p), ("index_start", _u64p),
                ("ids", _u32p), ("index_id", _u32p)]


class _CctResult(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_uint64), ("cap", ctypes.c_uint64),
        ("parent", _u32p), ("site", _u32p), ("node", _u32p), ("first_child", _u32p),
        ("n_children", _u32p), ("kind", _u8p), ("frac", _f64p), ("excl", _f64p), ("incl", _f64p),
        ("n_func", ctypes.c_uint32), ("n_call", ctypes.c_uint32), ("n_dag", ctypes.c_uint32),
        ("w_step1", _u64p), ("w", _u64p), ("func_active", _u8p), ("S_f", _u64p),
        ("scc_of", _u32p), ("dag_nontrivial", _u8p), ("dag_active", _u8p), ("W", _u64p),
        ("status", ctypes.c_int),
    ]


def build(force: bool = False) -> str:
    """Compile the oracle (gcc -O2 -ffp-contract=off: one IEEE op per written operation)."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(SRC) > os.path.getmtime(LIB_PATH):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-std=c11", "-shared", "-fPIC",
                               "-o", LIB_PATH, SRC, "-lpthread"])
    return LIB_PATH


@functools.lru_cache(None)
def _lib():
    build()
    lib = ctypes.CDLL(LIB_PATH)
    vp, u32, u64 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64
    lib.oracle_attribute.argtypes = [u32, vp, vp, vp, u64, vp, vp, vp]
    lib.oracle_attribute.restype = None
    lib.oracle_attribute_mt.argtypes = [u32, vp, vp, vp, u64, vp, vp, ctypes.c_int]
    lib.oracle_attribute_mt.restype = ctypes.c_int
    lib.oracle_rollup.argtypes = [u32, vp, vp, u32, vp, vp, vp, vp]
    lib.oracle_rollup.restype = None
    lib.oracle_inst_func.argtypes = [u32, vp, u32, vp, u32, vp, vp]
    lib.oracle_inst_func.restype = None
    lib.oracle_cct_mode.argtypes = [u32, vp, u32, vp, u32, vp, u32, vp, vp, vp, u64, ctypes.c_int]
    lib.oracle_cct_mode.restype = ctypes.POINTER(_CctResult)
    lib.oracle_attribute_profiles.argtypes = [u32, vp, vp, vp, u32, vp, u64, u32, vp, vp]
    lib.oracle_attribute_profiles.restype = None
    lib.oracle_profile_stats.argtypes = [u32, u32, vp, vp]
    lib.oracle_profile_stats.restype = None
    lib.oracle_sparse_build.argtypes = [vp, u32, u32, ctypes.c_int]
    lib.oracle_sparse_build.restype = ctypes.POINTER(_Sparse)
    lib.oracle_sparse_free.argtypes = [ctypes.POINTER(_Sparse)]
    lib.oracle_sparse_free.restype = None
    lib.oracle_block_counts.argtypes = [u32, vp, vp, vp]
    lib.oracle_block_counts.restype = None
    lib.oracle_cct_free.argtypes = [ctypes.POINTER(_CctResult)]
    lib.oracle_cct_free.restype = None
    lib.oracle_derive_u64.argtypes = [u64, vp, vp, vp]
    lib.oracle_derive_u64.restype = None
    lib.oracle_derive_f64.argtypes = [u64, vp, vp]
    lib.oracle_derive_f64.restype = None
    lib.oracle_cct_profiles.argtypes = [u64, vp, vp, vp, vp, u32, u32, vp, vp, vp]
    lib.oracle_cct_profiles.restype = None
    lib.oracle_profile_stats_f64.argtypes = [u32, u64, vp, vp]
    lib.oracle_profile_stats_f64.restype = None
    lib.oracle_blame.argtypes = [u32, vp, vp, vp, vp, vp, u32, u32, u32, vp, vp, vp, vp, vp]
    lib.oracle_blame.restype = ctypes.c_int
    return lib


def _c(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a, (a.ctypes.data if a.size else None)


def _records(rec) -> np.ndarray:
    rec = np.ascontiguousarray(rec)
    if rec.dtype.itemsize != 16:
        raise ValueError("records must be 16-byte items")
    return rec


# ---- D1 ---------------------------------------------------------------------------------
def attribute(st: dict, rec, rec_inst: bool = False, threads: int = 1):
    """D1: returns (H [n_inst,16] u64, U [16] u64, rec_inst [n] u32 or None)."""
    rec = _records(rec)
    n_inst = len(st["inst_addr"])
    addr, pa = _c(st["inst_addr"], np.uint64)
    ln, pl = _c(st["inst_len"], np.uint16)
    H = np.zeros((n_inst, SLOTS), np.uint64)
    U = np.zeros(SLOTS, np.uint64)
    ri = np.empty(len(rec), np.uint32) if rec_inst else None
    if threads > 1 and not rec_inst:
        _lib().oracle_attribute_mt(n_inst, pa, pl, rec.ctypes.data if len(rec) else None, len(rec),
                                   H.ctypes.data, U.ctypes.data, threads)
    else:
        _lib().oracle_attribute(n_inst, pa, pl, rec.ctypes.data if len(rec) else None, len(rec),
                                H.ctypes.data, U.ctypes.data, ri.ctypes.data if ri is not None and len(rec) else None)
    return H, U, ri


# ---- D2 ---------------------------------------------------------------------------------
def rollup(st: dict, H):
    """D2: per-scope inclusive histograms and sample-weighted class mix, by scope id."""
    n_inst, n_scope = len(st["inst_addr"]), len(st["scope_parent"])
    Hc, ph = _c(H, np.uint64)
    Hs = np.zeros((n_scope, SLOTS), np.uint64)
    MIX = np.zeros((n_scope, SLOTS), np.uint64)
    a_s, ps = _c(st["inst_scope"], np.uint32)
    a_c, pc = _c(st["inst_class"], np.uint8)
    a_p, pp = _c(st["scope_parent"], np.uint32)
    _lib().oracle_rollup(n_inst, ps, pc, n_scope, pp, ph, Hs.ctypes.data if n_scope else None,
                         MIX.ctypes.data if n_scope else None)
    return Hs, MIX


def inst_func(st: dict) -> np.ndarray:
    n_inst = len(st["inst_addr"])
    out = np.empty(n_inst, np.uint32)
    a = [_c(st[k], np.uint32) for k in ("inst_scope", "scope_parent", "func_scope")]
    _lib().oracle_inst_func(n_inst, a[0][1], len(st["scope_parent"]), a[1][1], len(st["func_scope"]),
                            a[2][1], out.ctypes.data if n_inst else None)
    return out


def scope_rows(st: dict, scope: str) -> np.ndarray:
    """Row ids of a scope set: 'INST' instruction ids, 'LINE'/'LOOP'/'INLINE' ascending scope
    ids of that kind, 'FUNC' function ids (the row order gpa_derive_metrics documents)."""
    kinds = {"LINE": KIND_LINE, "LOOP": KIND_LOOP, "INLINE": KIND_INLINE}
    if scope == "INST":
        return np.arange(len(st["inst_addr"]), dtype=np.uint32)
    if scope == "FUNC":
        return np.arange(len(st["func_scope"]), dtype=np.uint32)
    return np.nonzero(np.asarray(st["scope_kind"]) == kinds[scope])[0].astype(np.uint32)


def scope_hist(st: dict, H, scope: str):
    """(hist [rows,16], mix [rows,16]) of a scope set, from D2 (INST rows: H itself and the
    per-instruction class mix)."""
    H = np.asarray(H, np.uint64)
    if scope == "INST":
        S = H[:, :VALID].sum(1, dtype=np.uint64)
        mix = np.zeros_like(H)
        mix[np.arange(len(H)), np.asarray(st["inst_class"], np.int64)] = S
        return H.copy(), mix
    Hs, MIX = rollup(st, H)
    ids = scope_rows(st, scope)
    if scope == "FUNC":
        ids = np.asarray(st["func_scope"], np.int64)
    return Hs[ids], MIX[ids]


# ---- D3-D6 ------------------------------------------------------------------------------
def cct(st: dict, H, max_contexts: int = (1 << 63), exact: bool = False) -> dict:
    """D3-D6: the approximate GPU CCT (BFS numbering) and the Step 1-3 intermediates.
    exact=True: H holds exact execution counts; Step 2 and the guard are skipped (R24)."""
    n_inst, n_scope = len(st["inst_addr"]), len(st["scope_parent"])
    n_func, n_call = len(st["func_scope"]), len(st["call_inst"])
    a = {k: _c(st[k], np.uint32) for k in ("inst_scope", "scope_parent", "func_scope", "call_inst", "call_callee")}
    Hc, ph = _c(H, np.uint64)
    r = _lib().oracle_cct_mode(n_inst, a["inst_scope"][1], n_scope, a["scope_parent"][1], n_func,
                               a["func_scope"][1], n_call, a["call_inst"][1], a["call_callee"][1], ph, max_contexts,
                               1 if exact else 0)
    try:
        R = r.contents
        n, nd = int(R.n), int(R.n_dag)

        def arr(p, cnt, dt):
            if cnt == 0:
                return np.zeros(0, dt)
            return np.ctypeslib.as_array(p, shape=(cnt,)).astype(dt, copy=True)

        out = dict(
            n=n, status=int(R.status), n_dag=nd,
            parent=arr(R.parent, n, np.uint32), site=arr(R.site, n, np.uint32), node=arr(R.node, n, np.uint32),
            kind=arr(R.kind, n, np.uint8), first_child=arr(R.first_child, n, np.uint32),
            n_children=arr(R.n_children, n, np.uint32), frac=arr(R.frac, n, np.float64),
            excl=arr(R.excl, n * SLOTS, np.float64).reshape(n, SLOTS),
            incl=arr(R.incl, n * SLOTS, np.float64).reshape(n, SLOTS),
            w_step1=arr(R.w_step1, n_call, np.uint64), w=arr(R.w, n_call, np.uint64),
            func_active=arr(R.func_active, n_func, np.uint8),
            S_f=arr(R.S_f, n_func * SLOTS, np.uint64).reshape(n_func, SLOTS),
            scc_of=arr(R.scc_of, n_func, np.uint32), dag_nontrivial=arr(R.dag_nontrivial, nd, np.uint8),
            dag_active=arr(R.dag_active, nd, np.uint8), W=arr(R.W, nd, np.uint64))
    finally:
        _lib().oracle_cct_free(r)
    return out


def attribute_profiles(st: dict, rec, n_prof: int):
    """D8: per-profile function histograms Hp [n_prof+1, n_func, 16] and unattributed
    Up [n_prof+1, 16] (row n_prof collects stream ids >= n_prof)."""
    rec = _records(rec)
    n_inst, n_func = len(st["inst_addr"]), len(st["func_scope"])
    addr, pa = _c(st["inst_addr"], np.uint64)
    ln, pl = _c(st["inst_len"], np.uint16)
    ifn, pf = _c(inst_func(st), np.uint32)
    Hp = np.zeros((n_prof + 1, n_func, SLOTS), np.uint64)
    Up = np.zeros((n_prof + 1, SLOTS), np.uint64)
    if len(rec):
        _lib().oracle_attribute_profiles(n_inst, pa, pl, pf, n_func, rec.ctypes.data, len(rec), n_prof,
                                         Hp.ctypes.data if Hp.size else None, Up.ctypes.data)
    return Hp, Up


def attribute_profiles_inst(st: dict, rec, n_prof: int):
    """D8 at instruction level: Hp [n_prof+1, n_inst, 16], Up [n_prof+1, 16] (the per-function
    attribution with every instruction its own row)."""
    rec = _records(rec)
    n_inst = len(st["inst_addr"])
    addr, pa = _c(st["inst_addr"], np.uint64)
    ln, pl = _c(st["inst_len"], np.uint16)
    ident, pi = _c(np.arange(n_inst, dtype=np.uint32), np.uint32)
    Hp = np.zeros((n_prof + 1, n_inst, SLOTS), np.uint64)
    Up = np.zeros((n_prof + 1, SLOTS), np.uint64)
    if len(rec):
        _lib().oracle_attribute_profiles(n_inst, pa, pl, pi, n_inst, rec.ctypes.data, len(rec), n_prof,
                                         Hp.ctypes.data if Hp.size else None, Up.ctypes.data)
    return Hp, Up


def cct_ctx_func(R: dict) -> np.ndarray:
    """Function of each context of an oracle CCT (NONE for SCC contexts): FUNC contexts name a
    trivial DAG node (its single member), SCC_MEMBER contexts name the function."""
    dag_func = np.full(R["n_dag"], NONE, np.uint32)
    for f, X in enumerate(R["scc_of"]):
        if not R["dag_nontrivial"][X]:
            dag_func[X] = f
    out = np.full(R["n"], NONE, np.uint32)
    k, nd = R["kind"], R["node"]
    out[k == 0] = dag_func[nd[k == 0]]
    out[k == 2] = nd[k == 2]
    return out


def cct_profiles(R: dict, Hp) -> tuple:
    """D11: per-profile excl / incl cubes [P1, n, 16] over the aggregate tree R (from cct())."""
    Hp = np.ascontiguousarray(Hp, np.uint64)
    P1, n_func, n = Hp.shape[0], Hp.shape[1], R["n"]
    cf, pcf = _c(cct_ctx_func(R), np.uint32)
    fr, pfr = _c(R["frac"], np.float64)
    fc, pfc = _c(R["first_child"], np.uint32)
    nc, pnc = _c(R["n_children"], np.uint32)
    E = np.zeros((P1, n, SLOTS), np.float64)
    I = np.zeros((P1, n, SLOTS), np.float64)
    if n and P1:
        _lib().oracle_cct_profiles(n, pcf, pfr, pfc, pnc, P1, n_func, Hp.ctypes.data, E.ctypes.data, I.ctypes.data)
    return E, I


def cct_per_profile(st: dict, Hp_inst, exact: bool = False) -> dict:
    """D12 (reading R30): an approximate CCT for each profile ("for each GPU kernel invocation",
    P:872) from that profile's own instruction histogram Hp_inst[p] (D3-D6 per profile), then the
    trees unified by call path ("unify the tree of call paths from each profile into a
    single tree"): a unified context is a path present in at least one profile's tree; roots in
    DAG order, the children of a context in the order its trees give them (SCC members by
    function id, calls by call instruction), numbered breadth first.  Per profile p and unified
    context u: frac[u, p], excl[u, p, :], incl[u, p, :] are p's own tree values, 0 where p's tree
    lacks the path.  Plain Python over the per-profile trees (small inputs)."""
    Hp_inst = np.ascontiguousarray(Hp_inst, np.uint64)
    P = Hp_inst.shape[0]
    trees = [cct(st, Hp_inst[p], exact=exact) for p in range(P)]
    ci = np.asarray(st["call_inst"], np.int64)
    KIND_SCC = 1
    # unified context: (kind, node, parent uid, site, {p: context id in p's tree})
    roots = {}
    for p, R in enumerate(trees):
        for c in range(R["n"]):
            if R["parent"][c] == NONE:
                roots.setdefault(int(R["node"][c]), (int(R["kind"][c]), {}))[1][p] = c
    U = [(k, node, NONE, NONE, mem) for node, (k, mem) in sorted(roots.items())]
    i = 0
    while i < len(U):
        kind, node, _, _, mem = U[i]
        kids = {}
        for p, c in mem.items():
            R = trees[p]
            for d in range(int(R["first_child"][c]), int(R["first_child"][c] + R["n_children"][c])):
                site = int(R["site"][d])
                key = int(R["node"][d]) if kind == KIND_SCC else int(ci[site])  # members / call sites
                ent = kids.setdefault(key, [int(R["kind"][d]), int(R["node"][d]), site, {}])
                ent[3][p] = d
        for key in sorted(kids):
            k, nd, site, m = kids[key]
            U.append((k, nd, i, site, m))
        i += 1
    n = len(U)
    out = dict(n=n, n_profiles=P,
               kind=np.array([u[0] for u in U], np.uint8), node=np.array([u[1] for u in U], np.uint32),
               parent=np.array([u[2] for u in U], np.uint32), site=np.array([u[3] for u in U], np.uint32),
               frac=np.zeros((n, P), np.float64), excl=np.zeros((n, P, SLOTS), np.float64),
               incl=np.zeros((n, P, SLOTS), np.float64), trees=trees)
    for u, (_, _, _, _, mem) in enumerate(U):
        for p, c in mem.items():
            out["frac"][u, p] = trees[p]["frac"][c]
            out["excl"][u, p] = trees[p]["excl"][c]
            out["incl"][u, p] = trees[p]["incl"][c]
    return out


def profile_stats_f64(X, n_prof: int) -> np.ndarray:
    """D11: statistics of an fp64 cube [>= n_prof, rows, 16] over profiles 0..n_prof-1."""
    X = np.ascontiguousarray(X, np.float64)
    rows = X.shape[1]
    out = np.empty((rows, 6, SLOTS), np.float64)
    if rows:
        _lib().oracle_profile_stats_f64(n_prof, rows, X.ctypes.data, out.ctypes.data)
    return out


def profile_stats(Hp, n_prof: int) -> np.ndarray:
    """D8: [rows, 6, 16] = sum, min, mean, max, std (population), cv over profiles 0..n_prof-1."""
    Hp = np.ascontiguousarray(Hp, np.uint64)
    rows = Hp.shape[1]
    out = np.empty((rows, 6, SLOTS), np.float64)
    if rows:
        _lib().oracle_profile_stats(n_prof, rows, Hp.ctypes.data, out.ctypes.data)
    return out


def sparse_build(Hp, cms: bool) -> dict:
    """D9: CMS (cms=True) or PMS of the cube Hp [P, C, 16] (see gpa_oracle.c)."""
    Hp = np.ascontiguousarray(Hp, np.uint64)
    P, C = Hp.shape[0], Hp.shape[1]
    r = _lib().oracle_sparse_build(Hp.ctypes.data if Hp.size else None, P, C, 1 if cms else 0)
    try:
        S = r.contents
        nq, nv, ni = S.n_planes, S.n_values, S.n_index

        def arr(p, cnt, dt):
            return np.ctypeslib.as_array(p, shape=(cnt,)).astype(dt, copy=True) if cnt else np.zeros(0, dt)
        return dict(n_planes=nq, n_values=nv, n_index=ni, plane_off=arr(S.plane_off, nq + 1, np.uint64),
                    index_off=arr(S.index_off, nq + 1, np.uint64), vals=arr(S.vals, nv, np.uint64),
                    ids=arr(S.ids, nv, np.uint32), index_start=arr(S.index_start, ni, np.uint64),
                    index_id=arr(S.index_id, ni, np.uint32))
    finally:
        _lib().oracle_sparse_free(r)


def block_counts(n_inst: int, block_start, count) -> np.ndarray:
    """Exact per-instruction counts (slot 0) from basic-block execution counts."""
    bs, pb = _c(block_start, np.uint32)
    c, pc = _c(count, np.uint64)
    H = np.zeros((n_inst, SLOTS), np.uint64)
    if len(c):
        _lib().oracle_block_counts(len(c), pb, pc, H.ctypes.data)
    return H


# ---- D7 ---------------------------------------------------------------------------------
def derive_u64(V, MIX=None) -> np.ndarray:
    V = np.ascontiguousarray(V, np.uint64).reshape(-1, SLOTS)
    out = np.empty((len(V), NCOLS), np.float64)
    M = None if MIX is None else np.ascontiguousarray(MIX, np.uint64).reshape(-1, SLOTS)
    if len(V):
        _lib().oracle_derive_u64(len(V), V.ctypes.data, None if M is None else M.ctypes.data, out.ctypes.data)
    return out


def derive_f64(V) -> np.ndarray:
    V = np.ascontiguousarray(V, np.float64).reshape(-1, SLOTS)
    out = np.empty((len(V), NCOLS), np.float64)
    if len(V):
        _lib().oracle_derive_f64(len(V), V.ctypes.data, out.ctypes.data)
    return out


# ---- D10 --------------------------------------------------------------------------------
def blame(tr: dict) -> dict:
    """D10: GPU-idleness blame of a trace set (keys line_off, line_kind, line_scope, time, ctx,
    n_scopes, n_routines).  Returns num [S, R, kmax+1] u64, total [S], gpu_idle [S], blame and
    share [S, R] f64, kmax.  Raises ValueError on an invalid trace set."""
    lo, plo = _c(tr["line_off"], np.uint64)
    lk, plk = _c(tr["line_kind"], np.uint8)
    ls, pls = _c(tr["line_scope"], np.uint32)
    t, pt = _c(tr["time"], np.uint64)
    cx, pcx = _c(tr["ctx"], np.uint32)
    S, R = int(tr["n_scopes"]), int(tr["n_routines"])
    nl = len(lk)
    kmax = int(np.bincount(ls[lk == 1], minlength=S).max()) if (lk == 1).any() and S else 0
    kmax = max(kmax, 1)
    num = np.zeros((S, R, kmax + 1), np.uint64)
    total, idle = np.zeros(S, np.uint64), np.zeros(S, np.uint64)
    bl, sh = np.zeros((S, R), np.float64), np.zeros((S, R), np.float64)
    rc = _lib().oracle_blame(nl, plo, plk, pls, pt, pcx, S, R, kmax, num.ctypes.data, total.ctypes.data,
                             idle.ctypes.data, bl.ctypes.data, sh.ctypes.data)
    if rc != 0:
        raise ValueError("invalid trace set")
    return dict(num=num, total=total, gpu_idle=idle, blame=bl, share=sh, kmax=kmax)
