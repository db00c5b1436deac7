"""Seeded synthetic workloads for the PC-sample attribution path (INPUT GENERATION ONLY).

This module builds, from a seed, everything a run needs as *input*:

* a synthetic GPU load module's program structure (the arrays `gpa_load_structure`
  takes): functions laid out at 128-B-aligned relocated addresses with gaps,
  16-B instructions with classes, a scope tree of inlined code / loops / lines
   and direct call sites forming a call graph with recursive SCCs
  (P:874-879);
* the tables of the counter-based record generator (`gen_core.h`), so record k of a
  workload is a pure function of (seed, k): host (`gen_host.c`) and device (`gen_dev.cu`)
  builds are bit-identical and any shard can be produced on its own.

It holds none of the analysis method's arithmetic: no attribution, roll-up, CCT or metric
code.  Both the oracle side and the CUDA side of every parity test take their inputs from
here.  The recipe (shapes, distributions) is DESIGN.md §4.
"""
from __future__ import annotations

import ctypes
import dataclasses
import functools
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
NONE = 0xFFFFFFFF

RECORD_DTYPE = np.dtype([("pc", "<u8"), ("count", "<u4"), ("stall", "<u2"), ("stream", "<u2")])
assert RECORD_DTYPE.itemsize == 16

KIND_FUNCTION, KIND_INLINE, KIND_LOOP, KIND_LINE = 0, 1, 2, 3
CLASS_CALL, CLASS_SYNC = 14, 15

# instruction-class mix (about a third index arithmetic)
CLASS_P = np.array([0.33, 0.15, 0.10, 0.02, 0.02, 0.03, 0.09, 0.06, 0.08, 0.01, 0.03,
                    0.01, 0.01, 0.04, 0.00, 0.02])
CLASS_P = CLASS_P / CLASS_P.sum()

# per-class base distribution over the 12 stall reasons (R2 order:
# 0 issued, 1 inst_fetch, 2 exec_dep, 3 mem_dep, 4 texture, 5 sync, 6 const_mem,
# 7 pipe_busy, 8 mem_throttle, 9 not_selected, 10 other, 11 sleeping)
_DEFAULT = np.array([.30, .04, .20, .05, .005, .01, .02, .06, .01, .20, .04, .005])


def _stall_base(cls: int) -> np.ndarray:
    b = _DEFAULT.copy()
    if cls in (6, 9):            # global / local loads: memory dependency heavy
        b[3] += 0.9; b[8] += 0.15
    elif cls in (7, 12):         # stores / atomics: throttle
        b[8] += 0.5; b[3] += 0.2
    elif cls == 11:              # texture
        b[4] += 0.8
    elif cls == 8:               # shared
        b[3] += 0.3; b[7] += 0.2
    elif cls == 2:               # fp64: exec dependency / pipe busy
        b[2] += 0.5; b[7] += 0.4
    elif cls == 4:               # SFU
        b[7] += 0.3; b[2] += 0.3
    elif cls == 15:              # barriers
        b[5] += 1.2; b[11] += 0.1
    elif cls == 10:              # constant
        b[6] += 0.4
    elif cls in (13, 14):        # control / call
        b[1] += 0.3; b[10] += 0.1
    return b / b.sum()


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    seed: int
    records: int
    n_func: int
    n_kernels: int
    n_inst: int
    func_sizes: tuple = ()
    window: int = 6
    scc_sizes: tuple = ()
    n_self_rec: int = 0
    extra_in_frac: float = 0.1
    dup_site_frac: float = 0.02
    cross_home_frac: float = 0.1
    unsampled_call_frac: float = 0.3
    cold_func_frac: float = 0.0
    max_loop_depth: int = 3
    max_inline_depth: int = 0
    p_loop: float = 0.04
    p_inline: float = 0.0
    line_len_mean: float = 3.0
    split_line_frac: float = 0.15
    ctx_budget: int = 100
    full_stall: bool = False
    max_reasons: int = 4
    hot_plant: bool = False
    n_streams: int = 1
    burst_shift: int = 12
    p_misalign: float = 0.01
    p_corrupt_pc: float = 1e-4
    p_corrupt_stall: float = 1e-4
    permute_funcs: bool = True

    def scaled(self, records: int) -> "Config":
        return dataclasses.replace(self, records=int(records))


# BASELINE.json configs[0..4]; parameters not fixed there are DESIGN.md §4 choices.
CONFIGS = {
    "C1": Config("C1", seed=101, records=10_000, n_func=3, n_kernels=1, n_inst=200,
                 func_sizes=(96, 64, 40), window=1, extra_in_frac=0.0, dup_site_frac=0.0,
                 cross_home_frac=0.0, unsampled_call_frac=0.0, max_loop_depth=1, p_loop=0.06,
                 ctx_budget=3, permute_funcs=False),
    "C2": Config("C2", seed=202, records=10_000_000, n_func=25, n_kernels=5, n_inst=12_000,
                 window=3, max_inline_depth=6, p_inline=0.12, p_loop=0.05, ctx_budget=100),
    "C3": Config("C3", seed=303, records=100_000_000, n_func=2000, n_kernels=20, n_inst=100_000,
                 scc_sizes=(2, 3, 4, 6, 8, 16, 32, 64, 2, 3), n_self_rec=50, extra_in_frac=0.25,
                 cold_func_frac=0.05, max_inline_depth=3, p_inline=0.05, p_loop=0.05,
                 ctx_budget=1 << 22),
    "C4": Config("C4", seed=404, records=1_000_000_000, n_func=400, n_kernels=4, n_inst=200_000,
                 scc_sizes=(2, 2, 3, 3, 4, 5, 6, 8), n_self_rec=2, extra_in_frac=0.15,
                 unsampled_call_frac=0.2, cold_func_frac=0.03, max_inline_depth=3, p_inline=0.04,
                 ctx_budget=1 << 20, n_streams=384),
    "C5": Config("C5", seed=505, records=4_000_000_000, n_func=5000, n_kernels=50, n_inst=500_000,
                 scc_sizes=tuple([2, 3, 4, 5, 6, 8, 12, 16] * 8), n_self_rec=36, extra_in_frac=0.1,
                 unsampled_call_frac=0.2, cold_func_frac=0.03, max_inline_depth=3, p_inline=0.04,
                 ctx_budget=1 << 20, full_stall=True, hot_plant=True),
}


# ----------------------------------------------------------------------------------------
# native helpers (gen_host.c)
# ----------------------------------------------------------------------------------------
class GenTables(ctypes.Structure):
    _fields_ = [
        ("seed", ctypes.c_uint64), ("burst_shift", ctypes.c_uint32), ("n_kernels", ctypes.c_uint32),
        ("kern_prob", ctypes.c_void_p), ("kern_alias", ctypes.c_void_p),
        ("reach_off", ctypes.c_void_p), ("reach_prob", ctypes.c_void_p),
        ("reach_alias", ctypes.c_void_p), ("reach_inst", ctypes.c_void_p),
        ("stall_cum", ctypes.c_void_p), ("inst_addr", ctypes.c_void_p), ("inst_len", ctypes.c_void_p),
        ("n_probe", ctypes.c_uint32), ("probe_pc", ctypes.c_void_p),
        ("n_streams", ctypes.c_uint32), ("stream_first_burst", ctypes.c_void_p),
        ("corrupt_pc_thresh", ctypes.c_uint32), ("corrupt_stall_thresh", ctypes.c_uint32),
        ("misalign_thresh", ctypes.c_uint32), ("hot_inst", ctypes.c_uint32),
        ("hot_records", ctypes.c_uint64), ("hot_stride", ctypes.c_uint64),
    ]


def build_native(force: bool = False) -> None:
    """Compile gen/libgen_host.so (gcc) and gen/libgen_dev.so (nvcc, sm_100a)."""
    host = os.path.join(HERE, "libgen_host.so")
    dev = os.path.join(HERE, "libgen_dev.so")
    src_h = [os.path.join(HERE, f) for f in ("gen_host.c", "gen_core.h")]
    src_d = [os.path.join(HERE, f) for f in ("gen_dev.cu", "gen_core.h")]

    def stale(out, srcs):
        return force or not os.path.exists(out) or any(os.path.getmtime(s) > os.path.getmtime(out) for s in srcs)

    if stale(host, src_h):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", host,
                               os.path.join(HERE, "gen_host.c"), "-lpthread"])
    if stale(dev, src_d):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "-o", dev,
                               os.path.join(HERE, "gen_dev.cu")])


@functools.lru_cache(None)
def _host_lib():
    build_native()
    lib = ctypes.CDLL(os.path.join(HERE, "libgen_host.so"))
    lib.gen_records_host.argtypes = [ctypes.POINTER(GenTables), ctypes.c_uint64, ctypes.c_uint64,
                                     ctypes.c_void_p, ctypes.c_int]
    lib.gen_records_host.restype = ctypes.c_int
    lib.gen_build_alias.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
    lib.gen_build_alias.restype = ctypes.c_int
    return lib


@functools.lru_cache(None)
def _dev_lib():
    build_native()
    lib = ctypes.CDLL(os.path.join(HERE, "libgen_dev.so"))
    lib.gen_records_device.argtypes = [ctypes.POINTER(GenTables), ctypes.c_uint64, ctypes.c_uint64,
                                       ctypes.c_void_p, ctypes.c_void_p]
    lib.gen_records_device.restype = ctypes.c_int
    return lib


def alias_table(weights: np.ndarray):
    w = np.ascontiguousarray(weights, dtype=np.float64)
    prob = np.empty(len(w), np.uint32)
    alias = np.empty(len(w), np.uint32)
    rc = _host_lib().gen_build_alias(w.ctypes.data, len(w), prob.ctypes.data, alias.ctypes.data)
    if rc != 0:
        raise ValueError("alias table needs a positive total weight")
    return prob, alias


# ----------------------------------------------------------------------------------------
# structure synthesis
# ----------------------------------------------------------------------------------------
def _call_graph(cfg: Config, rng: np.random.Generator):
    """Units (a single function or an SCC group), their call edges and static path counts.

    Returns (n_func, kernels, edges [(caller_f, callee_f)], static context count)."""
    K = cfg.n_kernels
    n_nonk = cfg.n_func - K
    groups = [int(s) for s in cfg.scc_sizes]
    n_single = n_nonk - sum(groups)
    assert n_single >= cfg.n_self_rec >= 0, "config has too few functions for its SCCs"
    units = [("k", 1)] * K
    nonk = [("scc", s) for s in groups] + [("self", 1)] * cfg.n_self_rec + \
           [("one", 1)] * (n_single - cfg.n_self_rec)
    order = rng.permutation(len(nonk)) if cfg.permute_funcs else np.arange(len(nonk))
    units += [nonk[i] for i in order]
    members, f = [], 0
    for _, s in units:
        members.append(list(range(f, f + s)))
        f += s
    U = len(units)
    M = max(U - K, 1)
    home = [u if u < K else ((u - K) * K) // M for u in range(U)]
    paths = [0] * U
    total_ctx = 0
    edges = []

    def unit_ctx(u):
        kind, s = units[u]
        return 1 + s if kind in ("scc", "self") else 1

    for u in range(K):
        paths[u] = 1
        total_ctx += 1
    by_home = {h: [h] for h in range(K)}
    for u in range(K, U):
        h = home[u]
        cand = by_home[h][-cfg.window:]
        if cfg.window > 1 and h not in cand:
            cand = [h] + cand
        callers = [cand[rng.integers(len(cand))]]
        if rng.random() < cfg.extra_in_frac:
            for _ in range(int(rng.integers(1, 4))):
                if rng.random() < cfg.cross_home_frac:
                    callers.append(int(rng.integers(u)))
                else:
                    pool = by_home[h]
                    callers.append(pool[rng.integers(len(pool))])
        if cfg.dup_site_frac > 0:
            callers += [c for c in callers if rng.random() < cfg.dup_site_frac]
        p = sum(paths[c] for c in callers)
        if total_ctx + p * unit_ctx(u) > cfg.ctx_budget:       # keep the CCT bounded
            callers = [callers[0]]
            p = paths[callers[0]]
            if total_ctx + p * unit_ctx(u) > cfg.ctx_budget:
                callers = [h]
                p = 1
        paths[u] = p
        total_ctx += p * unit_ctx(u)
        for c in callers:
            cm = members[c][rng.integers(len(members[c]))]
            vm = members[u][rng.integers(len(members[u]))]
            edges.append((cm, vm))
        kind, s = units[u]
        if kind == "scc":                                       # internal cycle + chords
            ms = members[u]
            for a in range(s):
                edges.append((ms[a], ms[(a + 1) % s]))
            for _ in range(s // 2):
                edges.append((ms[rng.integers(s)], ms[rng.integers(s)]))
        elif kind == "self":
            edges.append((members[u][0], members[u][0]))
        by_home[h].append(u)
    return cfg.n_func, list(range(K)), edges, total_ctx


def _scope_tree(cfg, rng, lo, hi, fscope, parent_l, kind_l, inst_scope, inst_factor):
    """Recursive partition of a function's instruction range into loops / inlined code /
    lines.  Appends scopes to parent_l/kind_l, fills inst_scope and loop-trip factors."""

    def new_scope(parent, kind):
        parent_l.append(parent)
        kind_l.append(kind)
        return len(parent_l) - 1

    def rec(parent, lo, hi, loop_d, inl_d, factor):
        pos = lo
        lines_here = []
        while pos < hi:
            rem = hi - pos
            x = rng.random()
            if rem >= 6 and loop_d < cfg.max_loop_depth and x < cfg.p_loop:
                L = int(rng.integers(4, min(rem, 96) + 1))
                s = new_scope(parent, KIND_LOOP)
                trip = math.exp(rng.uniform(math.log(4), math.log(64)))
                rec(s, pos, pos + L, loop_d + 1, inl_d, factor * trip)
                pos += L
            elif rem >= 4 and inl_d < cfg.max_inline_depth and x < cfg.p_loop + cfg.p_inline:
                L = int(rng.integers(3, min(rem, 64) + 1))
                s = new_scope(parent, KIND_INLINE)
                rec(s, pos, pos + L, loop_d, inl_d + 1, factor)
                pos += L
            else:
                L = int(min(rem, rng.geometric(1.0 / cfg.line_len_mean)))
                if lines_here and rng.random() < cfg.split_line_frac:
                    s = lines_here[int(rng.integers(len(lines_here)))]   # non-contiguous line
                else:
                    s = new_scope(parent, KIND_LINE)
                    lines_here.append(s)
                inst_scope[pos:pos + L] = s
                inst_factor[pos:pos + L] = factor
                pos += L

    rec(fscope, lo, hi, 0, 0, 1.0)


@dataclasses.dataclass
class Workload:
    cfg: Config
    structure: dict           # arrays for gpa_load_structure / the oracle
    tables: dict              # arrays of the record generator
    meta: dict                # counts and facts about the workload
    _dev: dict = dataclasses.field(default_factory=dict, repr=False)

    # ---- record generation -------------------------------------------------------------
    def _ctables(self, arrs: dict, ptr) -> GenTables:
        t = self.tables
        return GenTables(
            seed=t["seed"], burst_shift=t["burst_shift"], n_kernels=len(t["kern_prob"]),
            kern_prob=ptr(arrs["kern_prob"]), kern_alias=ptr(arrs["kern_alias"]),
            reach_off=ptr(arrs["reach_off"]), reach_prob=ptr(arrs["reach_prob"]),
            reach_alias=ptr(arrs["reach_alias"]), reach_inst=ptr(arrs["reach_inst"]),
            stall_cum=ptr(arrs["stall_cum"]), inst_addr=ptr(arrs["inst_addr"]),
            inst_len=ptr(arrs["inst_len"]), n_probe=len(t["probe_pc"]), probe_pc=ptr(arrs["probe_pc"]),
            n_streams=len(t["stream_first_burst"]), stream_first_burst=ptr(arrs["stream_first_burst"]),
            corrupt_pc_thresh=t["corrupt_pc_thresh"], corrupt_stall_thresh=t["corrupt_stall_thresh"],
            misalign_thresh=t["misalign_thresh"], hot_inst=t["hot_inst"],
            hot_records=t["hot_records"], hot_stride=t["hot_stride"])

    def _arrays(self):
        t = self.tables
        return {k: t[k] for k in ("kern_prob", "kern_alias", "reach_off", "reach_prob", "reach_alias",
                                  "reach_inst", "stall_cum", "probe_pc", "stream_first_burst")} | \
            {"inst_addr": self.structure["inst_addr"], "inst_len": self.structure["inst_len"]}

    def records_host(self, k0: int = 0, n: int | None = None, threads: int | None = None,
                     out: np.ndarray | None = None) -> np.ndarray:
        """Records [k0, k0+n) of the workload stream as a RECORD_DTYPE array (host)."""
        n = self.cfg.records - k0 if n is None else int(n)
        if out is None:
            out = np.empty(n, RECORD_DTYPE)
        arrs = self._arrays()
        ct = self._ctables(arrs, lambda a: a.ctypes.data)
        th = threads or min(16, os.cpu_count() or 1)
        rc = _host_lib().gen_records_host(ctypes.byref(ct), k0, n, out.ctypes.data, th)
        if rc != 0:
            raise RuntimeError("gen_records_host failed")
        return out

    def records_device(self, out, k0: int = 0, n: int | None = None, stream=None):
        """Write records [k0, k0+n) into a CUDA tensor `out` (>= 16*n bytes, 16-B aligned)."""
        import torch
        n = self.cfg.records - k0 if n is None else int(n)
        dev = out.device
        key = str(dev)
        if key not in self._dev:
            tens = {k: torch.from_numpy(np.ascontiguousarray(v).view(np.uint8)).to(dev)
                    for k, v in self._arrays().items()}
            self._dev[key] = (tens, self._ctables(tens, lambda a: a.data_ptr()))
        _, ct = self._dev[key]
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        rc = _dev_lib().gen_records_device(ctypes.byref(ct), k0, n, out.data_ptr(), s.cuda_stream)
        if rc != 0:
            raise RuntimeError("gen_records_device failed")
        return out


def _build(cfg: Config) -> Workload:
    rng = np.random.default_rng(cfg.seed)
    n_func, kernels, edges, static_ctx = _call_graph(cfg, rng)

    # ---- function sizes (instructions); room for every call site ------------------------
    outdeg = np.zeros(n_func, np.int64)
    for c, _ in edges:
        outdeg[c] += 1
    if cfg.func_sizes:
        sizes = np.array(cfg.func_sizes, np.int64)
    else:
        raw = rng.lognormal(0.0, 0.8, n_func)
        sizes = np.maximum(np.round(raw / raw.sum() * cfg.n_inst).astype(np.int64), 8)
    sizes = np.maximum(sizes, outdeg + 4)
    diff = cfg.n_inst - int(sizes.sum())
    big = int(np.argmax(sizes))
    if diff > 0 or sizes[big] + diff >= outdeg[big] + 4:
        sizes[big] += diff
    N = int(sizes.sum())
    first = np.concatenate([[0], np.cumsum(sizes)])

    # ---- relocated layout: 16-B instructions, 128-B aligned function bases,
    #      gaps of 0..3 x 16 B before alignment -----------------------------------------------
    base = 0x10000
    inst_addr = np.empty(N, np.uint64)
    func_base = np.empty(n_func, np.uint64)
    func_end = np.empty(n_func, np.uint64)
    a = base
    for f in range(n_func):
        a = (a + 127) // 128 * 128
        func_base[f] = a
        inst_addr[first[f]:first[f + 1]] = a + 16 * np.arange(sizes[f], dtype=np.uint64)
        a += 16 * int(sizes[f])
        func_end[f] = a
        a += 16 * int(rng.integers(0, 4))
    inst_len = np.full(N, 16, np.uint16)

    # ---- scopes -------------------------------------------------------------------------------
    parent_l, kind_l = [], []
    inst_scope = np.empty(N, np.uint32)
    inst_factor = np.empty(N, np.float64)
    func_scope = np.empty(n_func, np.uint32)
    for f in range(n_func):
        parent_l.append(NONE)
        kind_l.append(KIND_FUNCTION)
        func_scope[f] = len(parent_l) - 1
        _scope_tree(cfg, rng, int(first[f]), int(first[f + 1]), int(func_scope[f]),
                    parent_l, kind_l, inst_scope, inst_factor)
    scope_parent = np.array(parent_l, np.uint32)
    scope_kind = np.array(kind_l, np.uint8)

    # ---- instruction classes and call sites -----------------------------------------------------
    inst_class = rng.choice(16, size=N, p=CLASS_P).astype(np.uint8)
    call_inst, call_callee = [], []
    used = set()
    for c, v in edges:
        lo, hi = int(first[c]), int(first[c + 1])
        while True:
            i = int(rng.integers(lo, hi))
            if i not in used:
                break
        used.add(i)
        call_inst.append(i)
        call_callee.append(v)
        inst_class[i] = CLASS_CALL
    order = np.argsort(np.array(call_inst, np.int64), kind="stable")
    call_inst = np.array(call_inst, np.uint32)[order]
    call_callee = np.array(call_callee, np.uint32)[order]
    hot_inst = 0
    if cfg.hot_plant:
        k0 = kernels[0]
        cands = [i for i in range(int(first[k0]), int(first[k0 + 1])) if i not in used]
        hot_inst = cands[len(cands) // 2]
        inst_class[hot_inst] = CLASS_SYNC

    # ---- sampling weights: loop trip factors x U(0.5,1.5); unsampled call sites; cold code --
    w = inst_factor * rng.uniform(0.5, 1.5, N)
    is_call = np.zeros(N, bool)
    is_call[call_inst] = True
    unsampled = call_inst[rng.random(len(call_inst)) < cfg.unsampled_call_frac]
    w[unsampled] = 0.0
    kern_set = set(kernels)
    cold = [f for f in range(n_func) if f not in kern_set and rng.random() < cfg.cold_func_frac]
    for f in cold:
        w[first[f]:first[f + 1]] = 0.0

    # ---- per-kernel reachable instructions (alias tables) -----------------------------------
    adj = [[] for _ in range(n_func)]
    for c, v in edges:
        adj[c].append(v)
    reach_off = [0]
    reach_prob, reach_alias, reach_inst = [], [], []
    kern_w = []
    for k in kernels:
        seen = {k}
        stack = [k]
        while stack:
            x = stack.pop()
            for y in adj[x]:
                if y not in seen:
                    seen.add(y)
                    stack.append(y)
        idx = np.concatenate([np.arange(first[f], first[f + 1]) for f in sorted(seen)])
        idx = idx[w[idx] > 0]
        p, al = alias_table(w[idx])
        reach_prob.append(p)
        reach_alias.append(al)
        reach_inst.append(idx.astype(np.uint32))
        reach_off.append(reach_off[-1] + len(idx))
        kern_w.append(rng.uniform(0.5, 2.0))
    kern_prob, kern_alias = alias_table(np.array(kern_w))

    # ---- stall-reason tables (31-bit cumulative thresholds) ----------------------------------
    bases = np.stack([_stall_base(c) for c in range(16)])
    base_p = bases[inst_class]
    g = rng.gamma(2.0, 1.0, size=(N, 12))                    # Dirichlet(alpha = 2) perturbation
    p = base_p * g
    if cfg.full_stall:
        p = p / p.sum(1, keepdims=True)
        p = 0.88 * p + 0.01                                  # every reason >= 1% everywhere
    else:
        keep = np.argsort(-p * rng.uniform(0.5, 1.5, size=p.shape), axis=1)[:, :cfg.max_reasons]
        mask = np.zeros_like(p, bool)
        np.put_along_axis(mask, keep, True, axis=1)
        p = np.where(mask, p, 0.0)
        p = p / p.sum(1, keepdims=True)
    cum = np.floor(np.cumsum(p, 1) * 2.0 ** 31)
    last_nz = 11 - np.argmax(p[:, ::-1] > 0, axis=1)
    cols = np.arange(12)[None, :]
    cum = np.where(cols >= last_nz[:, None], 2.0 ** 31, np.minimum(cum, 2.0 ** 31 - 1))
    stall_cum = cum.astype(np.uint32).reshape(-1)

    # ---- unmapped probe addresses: inter-function gaps, below / above the module ------------
    probes = [0, base - 1, int(func_end[-1]), int(func_end[-1]) + 12345, 0xFFFFFFFFFFFFFFFF]
    for f in range(n_func - 1):
        if func_base[f + 1] > func_end[f]:
            lo, hi = int(func_end[f]), int(func_base[f + 1])
            probes.append(lo)
            probes.append(int(rng.integers(lo, hi)))
    probes += [int(x) for x in rng.integers(0, base, 16)]
    probes += [int(func_end[-1]) + int(x) for x in rng.integers(0, 1 << 20, 16)]
    probe_pc = np.array(probes[:4096], np.uint64)

    # ---- streams: bursts of 2^burst_shift records, lognormal(0.5) stream lengths ------------
    n_bursts = max(1, -(-cfg.records // (1 << cfg.burst_shift)))
    if cfg.n_streams > 1:
        L = rng.lognormal(0.0, 0.5, cfg.n_streams)
        L = L / L.sum() * n_bursts
        Li = np.maximum(np.floor(L).astype(np.int64), 1 if n_bursts >= cfg.n_streams else 0)
        Li[int(np.argmax(Li))] += n_bursts - int(Li.sum())
        sfb = np.concatenate([[0], np.cumsum(Li)[:-1]]).astype(np.uint64)
    else:
        sfb = np.zeros(1, np.uint64)

    hot_records = (1 << 16) + 1 if cfg.hot_plant else 0
    hot_stride = max(1, cfg.records // hot_records) if hot_records else 1
    if hot_records and cfg.records < hot_records:
        hot_records = 0

    structure = dict(inst_addr=inst_addr, inst_len=inst_len, inst_class=inst_class,
                     inst_scope=inst_scope, scope_parent=scope_parent, scope_kind=scope_kind,
                     func_scope=func_scope, call_inst=call_inst, call_callee=call_callee)
    tables = dict(seed=cfg.seed, burst_shift=cfg.burst_shift,
                  kern_prob=kern_prob, kern_alias=kern_alias,
                  reach_off=np.array(reach_off, np.uint64),
                  reach_prob=np.concatenate(reach_prob), reach_alias=np.concatenate(reach_alias),
                  reach_inst=np.concatenate(reach_inst), stall_cum=stall_cum, probe_pc=probe_pc,
                  stream_first_burst=sfb,
                  corrupt_pc_thresh=int(cfg.p_corrupt_pc * 2 ** 32),
                  corrupt_stall_thresh=int(cfg.p_corrupt_stall * 2 ** 32),
                  misalign_thresh=int(cfg.p_misalign * 2 ** 32),
                  hot_inst=hot_inst, hot_records=hot_records, hot_stride=hot_stride)
    meta = dict(n_inst=N, n_func=n_func, n_scope=len(scope_parent), n_call=len(call_inst),
                n_line=int((scope_kind == KIND_LINE).sum()), n_loop=int((scope_kind == KIND_LOOP).sum()),
                n_inline=int((scope_kind == KIND_INLINE).sum()), static_contexts=static_ctx,
                kernels=kernels, cold_funcs=cold, hot_inst=hot_inst,
                reach_total=int(reach_off[-1]), func_first_inst=first)
    return Workload(cfg, structure, tables, meta)


@functools.lru_cache(maxsize=8)
def workload(name: str, records: int | None = None) -> Workload:
    """The seeded workload of config `name` (C1..C5), optionally with another record count
    (same structure and distributions; the stream is a prefix-free re-draw only in its
    record-count-dependent parts: stream boundaries and the hot-bin stride)."""
    cfg = CONFIGS[name]
    if records is not None:
        cfg = cfg.scaled(records)
    return _build(cfg)

