"""Measurements of the SURVEY §8f rows built beyond the north-star path (one JSON line each):
f1 per-profile histograms + cross-profile statistics on C4 (1e9 records, 384 profiles), and
f3 sparse PMS/CMS encoding of f1's cube, and
f4 GPU-idleness blame on the B3 trace set, and
f2 exact-count mode (block counts -> instructions -> exact-mode CCT) on C3's structure.
CUDA events around each call, median of K after W warm-ups."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
from paper_2109_06931_b200 import gpa

K, W = 5, 2
PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6535.7


def timed(fn):
    ts = []
    for r in range(W + K):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if r >= W:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def f1():
    w = gen.workload("C4")
    s = gpa.load_structure(w.structure, 0)
    n = w.cfg.records
    rec = torch.empty((n, 2), dtype=torch.int64, device="cuda")
    for k in range(0, n, 1 << 28):
        w.records_device(rec[k:k + (1 << 28)], k, min(1 << 28, n - k))
    P = 384
    PH = torch.zeros((P + 1, s.info["n_func"], 16), dtype=torch.int64, device="cuda")
    PU = torch.zeros((P + 1, 16), dtype=torch.int64, device="cuda")
    stats = torch.empty((s.info["n_func"], 6, 16), dtype=torch.float64, device="cuda")

    def run_attr():
        PH.zero_()
        PU.zero_()
        gpa.attribute_profiles(s, rec, P, PH, PU)

    ms_attr = timed(run_attr)
    ms_stats = timed(lambda: gpa.profile_stats(s, PH, P, stats))
    gbs = 16 * n / ms_attr / 1e6
    print(json.dumps({"row": "f1", "workload": "C4", "records": n, "profiles": P, "kernel": "k_attr_prof",
                      "attr_ms": ms_attr, "records_per_s": n / ms_attr * 1e3, "GBps": gbs, "frac": gbs / PEAK,
                      "stats_ms": ms_stats}), flush=True)
    f3(s, PH, P)
    # instruction level: (P+1) x n_inst x 16 u64 cube (9.9 GB at C4), all-L2 reductions
    PI = torch.zeros((P + 1, s.info["n_inst"], 16), dtype=torch.int64, device="cuda")

    def run_inst():
        PI.zero_()
        PU.zero_()
        gpa.attribute_profiles_inst(s, rec, P, PI, PU)

    ms_inst = timed(run_inst)
    st_inst = torch.empty((s.info["n_inst"], 6, 16), dtype=torch.float64, device="cuda")
    ms_inst_stats = timed(lambda: gpa.profile_stats_rows(PI, P, st_inst))
    del PI
    # CCT level over the aggregate tree
    H = torch.zeros((s.info["n_inst"], 16), dtype=torch.int64, device="cuda")
    U = torch.zeros(16, dtype=torch.int64, device="cuda")
    gpa.attribute_samples(s, rec, H, U)
    c = gpa.reconstruct_cct(s, H)
    E = torch.empty((P + 1, c.n, 16), dtype=torch.float64, device="cuda")
    I = torch.empty_like(E)
    ms_cct = timed(lambda: gpa.cct_profiles(s, c, PH, P, E, I))
    st_cct = torch.empty((c.n, 6, 16), dtype=torch.float64, device="cuda")
    ms_cct_stats = timed(lambda: gpa.profile_stats_f64(I, P, st_cct))
    print(json.dumps({"row": "f1-inst+cct", "workload": "C4", "profiles": P, "inst_attr_ms": ms_inst,
                      "inst_records_per_s": n / ms_inst * 1e3, "inst_GBps": 16 * n / ms_inst / 1e6,
                      "inst_stats_ms": ms_inst_stats, "contexts": c.n, "cct_profiles_ms": ms_cct,
                      "cct_stats_ms": ms_cct_stats}), flush=True)
    # a tree per profile unified by call path (R30): call-site weights from the records + build
    del E, I
    PW = torch.zeros((P + 1, max(s.info["n_call"], 1)), dtype=torch.int64, device="cuda")

    def run_w():
        PW.zero_()
        gpa.profile_call_weights(s, rec, P, PW)

    ms_w = timed(run_w)
    holder = []

    def run_multi():
        while holder:
            holder.pop().free()
        holder.append(gpa.reconstruct_cct_per_profile(s, PH, PW, P))

    ms_multi = timed(run_multi)
    print(json.dumps({"row": "f1-cct-per-profile", "workload": "C4", "profiles": P,
                      "call_weights_ms": ms_w, "call_weights_GBps": 16 * n / ms_w / 1e6,
                      "call_weights_frac": 16 * n / ms_w / 1e6 / PEAK,
                      "unified_contexts": holder[0].n, "aggregate_contexts": c.n,
                      "reconstruct_per_profile_ms": ms_multi}), flush=True)
    holder.pop().free()


def f3(s, PH, P):
    """Sparse PMS / CMS encoding of f1's cube (one build = count + scans + sync + write)."""
    for cms in (False, True):
        def run():
            gpa.sparse_build(s, PH, P, cms).free()
        ms = timed(run)
        sp = gpa.sparse_build(s, PH, P, cms)
        cube = PH.numel() * 8
        out = sp.n_values * 12 + sp.n_index * 12 + 16 * (sp.n_planes + 1)
        print(json.dumps({"row": "f3", "format": "CMS" if cms else "PMS", "cube_bytes": cube,
                          "n_values": sp.n_values, "n_index": sp.n_index, "ms": ms,
                          "GBps_cube_2pass_plus_out": (2 * cube + out) / ms / 1e6}), flush=True)
        sp.free()


def f2():
    w = gen.workload("C3", records=10)
    s = gpa.load_structure(w.structure, 0)
    n_inst = s.info["n_inst"]
    rng = np.random.default_rng(1)
    cuts = np.sort(rng.choice(np.arange(1, n_inst), n_inst // 6, replace=False))
    start = torch.from_numpy(np.concatenate([[0], cuts, [n_inst]]).astype(np.int32)).cuda()
    cnt = torch.from_numpy(rng.integers(0, 10 ** 6, len(cuts) + 1)).cuda()
    H = torch.zeros((n_inst, 16), dtype=torch.int64, device="cuda")

    def run():
        H.zero_()
        gpa.block_counts(s, start, cnt, H)
        c = gpa.reconstruct_cct(s, H, mode=gpa.WEIGHTS_EXACT)
        c.free()

    ms = timed(run)
    c = gpa.reconstruct_cct(s, H, mode=gpa.WEIGHTS_EXACT)
    print(json.dumps({"row": "f2", "workload": "C3 structure, random basic blocks", "blocks": len(cuts) + 1,
                      "contexts": c.n, "ms": ms}), flush=True)


def f4():
    """GPU-idleness blame over the B3 trace set (64 ranks x 14 lines, 31 M change points)."""
    from gen.trace import trace_set
    tr = trace_set("B3")
    S, R = tr["n_scopes"], tr["n_routines"]
    t = torch.from_numpy(tr["time"].view(np.int64)).cuda()
    c = torch.from_numpy(tr["ctx"].view(np.int32)).cuda()
    bl = torch.empty((S, R), dtype=torch.float64, device="cuda")
    sh = torch.empty_like(bl)
    n = len(tr["time"])
    ms = timed(lambda: gpa.idleness_blame(tr, t, c, bl, sh))
    print(json.dumps({"row": "f4", "workload": "B3", "events": n, "ranks": S, "ms": ms,
                      "events_per_s": n / ms * 1e3, "GBps_12B_per_event": 12 * n / ms / 1e6}), flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["f1", "f2", "f4"]
    for w in which:
        globals()[w]()
