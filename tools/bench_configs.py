"""Per-config measurements (every config, absolute numbers, the oracle beside it).

For each of C1..C5 at its BASELINE.json size, on one GPU: K_attr time (CUDA events, median of
5 after 2 warm-ups) with its HBM fraction; the whole step (zero + attribution + 5 scope
roll-ups/metrics + CCT + CCT metrics, as bench.py's step); and the oracle (D1 attribution on
one thread and on all host threads over a bounded prefix, plus the single-threaded rest of the
path on the full histogram).  Prints one markdown table.

    python tools/bench_configs.py [C1,C2,...]
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import gen
import oracle
from paper_2109_06931_b200 import gpa

SCOPES = ["INST", "LINE", "LOOP", "INLINE", "FUNC"]
try:
    PEAK = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    PEAK = 6650.0


def med(fn, k=5, w=2):
    ts = []
    for r in range(w + k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if r >= w:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def run(name):
    w = gen.workload(name)
    n = w.cfg.records
    s = gpa.load_structure(w.structure, 0)
    rec = torch.empty((n, 2), dtype=torch.int64, device="cuda")
    for k in range(0, n, 1 << 28):
        w.records_device(rec[k:k + (1 << 28)], k, min(1 << 28, n - k))
    ni = s.info["n_inst"]
    HU = torch.zeros(ni * 16 + 16, dtype=torch.int64, device="cuda")
    H, U = HU[:ni * 16].view(ni, 16), HU[ni * 16:]
    met = {sc: torch.empty((max(1, gpa.scope_row_count(s, sc)), 33), dtype=torch.float64, device="cuda")
           for sc in SCOPES}

    def attr():
        HU.zero_()
        gpa.attribute_samples(s, rec, H, U)

    plan = gpa.AttrPlan(s, rec, min(n, 1 << 22)) if n >= 4096 else None

    def attr_planned():  # a plan built once from the first 2^22 records, reused (gpa_attr_plan)
        HU.zero_()
        if plan is not None and plan.variant:
            plan.attribute(rec, H, U)
        else:
            gpa.attribute_samples(s, rec, H, U)

    def step():
        attr()
        gpa.derive_scopes(s, H, {sc: {"metrics": met[sc]} for sc in SCOPES})
        c = gpa.reconstruct_cct(s, H)
        cm = torch.empty((max(c.n, 1), 33), dtype=torch.float64, device="cuda")
        gpa.derive_metrics(s, "CCT_EXCL", cct=c, metrics=cm)
        gpa.derive_metrics(s, "CCT_INCL", cct=c, metrics=cm)
        torch.cuda.synchronize()
        c.free()

    t_attr = med(attr)
    t_plan = med(attr_planned)
    t_step = med(step)
    del rec
    torch.cuda.empty_cache()
    # oracle: D1 on a bounded prefix, 1 thread and all threads; the rest on the GPU's histogram
    cores = len(os.sched_getaffinity(0))
    m = min(n, 1 << 24)
    r = w.records_host(0, m, threads=cores)
    t0 = time.perf_counter()
    oracle.attribute(w.structure, r, threads=1)
    t1 = time.perf_counter()
    oracle.attribute(w.structure, r, threads=cores)
    t2 = time.perf_counter()
    Hh = H.cpu().numpy().view(np.uint64)
    t3 = time.perf_counter()
    for sc in SCOPES:
        h, mx = oracle.scope_hist(w.structure, Hh, sc)
        oracle.derive_u64(h, mx)
    R = oracle.cct(w.structure, Hh)
    oracle.derive_f64(R["excl"])
    oracle.derive_f64(R["incl"])
    t4 = time.perf_counter()
    return dict(name=name, n=n, t_attr=t_attr, gbs=16 * n / t_attr / 1e6, t_step=t_step, t_plan=t_plan,
                o1=m / (t1 - t0), oc=m / (t2 - t1), cores=cores, o_rest=(t4 - t3) * 1e3, ctx=R["n"])


if __name__ == "__main__":
    names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C1", "C2", "C3", "C4", "C5"]
    print(f"peak {PEAK} GB/s")
    print("| config | records | K_attr ms | GB/s (frac) | K_attr ms, reused plan (frac) | step ms | samples/s (step) | "
          "oracle D1 1 thread | oracle D1 all threads | oracle rest (1 thread) | CCT contexts |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for nm in names:
        d = run(nm)
        print(f"| {d['name']} | {d['n']:.3g} | {d['t_attr']:.3f} | {d['gbs']:.0f} ({d['gbs'] / PEAK:.3f}) | "
              f"{d['t_plan']:.3f} ({16 * d['n'] / d['t_plan'] / 1e6 / PEAK:.3f}) | {d['t_step']:.3f} | {d['n'] / d['t_step'] * 1e3:.3g} | {d['o1']:.3g}/s | {d['oc']:.3g}/s "
              f"({d['cores']}) | {d['o_rest']:.1f} ms | {d['ctx']} |", flush=True)
