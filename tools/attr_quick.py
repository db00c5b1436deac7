"""K_attr per config, GPU only (no oracle): CUDA-event median of the automatic call and of a call
with a reused plan, plus (--trace) the kernel timeline of one call from torch.profiler (CUPTI), so
launch gaps and the pre-pass / fold kernels show up next to the main kernel.

    python tools/attr_quick.py C2,C3,C4 [--trace] [--reps 7]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import gen
from paper_2109_06931_b200 import gpa

try:
    PEAK = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    PEAK = 6534.8


def med(fn, k, w=3):
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs")
    ap.add_argument("--trace", action="store_true")
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--records", type=int, default=0)
    a = ap.parse_args()
    for name in a.configs.split(","):
        w = gen.workload(name, records=a.records or None)
        n = w.cfg.records
        s = gpa.load_structure(w.structure, 0)
        rec = torch.empty((n, 2), dtype=torch.int64, device="cuda")
        for k in range(0, n, 1 << 28):
            w.records_device(rec[k:k + (1 << 28)], k, min(1 << 28, n - k))
        ni = s.info["n_inst"]
        HU = torch.zeros(ni * 16 + 16, dtype=torch.int64, device="cuda")
        H, U = HU[:ni * 16].view(ni, 16), HU[ni * 16:]

        def attr():
            HU.zero_()
            gpa.attribute_samples(s, rec, H, U)

        plan = gpa.AttrPlan(s, rec, n) if n >= 4096 else None

        def attr_planned():
            HU.zero_()
            if plan is not None and plan.variant:
                plan.attribute(rec, H, U)
            else:
                gpa.attribute_samples(s, rec, H, U)

        t = med(attr, a.reps)
        tp = med(attr_planned, a.reps)
        roof = 16 * n / PEAK / 1e6
        print(json.dumps(dict(config=name, records=n, kernel=gpa.attr_kernel_choice(s, n), attr_ms=round(t, 4),
                              frac=round(roof / t, 3), planned_ms=round(tp, 4), planned_frac=round(roof / tp, 3),
                              roofline_ms=round(roof, 4))), flush=True)
        if a.trace:
            from torch.profiler import ProfilerActivity, profile
            torch.cuda.synchronize()
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                attr()
                torch.cuda.synchronize()
            ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
            ev.sort(key=lambda e: e.time_range.start)
            t0 = ev[0].time_range.start if ev else 0
            for e in ev:
                print(f"  {e.time_range.start - t0:9.1f} us  {e.time_range.end - e.time_range.start:8.1f} us  {e.name[:90]}")
        del rec, plan
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
