"""Run reconstruct_cct (+ CCT metrics) a few times on a workload's histogram (for ncu launch
lists and host timing): python tools/prof_cct.py C3 [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
from paper_2109_06931_b200 import gpa

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
w = gen.workload(name, records=min(gen.workload(name).cfg.records, 200_000_000))
s = gpa.load_structure(w.structure, 0)
n = w.cfg.records
rec = torch.empty((n, 2), dtype=torch.int64, device="cuda")
for k in range(0, n, 1 << 28):
    w.records_device(rec[k:k + (1 << 28)], k, min(1 << 28, n - k))
H = torch.zeros((s.info["n_inst"], 16), dtype=torch.int64, device="cuda")
U = torch.zeros(16, dtype=torch.int64, device="cuda")
gpa.attribute_samples(s, rec, H, U)
torch.cuda.synchronize()
for r in range(reps):
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    c = gpa.reconstruct_cct(s, H)
    cm = torch.empty((max(c.n, 1), 33), dtype=torch.float64, device="cuda")
    gpa.derive_metrics(s, "CCT_EXCL", cct=c, metrics=cm)
    gpa.derive_metrics(s, "CCT_INCL", cct=c, metrics=cm)
    e1.record()
    torch.cuda.synchronize()
    print(f"rep {r}: {c.n} contexts, gpu {e0.elapsed_time(e1):.3f} ms, host {(time.perf_counter() - t0) * 1e3:.3f} ms")
    c.free()
if os.environ.get("TRACE"):
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        c = gpa.reconstruct_cct(s, H)
        cm = torch.empty((max(c.n, 1), 33), dtype=torch.float64, device="cuda")
        gpa.derive_metrics(s, "CCT_EXCL", cct=c, metrics=cm)
        gpa.derive_metrics(s, "CCT_INCL", cct=c, metrics=cm)
        torch.cuda.synchronize()
    ev = sorted((e for e in prof.events() if e.device_type.name == "CUDA"), key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start if ev else 0
    for e in ev:
        print(f"  {e.time_range.start - t0:9.1f} us  {e.time_range.end - e.time_range.start:8.1f} us  {e.name[:90]}")
    c.free()
