"""f1 function level only (gpa_attribute_profiles on C4: 1e9 records, 384 profiles), CUDA-event
median; for A/B of builds (tools/ab_libs.sh style).  python tools/f1_quick.py [records]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
from paper_2109_06931_b200 import gpa

n = int(sys.argv[1]) if len(sys.argv) > 1 else None
w = gen.workload("C4", records=n)
s = gpa.load_structure(w.structure, 0)
n = w.cfg.records
rec = torch.empty((n, 2), dtype=torch.int64, device="cuda")
for k in range(0, n, 1 << 28):
    w.records_device(rec[k:k + (1 << 28)], k, min(1 << 28, n - k))
P = 384
PH = torch.zeros((P + 1, s.info["n_func"], 16), dtype=torch.int64, device="cuda")
PU = torch.zeros((P + 1, 16), dtype=torch.int64, device="cuda")
ts = []
for r in range(9):
    PH.zero_()
    PU.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gpa.attribute_profiles(s, rec, P, PH, PU)
    e1.record()
    torch.cuda.synchronize()
    if r >= 2:
        ts.append(e0.elapsed_time(e1))
ms = statistics.median(ts)
print(json.dumps({"f1_ms": round(ms, 4), "frac": round(16 * n / ms / 1e6 / 6534.8, 3), "sum": int(PH.sum().item())}))
