"""A/B timing of the attribution kernel variants (GPA_ATTR_VARIANT) on one workload.
Each variant runs in a subprocess (the variant is read once per process)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, %r)
import gen
from paper_2109_06931_b200 import gpa
name, records, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
w = gen.workload(name, records=records)
s = gpa.load_structure(w.structure, 0)
n = w.cfg.records
rec = torch.empty((n, 2), dtype=torch.int64, device="cuda")
CH = 1 << 28
for k in range(0, n, CH):
    w.records_device(rec[k:k + CH], k, min(CH, n - k))
H = torch.zeros((s.info["n_inst"], 16), dtype=torch.int64, device="cuda")
U = torch.zeros(16, dtype=torch.int64, device="cuda")
ts = []
for r in range(reps + 2):
    H.zero_(); U.zero_()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); gpa.attribute_samples(s, rec, H, U); e1.record(); torch.cuda.synchronize()
    if r >= 2: ts.append(e0.elapsed_time(e1))
import hashlib
h = hashlib.sha1(H.cpu().numpy().tobytes() + U.cpu().numpy().tobytes()).hexdigest()
ms = sorted(ts)[len(ts) // 2]
print(json.dumps({"ms": ms, "min_ms": min(ts), "GBps": 16 * n / ms / 1e6, "rec_per_s": n / ms * 1e3, "sha1": h}))
''' % ROOT

if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "C5"
    records = int(sys.argv[2]) if len(sys.argv) > 2 else 4_000_000_000
    variants = sys.argv[3].split(",") if len(sys.argv) > 3 else ["1", "2", "3"]
    for v in variants:
        var, _, cfg = v.partition(":")
        env = dict(os.environ, GPA_ATTR_VARIANT=var, GPA_HOT_CFG=cfg or "0")
        out = subprocess.run([sys.executable, "-c", CHILD, name, str(records), "5"], env=env, capture_output=True,
                             text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-1500:].replace("\n", " | ")
        print(f"variant {v}: {line}", flush=True)
