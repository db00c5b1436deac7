"""Run one attribution call on a workload (for ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
from paper_2109_06931_b200 import gpa
name, records, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 2
w = gen.workload(name, records=records)
s = gpa.load_structure(w.structure, 0)
n = w.cfg.records
rec = torch.empty((n, 2), dtype=torch.int64, device="cuda")
CH = 1 << 28
for k in range(0, n, CH):
    w.records_device(rec[k:k + CH], k, min(CH, n - k))
H = torch.zeros((s.info["n_inst"], 16), dtype=torch.int64, device="cuda")
U = torch.zeros(16, dtype=torch.int64, device="cuda")
for _ in range(reps):
    H.zero_(); U.zero_()
    gpa.attribute_samples(s, rec, H, U)
torch.cuda.synchronize()
print("done")
