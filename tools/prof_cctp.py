"""Per-profile CCTs unified by call path (R30) on C4 (384 profiles), for ncu launch lists:
python tools/prof_cctp.py [records] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
from paper_2109_06931_b200 import gpa

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = gen.workload("C4", records=n)
s = gpa.load_structure(w.structure, 0)
rec = torch.empty((n, 2), dtype=torch.int64, device="cuda")
for k in range(0, n, 1 << 28):
    w.records_device(rec[k:k + (1 << 28)], k, min(1 << 28, n - k))
P = 384
PH = torch.zeros((P + 1, s.info["n_func"], 16), dtype=torch.int64, device="cuda")
PU = torch.zeros((P + 1, 16), dtype=torch.int64, device="cuda")
gpa.attribute_profiles(s, rec, P, PH, PU)
PW = torch.zeros((P + 1, max(s.info["n_call"], 1)), dtype=torch.int64, device="cuda")
gpa.profile_call_weights(s, rec, P, PW)
torch.cuda.synchronize()
for _ in range(reps):
    t = gpa.reconstruct_cct_per_profile(s, PH, PW, P)
    torch.cuda.synchronize()
    t.free()
print("done")
