"""One f1 instruction-level call on C4 (1e9 records, 384 profiles) for ncu: python tools/prof_f1inst.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
from paper_2109_06931_b200 import gpa
w = gen.workload("C4")
s = gpa.load_structure(w.structure, 0)
n = w.cfg.records
rec = torch.empty((n, 2), dtype=torch.int64, device="cuda")
for k in range(0, n, 1 << 28):
    w.records_device(rec[k:k + (1 << 28)], k, min(1 << 28, n - k))
P = 384
PI = torch.zeros((P + 1, s.info["n_inst"], 16), dtype=torch.int64, device="cuda")
PU = torch.zeros((P + 1, 16), dtype=torch.int64, device="cuda")
gpa.attribute_profiles_inst(s, rec, P, PI, PU)
torch.cuda.synchronize()
print("done")
