"""Small end-to-end run of every library entry point, for compute-sanitizer
(memcheck / racecheck / synccheck): python tools/sanitize.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
from paper_2109_06931_b200 import gpa

for kernel in (0, 1, 2, 3, 4):
    gpa.set_attr_kernel(kernel)
    for name, records in (("C1", 10_000), ("C2", 2_200_000)):
        w = gen.workload(name, records=records)
        s = gpa.load_structure(w.structure, 0)
        rec = torch.empty((records, 2), dtype=torch.int64, device="cuda")
        w.records_device(rec)
        H = torch.zeros((s.info["n_inst"], 16), dtype=torch.int64, device="cuda")
        U = torch.zeros(16, dtype=torch.int64, device="cuda")
        ri = torch.empty(records, dtype=torch.int32, device="cuda")
        gpa.attribute_samples(s, rec, H, U, ri)
        for sc in ("INST", "LINE", "LOOP", "INLINE", "FUNC"):
            n = max(1, gpa.scope_row_count(s, sc))
            gpa.derive_metrics(s, sc, H, scope_hist=torch.empty((n, 16), dtype=torch.int64, device="cuda"),
                               scope_mix=torch.empty((n, 16), dtype=torch.int64, device="cuda"),
                               metrics=torch.empty((n, 33), dtype=torch.float64, device="cuda"))
        for mode in (gpa.WEIGHTS_SAMPLES, gpa.WEIGHTS_EXACT):
            c = gpa.reconstruct_cct(s, H, mode=mode)
            m = torch.empty((max(1, c.n), 33), dtype=torch.float64, device="cuda")
            gpa.derive_metrics(s, "CCT_EXCL", cct=c, metrics=m)
            gpa.derive_metrics(s, "CCT_INCL", cct=c, metrics=m)
            c.free()
        P = 3
        PH = torch.zeros((P + 1, s.info["n_func"], 16), dtype=torch.int64, device="cuda")
        PU = torch.zeros((P + 1, 16), dtype=torch.int64, device="cuda")
        gpa.attribute_profiles(s, rec, P, PH, PU)
        gpa.profile_stats(s, PH, P, torch.empty((s.info["n_func"], 6, 16), dtype=torch.float64, device="cuda"))
        torch.cuda.synchronize()
        s.free()
print("sanitize run OK")
