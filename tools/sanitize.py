"""Small end-to-end run of every library entry point, for compute-sanitizer
(memcheck / racecheck / synccheck): python tools/sanitize.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
from paper_2109_06931_b200 import gpa

KERNELS = [int(k) for k in os.environ.get("SAN_KERNELS", "0,1,2,3,4").split(",")]
for kernel in KERNELS:
    gpa.set_attr_kernel(kernel)
    for name, records in (("C1", 10_000), ("C2", 2_200_000), ("C3", 300_000)):
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
            c = gpa.reconstruct_cct_async(s, H, mode=mode)  # device-side row count, finish
            m = torch.empty((max(1, c.capacity), 33), dtype=torch.float64, device="cuda")
            gpa.derive_metrics(s, "CCT_EXCL", cct=c, metrics=m)
            gpa.derive_metrics(s, "CCT_INCL", cct=c, metrics=m)
            c.finish()
            c.free()
        P = 3
        PH = torch.zeros((P + 1, s.info["n_func"], 16), dtype=torch.int64, device="cuda")
        PU = torch.zeros((P + 1, 16), dtype=torch.int64, device="cuda")
        gpa.attribute_profiles(s, rec, P, PH, PU)
        gpa.profile_stats(s, PH, P, torch.empty((s.info["n_func"], 6, 16), dtype=torch.float64, device="cuda"))
        for cms in (False, True):
            gpa.sparse_build(s, PH, P, cms).free()
        PI = torch.zeros((P + 1, s.info["n_inst"], 16), dtype=torch.int64, device="cuda")
        gpa.attribute_profiles_inst(s, rec, P, PI, PU)
        gpa.profile_stats_rows(PI, P, torch.empty((s.info["n_inst"], 6, 16), dtype=torch.float64, device="cuda"))
        c = gpa.reconstruct_cct(s, H)
        E = torch.empty((P + 1, max(1, c.n), 16), dtype=torch.float64, device="cuda")
        I = torch.empty_like(E)
        gpa.cct_profiles(s, c, PH, P, E, I)
        gpa.profile_stats_f64(I, P, torch.empty((max(1, c.n), 6, 16), dtype=torch.float64, device="cuda"))
        c.free()
        torch.cuda.synchronize()
        s.free()
    if kernel != KERNELS[0]:
        continue
    from gen.trace import trace_set
    for tname in ("B1", "B2"):
        tr = trace_set(tname)
        t = torch.from_numpy(tr["time"].view(np.int64)).cuda()
        cx = torch.from_numpy(tr["ctx"].view(np.int32)).cuda()
        S, R = tr["n_scopes"], tr["n_routines"]
        gpa.idleness_blame(tr, t, cx, torch.empty((S, R), dtype=torch.float64, device="cuda"),
                           torch.empty((S, R), dtype=torch.float64, device="cuda"),
                           torch.empty(S, dtype=torch.int64, device="cuda"), torch.empty(S, dtype=torch.int64, device="cuda"))
        torch.cuda.synchronize()
print("sanitize run OK")
