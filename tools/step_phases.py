"""Per-phase timing of one bench step (CUDA events + host clock) on a workload."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
from paper_2109_06931_b200 import gpa
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
records = int(sys.argv[2]) if len(sys.argv) > 2 else None
w = gen.workload(name, records=records)
s = gpa.load_structure(w.structure, 0)
n = w.cfg.records
rec = torch.empty((n, 2), dtype=torch.int64, device="cuda")
for k in range(0, n, 1 << 28):
    w.records_device(rec[k:k + (1 << 28)], k, min(1 << 28, n - k))
ni = s.info["n_inst"]
HU = torch.zeros(ni * 16 + 16, dtype=torch.int64, device="cuda")
H, U = HU[:ni * 16].view(ni, 16), HU[ni * 16:]
SC = ["INST", "LINE", "LOOP", "INLINE", "FUNC"]
met = {sc: torch.empty((max(1, gpa.scope_row_count(s, sc)), 33), dtype=torch.float64, device="cuda") for sc in SC}
st = torch.cuda.current_stream()
for rep in range(5):
    ev = []
    hs = []
    def mark(tag):
        e = torch.cuda.Event(enable_timing=True); e.record(st); ev.append((tag, e)); hs.append((tag, time.perf_counter()))
    torch.cuda.synchronize()
    mark("start")
    HU.zero_(); mark("zero")
    gpa.attribute_samples(s, rec, H, U); mark("attr")
    for sc in SC:
        gpa.derive_metrics(s, sc, H, metrics=met[sc]); mark(sc)
    c = gpa.reconstruct_cct(s, H); mark("cct")
    cm = torch.empty((max(c.n, 1), 33), dtype=torch.float64, device="cuda")
    gpa.derive_metrics(s, "CCT_EXCL", cct=c, metrics=cm); mark("cct_excl")
    gpa.derive_metrics(s, "CCT_INCL", cct=c, metrics=cm); mark("cct_incl")
    st.synchronize(); mark("sync")
    c.free(); mark("free")
    torch.cuda.synchronize()
    if rep == 4:
        e0 = ev[0][1]; h0 = hs[0][1]
        prev_d, prev_h = 0.0, 0.0
        for (tag, e), (_, h) in zip(ev, hs):
            d = e0.elapsed_time(e); hh = (h - h0) * 1e3
            print(f"{tag:10s} gpu {d:9.3f} ms (+{d - prev_d:7.3f})   host {hh:9.3f} ms (+{hh - prev_h:7.3f})")
            prev_d, prev_h = d, hh
