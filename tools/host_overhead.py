"""Per-call host enqueue time vs device time of gpa_attribute_samples for a mid-size call (C2,
1e7 records): K back-to-back calls, host time of the loop (no sync inside) and CUDA-event time of
the whole batch.  python tools/host_overhead.py [config] [records] [K]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
from paper_2109_06931_b200 import gpa

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000_000
K = int(sys.argv[3]) if len(sys.argv) > 3 else 200
w = gen.workload(name, records=n)
s = gpa.load_structure(w.structure, 0)
rec = torch.empty((n, 2), dtype=torch.int64, device="cuda")
w.records_device(rec)
H = torch.zeros((s.info["n_inst"], 16), dtype=torch.int64, device="cuda")
U = torch.zeros(16, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
for _ in range(20):
    gpa.attribute_samples(s, rec, H, U, stream=st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
t0 = time.perf_counter()
for _ in range(K):
    gpa.attribute_samples(s, rec, H, U, stream=st)
t1 = time.perf_counter()
e1.record()
torch.cuda.synchronize()
dev_ms = e0.elapsed_time(e1) / K
# the C ABI alone (ctypes call with prepared arguments)
args = (s.handle, rec.data_ptr(), n, H.data_ptr(), U.data_ptr(), None, st.cuda_stream)
t2 = time.perf_counter()
for _ in range(K):
    gpa._lib.gpa_attribute_samples(*args)
t3 = time.perf_counter()
torch.cuda.synchronize()
print(json.dumps({"config": name, "records": n, "calls": K, "host_us_per_call_binding": (t1 - t0) / K * 1e6,
                  "host_us_per_call_c_abi": (t3 - t2) / K * 1e6, "device_ms_per_call_back_to_back": dev_ms,
                  "frac_back_to_back": 16 * n / dev_ms / 1e6 / 6534.8}))
