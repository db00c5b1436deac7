"""Capture the DRAM traffic of the timed attribution kernel (bench.py's roofline.traffic) with ncu
and write profiles/k_attr_traffic_<cfg>.json, stamped with a hash of the kernel sources: bench.py
uses the capture only while the sources are unchanged (else traffic = null).  Run on a GPU box:

    python tools/capture_traffic.py [C5 [records]]
"""
import csv
import hashlib
import io
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SOURCES = ["paper_2109_06931_b200/csrc/k_attr.cu", "paper_2109_06931_b200/csrc/kern_common.cuh",
           "paper_2109_06931_b200/csrc/gpa_internal.cuh", "include/gpa.h"]


def source_hash() -> str:
    h = hashlib.sha1()
    for p in SOURCES:
        h.update(open(os.path.join(ROOT, p), "rb").read())
    return h.hexdigest()


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
    records = int(sys.argv[2]) if len(sys.argv) > 2 else None
    sys.path.insert(0, ROOT)
    import gen
    w = gen.workload(cfg, records=records)
    n = w.cfg.records
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "-k", "regex:k_attr_(code32|probe|direct|bins|hot|tma|stream)", "-c", "1", "--csv",
           sys.executable, os.path.join(ROOT, "tools", "prof_attr.py"), cfg, str(n), "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT).stdout
    rows = [r for r in csv.reader(io.StringIO(out)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6,
             "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}
    m = {r[mi]: float(r[vi].replace(",", "")) * scale.get(r[ui], 1) for r in rows}
    kernel = rows[0][ki].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
    rd, wr = m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]
    res = {"kernel": kernel, "config": cfg, "records": n, "dram_read": rd, "dram_write": wr,
           "dram_bytes_per_launch": rd + wr, "algorithmic_bytes": 16 * n,
           "traffic_over_algorithmic": (rd + wr) / (16 * n), "kernel_s_under_ncu": m.get("gpu__time_duration.sum"),
           "source_sha1": source_hash(), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "how": " ".join(cmd[:9]) + " tools/prof_attr.py (one call, cold L2; replayed per metric group)"}
    for d in ("profiles", "gpurun_out"):   # gpurun_out/: the copy that travels back from a GPU box
        os.makedirs(os.path.join(ROOT, d), exist_ok=True)
        json.dump(res, open(os.path.join(ROOT, d, f"k_attr_traffic_{cfg}.json"), "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
