"""Write the committed profile summaries (profiles/) from ncu outputs in gpurun_out/.

  python tools/profiles_from_ncu.py <round> <launches.csv> <full.ncu-rep> <config>
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    names = [r[ki] for r in rows]
    gen_idx = [i for i, n in enumerate(names) if "gen_kernel" in n]
    tail = rows[(max(gen_idx) + 1 if gen_idx else 0):]
    tot = collections.OrderedDict()
    for r in tail:
        n = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", ""))
        tot.setdefault(n, [0.0, 0])
        tot[n][0] += v
        tot[n][1] += 1
    s = sum(v[0] for v in tot.values())
    lines = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for n, (v, c) in sorted(tot.items(), key=lambda x: -x[1][0]):
        lines.append(f"| `{n}` | {c} | {v / 1e6:.3f} | {100 * v / s:.2f}% |")
    lines.append(f"| **all** | {len(tail)} | {s / 1e6:.3f} | 100% |")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    return tot, s


def full(rep, out_md, out_json, algo_bytes):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    hdr = rows[0]
    md = ["| section | metric | unit | value |", "|---|---|---|---|"]
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Value", "") and d.get("Section Name") in (
                "GPU Speed Of Light Throughput", "Memory Workload Analysis", "Compute Workload Analysis",
                "Scheduler Statistics", "Warp State Statistics", "Occupancy", "Launch Statistics"):
            md.append(f"| {d['Section Name']} | {d['Metric Name']} | {d['Metric Unit']} | {d['Metric Value']} |")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    d = dict(zip(rr[0], rr[2]))
    u = dict(zip(rr[0], rr[1]))

    def val(k):
        x = float(d[k].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u.get(k, ""), 1)
        return x * scale

    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    dur = val("gpu__time_duration.sum") if u.get("gpu__time_duration.sum") == "ns" else None
    keys = [k for k in sorted(d) if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")]
    md += ["", "| raw metric | unit | value |", "|---|---|---|"]
    for k in ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "smsp__inst_executed.sum",
              "smsp__inst_executed_op_global_red.sum", "smsp__inst_executed_op_shared_atom.sum",
              "lts__t_sectors_srcunit_tex_op_red.sum", "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed",
              "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum"] + keys:
        if k in d:
            md.append(f"| `{k}` | {u.get(k, '')} | {d[k]} |")
    with open(out_md, "w") as f:
        f.write("\n".join(md) + "\n")
    js = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr, "algorithmic_bytes": algo_bytes,
          "traffic_over_algorithmic": (rd + wr) / algo_bytes, "source": os.path.basename(rep)}
    with open(out_json, "w") as f:
        json.dump(js, f, indent=1)
    return js


if __name__ == "__main__":
    rnd, lcsv, rep, cfg = sys.argv[1:5]
    algo = int(sys.argv[5]) if len(sys.argv) > 5 else 64_000_000_000
    P = os.path.join(ROOT, "profiles")
    tot, s = launches(lcsv, os.path.join(P, f"{rnd}_launches_{cfg}.md"))
    kname = sys.argv[6] if len(sys.argv) > 6 else "k_attr_bins"
    js = full(rep, os.path.join(P, f"{rnd}_{kname}_{cfg}.md"), os.path.join(P, f"{rnd}_{kname}_{cfg}_traffic.json"), algo)
    print(json.dumps(js))
