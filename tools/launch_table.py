"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum CSV (second half of the
launches = the last of two identical calls): python tools/launch_table.py file.csv [fraction]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr, data = rows[start], rows[start + 1:]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
data = data[int(len(data) * (1 - frac)):]
agg = collections.OrderedDict()
for r in data:
    n = r[ki].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("void ", "")
    n = n.split("(")[0].split("<")[0]
    agg.setdefault(n, [0, 0.0])
    agg[n][0] += 1
    agg[n][1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"| kernel | launches | us | share |\n|---|---|---|---|")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| {k.split('::')[-1]} | {v[0]} | {v[1] / 1e3:.1f} | {v[1] / tot * 100:.1f} % |")
print(f"| total | {sum(v[0] for v in agg.values())} | {tot / 1e3:.1f} | |")
