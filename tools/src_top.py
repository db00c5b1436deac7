"""Top stalled SASS instructions of an ncu --page source --csv export (tools/ncu_src.sh)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n_top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
data = [r for r in rows[2:] if len(r) == len(h)]
S = "Warp Stall Sampling (All Samples)"
tot = sum(int(r[idx[S]]) for r in data)
print("total samples", tot, "instructions", len(data))
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
agg = {c: sum(int(r[idx[c]] or 0) for r in data) for c in cols}
print(" ".join(f"{c[6:]}={v/tot*100:.1f}%" for c, v in sorted(agg.items(), key=lambda x: -x[1]) if v))
for r in sorted(data, key=lambda r: -int(r[idx[S]]))[:n_top]:
    s = int(r[idx[S]])
    det = " ".join(f"{c[6:]}={r[idx[c]]}" for c in cols if r[idx[c]] not in ("0", "") and int(r[idx[c]]) > s // 20)
    print(f"{r[0][-5:]} {s/tot*100:5.1f}% {r[1].strip()[:64]:64s} {det}")
