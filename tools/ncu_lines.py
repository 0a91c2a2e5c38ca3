"""Aggregate an ncu source page (cuda,sass CSV) per CUDA source line.

usage: ncu -i X.ncu-rep --page source --csv --print-source=cuda,sass > s.csv
       python tools/ncu_lines.py s.csv [N]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = next(r for r in rows if r and r[0] == "Line No")
start = rows.index(hdr) + 1
samp = hdr.index("Warp Stall Sampling (All Samples)")
cols = ["L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive", "Instructions Executed"]
stalls = [h for h in hdr if h.startswith("stall_") and "Not" not in h]
ix = {c: hdr.index(c) for c in cols + stalls}
agg = collections.defaultdict(collections.Counter)
src = {}
cur = None


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


for r in rows[start:]:
    if len(r) < samp + 1:
        continue
    if r[0]:
        cur = int(r[0]) if r[0].isdigit() else cur
        src[cur] = r[1]
        continue
    agg[cur]["s"] += num(r[samp])
    for c in cols + stalls:
        agg[cur][c] += num(r[ix[c]])
tot = sum(a["s"] for a in agg.values()) or 1.0
print("samples", tot, "shared wavefronts", sum(a[cols[0]] for a in agg.values()),
      "excessive", sum(a[cols[1]] for a in agg.values()))
for ln in sorted(agg, key=lambda l: -agg[l]["s"])[:n]:
    a = agg[ln]
    top = sorted(stalls, key=lambda x: -a[x])[:3]
    print(f"{ln:5} {a['s'] / tot * 100:5.1f}% wf={a[cols[0]]:.1e} exc={a[cols[1]]:.1e} "
          + " ".join(f"{t[6:]}={a[t] / max(a['s'], 1) * 100:.0f}%" for t in top)
          + "  | " + src.get(ln, "").strip()[:70])
