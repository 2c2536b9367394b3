"""Summarise an `ncu --page source --csv` dump: top SASS lines by stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        s = int(r[idx["Warp Stall Sampling (All Samples)"]])
    except ValueError:
        continue
    st = sorted(((int(r[idx[c]] or 0), c) for c in stall_cols), reverse=True)[:2]
    data.append((s, r[idx["Address"]][-5:], r[idx["Source"]].strip()[:60], st))
tot = sum(d[0] for d in data)
print("total samples", tot)
for s, a, src, st in sorted(data, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{100*s/tot:5.1f}% {a} {src:60s} {st}")
