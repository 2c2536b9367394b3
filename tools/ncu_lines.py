"""Per-CUDA-source-line summary of an `ncu --page source --csv --print-source
cuda,sass` dump: stall samples, warp instructions and shared wavefronts.

    python tools/ncu_lines.py dump.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fname = ""
hdr = None
agg = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        # second "Source" column is the SASS text; the first is the CUDA line
        continue
    if hdr is None or not r or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        s = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        ins = int(r[hdr["Instructions Executed"]] or 0)
        wf = int(r[hdr["L1 Wavefronts Shared"]] or 0)
    except (ValueError, KeyError, IndexError):
        continue
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    st = sorted(((int(r[hdr[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    agg.append((s, ins, wf, f"{fname}:{r[0]}", r[1].strip()[:70], st))
ts = sum(a[0] for a in agg) or 1
ti = sum(a[1] for a in agg) or 1
tw = sum(a[2] for a in agg) or 1
print(f"samples {ts}  warp-instr {ti}  smem wavefronts {tw}")
for s, ins, wf, loc, src, st in sorted(agg, reverse=True)[:top]:
    print(f"{100*s/ts:5.1f}% smp {100*ins/ti:5.1f}% ins {100*wf/tw:5.1f}% wf  {loc:22s} {src:70s} {[(c, n) for n, c in st if n]}")
