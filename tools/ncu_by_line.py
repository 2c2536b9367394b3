"""Aggregate an `ncu --page source --csv --print-source sass` dump per CUDA
source line, using the address -> line map of `nvdisasm -g` on the same cubin.

    python tools/ncu_by_line.py <sass.csv> <nvdisasm -g output> <function substring> [top]

Prints, per source line: warp-stall samples (share), warp instructions
executed, shared-memory wavefronts (and excess), the top stall reasons.  The
SASS text of a few addresses is compared with the disassembly first (the
cubin must be the one that was profiled).
"""
import csv
import re
import sys
from collections import defaultdict


def line_map(dis_path, func):
    amap, text = {}, {}
    cur = None
    inside = False
    for ln in open(dis_path):
        if ln.startswith(".text.") and ln.rstrip().endswith(":"):
            inside = func in ln
            continue
        if not inside:
            continue
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", ln)
        if m:
            a = int(m.group(1), 16)
            amap[a] = cur
            text[a] = m.group(2)
    return amap, text


def main():
    sass_csv, dis, func = sys.argv[1], sys.argv[2], sys.argv[3]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    amap, text = line_map(dis, func)
    rows = list(csv.reader(open(sass_csv)))
    # first kernel only (the dump may hold several); addresses relative to its start
    ends = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
    if len(ends) > 1:
        rows = rows[: ends[1]]
    hdr = rows[1]
    base = int(rows[2][0], 16)
    ix = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = defaultdict(lambda: defaultdict(float))
    mism = 0
    n = 0
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        try:
            a = int(r[ix["Address"]], 16) - base
        except ValueError:
            continue
        n += 1
        src = r[ix["Source"]].strip().rstrip(";").strip()
        if a in text and n % 50 == 1:
            t0 = re.sub(r"\s+", " ", text[a])
            t1 = re.sub(r"\s+", " ", src)
            if t0.split(" ")[0].lstrip("@!P0123456789T ") != t1.split(" ")[0].lstrip("@!P0123456789T "):
                mism += 1
        key = amap.get(a)
        d = agg[key]

        def num(c):
            try:
                return float(r[ix[c]] or 0)
            except (ValueError, KeyError):
                return 0.0

        d["samples"] += num("Warp Stall Sampling (All Samples)")
        d["inst"] += num("Instructions Executed")
        d["wf"] += num("L1 Wavefronts Shared")
        d["wfx"] += num("L1 Wavefronts Shared Excessive")
        for c in stalls:
            d[c] += num(c)
    if mism:
        print(f"WARNING: {mism} sampled addresses disagree with the disassembly (different cubin?)")
    tot = sum(d["samples"] for d in agg.values()) or 1
    toti = sum(d["inst"] for d in agg.values()) or 1
    print(f"total stall samples {tot:.0f}, warp instructions {toti:.3e}")
    for key, d in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
        st = sorted(((d[c], c[6:]) for c in stalls), reverse=True)[:3]
        sts = " ".join(f"{c}:{100 * v / max(d['samples'], 1):.0f}%" for v, c in st if v)
        loc = f"{key[0]}:{key[1]}" if key else "?"
        print(f"{100 * d['samples'] / tot:5.1f}% inst {100 * d['inst'] / toti:5.1f}% wf {d['wf']:.2e} (x{d['wfx']:.1e})  {loc:22s} {sts}")


if __name__ == "__main__":
    main()
