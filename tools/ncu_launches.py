"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv`) per kernel family.

    python tools/ncu_launches.py gpurun_out/launches.csv [--steps K] [--json out.json]

Launches are cold-cache and serialised under ncu: compare SHARES of the step,
not absolute times.  With --steps, only the last K sorts are used (one sort =
the launches from a prepass_kernel to the next).
"""
import argparse
import csv
import json
import re
from collections import OrderedDict, defaultdict

FAMILY = [
    ("prepass", r"prepass"), ("sample", r"sample_kernel"), ("classify", r"classify"),
    ("boundaries", r"boundaries"), ("stripe_fix", r"stripe_fix"), ("permute", r"permute"),
    ("cleanup", r"cleanup"), ("schedule", r"schedule"), ("basecase", r"basecase|count_"),
    ("reverse", r"reverse"), ("plan", r"entry_kernel|driver_kernel"),
]


def family(name):
    for f, pat in FAMILY:
        if re.search(pat, name):
            return f
    return "other:" + name.split("(")[0][-40:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--json")
    a = ap.parse_args()
    rows = [r for r in csv.reader(l for l in open(a.csv) if l.startswith('"'))]
    hdr = rows[0]
    I = {h: i for i, h in enumerate(hdr)}
    launches = OrderedDict()
    for r in rows[1:]:
        lid = int(r[I["ID"]])
        d = launches.setdefault(lid, {"name": r[I["Kernel Name"]], "grid": r[I["Grid Size"]]})
        v = float(r[I["Metric Value"]].replace(",", ""))
        d[r[I["Metric Name"]]] = v
    ids = list(launches)
    starts = [i for i in ids if re.search(r"entry_kernel", launches[i]["name"])] or \
        [i for i in ids if re.search(r"presample_kernel|prepass_kernel", launches[i]["name"])]
    sel = ids[starts[-a.steps]:] if len(starts) >= a.steps else ids
    fam = defaultdict(lambda: {"launches": 0, "ms": 0.0, "dram_read": 0.0, "dram_write": 0.0})
    for i in sel:
        d = launches[i]
        f = fam[family(d["name"])]
        f["launches"] += 1
        f["ms"] += d.get("gpu__time_duration.sum", 0) / 1e6
        f["dram_read"] += d.get("dram__bytes_read.sum", 0)
        f["dram_write"] += d.get("dram__bytes_write.sum", 0)
    tot = sum(f["ms"] for f in fam.values())
    out = {}
    print(f"{'family':12s} {'launch':>6s} {'ms/step':>9s} {'share':>6s} {'DRAM GB/step':>12s} {'GB/s':>8s}")
    for k, f in sorted(fam.items(), key=lambda kv: -kv[1]["ms"]):
        ms = f["ms"] / a.steps
        gb = (f["dram_read"] + f["dram_write"]) / a.steps / 1e9
        print(f"{k:12s} {f['launches'] // a.steps:6d} {ms:9.3f} {100 * f['ms'] / tot:5.1f}% {gb:12.3f} "
              f"{gb / (ms / 1e3) if ms else 0:8.0f}")
        out[k] = {"launches_per_step": f["launches"] // a.steps, "ms_per_step": ms,
                  "share": f["ms"] / tot, "dram_bytes_per_step": gb * 1e9,
                  "dram_bytes_per_launch": gb * 1e9 / max(1, f["launches"] // a.steps)}
    print(f"total {tot / a.steps:.3f} ms/step (serialised, cold-cache)")
    if a.json:
        json.dump(out, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
