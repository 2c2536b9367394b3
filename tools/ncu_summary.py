"""Summarise `ncu --set full` reports (one launch each) for profiles/:
duration, DRAM bytes and throughput, issue/occupancy, shared-memory
wavefronts and conflicts, top stall reasons, registers.

    python tools/ncu_summary.py rep1.ncu-rep|raw1.csv [...] > profiles/r1_ncu_full_summary.txt
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("kernel", "Kernel Name"), ("grid", "launch__grid_size"), ("block", "launch__block_size"),
    ("regs/thread", "launch__registers_per_thread"),
    ("duration ms", "gpu__time_duration.sum"),
    ("dram read GB", "dram__bytes_read.sum"), ("dram write GB", "dram__bytes_write.sum"),
    ("dram busy %", "dram__cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("warp instr", "smsp__inst_executed.sum"),
    ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("smem wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    ("smem conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    ("L2 hit %", "lts__t_sector_hit_rate.pct"),
]
STALLS = ["barrier", "short_scoreboard", "long_scoreboard", "wait", "math_pipe_throttle", "mio_throttle",
          "not_selected", "lg_throttle", "membar", "sleeping", "branch_resolving"]


def main():
    for rep in sys.argv[1:]:
        if rep.endswith(".csv"):  # an exported `--page raw --csv`
            raw = open(rep).read()
        else:
            raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        h, units = rows[0], rows[1]
        for r in rows[2:]:
            print(f"== {rep.split('/')[-1]}")
            for name, m in METRICS:
                if m in h:
                    v = r[h.index(m)]
                    u = units[h.index(m)]
                    if name.endswith("GB") and u in ("byte", "Gbyte", "Mbyte", "Kbyte"):
                        scale = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}[u]
                        v = f"{float(v.replace(',', '')) * scale:.3f}"
                    elif name == "duration ms" and u in ("nsecond", "usecond", "msecond"):
                        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}[u]
                        v = f"{float(v.replace(',', '')) * scale:.3f}"
                    print(f"  {name:18s} {v}")
            try:
                rd = float(r[h.index("dram__bytes_read.sum")].replace(",", ""))
                wr = float(r[h.index("dram__bytes_write.sum")].replace(",", ""))
                t = float(r[h.index("gpu__time_duration.sum")].replace(",", ""))
                us = units[h.index("dram__bytes_read.sum")]
                ut = units[h.index("gpu__time_duration.sum")]
                b = (rd + wr) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[us]
                s = t * {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}[ut]
                print(f"  {'dram GB/s':18s} {b / s / 1e9:.0f}")
            except (ValueError, KeyError):
                pass
            st = []
            for sname in STALLS:
                m = f"smsp__average_warps_issue_stalled_{sname}_per_issue_active.ratio"
                if m in h:
                    st.append((float(r[h.index(m)] or 0), sname))
            print("  stalls per issue  " + ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:6]))


if __name__ == "__main__":
    main()
