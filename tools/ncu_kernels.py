"""Per-kernel summary of an ncu report: time, DRAM bytes/throughput,
occupancy, issue activity and the top stall reasons.
    python tools/ncu_kernels.py report.ncu-rep"""
import csv
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
col = {n: i for i, n in enumerate(h)}
want = [("time_us", "gpu__time_duration.sum"), ("rd_GB", "dram__bytes_read.sum"), ("wr_GB", "dram__bytes_write.sum"),
        ("dram%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        ("warps%", "sm__warps_active.avg.pct_of_peak_sustained_active"), ("regs", "launch__registers_per_thread"),
        ("issue%", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        ("fp64%", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        ("winst", "smsp__inst_executed.sum")]
for r in rows[2:]:
    name = r[col["Kernel Name"]].split("(")[0].replace("void ", "")[:34]
    vals = []
    for lab, m in want:
        v = r[col[m]] if m in col else "?"
        vals.append(f"{lab}={v}")
    st = [(h[i], float(r[i])) for i in range(len(h)) if "smsp__average_warps_issue_stalled" in h[i]
          and h[i].endswith("per_issue_active.ratio") and r[i] not in ("", "n/a")]
    st.sort(key=lambda x: -x[1])
    print(f"{name:34s} " + " ".join(vals))
    print(" " * 35 + "stalls " + ", ".join(f"{a.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={b:.2f}" for a, b in st[:5]))
