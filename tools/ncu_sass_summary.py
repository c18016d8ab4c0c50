"""Summarise an ncu source page (SASS) for one kernel: instruction mix by
opcode and the hottest stall sites.  Usage:
    python tools/ncu_sass_summary.py report.ncu-rep <kernel-regex> [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
lines = raw.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
ci = h.index("Source"); ii = h.index("Instructions Executed"); si = h.index("Warp Stall Sampling (All Samples)")
ti = h.index("Thread Instructions Executed")
by_op = collections.Counter(); samples = []
tot_i = tot_t = 0
for r in rows[1:]:
    if len(r) <= max(ci, ii, si):
        continue
    src = r[ci].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    try:
        n = int(r[ii]); s = int(r[si]); t = int(r[ti])
    except ValueError:
        continue
    by_op[op] += n; tot_i += n; tot_t += t
    samples.append((s, r[0], src))
print(f"warp instructions {tot_i:,}  thread instructions {tot_t:,}")
for op, n in by_op.most_common(top):
    print(f"  {op:12s} {n:14,d} {100*n/tot_i:5.1f}%")
samples.sort(reverse=True)
print("hottest stall sites:")
for s, a, src in samples[:top]:
    print(f"  {s:7d} {a[-6:]} {src}")
