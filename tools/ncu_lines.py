"""Instructions executed and stall samples per CUDA source line for one kernel.
    python tools/ncu_lines.py report.ncu-rep <kernel-regex> [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
h = rows[hi]
ii, si = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
agg = collections.defaultdict(lambda: [0, 0])
cur = None
for r in rows[hi + 1:]:
    if not r or r[0] in ("File Path", "Function Name", "Line No"):
        continue
    if r[0]:
        cur = (r[0], r[1].strip()[:95])
    try:
        agg[cur][0] += int(r[ii])
        agg[cur][1] += int(r[si])
    except (ValueError, IndexError):
        pass
tot = sum(v[0] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0]:>13,d} {100 * v[0] / tot:5.1f}% stall={v[1]:6d}  L{k[0]}: {k[1]}")
