"""Mean device time per kernel name from an ncu --metrics gpu__time_duration.sum
--csv launch list.   python tools/launch_times.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
acc = collections.defaultdict(list)
for r in rows[hdr + 1:]:
    v = float(r[vi].replace(",", ""))
    if r[ui] == "nsecond":
        v /= 1e3
    elif r[ui] == "msecond":
        v *= 1e3
    acc[r[ki].split("(")[0].replace("void ", "")].append(v)
tot = 0.0
for k, v in acc.items():
    m = sum(v) / len(v)
    tot += sum(v)
    print(f"{k[:50]:50s} n={len(v):3d} mean_ns={m:9.0f}")
print(f"total_ns={tot:.0f}")
