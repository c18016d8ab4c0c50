"""DRAM bytes and time per kernel launch from an ncu --set full report ->
profiles/ncu_traffic.json (read by bench.py for roofline.traffic).
    python tools/ncu_traffic.py report.ncu-rep "command line" > profiles/ncu_traffic.json"""
import csv
import json
import re
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units = rows[0], rows[1]
col = {n: i for i, n in enumerate(h)}
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1.0, "us": 1e3, "ms": 1e6,
         "s": 1e9}


def val(r, metric):
    i = col[metric]
    return float(r[i]) * SCALE.get(units[i], 1.0)


acc = {}
for r in rows[2:]:
    full = r[col["Kernel Name"]]
    name = re.sub(r"^void ", "", full.split("(")[0])
    short = re.sub(r"<.*", "", name).replace("nmk::", "").replace("cub::", "cub_")
    rd = val(r, "dram__bytes_read.sum")
    wr = val(r, "dram__bytes_write.sum")
    t = val(r, "gpu__time_duration.sum")   # ns
    a = acc.setdefault(short, {"name": name, "launches": 0, "read": 0.0, "write": 0.0, "time_ns": 0.0})
    a["launches"] += 1
    a["read"] += rd
    a["write"] += wr
    a["time_ns"] += t
out = {"source": "ncu --set full --clock-control none: " + (sys.argv[2] if len(sys.argv) > 2 else ""),
       "kernels": {}, "dram_bytes_per_launch": {}}
for short, a in acc.items():
    n = a["launches"]
    out["kernels"][short] = {"name": a["name"], "launches": n, "dram_read_bytes": a["read"] / n,
                             "dram_write_bytes": a["write"] / n, "time_ms": a["time_ns"] / n / 1e6}
    out["dram_bytes_per_launch"][short] = (a["read"] + a["write"]) / n
print(json.dumps(out, indent=1))
