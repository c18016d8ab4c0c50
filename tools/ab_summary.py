"""Summarise tools/ab_cfg.py output: mean step ms and per-phase ms per (case, variant)."""
import ast
import collections
import re
import sys

acc = collections.defaultdict(list)
for line in sys.stdin:
    m = re.match(r"(.{16}) (\S+)\s+step ([\d.]+) ms\s+([\d.]+) GB/s (\{.*\})", line)
    if not m:
        continue
    acc[(m.group(1).strip(), m.group(2))].append((float(m.group(3)), ast.literal_eval(m.group(5))))
for (case, var), rows in sorted(acc.items()):
    step = sum(r[0] for r in rows) / len(rows)
    ph = {k: round(sum(r[1][k] for r in rows) / len(rows), 4) for k in rows[0][1]}
    print(f"{case:16s} {var:24s} step {step:.4f}  {ph}")
