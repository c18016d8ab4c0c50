#!/bin/bash
# GPU box: bench.py across workloads, one JSON line per run into gpurun_out/bench_suite.jsonl
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
out=gpurun_out/bench_suite.jsonl; : > $out
run() { echo "== $*" >&2; timeout ${BENCH_TIMEOUT:-900} python bench.py "$@" 2> gpurun_out/bench_err_$(echo "$*" | tr ' -' '__').log | tail -1 >> $out; echo "rc=$? $*" >&2; }
for spec in "$@"; do run $spec; done
python - <<'PY'
import json
for l in open("gpurun_out/bench_suite.jsonl"):
    l = l.strip()
    if not l.startswith("{"): print("??", l[:200]); continue
    d = json.loads(l)
    if d.get("impl") == "reference":
        print("REF", d["config"]["workload"][:40], round(d["value"], 4), d["cpu_baseline"].get("workers_1_gbs"), d.get("full_size_once", {}).get("gbs")); continue
    r = d["roofline"]; e = d.get("e2e") or {}; s = d.get("series_e2e") or {}
    print(d["config"]["workload"][:40], "N", d["n_gpus"], "val %.1f" % d["value"], "ms %.4f" % d["ms_per_step"],
          "phase", {k: round(v, 4) for k, v in d["phase_ms"].items()}, "roof %s %.3f" % (r["kernel"][:12], r["frac"]),
          "step1p %.3f" % d["roofline_all"]["step"]["single_pass_frac"], "e2e", e.get("value"), "series", s.get("value"),
          "cpu", (d.get("cpu_baseline") or {}).get("value"), "clk", d["clocks"])
PY
