#!/bin/bash
# GPU box: round-2 evidence for the cfg2 bench step (run after bench.py exits 0 without ncu).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pre_bench.json 2> gpurun_out/pre_bench.err || exit 1
# 1. launch list of the bench command (cold, serialised per-launch times)
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv \
    --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/ncu_launch.log 2>&1
# 2. full capture of one eager step (the second of tools/one_step.py's two steps)
ncu -f --set full --clock-control none --import-source on -k regex:"k_" -s 10 -c 8 -o /tmp/r2_cfg2 \
    python tools/one_step.py cfg2 > gpurun_out/ncu_full.log 2>&1
python tools/ncu_kernels.py /tmp/r2_cfg2.ncu-rep > gpurun_out/r2_ncu_full_kernels.txt
python tools/ncu_traffic.py /tmp/r2_cfg2.ncu-rep "ncu --set full --clock-control none --import-source on -k regex:k_ -s 10 -c 8 python tools/one_step.py cfg2 (round 2, cfg2 512^3 f64, B=8)" > gpurun_out/r2_ncu_traffic.json
for k in k_minmax k_hist_dev k_encode_keyed k_dec_chunks; do
  python tools/ncu_sass_summary.py /tmp/r2_cfg2.ncu-rep "$k" 20 > gpurun_out/r2_${k}_sass.txt 2>&1
  python tools/ncu_lines.py /tmp/r2_cfg2.ncu-rep "$k" 25 > gpurun_out/r2_${k}_lines.txt 2>&1
done
cuobjdump -sass paper_1703_02438_b200/libnmkgpu.so > /tmp/all.sass
python - <<'PY' > gpurun_out/r2_sass_opcodes.txt
import re, collections
txt = open("/tmp/all.sass").read()
funcs = re.split(r"\n\s+Function : ", txt)
want = {"k_minmax<double>": "k_minmaxIdE", "k_hist_dev<double,0>": "k_hist_devIdLi0E", "k_encode_keyed<double,8,0>": "k_encode_keyedIdLi8ELb0E",
        "k_dec_chunks<double,8,6>": "k_dec_chunksIdLi8ELi6E", "k_inflate": "k_inflate", "k_deflate_segments": "k_deflate_segments"}
for label, tag in want.items():
    for f in funcs:
        head = f.split("\n", 1)[0]
        if tag in head:
            ops = collections.Counter(m.group(1).split(".")[0] for m in re.finditer(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", f))
            keys = ["UBLKCP", "SYNCS", "LDG", "LDGSTS", "STG", "LDS", "STS", "ATOMS", "RED", "REDUX", "MATCH", "FMUL2", "FFMA2", "FADD2", "DMUL", "DADD", "DFMA", "MUFU", "SHFL", "VOTE"]
            print(label, head.strip()[:90])
            print("   ", {k: ops[k] for k in keys if ops[k]})
            break
PY
ls -la gpurun_out
