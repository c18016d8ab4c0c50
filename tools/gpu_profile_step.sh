#!/bin/bash
# GPU box: full ncu capture of one hinted sync-free step of a workload, summarised into gpurun_out/
# usage: bash tools/gpu_profile_step.sh <tag> <one_step.py args...>   (kernels for line/SASS pages: $KERNELS)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
tag=$1; shift
python tools/one_step.py "$@" > gpurun_out/${tag}_plain.log 2>&1 || { tail -5 gpurun_out/${tag}_plain.log; exit 1; }
ncu -f --set full --clock-control none --import-source on -k regex:"k_" -s 10 -c 8 -o /tmp/${tag} \
    python tools/one_step.py "$@" > gpurun_out/${tag}_ncu.log 2>&1
python tools/ncu_kernels.py /tmp/${tag}.ncu-rep > gpurun_out/${tag}_kernels.txt
for k in ${KERNELS:-k_minmax k_hist_dev k_encode_keyed k_dec_chunks}; do
  python tools/ncu_lines.py /tmp/${tag}.ncu-rep "$k" 25 > gpurun_out/${tag}_${k}_lines.txt 2>&1
done
cat gpurun_out/${tag}_kernels.txt
