#!/bin/bash
# GPU box: run a subset of GPU tests, logs to gpurun_out/
# usage: bash tools/gpu_run_tests.sh "<pytest args>" [logname]
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
free -g | head -2; nproc
log=gpurun_out/${2:-tests}.log
timeout ${TEST_TIMEOUT:-1500} python -m pytest $1 -q -rfE --durations=15 > $log 2>&1; echo rc=$?
tail -25 $log
