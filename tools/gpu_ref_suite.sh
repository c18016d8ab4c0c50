#!/bin/bash
# GPU box: the reference test suite against the drop-in + our GPU tests
mkdir -p $GRAFT_REPO_ROOT/gpurun_out
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm --format=csv
cd /tmp && PYTHONPATH=$GRAFT_REPO_ROOT/tests timeout 1200 python -m pytest -p ref_dropin -q $GRAFT_REPO_ROOT/oracle/_ref/tests/ -p no:cacheprovider --rootdir=$GRAFT_REPO_ROOT/oracle/_ref -rfE --tb=short > $GRAFT_REPO_ROOT/gpurun_out/ref_suite.log 2>&1; echo rc=$?
tail -5 $GRAFT_REPO_ROOT/gpurun_out/ref_suite.log
cd $GRAFT_REPO_ROOT && timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo gpu_rc=$?; tail -3 gpurun_out/gpu_tests.log
