#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=${1:-c3}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_child_chains3|k_child_step2" -s 2 -c 2 -o gpurun_out/${T}_c3 python tools/trace_run.py random_20000 0 > gpurun_out/${T}_c3.log 2>&1
exit 0
