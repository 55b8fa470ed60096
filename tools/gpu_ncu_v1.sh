#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=${1:-v1}
timeout 900 ncu --set full --import-source on --clock-control none -k k_child_step -s 1 -c 1 -o gpurun_out/${T}_v1 python tools/trace_run.py random_20000 0 > gpurun_out/${T}_v1.log 2>&1
exit 0
