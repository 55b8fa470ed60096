#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=${1:-rt}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_refine_warp" -s 6 -c 1 -o gpurun_out/${T}_root python tools/trace_run.py random_20000 0 > gpurun_out/${T}_root.log 2>&1
exit 0
