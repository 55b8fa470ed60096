#!/bin/bash
# one ncu --set full capture of a k_wvectors_pair launch (and a k_child_step2) during tools/trace_run.py; tag $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=${1:-np}
timeout 300 python tools/trace_run.py random_20000 0 > /dev/null 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_wvectors_pair -s 3 -c 1 -o gpurun_out/${T}_pair python tools/trace_run.py random_20000 0 > gpurun_out/${T}_pair.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_child_step2 -s 1 -c 1 -o gpurun_out/${T}_child2 python tools/trace_run.py random_20000 0 > gpurun_out/${T}_child2.log 2>&1
exit 0
