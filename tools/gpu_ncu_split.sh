#!/bin/bash
# ncu --set full of one single-warp vector piece (k_wvectors_split, a level-2 piece: both its launches); tag $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
T=${1:-n}
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wvectors_split -s 6 -c 2 -o gpurun_out/${T}_prof_wsplit $CMD > gpurun_out/${T}_ncu_wsplit.log 2>&1
tail -3 gpurun_out/${T}_ncu_wsplit.log
exit 0
