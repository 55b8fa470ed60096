#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
for c in random_20000 glued_wilkinson_21000 clement_50000 random_100000; do
  timeout 300 python tools/trace_run.py $c 2 2> gpurun_out/tiers_$c.txt
done
exit 0
