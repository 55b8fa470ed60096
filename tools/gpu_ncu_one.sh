#!/bin/bash
# one ncu --set full capture: $1 = tag, $2 = kernel (-k argument), $3 = launches to skip
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/$1_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k $2 -s $3 -c 1 -o gpurun_out/$1_prof $CMD > gpurun_out/$1_ncu.log 2>&1
exit 0
