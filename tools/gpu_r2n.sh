#!/bin/bash
# gpu_r2.sh then one ncu --set full capture: $1 tag, $2 run tests (1/0), $3 kernel regex, $4 skip, $5 count
cd "$GRAFT_REPO_ROOT" || cd /root/repo
bash tools/gpu_r2.sh $1 $2
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c ${5:-1} -o gpurun_out/$1_prof $CMD > gpurun_out/$1_ncufull.log 2>&1
exit 0
