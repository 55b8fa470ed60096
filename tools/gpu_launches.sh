#!/bin/bash
# ncu launch lists (gpu__time_duration) of one random-20000 solve per refinement setting
# COMBOS="chunk:M ..." (MRRR_RW_CHUNK, MRRR_RW_M); tag = $1
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
T=${1:-l}
for cm in ${COMBOS:-0:0}; do
  c=${cm%%:*}; m=${cm##*:}
  export MRRR_RW_CHUNK=$c MRRR_RW_M=$m
  timeout 300 python tools/diag_solve.py random:20000 > gpurun_out/${T}_plain_$c_$m.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${T}_launches_${c}_$m.csv python tools/diag_solve.py random:20000 > gpurun_out/${T}_ncu_${c}_$m.log 2>&1
  timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_${c}_$m.json 2> gpurun_out/${T}_bench_${c}_$m.err
done
exit 0
