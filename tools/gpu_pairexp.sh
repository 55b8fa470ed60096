#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
for mc in 32 128 512; do
  for c in random_20000 glued_wilkinson_21000 random_100000; do
    MRRR_PAIR_MAXCL=$mc timeout 900 python bench.py --config $c --steps 4 --warmup 2 --no-cpu --no-e2e > gpurun_out/$1_${c}_$mc.json 2> gpurun_out/$1_${c}_$mc.err
  done
done
exit 0
