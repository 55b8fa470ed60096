#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
for tc in 8 4 16; do
  for c in random_20000 glued_wilkinson_21000 random_100000; do
    MRRR_RW_CHUNK=$tc MRRR_RW_ROOT_CHUNK=32 timeout 900 python bench.py --config $c --steps 4 --warmup 2 --no-cpu --no-e2e > gpurun_out/$1_${c}_$tc.json 2> gpurun_out/$1_${c}_$tc.err
  done
done
exit 0
