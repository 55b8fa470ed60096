#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
for rc in 32 16 8; do
  for c in random_20000 random_100000; do
    MRRR_RW_ROOT_CHUNK=$rc timeout 900 python bench.py --config $c --steps 4 --warmup 2 --no-cpu --no-e2e > gpurun_out/$1_${c}_$rc.json 2> gpurun_out/$1_${c}_$rc.err
  done
done
exit 0
