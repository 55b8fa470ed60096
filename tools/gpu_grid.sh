#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
mkdir -p gpurun_out
for gf in 4 2 8 16; do
  for c in random_20000 random_100000; do
    MRRR_GRID_FACTOR=$gf timeout 900 python bench.py --config $c --steps 4 --warmup 2 --no-cpu --no-e2e > gpurun_out/$1_${c}_$gf.json 2> gpurun_out/$1_${c}_$gf.err
  done
done
exit 0
